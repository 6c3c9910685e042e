// Micro-benchmark of the line-FFT building block (ffst_fft.cuh) at n = 4096, float32:
// batched 4096-point C2C rows, HBM in -> HBM out, no window, no scheduling.  Measurement only.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_1202_1773_b200/csrc/ffst_fft.cuh"
using namespace ffst;
constexpr int N = 4096;
using C = float2;

template <int NT, int MINB, bool TWS>
__global__ void __launch_bounds__(NT, MINB) k_rows(const C* __restrict__ in, C* __restrict__ out, int rows, const C* tw) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  C* sm = reinterpret_cast<C*>(sm_raw);
  constexpr int TH = 256, LPB = NT / TH;
  const int line = threadIdx.x / TH, t = threadIdx.x % TH;
  C* scr = sm + line * Pad<float>::len(N);
  const C* twp = tw;
  if constexpr (TWS) {
    C* st = sm + LPB * Pad<float>::len(N);
    for (int i = threadIdx.x; i < N; i += NT) st[i] = tw[i];
    __syncthreads();
    twp = st;
  }
  for (int r0 = blockIdx.x * LPB; r0 < rows; r0 += gridDim.x * LPB) {
    const int r = r0 + line;
    const C* src = in + (size_t)(r < rows ? r : 0) * N;
    C v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __ldcs(src + t + q * TH);
    LineFFT<float, N, false, N, TWS>::run(v, scr, t, twp);
    if (r < rows) {
#pragma unroll
      for (int q = 0; q < 16; ++q) __stcs(out + (size_t)r * N + t + q * TH, v[q]);
    }
    __syncthreads();
  }
}

// software-pipelined: the next line's 16 loads are issued before the current line's FFT
template <int NT, int MINB, bool TWS, bool TWG = false, bool TW2 = false>
__global__ void __launch_bounds__(NT, MINB) k_rows_pf(const C* __restrict__ in, C* __restrict__ out, int rows, const C* tw) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  C* sm = reinterpret_cast<C*>(sm_raw);
  constexpr int TH = 256, LPB = NT / TH;
  const int line = threadIdx.x / TH, t = threadIdx.x % TH;
  C* scr = sm + line * Pad<float>::len(N);
  const C* twp = tw;
  if constexpr (TWS) {
    C* st = sm + LPB * Pad<float>::len(N);
    for (int i = threadIdx.x; i < N; i += NT) st[i] = tw[i];
    __syncthreads();
    twp = st;
  }
  if constexpr (TW2) {                     // hi[m] = w^(64 m), lo[m] = w^m
    C* st = sm + LPB * Pad<float>::len(N);
    for (int i = threadIdx.x; i < N / 64; i += NT) st[i] = tw[64 * i];
    for (int i = threadIdx.x; i < 64; i += NT) st[N / 64 + i] = tw[i];
    __syncthreads();
    twp = st;
  }
  const int step = gridDim.x * LPB;
  int r = blockIdx.x * LPB + line;
  C nx[16];
  {
    const C* src = in + (size_t)(r < rows ? r : 0) * N;
#pragma unroll
    for (int q = 0; q < 16; ++q) nx[q] = __ldcs(src + t + q * TH);
  }
  for (int r0 = blockIdx.x * LPB; r0 < rows; r0 += step) {
    C v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = nx[q];
    const int rn = r + step;
    const C* srcn = in + (size_t)(rn < rows ? rn : 0) * N;
#pragma unroll
    for (int q = 0; q < 16; ++q) nx[q] = __ldcs(srcn + t + q * TH);
    LineFFT<float, N, false, N, TWS || TWG || TW2, 16, TW2>::run(v, scr, t, twp);
    if (r < rows) {
#pragma unroll
      for (int q = 0; q < 16; ++q) __stcs(out + (size_t)r * N + t + q * TH, v[q]);
    }
    __syncthreads();
    r = rn;
  }
}

// loads only / stores only references
__global__ void k_copy(const float4* __restrict__ in, float4* __restrict__ out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

int main(int argc, char** argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 4096 * 4;   // default 4 planes of 4096^2 complex: 537 MB in / out
  const size_t bytes = (size_t)rows * N * sizeof(C);
  C *in, *out, *tw;
  cudaMalloc(&in, bytes); cudaMalloc(&out, bytes); cudaMalloc(&tw, N * sizeof(C));
  cudaMemset(in, 0, bytes);
  C htw[N];
  for (int m = 0; m < N; ++m) { double a = 2 * 3.14159265358979323846 * m / N; htw[m] = make_float2((float)cos(a), (float)-sin(a)); }
  cudaMemcpy(tw, htw, sizeof(htw), cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    const int reps = rows < 4096 ? 200 : 10;
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    cudaError_t err = cudaGetLastError();
    printf("%-40s %8.3f ms  %7.0f GB/s  %6.1f ns/line  %s\n", name, ms, 2.0 * bytes / ms / 1e6, ms * 1e6 / rows,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  timeit("copy (float4, cs)", [&] { k_copy<<<sms * 8, 512>>>((const float4*)in, (float4*)out, bytes / 16); });
#define RUN(NT, MINB, TWS)                                                                                   \
  {                                                                                                          \
    const size_t smem = (NT / 256) * Pad<float>::len(N) * sizeof(C) + (TWS ? N * sizeof(C) : 0);            \
    cudaFuncSetAttribute(k_rows<NT, MINB, TWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rows<NT, MINB, TWS>, NT, smem);          \
    char name[96]; snprintf(name, sizeof name, "rows NT=%d minB=%d tws=%d (%d CTA/SM)", NT, MINB, TWS, nb);  \
    timeit(name, [&] { k_rows<NT, MINB, TWS><<<sms * nb, NT, smem>>>(in, out, rows, tw); });                  \
  }
  RUN(256, 1, false) RUN(256, 2, false) RUN(256, 3, false) RUN(256, 4, false)
  RUN(256, 2, true) RUN(256, 3, true) RUN(512, 1, false) RUN(512, 2, false)
#define RUNPF(NT, MINB, TWS)                                                                                 \
  {                                                                                                          \
    const size_t smem = (NT / 256) * Pad<float>::len(N) * sizeof(C) + (TWS ? N * sizeof(C) : 0);            \
    cudaFuncSetAttribute(k_rows_pf<NT, MINB, TWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rows_pf<NT, MINB, TWS>, NT, smem);       \
    char name[96]; snprintf(name, sizeof name, "rows-pf NT=%d minB=%d tws=%d (%d CTA/SM)", NT, MINB, TWS, nb); \
    timeit(name, [&] { k_rows_pf<NT, MINB, TWS><<<sms * nb, NT, smem>>>(in, out, rows, tw); });               \
  }
  RUNPF(256, 1, false) RUNPF(256, 2, false) RUNPF(256, 2, true) RUNPF(256, 3, false)
  {
    const size_t smem = Pad<float>::len(N) * sizeof(C);
    cudaFuncSetAttribute(k_rows_pf<256, 2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    timeit("rows-pf twg (products, global table)", [&] { k_rows_pf<256, 2, false, true><<<sms * 2, 256, smem>>>(in, out, rows, tw); });
  }
  {
    const size_t smem = Pad<float>::len(N) * sizeof(C) + (N / 64 + 64) * sizeof(C);
    cudaFuncSetAttribute(k_rows_pf<256, 2, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    timeit("rows-pf tw2 (two-level shared table)", [&] { k_rows_pf<256, 2, false, false, true><<<sms * 2, 256, smem>>>(in, out, rows, tw); });
    cudaFuncSetAttribute(k_rows<256, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  return 0;
}
