// Microbenchmark: the inverse pass-1 access pattern (each CTA reads 64 KB row blocks with
// 16 x 16-byte loads per thread, 8 threads per 2 KB row), with an optional compute delay.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) kload(const float4* __restrict__ src, size_t nblk, int* ctr, int delay_ns,
                                               int mode, float* sink, unsigned long long* lat) {
  __shared__ int s_it;
  float acc = 0.f;
  unsigned long long tot = 0; int cnt = 0;
  for (;;) {
    if (threadIdx.x == 0) s_it = atomicAdd(ctr, 1);
    __syncthreads();
    int it = s_it;
    __syncthreads();
    if (it >= (int)nblk) break;
    const float4* base = src + (size_t)it * 4096;   // 64 KB block
    const int line = threadIdx.x / 8, t = threadIdx.x % 8;
    unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    float4 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const float4* a = base + line * 128 + t + q * 8;
      if (mode == 0) v[q] = __ldcs(a); else if (mode == 1) v[q] = __ldg(a); else v[q] = __ldcg(a);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) acc += v[q].x + v[q].y + v[q].z + v[q].w;
    unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    tot += t1 - t0; cnt++;
    if (delay_ns > 0) { unsigned long long s; do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s)); } while (s - t1 < (unsigned)delay_ns); }
  }
  if (acc == 12345.f) sink[0] = acc;
  if (threadIdx.x == 0 && cnt) atomicAdd(lat, tot / cnt);
}
int main() {
  const size_t bytes = 512ull << 20, nblk = bytes / 65536;
  float4* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  int* ctr; cudaMalloc(&ctr, 4); float* sink; cudaMalloc(&sink, 4);
  unsigned long long* lat; cudaMalloc(&lat, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int delay : {0, 2000, 5000, 10000}) {
      for (int grid_mult : {2}) {
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemset(ctr, 0, 4); cudaMemset(lat, 0, 8);
          cudaEventRecord(e0);
          kload<<<nsm * grid_mult, 256>>>(src, nblk, ctr, delay, mode, sink, lat);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
        }
        unsigned long long l; cudaMemcpy(&l, lat, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s) delay %5d ns grid %d: %.3f ms  %.0f GB/s  avg load phase %.2f us\n", mode,
               mode == 0 ? "cs" : mode == 1 ? "ldg" : "cg", delay, nsm * grid_mult, ms, bytes / ms / 1e6,
               (double)l / (nsm * grid_mult) / 1e3);
      }
    }
  return 0;
}
