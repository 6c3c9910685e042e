// ffst_tiny.cuh — fused kernels for small images (n <= 64): one CTA per (plane, image) holds the
// whole n x n problem in shared memory, so a forward transform is ONE launch and an inverse TWO
// (BASELINE configs[0], 64 x 64 float64, where the persistent two-pass schedule
// is launch / latency bound).
//
//   forward  (eq:shearletTransform): CTA (i, b): F = fft2(f_b) (rows, columns),
//            X = psi_i * F with psi_i evaluated on the fly on the whole natural-order grid,
//            c_i = ifft2(X) / n^2 -> coefficient plane (complex: no Hermitian decomposition needed)
//   inverse  (eq:inverseShearletTransform): CTA (i, b): part_{b,i} =
//            Re ifft2(psi_i * fft2(c_i)) / n^2 (the inverse is linear in the planes); then
//            tiny_sum: f_b = sum_i part_{b,i}, added in plane order (deterministic)
//
// Shared layout: the plane [n][n + 1] complex (one pad element per row: conflict-free column
// lines), plus each line group's FFT scratch.
#pragma once
#include "ffst_kernels.cuh"

namespace ffst {

template <typename T, int N>
struct Tiny {
  using C = cpx<T>;
  static constexpr int NT = 512;   // (the window and the plane I/O run on all threads, the line FFTs on N * TH)
  // 8 elements per thread from n = 64 on: the n lines of a pass then occupy all 512 threads (64 x 8)
  // instead of half of them (radix-8 passes: half the serial work per thread)
  static constexpr int EM = N >= 64 ? 8 : 16;
  static constexpr int E = RadixPlan<N, EM>::E, TH = N / E;
  static constexpr int LPR = NT / TH < N ? NT / TH : N;      // lines per round
  static constexpr int ROUNDS = N / LPR;
  static constexpr int LD = N + 1;                          // row stride of the plane in shared memory
  static constexpr int SCR = Pad<T, EM>::len(N);
  static constexpr size_t SMEM = (size_t)(N * LD + LPR * SCR) * sizeof(C);

  // 1-D FFTs of all rows (ROW) or columns of the shared plane, in place; INV: inverse sign.
  template <bool ROW, bool INV>
  static __device__ __forceinline__ void lines(C* pl, C* scr, const C* tw) {
    const int line = threadIdx.x / TH, t = threadIdx.x % TH;
    const bool act = line < LPR;
#pragma unroll 1
    for (int rd = 0; rd < ROUNDS; ++rd) {
      const int l = rd * LPR + (act ? line : 0);
      if (act) {                                   // (inactive threads are whole warps, or TH = 1: no sync)
        C r[E];
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const int m = t + q * TH;
          r[q] = ROW ? pl[l * LD + m] : pl[m * LD + l];
        }
        LineFFT<T, N, INV, N, false, EM>::run(r, scr + line * SCR, t, tw);
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const int m = t + q * TH;
          if (ROW) pl[l * LD + m] = r[q];
          else pl[m * LD + l] = r[q];
        }
      }
      __syncthreads();
    }
  }
};

// grid (eta_l, batch), Tiny::NT threads
template <typename T, int N>
__global__ void __launch_bounds__(512) tiny_fwd_kernel(KParams p) {
  using TY = Tiny<T, N>;
  using C = cpx<T>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* pl = reinterpret_cast<C*>(smem_raw);
  C* scr = pl + N * TY::LD;
  const int lp = blockIdx.x, b = blockIdx.y;
  const C* tw = static_cast<const C*>(p.tw);
  const T* img = static_cast<const T*>(p.img) + (size_t)b * N * N;
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) pl[(e / N) * TY::LD + e % N] = mk<T>(img[e], T(0));
  __syncthreads();
  TY::template lines<true, false>(pl, scr, tw);          // F = fft2(f): rows (omega_1) ...
  TY::template lines<false, false>(pl, scr, tw);         // ... then columns (omega_2)
  const PlaneDev P = p.planes[lp];
  const Radial<T> R = radial_of<T, N>(p);
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
    const int r = e / N, c = e % N;
    const T w = window<T>(P, centred(c, N), centred(r, N), R);
    C& v = pl[r * TY::LD + c];
    v = cscale<T>(v, w);
  }
  __syncthreads();
  TY::template lines<true, true>(pl, scr, tw);           // c = ifft2(psi * F)
  TY::template lines<false, true>(pl, scr, tw);
  const T s = T(1) / (T(N) * T(N));
  C* out = static_cast<C*>(p.coeff) + ((size_t)b * p.eta_l + lp) * N * N;
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) out[e] = cscale<T>(pl[(e / N) * TY::LD + e % N], s);
}

// grid (eta_l, batch): part[b][i] = Re ifft2(psi_i * fft2(c_i)) / n^2
template <typename T, int N>
__global__ void __launch_bounds__(512) tiny_inv_kernel(KParams p) {
  using TY = Tiny<T, N>;
  using C = cpx<T>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* pl = reinterpret_cast<C*>(smem_raw);
  C* scr = pl + N * TY::LD;
  const int lp = blockIdx.x, b = blockIdx.y;
  const C* tw = static_cast<const C*>(p.tw);
  const C* in = static_cast<const C*>(p.coeff) + ((size_t)b * p.eta_l + lp) * N * N;
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) pl[(e / N) * TY::LD + e % N] = in[e];
  __syncthreads();
  TY::template lines<true, false>(pl, scr, tw);          // fft2(c_i)
  TY::template lines<false, false>(pl, scr, tw);
  const PlaneDev P = p.planes[lp];
  const Radial<T> R = radial_of<T, N>(p);
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
    const int r = e / N, c = e % N;
    const T w = window<T>(P, centred(c, N), centred(r, N), R);
    C& v = pl[r * TY::LD + c];
    v = cscale<T>(v, w);
  }
  __syncthreads();
  TY::template lines<true, true>(pl, scr, tw);           // ifft2
  TY::template lines<false, true>(pl, scr, tw);
  const T s = T(1) / (T(N) * T(N));
  T* part = static_cast<T*>(p.part) + ((size_t)b * p.eta_l + lp) * N * N;
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) part[e] = pl[(e / N) * TY::LD + e % N].x * s;
}

// f_b = sum_i part[b][i] in plane order; grid (ceil(n^2 / 256), batch)
template <typename T, int N>
__global__ void __launch_bounds__(256) tiny_sum_kernel(KParams p) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.y;
  if (e >= N * N) return;
  const T* part = static_cast<const T*>(p.part) + (size_t)b * p.eta_l * N * N + e;
  T s = T(0);
  int i = 0;
  for (; i + 8 <= p.eta_l; i += 8) {               // eight loads in flight, added in plane order
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = part[(size_t)(i + u) * N * N];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; i < p.eta_l; ++i) s += part[(size_t)i * N * N];
  static_cast<T*>(p.img_out)[(size_t)b * N * N + e] = s;
}

}  // namespace ffst
