// ffst_user.cuh — plan-time kernels of the user-spectra mode (P:L2209-2224:
// "precomputed shearlet spectra ... used for the computation of the transform").
//
// The user hands eta real n x n spectra (rows omega_2, columns omega_1; centred or natural bin
// order).  At plan creation these kernels
//   * reduce the Parseval admission check of P:L2219-2220, max |sum_i psi_i^2 - 1|, and the
//     largest point-asymmetry max |psi_i(u) - psi_i(-u)| off the Nyquist lines (the even-n
//     decomposition of DESIGN.md 6.2 needs psi_i = sym_i + anti_i with anti_i on the Nyquist
//     row / column only, i.e. real-valued shearlets);
//   * write the symmetric part sym_i of every local plane into the Hermitian-half table the
//     persistent kernels read instead of evaluating the window: [eta_l][n/2+1][n], column
//     c <-> u1 = c (c = n/2: u1 = -n/2), row = natural bin of u2;
//   * record per plane the column hull where sym_i != 0 (the pruning range) and the anti part on
//     the Nyquist row / column (2n values, the plan's nyq_anti table for the Nyquist planes).
// Generic in n (run once per plan, not on the transform path).
#pragma once
#include "ffst_internal.h"
#include "ffst_math.cuh"

namespace ffst {


namespace user {

// u in -n/2 .. n/2-1 -> element of one plane in the caller's layout
__device__ __forceinline__ size_t at(const UserPrep& u, int u1, int u2) {
  const int H = u.n >> 1;
  if (u.centred) return (size_t)(u2 + H) * u.n + (u1 + H);
  return (size_t)(u2 < 0 ? u2 + u.n : u2) * u.n + (u1 < 0 ? u1 + u.n : u1);
}
// -u on the periodic grid: -(-n/2) = -n/2
__device__ __forceinline__ int neg(int v, int H) { return v == -H ? -H : -v; }

__device__ __forceinline__ void max_bits(unsigned long long* dst, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(dst, (unsigned long long)__double_as_longlong(v));
}

template <typename T>
__global__ void __launch_bounds__(256) stats_kernel(UserPrep u) {
  const T* psi = static_cast<const T*>(u.psi);
  const int n = u.n, H = n >> 1;
  const size_t plane = (size_t)n * n;
  double tight = 0.0, asym = 0.0;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < plane; e += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), m = (int)(e - (size_t)r * n);
    const int u1 = centred(m, n), u2 = centred(r, n);
    const size_t a = at(u, u1, u2), b = at(u, neg(u1, H), neg(u2, H));
    const bool interior = u1 != -H && u2 != -H;
    double s = 0.0;
    for (int i = 0; i < u.eta; ++i) {
      const double v = (double)psi[i * plane + a];
      s += v * v;
      if (interior) asym = fmax(asym, fabs(v - (double)psi[i * plane + b]));
    }
    tight = fmax(tight, fabs(s - 1.0));
  }
  for (int o = 16; o > 0; o >>= 1) {
    tight = fmax(tight, __shfl_xor_sync(0xffffffffu, tight, o));
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
  }
  if ((threadIdx.x & 31) == 0) {
    max_bits(u.stats + 0, tight);
    max_bits(u.stats + 1, asym);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) sym_kernel(UserPrep u) {
  const T* psi = static_cast<const T*>(u.psi);
  T* usym = static_cast<T*>(u.usym);
  const int n = u.n, H = n >> 1;
  const size_t plane = (size_t)n * n;
  const size_t total = (size_t)u.eta_l * (H + 1) * n;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  // rounded up so whole warps iterate together (warp-level hull reduction when n >= 32:
  // 32 consecutive threads then share one (plane, column))
  const size_t rounded = (total + 31) / 32 * 32;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < rounded; e += stride) {
    const bool act = e < total;
    int l = 0, c = 0;
    T v = T(0);
    if (act) {
      const int rb = (int)(e % n);
      const size_t lc = e / n;
      c = (int)(lc % (H + 1));
      l = (int)(lc / (H + 1));
      const int gi = u.shard_rank + l * u.shard_count;
      const T* P = psi + (size_t)gi * plane;
      const int u1 = c == H ? -H : c, u2 = centred(rb, n);
      v = P[at(u, u1, u2)];
      if (u1 == -H || u2 == -H) v = T(0.5) * (v + P[at(u, neg(u1, H), neg(u2, H))]);   // sym on the Nyquist lines
      usym[e] = v;
    }
    const bool nz = act && v != T(0);
    if (n >= 32) {
      const unsigned any = __ballot_sync(0xffffffffu, nz);
      if (any && (threadIdx.x & 31) == __ffs(any) - 1) {
        atomicMin(u.hull + 2 * l, c);
        atomicMax(u.hull + 2 * l + 1, c);
      }
    } else if (nz) {
      atomicMin(u.hull + 2 * l, c);
      atomicMax(u.hull + 2 * l + 1, c);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) anti_kernel(UserPrep u) {
  const T* psi = static_cast<const T*>(u.psi);
  T* anti = static_cast<T*>(u.anti);
  const int n = u.n, H = n >> 1;
  const size_t plane = (size_t)n * n;
  const size_t total = (size_t)u.eta_l * 2 * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int bin = (int)(e % n);
    const int which = (int)((e / n) % 2);
    const int l = (int)(e / (2 * (size_t)n));
    const T* P = psi + (size_t)(u.shard_rank + l * u.shard_count) * plane;
    const int w = centred(bin, n);
    // anti(u) = (psi(u) - psi(-u)) / 2 on the row u2 = -n/2 (which 0) / column u1 = -n/2 (which 1)
    const T a = which == 0 ? P[at(u, w, -H)] - P[at(u, neg(w, H), -H)]
                           : P[at(u, -H, w)] - P[at(u, -H, neg(w, H))];
    anti[e] = T(0.5) * a;
  }
}

}  // namespace user

template <typename T>
cudaError_t user_prepare_(const UserPrep& u, int grid, cudaStream_t s) {
  user::stats_kernel<T><<<grid, 256, 0, s>>>(u);
  if (u.usym == nullptr) return cudaGetLastError();   // admission numbers only
  user::sym_kernel<T><<<grid, 256, 0, s>>>(u);
  user::anti_kernel<T><<<grid, 256, 0, s>>>(u);
  return cudaGetLastError();
}

}  // namespace ffst
