// ffst_generic.cuh — the FFST for ARBITRARY image sizes n (odd, or even but not a power of two;
// SURVEY 8(f) f3): "it is possible to compute the shearlet transform for arbitrary image sizes"
// (Sec. 3.8), with the grid of Sec. 3.5.2 (odd n as is, even n on the odd
// grid n + 1 with the last row / column dropped).
//
// Full complex 2-D transforms: no Hermitian halving and no even-n sym / anti split
// -- the window psi_i(Delta u) is evaluated on the fly on the whole natural-order grid, so odd n
// (point-symmetric grid, real coefficients) and even n (Nyquist row / column included) are the
// same code.  Every 1-D DFT of length L = n is a Bluestein convolution through power-of-two FFTs
// of length M >= 2L - 1 (the LineFFT building block of ffst_fft.cuh):
//   X[k] = conj(w_k) * IFFT_M( FFT_M(x * conj(w)) * FFT_M(b) )[k] / M,  w_m = exp(i pi m^2 / L),
//   b_t = w_t for |t| < L (indices mod M), 0 elsewhere;  FFT_M(b) is a plan table.
// The inverse DFT is conj(DFT(conj x)).  Lines are always contiguous rows; the other axis is
// reached through a tiled transpose kernel (32 x 32 shared-memory tiles).
//
// Layouts (per image; natural frequency bins, rows = omega_2, columns = omega_1):
//   Ft  [n][n]  F transposed: Ft[c][r] = F[r][c], F = DFT2(f)
//   Wt  [chunk planes][n][n]  first-pass lines (transposed), W [chunk planes][n][n] second-pass rows
//   At  [n][n]  the adjoint's accumulator, transposed (At[c][r] = A[r][c])
#pragma once
#include "ffst_fft.cuh"
#include "ffst_internal.h"

namespace ffst {

// The generic path's tables and workspace (device pointers) -- a part of KParams-like state.
struct GenParams {
  int n, M, eta_l, batch;
  const PlaneDev* planes;      // [eta_l]
  const void* rtab;            // radial table (rows j < j0: psi1, row j0: varphi; smooth rows after)
  int j0, variant;
  const void* usr;             // user spectra: [eta_l][n][n] T natural order, else nullptr
  const void* chirp;           // cpx<T>[n]: conj(w_m) = exp(-i pi m^2 / n)
  const void* bhat;            // cpx<T>[M]: FFT_M(b)
  const void* twm;             // cpx<T>[M]: exp(-2 pi i m / M)
};

// natural bin -> centred frequency, Omega = {-floor(n/2) .. ceil(n/2)-1}
__device__ __forceinline__ int centred_any(int bin, int n) { return bin < ((n + 1) >> 1) ? bin : bin - n; }

template <typename T>
__device__ __forceinline__ T gen_window(const GenParams& g, const PlaneDev& P, int lp, int c, int r) {
  if (g.usr) return static_cast<const T*>(g.usr)[((size_t)lp * g.n + r) * g.n + c];
  Radial<T> R{static_cast<const T*>(g.rtab), g.n / 2 + 1, g.j0};
  if (g.variant == 1) R.smooth = static_cast<const T*>(g.rtab) + (size_t)(g.j0 + 1) * (g.n / 2 + 1);
  return window<T>(P, centred_any(c, g.n), centred_any(r, g.n), R);
}

// One Bluestein DFT of a line held in registers by the TH = M/E threads of a line group:
// in: x[t + q*TH] for indices < L (zero above); out: X[t + q*TH] for indices < L.
// INVDFT: sign +.  Unnormalised.
template <typename T, int M>
struct Bluestein {
  // M >= 256: twiddles from a two-level shared table (as the power-of-two kernels, ffst_kernels.cuh)
  static constexpr bool TW2 = M >= 256;
  using LF = LineFFT<T, M, false, M, TW2, 16, TW2>;
  using LI = LineFFT<T, M, true, M, TW2, 16, TW2>;
  static constexpr int E = LF::E, TH = M / E;
  static __device__ __forceinline__ cpx<T>* tw2tab() {
    __shared__ cpx<T> tab[TW2 ? M / 64 + 64 : 1];
    return tab;
  }
  static __device__ __forceinline__ void tw2_fill(const GenParams& g) {
    if constexpr (TW2) {
      const cpx<T>* tw = static_cast<const cpx<T>*>(g.twm);
      for (int i = threadIdx.x; i < M / 64 + 64; i += blockDim.x) tw2tab()[i] = i < M / 64 ? tw[64 * i] : tw[i - M / 64];
      __syncthreads();
    }
  }
  template <bool INVDFT>
  static __device__ __forceinline__ void run(cpx<T> (&r)[E], int L, cpx<T>* scr, int t, const GenParams& g) {
    const cpx<T>* ch = static_cast<const cpx<T>*>(g.chirp);
    const cpx<T>* bh = static_cast<const cpx<T>*>(g.bhat);
    const cpx<T>* tw = TW2 ? tw2tab() : static_cast<const cpx<T>*>(g.twm);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int m = t + q * TH;
      cpx<T> v = r[q];
      if (INVDFT) v.y = -v.y;
      r[q] = m < L ? cmul<T>(v, __ldg(ch + m)) : czero<T>();
    }
    LF::run(r, scr, t, tw);
#pragma unroll
    for (int q = 0; q < E; ++q) r[q] = cmul<T>(r[q], __ldg(bh + t + q * TH));
    SyncOf<TH>::sync();
    LI::run(r, scr, t, tw);
    const T s = T(1) / T(M);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int k = t + q * TH;
      cpx<T> v = k < L ? cscale<T>(cmul<T>(r[q], __ldg(ch + (k < L ? k : 0))), s) : czero<T>();
      if (INVDFT) v.y = -v.y;
      r[q] = v;
    }
    SyncOf<TH>::sync();
  }
};

enum { GEN_SPEC = 0, GEN_PLAIN = 1, GEN_FWD_COL = 2, GEN_INV_COL = 3, GEN_FINAL = 4 };

// Row passes.  grid (ceil(lines / LPB), count): blockIdx.y = matrix (image, or image x chunk
// plane), each line group one row of n.
//   GEN_SPEC     real image rows -> DFT -> dst (complex)
//   GEN_PLAIN    complex rows -> DFT (INVDFT: IDFT * scale) -> dst
//   GEN_FWD_COL  row c of Ft[b] times psi_p(c, r) -> IDFT -> Wt[b, p] row c       (blockIdx.y = b * np + p)
//   GEN_INV_COL  sum over the chunk planes of psi_p(c, r) * DFT(Wt[b, p] row c) -> At[b] row c (+=)
//   GEN_FINAL    complex rows -> IDFT * scale -> real part -> dst (real)
// cube_side: 0 plain matrix indexing mat; 1 / 2: the src / dst is the coefficient cube, matrix
// mat = b * np + p maps to cube plane (b * cube_eta + p0 + p).
template <typename T, int M, int MODE, bool INVDFT>
__global__ void __launch_bounds__(256) gen_rows_kernel(GenParams g, const void* src, void* dst, int np, int p0,
                                                       int first, T scale, int cube_side, int cube_eta) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using B = Bluestein<T, M>;
  using C = cpx<T>;
  constexpr int TH = B::TH, E = B::E;
  constexpr int LPB = TH >= 256 ? 1 : 256 / TH;
  const int n = g.n;
  const int line = threadIdx.x / TH, t = threadIdx.x % TH;
  const int row = blockIdx.x * LPB + line;
  const bool act = row < n;
  const int rr = act ? row : 0;
  C* scr = reinterpret_cast<C*>(smem_raw) + line * Pad<T>::len(M);
  const size_t nn = (size_t)n * n;
  B::tw2_fill(g);
  C r[E];
  if constexpr (MODE == GEN_INV_COL) {
    const int b = blockIdx.y;
    C acc[E];
#pragma unroll
    for (int q = 0; q < E; ++q) acc[q] = czero<T>();
#pragma unroll 1
    for (int p = 0; p < np; ++p) {
      const C* s = static_cast<const C*>(src) + ((size_t)b * np + p) * nn + (size_t)rr * n;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int m = t + q * TH;
        r[q] = m < n ? s[m] : czero<T>();
      }
      B::template run<false>(r, n, scr, t, g);
      const int lp = p0 + p;
      const PlaneDev P = g.planes[lp];
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int k = t + q * TH;
        if (act && k < n) {
          const T w = gen_window<T>(g, P, lp, rr, k);     // row rr of At = column rr of A: c = rr, r = k
          acc[q].x += w * r[q].x;
          acc[q].y += w * r[q].y;
        }
      }
    }
    if (act) {
      C* d = static_cast<C*>(dst) + (size_t)b * nn + (size_t)rr * n;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int k = t + q * TH;
        if (k < n) d[k] = first ? acc[q] : cadd<T>(d[k], acc[q]);
      }
    }
    return;
  } else {
    const int mat = blockIdx.y;
    const int cmat = cube_eta > 0 ? (mat / np) * cube_eta + p0 + mat % np : mat;
    const int smat = cube_side == 1 ? cmat : mat, dmat = cube_side == 2 ? cmat : mat;
    if constexpr (MODE == GEN_SPEC) {
      const T* s = static_cast<const T*>(src) + (size_t)mat * nn + (size_t)rr * n;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int m = t + q * TH;
        r[q] = mk<T>(m < n ? s[m] : T(0), T(0));
      }
    } else if constexpr (MODE == GEN_FWD_COL) {
      const int b = mat / np, p = mat % np, lp = p0 + p;
      const PlaneDev P = g.planes[lp];
      const C* s = static_cast<const C*>(src) + (size_t)b * nn + (size_t)rr * n;   // row rr of Ft = column rr of F
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int m = t + q * TH;
        C v = czero<T>();
        if (act && m < n) {
          const T w = gen_window<T>(g, P, lp, rr, m);
          if (w != T(0)) v = cscale<T>(s[m], w);
        }
        r[q] = v;
      }
    } else {
      const C* s = static_cast<const C*>(src) + (size_t)smat * nn + (size_t)rr * n;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int m = t + q * TH;
        r[q] = m < n ? s[m] : czero<T>();
      }
    }
    B::template run<INVDFT>(r, n, scr, t, g);
    if (!act) return;
    if constexpr (MODE == GEN_FINAL) {
      T* d = static_cast<T*>(dst) + (size_t)dmat * nn + (size_t)rr * n;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int k = t + q * TH;
        if (k < n) d[k] = r[q].x * scale;
      }
    } else {
      C* d = static_cast<C*>(dst) + (size_t)dmat * nn + (size_t)rr * n;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int k = t + q * TH;
        if (k < n) d[k] = cscale<T>(r[q], scale);
      }
    }
  }
}

// Batched transpose of n x n complex matrices: dst[m][c][r] = src[m][r][c]; 32 x 32 tiles,
// grid (ceil(n/32), ceil(n/32), matrices), 32 x 8 threads.
template <typename T>
__global__ void __launch_bounds__(256) gen_transpose_kernel(const cpx<T>* src, cpx<T>* dst, int n) {
  __shared__ cpx<T> tile[32][33];
  const size_t off = (size_t)blockIdx.z * n * n;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int r = r0 + ty + k, c = c0 + tx;
    if (r < n && c < n) tile[ty + k][tx] = src[off + (size_t)r * n + c];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int c = c0 + ty + k, r = r0 + tx;
    if (r < n && c < n) dst[off + (size_t)c * n + r] = tile[tx][ty + k];
  }
}

// Spectra export of the generic path (tests / diagnostics): psi[i][row][col], natural or centred.
template <typename T>
__global__ void gen_spectra_kernel(GenParams g, T* psi, int centred_layout) {
  const int n = g.n;
  const size_t total = (size_t)g.eta_l * n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / ((size_t)n * n));
    const int rem = (int)(e - (size_t)i * n * n);
    int row = rem / n, col = rem - row * n;
    if (centred_layout) {                      // omega = 0 at (floor(n/2), floor(n/2)) (fftshift)
      row = (row - n / 2 + n) % n;
      col = (col - n / 2 + n) % n;
    }
    psi[e] = gen_window<T>(g, g.planes[i], i, col, row);
  }
}

// User spectra (any layout, any symmetry) -> the plan's natural-order table of the local planes.
template <typename T>
__global__ void gen_user_copy_kernel(const T* psi, T* out, int n, const int* gidx, int eta_l, int centred_layout) {
  const size_t total = (size_t)eta_l * n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(e / ((size_t)n * n));
    const int rem = (int)(e - (size_t)l * n * n);
    int r = rem / n, c = rem - r * n;
    if (centred_layout) { r = (r + n / 2) % n; c = (c + n / 2) % n; }
    out[e] = psi[((size_t)gidx[l] * n + r) * n + c];
  }
}

// Admission numbers of a generic-path system over the caller's eta planes: max |sum_i psi_i^2 - 1|
// and the point asymmetry max |psi_i(u) - psi_i(-u)| off the Nyquist lines
// (informational here: the full complex path needs no symmetry).  stats: bit patterns of doubles.
template <typename T>
__global__ void gen_user_stats_kernel(const T* psi, int n, int eta, int centred_layout, unsigned long long* stats) {
  const size_t nn = (size_t)n * n;
  double tight = 0.0, asym = 0.0;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < nn; e += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), c = (int)(e % n);
    // natural bins of this storage position, and of its mirror -u
    // (centred storage index s holds frequency s - floor(n/2), i.e. natural bin (s - n/2) mod n)
    const int rn = centred_layout ? (r - n / 2 + n) % n : r, cn = centred_layout ? (c - n / 2 + n) % n : c;
    const int rm = (n - rn) % n, cm = (n - cn) % n;
    const int rs = centred_layout ? (rm + n / 2) % n : rm, cs = centred_layout ? (cm + n / 2) % n : cm;
    const bool nyq = (n % 2 == 0) && (rn == n / 2 || cn == n / 2);
    double s = 0.0;
    for (int i = 0; i < eta; ++i) {
      const double v = (double)psi[(size_t)i * nn + e];
      s += v * v;
      if (!nyq) asym = fmax(asym, fabs(v - (double)psi[(size_t)i * nn + (size_t)rs * n + cs]));
    }
    tight = fmax(tight, fabs(s - 1.0));
  }
  atomicMax(stats, (unsigned long long)__double_as_longlong(tight));
  atomicMax(stats + 1, (unsigned long long)__double_as_longlong(asym));
}

}  // namespace ffst
