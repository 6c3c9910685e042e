// ffst_gen_launch.cuh — host launchers of the arbitrary-n path (ffst_generic.cuh): runtime M ->
// compile-time Bluestein length dispatch.
#pragma once
#include "ffst_generic.cuh"

namespace ffst {

template <typename T, int M, int MODE, bool INV>
static cudaError_t gen_rows_M(const GenParams& g, const void* src, void* dst, int np, int p0, int first, T scale,
                              int cube_side, int cube_eta, int mats, cudaStream_t s) {
  using B = Bluestein<T, M>;
  constexpr int LPB = B::TH >= 256 ? 1 : 256 / B::TH;
  const size_t smem = (size_t)LPB * Pad<T>::len(M) * sizeof(cpx<T>);
  auto k = gen_rows_kernel<T, M, MODE, INV>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<dim3((g.n + LPB - 1) / LPB, mats), LPB * B::TH, smem, s>>>(g, src, dst, np, p0, first, scale, cube_side,
                                                                 cube_eta);
  return cudaGetLastError();
}

template <typename T, int MODE, bool INV>
static cudaError_t gen_rows_any(const GenParams& g, const void* src, void* dst, int np, int p0, int first, T scale,
                                int cube_side, int cube_eta, int mats, cudaStream_t s) {
#define FFST_GM(MM) \
  case MM: return gen_rows_M<T, MM, MODE, INV>(g, src, dst, np, p0, first, scale, cube_side, cube_eta, mats, s);
  switch (g.M) {
    FFST_GM(16) FFST_GM(32) FFST_GM(64) FFST_GM(128) FFST_GM(256) FFST_GM(512) FFST_GM(1024) FFST_GM(2048)
    FFST_GM(4096)
    default: return cudaErrorInvalidValue;
  }
#undef FFST_GM
}

template <typename T>
cudaError_t launch_gen_rows_impl(int op, const GenParams& g, const void* src, void* dst, int np, int p0, int first,
                                 double scale, int cube_side, int cube_eta, int mats, cudaStream_t s) {
  const T sc = (T)scale;
  switch (op) {
    case GEN_OP_SPEC: return gen_rows_any<T, GEN_SPEC, false>(g, src, dst, np, p0, first, sc, cube_side, cube_eta, mats, s);
    case GEN_OP_DFT: return gen_rows_any<T, GEN_PLAIN, false>(g, src, dst, np, p0, first, sc, cube_side, cube_eta, mats, s);
    case GEN_OP_IDFT: return gen_rows_any<T, GEN_PLAIN, true>(g, src, dst, np, p0, first, sc, cube_side, cube_eta, mats, s);
    case GEN_OP_FWD_COL: return gen_rows_any<T, GEN_FWD_COL, true>(g, src, dst, np, p0, first, sc, cube_side, cube_eta, mats, s);
    case GEN_OP_INV_COL: return gen_rows_any<T, GEN_INV_COL, false>(g, src, dst, np, p0, first, sc, cube_side, cube_eta, mats, s);
    case GEN_OP_FINAL: return gen_rows_any<T, GEN_FINAL, true>(g, src, dst, np, p0, first, sc, cube_side, cube_eta, mats, s);
    default: return cudaErrorInvalidValue;
  }
}

#define FFST_GEN_INSTANTIATE(T)                                                                                 \
  template <> cudaError_t launch_gen_rows<T>(int op, const GenParams& g, const void* src, void* dst, int np,    \
                                             int p0, int first, double scale, int cube_side, int cube_eta,     \
                                             int mats, cudaStream_t s) {                                       \
    return launch_gen_rows_impl<T>(op, g, src, dst, np, p0, first, scale, cube_side, cube_eta, mats, s);       \
  }                                                                                                            \
  template <> cudaError_t launch_gen_transpose<T>(const void* src, void* dst, int n, int mats, cudaStream_t s) { \
    gen_transpose_kernel<T><<<dim3((n + 31) / 32, (n + 31) / 32, mats), 256, 0, s>>>(                          \
        static_cast<const cpx<T>*>(src), static_cast<cpx<T>*>(dst), n);                                        \
    return cudaGetLastError();                                                                                 \
  }                                                                                                            \
  template <> cudaError_t launch_gen_spectra<T>(const GenParams& g, void* psi, int centred, cudaStream_t s) {   \
    gen_spectra_kernel<T><<<148 * 8, 256, 0, s>>>(g, static_cast<T*>(psi), centred);                           \
    return cudaGetLastError();                                                                                 \
  }                                                                                                            \
  template <> cudaError_t launch_gen_user<T>(const void* psi, void* out, int n, const int* gidx, int eta_l,     \
                                             int eta, int centred, unsigned long long* stats, cudaStream_t s) { \
    if (out != nullptr) {                                                                                      \
      gen_user_copy_kernel<T><<<148 * 8, 256, 0, s>>>(static_cast<const T*>(psi), static_cast<T*>(out), n,      \
                                                      gidx, eta_l, centred);                                   \
      cudaError_t e = cudaGetLastError();                                                                      \
      if (e != cudaSuccess) return e;                                                                          \
    }                                                                                                          \
    gen_user_stats_kernel<T><<<148 * 4, 256, 0, s>>>(static_cast<const T*>(psi), n, eta, centred, stats);      \
    return cudaGetLastError();                                                                                 \
  }

}  // namespace ffst
