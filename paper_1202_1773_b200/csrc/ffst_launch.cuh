// ffst_launch.cuh — host launchers: runtime n -> compile-time N dispatch.
#pragma once
#include <algorithm>
#include "ffst_tiny.cuh"
#include "ffst_user.cuh"

namespace ffst {

constexpr int NYQ_GROUPS_MAX = 64;   // stage-1 CTAs per (direction, image) of the Nyquist correction

template <typename T> struct MaxN;
template <> struct MaxN<float> { static constexpr int v = 4096; };
template <> struct MaxN<double> { static constexpr int v = 2048; };

// Opt in to the dynamic shared memory a kernel needs (always: static + dynamic may exceed
// the 48 KB default even when the dynamic part alone does not).
template <typename K>
static cudaError_t set_smem(K kernel, size_t bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

#define FFST_CHECK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

template <typename T, int N> struct Launch {
  using G = Geo<T, N>;
  static Geometry geometry() {
    Geometry g{};
    g.nt = G::NT; g.gc = G::GC; g.rp2 = G::RP2; g.rpi = G::RPI; g.gr = G::GR; g.lpc = G::LPC; g.igc = G::IGC;
    g.smem_fwd = G::SMEM_FWD; g.smem_inv = G::SMEM_INV; g.smem_aux = G::SMEM_AUX;
    g.colpad = G::GC; g.ncpf = G::NCPF; g.tparts = G::TPARTS;
    return g;
  }
  static cudaError_t spectrum(const KParams& p, int batch, cudaStream_t s) {
    FFST_CHECK(set_smem(spec_rows_kernel<T, N>, G::SMEM_INV));
    spec_rows_kernel<T, N><<<dim3(N / G::RPS, batch), G::NT, G::SMEM_INV, s>>>(p);
    FFST_CHECK(cudaGetLastError());
    FFST_CHECK(set_smem(spec_cols_kernel<T, N>, G::SMEM_AUX));
    spec_cols_kernel<T, N><<<dim3((N / 2 + 1 + G::LPC - 1) / G::LPC, batch), G::NT, G::SMEM_AUX, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t nyq_fwd(const KParams& p, int batch, cudaStream_t s) {
    FFST_CHECK(set_smem(nyq_fwd_kernel<T, N>, G::SMEM_NYQ));
    nyq_fwd_kernel<T, N><<<dim3((p.n_nyq + G::LPC - 1) / G::LPC, 2, batch), G::NT, G::SMEM_NYQ, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t fwd_main(const KParams& p, int grid, cudaStream_t s) {
    FFST_CHECK(set_smem(fwd_main_kernel<T, N>, G::SMEM_FWD));
    fwd_main_kernel<T, N><<<grid, G::NT, G::SMEM_FWD, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t inv_main(const KParams& p, int grid, cudaStream_t s) {
    FFST_CHECK(set_smem(inv_main_kernel<T, N>, G::SMEM_INV));
    inv_main_kernel<T, N><<<grid, G::NT, G::SMEM_INV, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t nyq_inv(const KParams& p, int batch, cudaStream_t s) {
    const int rounds = (p.n_nyq + G::LPC - 1) / G::LPC;
    const int groups = rounds < NYQ_GROUPS_MAX ? rounds : NYQ_GROUPS_MAX;
    FFST_CHECK(set_smem(nyq_inv_kernel<T, N>, G::SMEM_NYQ));
    nyq_inv_kernel<T, N><<<dim3(2, batch, groups), G::NT, G::SMEM_NYQ, s>>>(p);
    FFST_CHECK(cudaGetLastError());
    // stage 2: one line per CTA (THC threads; at least a warp)
    const int nt = G::THC < 32 ? 32 : G::THC;
    const size_t sm = (size_t)(nt / G::THC) * G::SMC * sizeof(cpx<T>);
    FFST_CHECK(set_smem(nyq_fin_kernel<T, N>, sm));
    nyq_fin_kernel<T, N><<<dim3(2, batch), nt, sm, s>>>(p, groups);
    return cudaGetLastError();
  }
  // final pass, split so the Nyquist correction can run beside the column pass (it is only
  // needed by the row pass): which = 0 column pass, 1 row pass
  static cudaError_t nyq_compact_sums(const KParams& p, int batch, cudaStream_t s) {
    nyq_compact_sums_kernel<T, N><<<dim3(p.n_nyq, batch), 256, 0, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t final_(const KParams& p, int batch, int which, cudaStream_t s) {
    if (which == 0) {
      FFST_CHECK(set_smem(fin_cols_kernel<T, N>, G::SMEM_FWD));
      // columns per CTA: GC, halved while the grid would not cover the SMs (config 1: one CTA
      // walked all 33 columns x 16 accumulator lanes, 66 us)
      int cpb = G::GC;
      while (cpb > 1 && ((N / 2 + cpb) / cpb) * batch < 148) cpb = (cpb + 1) / 2;
      fin_cols_kernel<T, N><<<dim3((N / 2 + cpb) / cpb, batch), G::NT, G::SMEM_FWD, s>>>(p, cpb);
      return cudaGetLastError();
    }
    FFST_CHECK(set_smem(fin_rows_kernel<T, N>, G::SMEM_FWD));
    fin_rows_kernel<T, N><<<dim3((N + G::RPF - 1) / G::RPF, batch), G::NT, G::SMEM_FWD, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t spectra(const KParams& p, void* psi, int centred, cudaStream_t s) {
    const size_t total = (size_t)p.eta_l * N * N;
    int grid = (int)((total + 255) / 256);
    if (grid > 148 * 32) grid = 148 * 32;
    if (grid < 1) grid = 1;
    spectra_kernel<T, N><<<grid, 256, 0, s>>>(p, static_cast<T*>(psi), centred);
    return cudaGetLastError();
  }
  // fused small-n path (n <= 64): which = 0 forward, 1 inverse (two launches)
  static cudaError_t tiny(const KParams& p, int batch, int which, cudaStream_t s) {
    if constexpr (N <= 64) {
      using TY = Tiny<T, N>;
      if (which == 0) {
        FFST_CHECK(set_smem(tiny_fwd_kernel<T, N>, TY::SMEM));
        tiny_fwd_kernel<T, N><<<dim3(p.eta_l, batch), TY::NT, TY::SMEM, s>>>(p);
        return cudaGetLastError();
      }
      FFST_CHECK(set_smem(tiny_inv_kernel<T, N>, TY::SMEM));
      tiny_inv_kernel<T, N><<<dim3(p.eta_l, batch), TY::NT, TY::SMEM, s>>>(p);
      FFST_CHECK(cudaGetLastError());
      tiny_sum_kernel<T, N><<<dim3((N * N + 255) / 256, batch), 256, 0, s>>>(p);
      return cudaGetLastError();
    } else {
      return cudaErrorInvalidValue;
    }
  }
  static int max_active(int which) {
    int nb = 0;
    if (which == 0) {
      if (set_smem(fwd_main_kernel<T, N>, G::SMEM_FWD) != cudaSuccess) return 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fwd_main_kernel<T, N>, G::NT, G::SMEM_FWD);
    } else {
      if (set_smem(inv_main_kernel<T, N>, G::SMEM_INV) != cudaSuccess) return 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, inv_main_kernel<T, N>, G::NT, G::SMEM_INV);
    }
    return nb;
  }
};

#define FFST_DISPATCH(T, n, CALL, FAIL)                                  \
  switch (n) {                                                           \
    case 4: return Launch<T, 4>::CALL;                                   \
    case 8: return Launch<T, 8>::CALL;                                   \
    case 16: return Launch<T, 16>::CALL;                                 \
    case 32: return Launch<T, 32>::CALL;                                 \
    case 64: return Launch<T, 64>::CALL;                                 \
    case 128: return Launch<T, 128>::CALL;                               \
    case 256: return Launch<T, 256>::CALL;                               \
    case 512: return Launch<T, 512>::CALL;                               \
    case 1024: return Launch<T, 1024>::CALL;                             \
    case 2048: return Launch<T, 2048>::CALL;                             \
    case 4096: if constexpr (MaxN<T>::v >= 4096) return Launch<T, (MaxN<T>::v >= 4096 ? 4096 : 2048)>::CALL; \
      else return FAIL;                                                  \
    default: return FAIL;                                                \
  }

#define FFST_INSTANTIATE(T)                                                                                    \
  template <> Geometry geometry<T>(int n) { FFST_DISPATCH(T, n, geometry(), Geometry{}) }                      \
  template <> cudaError_t launch_spectrum<T>(const KParams& p, int b, cudaStream_t s) {                        \
    FFST_DISPATCH(T, p.n, spectrum(p, b, s), cudaErrorInvalidValue) }                                          \
  template <> cudaError_t launch_nyq_fwd<T>(const KParams& p, int b, cudaStream_t s) {                         \
    FFST_DISPATCH(T, p.n, nyq_fwd(p, b, s), cudaErrorInvalidValue) }                                           \
  template <> cudaError_t launch_fwd_main<T>(const KParams& p, int g, cudaStream_t s) {                        \
    FFST_DISPATCH(T, p.n, fwd_main(p, g, s), cudaErrorInvalidValue) }                                          \
  template <> cudaError_t launch_inv_main<T>(const KParams& p, int g, cudaStream_t s) {                        \
    FFST_DISPATCH(T, p.n, inv_main(p, g, s), cudaErrorInvalidValue) }                                          \
  template <> cudaError_t launch_nyq_compact_sums<T>(const KParams& p, int b, cudaStream_t s) {                \
    FFST_DISPATCH(T, p.n, nyq_compact_sums(p, b, s), cudaErrorInvalidValue) }                                  \
  template <> cudaError_t launch_nyq_inv<T>(const KParams& p, int b, cudaStream_t s) {                         \
    FFST_DISPATCH(T, p.n, nyq_inv(p, b, s), cudaErrorInvalidValue) }                                           \
  template <> cudaError_t launch_final<T>(const KParams& p, int b, int which, cudaStream_t s) {                \
    FFST_DISPATCH(T, p.n, final_(p, b, which, s), cudaErrorInvalidValue) }                                            \
  template <> cudaError_t launch_spectra_export<T>(const KParams& p, void* psi, int c, cudaStream_t s) {       \
    FFST_DISPATCH(T, p.n, spectra(p, psi, c, s), cudaErrorInvalidValue) }                                      \
  template <> cudaError_t launch_tiny<T>(const KParams& p, int b, int which, cudaStream_t s) {                 \
    FFST_DISPATCH(T, p.n, tiny(p, b, which, s), cudaErrorInvalidValue) }                                       \
  template <> cudaError_t launch_expand_compact<T>(const KParams& p, const void* re, const void* gh, void* out,  \
                                                   int batch, cudaStream_t s) {                                 \
    const long long pairs = (long long)batch * p.eta_l * p.n * p.n / 2;                                       \
    const int grid = (int)std::min<long long>((pairs + 255) / 256, 148LL * 16);                                \
    expand_compact_kernel<T><<<grid < 1 ? 1 : grid, 256, 0, s>>>(p.planes, p.n, p.eta_l, p.n_nyq,             \
        static_cast<const T*>(re), static_cast<const T*>(gh), static_cast<cpx<T>*>(out), pairs);              \
    return cudaGetLastError(); }                                                                               \
  template <> cudaError_t launch_user_prepare<T>(const UserPrep& u, int grid, cudaStream_t s) {              \
    return user_prepare_<T>(u, grid, s); }                                                                     \
  template <> int max_active_main<T>(int n, int device, int which) {                                           \
    (void)device; FFST_DISPATCH(T, n, max_active(which), 0) }

}  // namespace ffst
