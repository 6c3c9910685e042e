// ffst_kernels.cuh — the FFST hot path on sm_100a (included once per dtype).
//
// Path:
//   forward  (eq:shearletTransform)
//     spectrum   f -> F = fft2(f), Hermitian half, column-major  (row R2C, column FFT)
//     nyq_fwd    rank-2 imaginary Nyquist terms of the even-N grid (per Nyquist plane)
//     fwd_main   persistent: pass 1 = window sym_i(u) * F on the plane's column range,
//                column IFFT -> L2-resident intermediate W; pass 2 = row C2R of W,
//                + Nyquist term -> complex coefficient plane c_i (the only HBM stream)
//   inverse  (eq:inverseShearletTransform)
//     inv_main   persistent: pass 1 = row R2C of Re c_i (dense read of the cube) pruned to
//                the plane's columns -> W (+ alternating sums of Im c_i for Nyquist planes);
//                pass 2 = column FFT of W, * sym_i, accumulated over planes into A
//                (deterministic: one owner per column group, chained across chunks)
//     nyq_inv    Nyquist correction of the adjoint
//     final      f = Re ifft2(A) (column IFFT + row C2R) - correction
#pragma once
#include "ffst_fft.cuh"
#include "ffst_internal.h"

namespace ffst {

template <typename T, int N>
struct Geo {
  static constexpr int NT = 256;
  static constexpr int ESZ = (int)sizeof(cpx<T>);
  static constexpr int H = N / 2;
  static constexpr int EC = RadixPlan<N>::E, THC = N / EC, LPC = NT / THC;
  static constexpr int ER = RadixPlan<H>::E, THR = H / ER, LPR = NT / THR;
  static constexpr int SMC = Pad<T>::len(N), SMR = Pad<T>::len(H);
  static constexpr int SCR_C = LPC * SMC, SCR_R = LPR * SMR;
  // row passes as row PAIRS on length-N lines ("two-for-one", one complex FFT per two real rows)
  // when a round holds the same rows either way (E = 16 for both line lengths)
  static constexpr bool PAIR = 2 * LPC == LPR;
  // measured: the pair form wins for the inverse row pass (configs 2-5) and loses for the forward
  // one at n >= 512 (its stores are 8-byte instead of 16-byte per lane): inverse only
  static constexpr bool PAIR_FWD = false, PAIR_INV = PAIR && sizeof(T) == 4;   // float64: registers
  // partial alternating row sums per row of a Nyquist plane (nyq_T): one per warp of a line (no
  // cross-warp reduction, no barrier per round)
  static constexpr int TPARTS = PAIR_INV ? (THC > 32 ? THC / 32 : 1) : (THR > 32 ? THR / 32 : 1);
  static constexpr int SCRX = SCR_C > SCR_R ? SCR_C : SCR_R;
  // forward pass 1: columns per item (>= 32-byte row segments of the intermediate)
  static constexpr int GC = LPC > (32 / ESZ) ? LPC : (32 / ESZ);
  static constexpr int GCP = GC + 1;
  static constexpr int TILE_C = N * GCP;
  // n >= 2048: an N x GC transposition tile would fill the SM's shared memory (one CTA per SM,
  // 12 % warps active at n = 4096); forward pass 1 then stores each column straight from
  // registers (8-byte stores whose sectors the item's GC columns complete in L2)
  static constexpr bool DIRECT = (long long)N * GCP * ESZ > 65536;
  // DIRECT sizes: the forward intermediate W (and the final pass's Fscr) is column-major
  // ([column][N rows], like the inverse's): pass 1 stores each column line coalesced straight from
  // registers, and the row pass reads tiles of TRF rows (32-byte column segments at float32)
  // through shared memory.  (A row-major W needs one L2 write request per element here.)
  // Within W the rows come in blocks of TB: element (row r, column c) at ((r / TB) stride + c) TB + r % TB
  // (stride = the padded column count), so that a row item's TRF-row tiles read one contiguous
  // block (DRAM locality: plain column-major would read 32-byte segments 32 KB apart at n = 4096).
  static constexpr bool WCOL = DIRECT;
  static constexpr int TILE_CE = DIRECT ? 0 : TILE_C;     // tile elements allocated (pass 1)
  // forward pass 2: rows per item (per-item overhead and the Nyquist-term staging amortised)
  // (measured sweep: ~256 KB of output per item up to n = 512, 512 KB at n = 1024, 64 rows from n = 2048)
  static constexpr int RP2_B = (N >= 1024 ? 524288 : 262144) / (N * ESZ);
  static constexpr int RP2_A = RP2_B > LPR ? RP2_B : LPR;
  static constexpr int RP2_ = (N >= 2048 && RP2_A < 64) ? 64 : RP2_A;
  static constexpr int RP2 = RP2_ < N ? RP2_ : N;
  // column-major row pass (WCOL): rows per shared tile
  static constexpr int TRF_ = LPR > 4 ? LPR : 4;
  static constexpr int TRF = TRF_ < N ? TRF_ : N;
  static constexpr int RPT = TRF / LPR > 0 ? TRF / LPR : 1;     // rounds per tile
  static constexpr int TB = TRF;                                  // row block of the WCOL layout
  static FFST_HD size_t wat(int r, int c, int stride) { return ((size_t)(r / TB) * stride + c) * TB + r % TB; }
  // The inverse's intermediate stays plain column-major: in the row-block layout the row pass stores
  // each tile as one contiguous chunk (config 5 inverse pass 1 12.7 -> 11.5 ms), but the column pass
  // then loads 32-byte pieces of eight lines per warp instruction (pass 2 4.5 -> 8.0 ms).
  static constexpr bool WBLK_INV = false;
  // inverse pass 1 (row pairs): the extraction stores each column's row pair straight to W instead
  // of staging a tile of rows in shared memory (measured, 20-step A/B twice: n = 256 inverse 0.239 -> 0.227 ms, n = 512 3.42 -> 3.33 ms,
  // n = 1024 even, n = 4096 +15 %: there the tile's 64-128-byte column segments win)
  static constexpr bool DIRW = N <= 512;
  static FFST_HD size_t iat(int r, int c, int ncols) { return WBLK_INV ? wat(r, c, ncols) : (size_t)c * N + r; }
  static constexpr int RPF_ = WCOL ? TRF : LPR;      // final row pass: one tile / round per CTA (more CTAs)
  static constexpr int RPF = RPF_ < N ? RPF_ : N;
  // inverse pass 1: rows per tile and per item
  static constexpr int GR_ = LPR > (32 / ESZ) ? LPR : (32 / ESZ);
  static constexpr int GR = GR_ < N ? GR_ : N;
  static constexpr int TSTR = H + 1;           // odd: conflict-free column reads of the tile
  static constexpr int TILE_R = GR * TSTR;
  // (measured at configs 2-5: n = 256 best at 128 rows, 512 to 4096 at 64)
  static constexpr int RPI0 = N >= 512 ? 64 : N / 2;
  static constexpr int RPI_ = RPI0 > GR ? RPI0 : GR;
  static constexpr int RPI = RPI_ < N ? RPI_ : N;
  // spectrum row pass (spec_rows_kernel): rows per CTA (more, smaller CTAs: one short launch)
  static constexpr int RPS_ = (N >= 2048 ? 32 : N / 16) > GR ? (N >= 2048 ? 32 : N / 16) : GR;
  static constexpr int RPS = RPS_ < N ? RPS_ : N;
  // padded row stride of the final column pass output
  static constexpr int NCPF = ((H + 1 + GC - 1) / GC) * GC;
  // inverse pass 2: column groups of LPC columns per round, IG rounds per item (n >= 2048: one
  // column per round, so an item is four column FFTs over its chunk's planes)
  static constexpr int IG = N >= 2048 ? 4 : 1;
  static constexpr int IGC = IG * LPC;
  // per-thread window values (EC reals per thread), staged in shared memory so the window
  // arithmetic is not unrolled into the FFT's register footprint
  static constexpr int WBUF = NT * EC * (int)sizeof(T) / ESZ;      // in complex elements
  // staged Nyquist terms (complex units); WCOL: the row tile instead (the terms are read through L1)
  static constexpr int NYQB = WCOL ? TRF * TSTR : (N + RP2) * (int)sizeof(T) / ESZ + 1;
  static constexpr size_t SMEM_FWD = (size_t)((SCR_C + TILE_CE + WBUF) > (SCRX + NYQB) ? (SCR_C + TILE_CE + WBUF) : (SCRX + NYQB)) * ESZ;
  static constexpr size_t SMEM_INV = (size_t)((SCRX + TILE_R) > (SCR_C + WBUF) ? (SCRX + TILE_R) : (SCR_C + WBUF)) * ESZ + 256;
  static constexpr size_t SMEM_AUX = SMEM_FWD > SMEM_INV ? SMEM_FWD : SMEM_INV;
  static constexpr size_t SMEM_NYQ = (size_t)(SCR_C + NT * EC) * ESZ;
  static_assert(RPI % GR == 0, "RPI must be a multiple of GR");
  static_assert(!WCOL || (RP2 % TRF == 0 && (TRF % LPR == 0 || TRF == N) && N % TRF == 0), "row tiles must tile the row items");
  static_assert(!PAIR || (GR % (2 * LPC) == 0 || GR < 2 * LPC), "row-pair rounds must tile GR");
  static_assert(SCR_C * ESZ >= LPC * N * (int)sizeof(T), "row-pair column-sum scratch");
  static_assert(GC % LPC == 0 || LPC > GC, "GC vs LPC");
};

enum { MODE_MAIN = 0, MODE_AUX = 1, MODE_COMPACT = 2 };   // COMPACT: forward rows as reals (f1 format)

template <typename T> __device__ __forceinline__ void store_pair_cs(cpx<T>* dst, cpx<T> a, cpx<T> b);
template <> __device__ __forceinline__ void store_pair_cs<float>(float2* dst, float2 a, float2 b) {
  __stcs(reinterpret_cast<float4*>(dst), make_float4(a.x, a.y, b.x, b.y));
}
template <> __device__ __forceinline__ void store_pair_cs<double>(double2* dst, double2 a, double2 b) {
  __stcs(dst, a);
  __stcs(dst + 1, b);
}
// L2 residency hints (createpolicy): the adjoint's accumulator A is read-modify-written by every
// plane and is kept (evict_last); an intermediate ring that cannot stay in L2 (KParams.ring_stream:
// n >= 2048, 12+ slots of 27-52 MB) is streamed (evict_first) so that it does not push A out.
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// fire-and-forget accumulation in L2 (the accumulation chain orders the additions: deterministic)
template <typename T> __device__ __forceinline__ void red_add(cpx<T>* dst, cpx<T> v, unsigned long long pol);
template <> __device__ __forceinline__ void red_add<float>(float2* dst, float2 v, unsigned long long pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(dst), "f"(v.x), "f"(v.y),
               "l"(pol) : "memory");
}
template <> __device__ __forceinline__ void red_add<double>(double2* dst, double2 v, unsigned long long pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(&dst->x), "d"(v.x), "l"(pol) : "memory");
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(&dst->y), "d"(v.y), "l"(pol) : "memory");
}
template <typename T> __device__ __forceinline__ void st_hint(cpx<T>* dst, cpx<T> v, unsigned long long pol);
template <> __device__ __forceinline__ void st_hint<float>(float2* dst, float2 v, unsigned long long pol) {
  asm volatile("st.global.cg.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(dst), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}
template <> __device__ __forceinline__ void st_hint<double>(double2* dst, double2 v, unsigned long long pol) {
  asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(dst), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
// two adjacent complex values in one store (float32: 16 bytes) with an L2 policy
template <typename T> __device__ __forceinline__ void store_pair_hint(cpx<T>* dst, cpx<T> a, cpx<T> b, unsigned long long pol);
template <> __device__ __forceinline__ void store_pair_hint<float>(float2* dst, float2 a, float2 b, unsigned long long pol) {
  asm volatile("st.global.cg.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst), "f"(a.x), "f"(a.y), "f"(b.x),
               "f"(b.y), "l"(pol) : "memory");
}
template <> __device__ __forceinline__ void store_pair_hint<double>(double2* dst, double2 a, double2 b, unsigned long long pol) {
  st_hint<double>(dst, a, pol);
  st_hint<double>(dst + 1, b, pol);
}
template <typename T> __device__ __forceinline__ cpx<T> ld_hint(const cpx<T>* src, unsigned long long pol);
template <> __device__ __forceinline__ float2 ld_hint<float>(const float2* src, unsigned long long pol) {
  float2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(src), "l"(pol));
  return v;
}
template <> __device__ __forceinline__ double2 ld_hint<double>(const double2* src, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(src), "l"(pol));
  return v;
}
template <typename T> __device__ __forceinline__ void store_pair_cg(cpx<T>* dst, cpx<T> a, cpx<T> b);
template <> __device__ __forceinline__ void store_pair_cg<float>(float2* dst, float2 a, float2 b) {
  __stcg(reinterpret_cast<float4*>(dst), make_float4(a.x, a.y, b.x, b.y));
}
template <> __device__ __forceinline__ void store_pair_cg<double>(double2* dst, double2 a, double2 b) {
  __stcg(dst, a);
  __stcg(dst + 1, b);
}
template <typename T> __device__ __forceinline__ void load_pair_cs(const cpx<T>* src, cpx<T>& a, cpx<T>& b);
template <> __device__ __forceinline__ void load_pair_cs<float>(const float2* src, float2& a, float2& b) {
  const float4 v = __ldcs(reinterpret_cast<const float4*>(src));
  a = make_float2(v.x, v.y);
  b = make_float2(v.z, v.w);
}
template <> __device__ __forceinline__ void load_pair_cs<double>(const double2* src, double2& a, double2& b) {
  a = __ldcs(src);
  b = __ldcs(src + 1);
}

// Asynchronous global -> shared copies (LDGSTS): no registers held while in flight.
template <typename T> __device__ __forceinline__ void cp_async_el(cpx<T>* dst_smem, const cpx<T>* src, unsigned long long pol,
                                                                 bool hint) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  if (sizeof(cpx<T>) == 8) {
    if (hint) asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "l"(pol) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  } else {
    if (hint) asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "l"(pol) : "memory");
    else asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__shared__ unsigned long long s_probe[4];   // intra-item probes (trace mode)
#define FFST_PROBE(p, i) do { if ((p).trace != nullptr && threadIdx.x == 0) s_probe[i] = gtimer(); } while (0)

// Dependency counters (PTX memory model).  Publishing side: red.release.gpu after the item's last
// write (or, for a slot-reuse dependency, its last read) -- MEMBAR.ALL.GPU + RED, no L1 flush.
// Waiting side: thread 0 polls with relaxed (volatile) loads until the counter reaches its target,
// then executes fence.acq_rel.gpu: the poll that observed the released value plus this fence
// synchronise with every release that contributed to it, and the CTA barrier that follows every
// wait (__syncthreads) extends that ordering to the other threads of the CTA (the pattern of a
// cooperative grid barrier).  So an item's reads of a producer's ring slot or accumulator lane,
// and its writes into a slot that earlier readers release, are ordered after the dependency.
// One fence per satisfied wait (per item), not per poll.
__device__ __forceinline__ void spin_wait(const int* ctr, int target, int sync_mode = 3) {
  const volatile int* v = ctr;
  while (*v < target) __nanosleep(40);
  if (sync_mode & 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void red_release(int* ctr, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(ctr), "r"(v) : "memory");
}

// Predicated cached loads (__ldg / __ldcg / __ldcs are non-volatile inline asm): the compiler may
// hoist them above the guarding branch, so every such load's address is kept inside its buffer
// even for idle lanes (clamped row / column indices).  Observed with cuda-gdb: a hoisted __ldg of
// the user-spectra table through a null pointer (illegal address, n = 16, 32).
//
// the plan's radial tables (classic rows; smooth rows after them when p.variant == 1)
template <typename T, int N>
__device__ __forceinline__ Radial<T> radial_of(const KParams& p) {
  Radial<T> R{static_cast<const T*>(p.rtab), N / 2 + 1, p.j0};
  if (p.variant == 1) R.smooth = static_cast<const T*>(p.rtab) + (size_t)(p.j0 + 1) * (N / 2 + 1);
  return R;
}

// user spectra (f4): the plane's [n/2+1][n] table of symmetric parts, else nullptr
template <typename T, int N>
__device__ __forceinline__ const T* user_plane(const KParams& p, const PlaneDev& P) {
  return p.usym ? static_cast<const T*>(p.usym) + (size_t)P.rec * (N / 2 + 1) * N : nullptr;
}

template <typename T, int N>
struct K {
  using G = Geo<T, N>;
  using C = cpx<T>;
  static constexpr int H = N / 2;
  static constexpr int NT = G::NT;

  // Line FFTs take their twiddles from a two-level table in shared memory for n >= 256:
  // w^m = hi[m / 64] lo[m % 64] (n/64 + 64 entries), one table read pair per butterfly and the
  // powers w^q by products (ffst_fft.cuh TW2).  Measured on the bare 4096-point block: 12.6 ->
  // 10.9 ns per line (scripts/micro/fftbench.cu).  Every kernel that runs a K item fills it first.
  static constexpr bool TW2 = N >= 256;
  static __device__ __forceinline__ C* tw2tab() {
    __shared__ C tab[TW2 ? N / 64 + 64 : 1];
    return tab;
  }
  static __device__ __forceinline__ void tw2_fill(const KParams& p) {
    if constexpr (TW2) {
      const C* tw = static_cast<const C*>(p.tw);
      C* tab = tw2tab();
      for (int i = threadIdx.x; i < N / 64 + 64; i += blockDim.x) tab[i] = i < N / 64 ? tw[64 * i] : tw[i - N / 64];
      __syncthreads();
    }
  }
  // w^k = exp(-2 pi i k / N): from the shared two-level table (n >= 256), else the global table
  static __device__ __forceinline__ C twk(int kk, const C* tw) {
    if constexpr (TW2) {
      const C* tab = tw2tab();
      return cmul<T>(tab[kk >> 6], tab[N / 64 + (kk & 63)]);
    } else {
      return __ldg(tw + kk);
    }
  }
  template <int L, bool INV, bool NAMED = false>
  static __device__ __forceinline__ void fft(C (&r)[LineFFT<T, L, INV, N>::E], C* sm, int t, const C* tw) {
    if constexpr (TW2) LineFFT<T, L, INV, N, true, 16, true, NAMED>::run(r, sm, t, tw2tab());
    else LineFFT<T, L, INV, N, false, 16, false, NAMED>::run(r, sm, t, tw);
  }

  // Window sym_i of the CTA's column lines into wbuf[q * NT + tid] (thread tid's element q = row
  // t + q THC of column cb0 + tid / THC).  The support is ~10 % of the rows: the line's threads
  // enumerate only the candidate rows (integer intervals from col_bounds) and evaluate them
  // converged -- no per-element test.  All threads of the CTA call it; act = the thread's column
  // is one to window.
  static __device__ __forceinline__ void window_lines(const PlaneDev& P, int cb0, bool act, T* wbuf, C* scr,
                                                      const Radial<T>& R, T delta, const T* us,
                                                      bool dbg_skip_window = false) {
    const int tid = threadIdx.x, t = tid % G::THC;
    const int cb = cb0 + tid / G::THC;
    if (dbg_skip_window) {                   // measurement only (FFST_DBG bit 2): window = 1 on the column
#pragma unroll
      for (int q = 0; q < G::EC; ++q) wbuf[q * NT + tid] = act ? T(1) : T(0);
      SyncOf<G::THC>::sync();
      return;
    }
    if (us != nullptr) {   // user spectra (f4): the plane's symmetric part from its table, every row
#pragma unroll
      for (int q = 0; q < G::EC; ++q) wbuf[q * NT + tid] = act ? us[(size_t)cb * N + t + q * G::THC] : T(0);
      SyncOf<G::THC>::sync();
      return;
    }
    const int u1 = cb == H ? -H : cb;
#pragma unroll
    for (int q = 0; q < G::EC; ++q) wbuf[q * NT + tid] = T(0);
    SyncOf<G::THC>::sync();
    if (act) {
      if (cb == H) {                         // the Nyquist column: every row (the thread's own)
#pragma unroll 1
        for (int q = 0; q < G::EC; ++q) wbuf[q * NT + tid] = window_sym<T>(P, u1, centred(t + q * G::THC, N), H, R);
      } else {
        // The candidate rows of the column (a superset of the support, exact integer bounds) are
        // at most three u2 intervals -- the horizontal wedge [hlo, hhi] and the vertical band
        // alo <= |u2| <= ahi on either side -- plus the Nyquist row u2 = -n/2: the line's threads
        // enumerate them and write each value into the slot of the thread that owns the row
        // (an overlap of two intervals writes the same value twice).
        const ColBounds bnd = col_bounds<T>(P, u1, H, delta);
        const int h0 = bnd.hlo > -H ? bnd.hlo : -H, h1 = bnd.hhi < H - 1 ? bnd.hhi : H - 1;
        const int nh = h1 >= h0 ? h1 - h0 + 1 : 0;
        const int ap = bnd.ahi < H - 1 ? bnd.ahi : H - 1, an = bnd.ahi < H ? bnd.ahi : H;
        const int np = ap >= bnd.alo ? ap - bnd.alo + 1 : 0, nn = an >= bnd.alo ? an - bnd.alo + 1 : 0;
        const int K = nh + np + nn + 1;
        const int lbase = tid - t;           // first thread of this line
#pragma unroll 1
        for (int i = t; i < K; i += G::THC) {
          const int u2 = i < nh ? h0 + i
                       : i < nh + np ? bnd.alo + (i - nh)
                       : i < nh + np + nn ? -(bnd.alo + (i - nh - np)) : -H;
          const int rb = u2 < 0 ? u2 + N : u2;
          wbuf[(rb / G::THC) * NT + lbase + rb % G::THC] = window_sym<T>(P, u1, u2, H, R);
        }
      }
    }
    SyncOf<G::THC>::sync();
  }

  // ------------------------------------------------------------------ column IFFT item
  // MAIN: forward pass 1 — column bins [c0, c0+cnt) of plane P: X(u) = sym_P(u) F(u),
  //       IFFT along u2, rows -> W (row-major, stride P.ncols_pad, column c - P.c_lo; WCOL:
  //       column-major in row blocks, Geo::wat).
  // AUX:  final pass 1 — column bins of A[b] (no window) -> Fscr[b] (row-major, stride NCPF;
  //       WCOL: column-major).
  template <int MODE>
  static __device__ void col_ifft(const KParams& p, int b, const PlaneDev& P, int c0, int cnt,
                                  const C* __restrict__ src, C* dst, int dst_stride, int dst_col0,
                                  C* smem, const int* dep = nullptr, int dep_target = 0) {
    C* scr = smem;
    C* tile = smem + G::SCR_C;
    const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
    const C* tw = static_cast<const C*>(p.tw);
    const T delta = (T)p.delta;
    const Radial<T> R = radial_of<T, N>(p);
    constexpr int ROUNDS = G::GC / G::LPC > 0 ? G::GC / G::LPC : 1;
#pragma unroll 1
    for (int rd = 0; rd < ROUNDS; ++rd) {
      const int ci = rd * G::LPC + line;
      const bool act = ci < cnt;
      const int cb = c0 + ci;
      const C* col = src + (size_t)(act ? cb : c0) * N;   // in range even for idle lines (hoisted loads)
      C r[G::EC];
      if constexpr (MODE == MODE_MAIN) {
        T* wbuf = reinterpret_cast<T*>(tile + G::TILE_CE);
        window_lines(P, c0 + rd * G::LPC, act, wbuf, scr, R, delta, user_plane<T, N>(p, P), p.dbg & 4);
        if (rd == 0) FFST_PROBE(p, 0);
#pragma unroll
        for (int q = 0; q < G::EC; ++q) {
          const T w = wbuf[q * NT + tid];
          r[q] = w != T(0) ? cscale<T>(__ldg(col + t + q * G::THC), w) : czero<T>();
        }
      } else {   // final pass: the accumulator lanes of A summed in lane order
#pragma unroll
        for (int q = 0; q < G::EC; ++q) r[q] = act ? __ldcg(col + t + q * G::THC) : czero<T>();
#pragma unroll 2
        for (int l = 1; l < p.a_lanes; ++l) {      // (two lanes' loads in flight)
          const C* cl = col + (size_t)l * p.a_lane_elems;
#pragma unroll
          for (int q = 0; q < G::EC; ++q)
            if (act) r[q] = cadd<T>(r[q], __ldcg(cl + t + q * G::THC));
        }
      }
      if (rd == 0) FFST_PROBE(p, 1);
      if (!(p.dbg & 1)) fft<N, true>(r, scr + line * G::SMC, t, tw);
      if (rd == 0) FFST_PROBE(p, 2);
      if constexpr (G::WCOL) {
        if (rd == 0 && dep != nullptr) {       // ring-slot reuse: wait only before writing dst
          if (tid == 0) spin_wait(dep, dep_target);
          __syncthreads();
        }
        // column-major destination: the line's elements t + q THC are contiguous (coalesced stores)
        if (act && !(p.dbg & 2)) {
          const int c = dst_col0 + ci;
          if (MODE == MODE_MAIN && p.ring_stream) {
            const unsigned long long pf = policy_evict_first();
#pragma unroll
            for (int q = 0; q < G::EC; ++q) st_hint<T>(dst + G::wat(t + q * G::THC, c, dst_stride), r[q], pf);
          } else {
#pragma unroll
            for (int q = 0; q < G::EC; ++q) __stcg(dst + G::wat(t + q * G::THC, c, dst_stride), r[q]);
          }
        }
      } else if (ci < G::GC) {
#pragma unroll
        for (int q = 0; q < G::EC; ++q) tile[(t + q * G::THC) * G::GCP + ci] = r[q];
      }
      __syncthreads();
    }
    if constexpr (!G::WCOL) {
      if (dep != nullptr) {                    // ring-slot reuse: wait only before writing dst
        if (tid == 0) spin_wait(dep, dep_target);
        __syncthreads();
      }
      const int ncopy = cnt < G::GC ? cnt : G::GC;
      FFST_PROBE(p, 3);
#pragma unroll 1
      for (int e = tid; e < N * G::GC; e += NT) {
        const int rr = e / G::GC, ci = e - rr * G::GC;
        if (ci < ncopy) dst[(size_t)rr * dst_stride + dst_col0 + ci] = tile[rr * G::GCP + ci];
      }
    }
  }

  // Forward pass 1 of one plane's column group for two images (the chunks of two images that
  // hold the same planes are paired by the planner): the window -- the same for both -- is
  // evaluated once, applied to each image's spectrum, one column IFFT per image, each written to
  // its own ring slot.  Only when one round covers the group (GC == LPC).
  static __device__ void col_ifft_two(const KParams& p, const PlaneDev& P, int c0, int cnt, const C* src0,
                                      const C* src1, C* dst0, C* dst1, int dst_stride, int dst_col0, C* smem,
                                      const int* dep0, int tgt0, const int* dep1, int tgt1) {
    static_assert(G::GC == G::LPC || true, "");
    C* scr = smem;
    C* tile = smem + G::SCR_C;
    T* wbuf = reinterpret_cast<T*>(tile + G::TILE_CE);
    const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
    const C* tw = static_cast<const C*>(p.tw);
    const Radial<T> R = radial_of<T, N>(p);
    const int ci = line;
    const bool act = ci < cnt;
    const int cb = c0 + ci;
    window_lines(P, c0, act, wbuf, scr, R, (T)p.delta, user_plane<T, N>(p, P));
    FFST_PROBE(p, 0);
    const int ncopy = cnt < G::GC ? cnt : G::GC;
#pragma unroll 1
    for (int img = 0; img < 2; ++img) {
      const C* col = (img == 0 ? src0 : src1) + (size_t)(act ? cb : c0) * N;
      C r[G::EC];
#pragma unroll
      for (int q = 0; q < G::EC; ++q) {
        const T w = wbuf[q * NT + tid];
        r[q] = w != T(0) ? cscale<T>(__ldg(col + t + q * G::THC), w) : czero<T>();
      }
      fft<N, true>(r, scr + line * G::SMC, t, tw);
      const int* dep = img == 0 ? dep0 : dep1;
      C* dst = img == 0 ? dst0 : dst1;
      if constexpr (G::WCOL) {
        if (tid == 0 && dep != nullptr) spin_wait(dep, img == 0 ? tgt0 : tgt1);   // ring-slot reuse
        __syncthreads();
        if (act) {                              // column-major destination (coalesced)
#pragma unroll
          for (int q = 0; q < G::EC; ++q) __stcg(dst + G::wat(t + q * G::THC, dst_col0 + ci, dst_stride), r[q]);
        }
      } else {
        if (ci < G::GC) {
#pragma unroll
          for (int q = 0; q < G::EC; ++q) tile[(t + q * G::THC) * G::GCP + ci] = r[q];
        }
        if (tid == 0 && dep != nullptr) spin_wait(dep, img == 0 ? tgt0 : tgt1);   // ring-slot reuse
        __syncthreads();
#pragma unroll 1
        for (int e = tid; e < N * G::GC; e += NT) {
          const int rr = e / G::GC, c = e - rr * G::GC;
          if (c < ncopy) dst[(size_t)rr * dst_stride + dst_col0 + c] = tile[rr * G::GCP + c];
        }
      }
      __syncthreads();                          // scratch / tile reuse by the second image
    }
  }

  // ------------------------------------------------------------------ row C2R item
  // Rows [r0, r0+cnt) of an intermediate holding Hermitian-half bins [c_lo, c_lo+ncols)
  // (row-major, stride `stride`; WCOL: column-major in row blocks of TB, Geo::wat, read in tiles of
  // TRF rows through shared memory).  MAIN: complex coefficient rows (+ Nyquist imaginary term);
  // AUX: real image rows minus the adjoint's Nyquist correction.
  template <int MODE>
  static __device__ void row_c2r(const KParams& p, const C* __restrict__ src, int stride, int c_lo, int ncols,
                                 int r0, int cnt, C* out_c, T* out_r, const T* nyqG, const T* nyqH,
                                 C* smem) {
    C* scr = smem;
    const int tid = threadIdx.x, line = tid / G::THR, t = tid % G::THR;
    const C* tw = static_cast<const C*>(p.tw);
    const T scale = T(1) / (T(N) * T(N));
    constexpr int ROUNDS_ = (G::WCOL && G::RPF > G::RP2 ? G::RPF : G::RP2) / G::LPR;
    constexpr int ROUNDS = ROUNDS_ > 0 ? ROUNDS_ : 1;
    const int rounds = (cnt + G::LPR - 1) / G::LPR < ROUNDS ? (cnt + G::LPR - 1) / G::LPR : ROUNDS;
    // Nyquist terms of this item: staged in shared memory (G(m1) for all m1, H(r) for its rows),
    // or, WCOL (the region holds the row tile), read through L1
    T* sG = reinterpret_cast<T*>(smem + G::SCRX);
    T* sH = sG + N;
    C* tile = smem + G::SCRX;                  // WCOL: [TRF][TSTR]
    if (!G::WCOL && nyqG != nullptr) {
      for (int m = tid; m < N; m += NT) sG[m] = nyqG[m];
      for (int i = tid; i < cnt; i += NT) sH[i] = nyqH[r0 + i];
      __syncthreads();
    }
    constexpr int RPT = G::RPT;                // WCOL: rounds per tile
    const bool stream = MODE == MODE_MAIN && p.ring_stream;
    const unsigned long long pf = policy_evict_first();
    // WCOL: each line owns RPT rows of every TRF-row tile (rows tl TRF + line RPT + j, j < RPT) and
    // gathers them itself (cp.async, column segments of one row block -> its tile rows), so the
    // lines of the CTA synchronise only with themselves (named barriers) and run out of step.
    C* ltile = tile + line * RPT * G::TSTR;
    auto issue_tile = [&](int tl) {
      const int rb = tl * G::TRF + line * RPT;                 // first row (in the item) of the line's block
#pragma unroll 4
      for (int e = t; e < ncols * RPT; e += G::THR) {
        const int kk = e / RPT, rr = e - kk * RPT;
        if (rb + rr < cnt) cp_async_el<T>(ltile + rr * G::TSTR + c_lo + kk, src + G::wat(r0 + rb + rr, kk, stride), pf, stream);
      }
      cp_async_commit();
    };
    if constexpr (G::WCOL) {
      // the line's tile rows are indexed by the bin k = 0..H: zero outside the plane's bins (the copies
      // never touch them), so the rounds read them without range tests
      for (int e = t; line * RPT < G::TRF && e < (G::H + 1 - ncols) * RPT; e += G::THR) {
        const int rr = e % RPT, j = e / RPT;
        ltile[rr * G::TSTR + (j < c_lo ? j : j + ncols)] = czero<T>();
      }
      issue_tile(0);
    }
#pragma unroll 1
    for (int rd = 0; rd < rounds; ++rd) {
      const int ri = G::WCOL ? (rd / RPT) * G::TRF + line * RPT + rd % RPT : rd * G::LPR + line;
      const bool act = ri < cnt;
      const int r = r0 + (act ? ri : 0);
      C z[G::ER], zm[G::ER];
      if constexpr (G::WCOL) {
        if (rd % RPT == 0) {                   // this round's rows have landed
          cp_async_wait_all();
          SyncOf<G::THR, true>::sync();
        }
        const C* trow = ltile + (rd % RPT) * G::TSTR;
#pragma unroll
        for (int q = 0; q < G::ER; ++q) {     // (line-uniform test: lines past the tile read nothing)
          z[q] = act ? trow[t + q * G::THR] : czero<T>();
          zm[q] = act ? trow[H - t - q * G::THR] : czero<T>();
        }
        if (rd % RPT == RPT - 1 && rd + 1 < rounds) {   // every read of the line's rows done: the next
          SyncOf<G::THR, true>::sync();                 // ones stream in behind this round's FFT
          issue_tile(rd / RPT + 1);
        }
      } else {
        const C* row = src + (size_t)r * stride - c_lo;
        // phase 1: issue every load of the round (no use in between: all in flight together)
#pragma unroll
        for (int q = 0; q < G::ER; ++q) {
          const int k = t + q * G::THR, km = H - k;
          const bool ik = act && k >= c_lo && k < c_lo + ncols, ikm = act && km >= c_lo && km < c_lo + ncols;
          z[q] = ik ? __ldcg(row + (ik ? k : c_lo)) : czero<T>();
          zm[q] = ikm ? __ldcg(row + (ikm ? km : c_lo)) : czero<T>();
        }
      }
      // phase 2: Hermitian pre-processing of the half-length C2R
#pragma unroll
      for (int q = 0; q < G::ER; ++q) {
        const int k = t + q * G::THR;
        const C xk = z[q], xm = zm[q];
        const C a = cadd_conj<T>(xk, xm);                   // xk + conj(xm)
        const C d = csub_conj<T>(xk, xm);                   // xk - conj(xm)
        const C e = cmulc<T>(d, twk(k, tw));                // d * exp(+2 pi i k / N)
        z[q] = cadd_i<T>(a, e);                             // a + i e
      }
      if (rd == 0) FFST_PROBE(p, 0);
      if (!(p.dbg & 1)) fft<H, true, true>(z, scr + line * G::SMR, t, tw);
      if (rd == 0) FFST_PROBE(p, 1);
      if (act) {
        const T sr = (r & 1) ? T(-1) : T(1);
        // (cached loads may be hoisted above their guard: valid addresses without Nyquist terms too)
        const T* gsafe = nyqG != nullptr ? nyqG : reinterpret_cast<const T*>(tw);
        const T* hsafe = nyqG != nullptr ? nyqH : reinterpret_cast<const T*>(tw);
        T hr = T(0);
        if (nyqG != nullptr) hr = G::WCOL ? __ldg(hsafe + r) : sH[ri];
#pragma unroll
        for (int q = 0; q < G::ER; ++q) {
          const int m1 = 2 * (t + q * G::THR);
          const C xs = cscale<T>(z[q], scale);
          const T x0 = xs.x, x1 = xs.y;
          T c0 = T(0), c1 = T(0);
          if (MODE != MODE_COMPACT && nyqG != nullptr) {
            T g0, g1;
            if constexpr (G::WCOL) {
                            const cpx<T> gg = __ldg(reinterpret_cast<const cpx<T>*>(gsafe + m1));
              g0 = gg.x; g1 = gg.y;
            } else {
              g0 = sG[m1]; g1 = sG[m1 + 1];
            }
            const C cc = cfma_real<T>(sr, mk<T>(g0, g1), mk<T>(hr, -hr));
            c0 = cc.x;
            c1 = cc.y;
          }
          if constexpr (MODE == MODE_MAIN) {
            if (!(p.dbg & 2)) store_pair_cs<T>(out_c + (size_t)r * N + m1, mk<T>(x0, c0), mk<T>(x1, c1));
          } else if constexpr (MODE == MODE_COMPACT) {   // real part only; the Nyquist term is (G, H)
            __stcs(reinterpret_cast<cpx<T>*>(out_r + (size_t)r * N + m1), mk<T>(x0, x1));
          } else {
            cpx<T> v = mk<T>(x0 - c0, x1 - c1);
            *reinterpret_cast<cpx<T>*>(out_r + (size_t)r * N + m1) = v;
          }
        }
      }
      SyncOf<G::THR, true>::sync();
    }
  }

  // ------------------------------------------------------------------ row R2C item
  // Rows [r0, r0+cnt): MAIN reads Re of a coefficient plane (and, for Nyquist planes,
  // the alternating sums of Im); AUX reads a real image.  R2C along m1, keeps bins
  // [c_lo, c_lo+ncols) -> dst column-major (dst[(k - c_lo) * N + r]).
  template <int MODE>
  static __device__ void row_r2c(const KParams& p, const C* __restrict__ src_c, const T* __restrict__ src_r,
                                 int c_lo, int ncols, int r0, int cnt, C* dst, int nyq_b, int nyq_idx,
                                 int nyq_group, C* smem, const int* dep = nullptr, int dep_target = 0) {
    C* scr = smem;
    C* tile = smem + G::SCRX;
    const int tid = threadIdx.x, line = tid / G::THR, t = tid % G::THR;
    const C* tw = static_cast<const C*>(p.tw);
    const bool nyq = MODE == MODE_MAIN && nyq_idx >= 0;
    // MAIN: the lines of the CTA synchronise only with themselves inside a tile (named barriers);
    // the whole CTA meets at the tile stores
    constexpr bool NL = MODE == MODE_MAIN;
    T sacc[G::ER][2];
#pragma unroll
    for (int q = 0; q < G::ER; ++q) sacc[q][0] = sacc[q][1] = T(0);
    constexpr int ROUNDS = G::GR / G::LPR > 0 ? G::GR / G::LPR : 1;
    const int ntiles = (cnt + G::GR - 1) / G::GR;
#pragma unroll 1
    for (int ti = 0; ti < ntiles; ++ti) {
      const int rt0 = r0 + ti * G::GR;
#pragma unroll 1
      for (int rd = 0; rd < ROUNDS; ++rd) {
        const int ri = rd * G::LPR + line;              // row inside the tile
        const bool act = ri < G::GR && ti * G::GR + ri < cnt;
        const int r = rt0 + ri;
        C z[G::ER];
        T trow = T(0);
        const T sr = (r & 1) ? T(-1) : T(1);
        if constexpr (MODE == MODE_MAIN) {
          // phase 1: issue all loads of the round; phase 2: split real / imaginary parts
          C va[G::ER], vb[G::ER];
#pragma unroll
          for (int q = 0; q < G::ER; ++q) {
            if (act) {
              load_pair_cs<T>(src_c + (size_t)(act ? r : r0) * N + 2 * (t + q * G::THR), va[q], vb[q]);
            } else {
              va[q] = czero<T>();
              vb[q] = czero<T>();
            }
          }
#pragma unroll
          for (int q = 0; q < G::ER; ++q) z[q] = mk<T>(va[q].x, vb[q].x);
          if (nyq) {
#pragma unroll
            for (int q = 0; q < G::ER; ++q) {
              sacc[q][0] += sr * va[q].y;
              sacc[q][1] += sr * vb[q].y;
              trow += va[q].y - vb[q].y;
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < G::ER; ++q)
            z[q] = act ? *reinterpret_cast<const cpx<T>*>(src_r + (size_t)(act ? r : r0) * N + 2 * (t + q * G::THR)) : czero<T>();
        }
        if (ti == 0 && rd == 0) FFST_PROBE(p, 0);
        fft<H, false, NL>(z, scr + line * G::SMR, t, tw);
        if (ti == 0 && rd == 0) FFST_PROBE(p, 1);
        if (nyq) {
          // alternating row sum t(r) = sum_m1 (-1)^m1 Im c(r, m1): one partial per warp of the line
          // (G::TPARTS, summed in order by nyq_inv_kernel)
          T v = trow;
#pragma unroll
          for (int o = (G::THR < 32 ? G::THR : 32) / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if ((t & 31) == 0 && act)
            static_cast<T*>(p.nyq_T)[(((size_t)nyq_b * p.n_nyq + nyq_idx) * G::TPARTS + (t >> 5)) * N + r] = v;
        }
        C* sl = scr + line * G::SMR;
        SyncOf<G::THR, NL>::sync();
#pragma unroll
        for (int q = 0; q < G::ER; ++q) sl[Pad<T>::at(t + q * G::THR)] = z[q];
        SyncOf<G::THR, NL>::sync();
        if (act) {
#pragma unroll 1
          for (int kk = t; kk < ncols; kk += G::THR) {
            const int k = c_lo + kk;                         // 0..H
            const C zk = sl[Pad<T>::at(k == H ? 0 : k)];
            const C zm = sl[Pad<T>::at(k == 0 ? 0 : H - k)];
            const C a = mk<T>(zk.x + zm.x, zk.y - zm.y);    // Z[k] + conj(Z[H-k])
            const C d = mk<T>(zk.x - zm.x, zk.y + zm.y);    // Z[k] - conj(Z[H-k])
            const C e = cmul<T>(d, twk(k, tw));              // W^k d
            tile[ri * G::TSTR + kk] = mk<T>(T(0.5) * (a.x + e.y), T(0.5) * (a.y - e.x));   // (a - i e)/2
          }
        }
        SyncOf<G::THR, NL>::sync();
        if (ti == 0 && rd == 0) FFST_PROBE(p, 2);
      }
      if (dep != nullptr && ti == 0 && tid == 0) spin_wait(dep, dep_target);   // slot reuse: before the first write
      __syncthreads();
      const int rows_here = cnt - ti * G::GR < G::GR ? cnt - ti * G::GR : G::GR;
#pragma unroll 1
      for (int e = tid; e < ncols * G::GR; e += NT) {
        const int kk = e / G::GR, ri = e - kk * G::GR;
        if (ri < rows_here) dst[MODE == MODE_MAIN ? G::iat(rt0 + ri, kk, ncols) : (size_t)kk * N + rt0 + ri] = tile[ri * G::TSTR + kk];
      }
      __syncthreads();
      if (ti == 0) FFST_PROBE(p, 3);
    }
    if (nyq) {
      // partial alternating column sums s(m1) = sum_r (-1)^r Im c(r, m1) over this item's rows
      T* red = reinterpret_cast<T*>(scr);                  // [LPR][N] scalars (fits SCR_R)
#pragma unroll
      for (int q = 0; q < G::ER; ++q) {
        const int m1 = 2 * (t + q * G::THR);
        red[line * N + m1] = sacc[q][0];
        red[line * N + m1 + 1] = sacc[q][1];
      }
      __syncthreads();
      T* outp = static_cast<T*>(p.nyq_S) + (((size_t)nyq_b * p.n_nyq + nyq_idx) * p.n_rowitems + nyq_group) * N;
#pragma unroll 1
      for (int m = tid; m < N; m += NT) {
        T s = T(0);
        for (int l = 0; l < G::LPR; ++l) s += red[l * N + m];
        outp[m] = s;
      }
      __syncthreads();
    }
  }


  // ------------------------------------------------------------------ row passes, two rows per line
  // Forward pass 2 (PAIR): rows ra, ra+1 of the intermediate are Hermitian (sym part); one complex
  // inverse FFT of Z = Ta + i Tb over all N bins (bins above H from the mirror) gives the two real
  // rows -- no half-length pre-processing twiddles.  Same output and Nyquist term as row_c2r.
  static __device__ void row_c2r_pair(const KParams& p, const C* __restrict__ src, int stride, int c_lo, int ncols,
                                      int r0, int cnt, C* out_c, const T* nyqG, const T* nyqH, C* smem) {
    C* scr = smem;
    const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
    const C* tw = static_cast<const C*>(p.tw);
    const T scale = T(1) / (T(N) * T(N));
    constexpr int RPR = 2 * G::LPC;
    T* sG = reinterpret_cast<T*>(smem + G::SCRX);
    T* sH = sG + N;
    if (nyqG != nullptr) {
      for (int m = tid; m < N; m += NT) sG[m] = nyqG[m];
      for (int i = tid; i < cnt; i += NT) sH[i] = nyqH[r0 + i];
      __syncthreads();
    }
    const unsigned nc = (unsigned)ncols;
#pragma unroll 1
    for (int rd = 0; rd * RPR < cnt; ++rd) {
      const int ri = rd * RPR + 2 * line;
      const bool act = ri < cnt;
      const int ra = r0 + (act ? ri : 0);
      const C* wa = src + (size_t)ra * stride - c_lo;
      const C* wb = wa + stride;
      C z[G::EC];
#pragma unroll
      for (int q = 0; q < G::EC; ++q) {
        const int c = t + q * G::THC;
        const bool up = c > H;
        const int k = up ? N - c : c;
        C a = czero<T>(), b = czero<T>();
        if (act && (unsigned)(k - c_lo) < nc) {
          const int kk = (unsigned)(k - c_lo) < nc ? k : c_lo;   // in range even if hoisted
          a = __ldcg(wa + kk);
          b = __ldcg(wb + kk);
        }
        z[q] = up ? mk<T>(a.x + b.y, b.x - a.y) : mk<T>(a.x - b.y, a.y + b.x);
      }
      if (rd == 0) FFST_PROBE(p, 0);
      fft<N, true>(z, scr + line * G::SMC, t, tw);
      if (rd == 0) FFST_PROBE(p, 1);
      if (act) {
        C* oa = out_c + (size_t)ra * N;
        C* ob = oa + N;
        if (nyqG != nullptr) {
          const T sa = (ra & 1) ? T(-1) : T(1);
          const T ha = sH[ri], hb = sH[ri + 1];
#pragma unroll
          for (int q = 0; q < G::EC; ++q) {
            const int m1 = t + q * G::THC;
            const T sm = (m1 & 1) ? T(-1) : T(1);
            const T g = sG[m1];
            __stcs(oa + m1, mk<T>(z[q].x * scale, sa * g + sm * ha));
            __stcs(ob + m1, mk<T>(z[q].y * scale, -sa * g + sm * hb));
          }
        } else {
#pragma unroll
          for (int q = 0; q < G::EC; ++q) {
            const int m1 = t + q * G::THC;
            __stcs(oa + m1, mk<T>(z[q].x * scale, T(0)));
            __stcs(ob + m1, mk<T>(z[q].y * scale, T(0)));
          }
        }
      }
      SyncOf<G::THC>::sync();
    }
  }

  // Inverse pass 1 (PAIR): Z = Re c(ra, .) + i Re c(ra+1, .), one forward FFT; the rows' spectra
  // Xa[k] = (Z[k] + conj Z[N-k])/2, Xb[k] = (Z[k] - conj Z[N-k])/(2i) for the plane's bins -> tile
  // -> W (column-major), plus the alternating sums of Im c for Nyquist planes.  Same results as
  // row_r2c<MODE_MAIN>.
  // REAL: the rows are reals (compact format, f1): src_c is read as T rows, no Nyquist sums.
  template <bool REAL = false>
  static __device__ void row_r2c_pair(const KParams& p, const C* __restrict__ src_c, int c_lo, int ncols, int r0,
                                      int cnt, C* dst, int nyq_b, int nyq_idx, int nyq_group, C* smem,
                                      const int* dep = nullptr, int dep_target = 0) {
    C* scr = smem;
    C* tile = smem + G::SCRX;
    T* red = reinterpret_cast<T*>(tile + G::TILE_R);        // NT/32 scalars past the tile
    const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
    const C* tw = static_cast<const C*>(p.tw);
    const bool nyq = !REAL && nyq_idx >= 0 && !(p.dbg & 8);
    constexpr int RPR = 2 * G::LPC;
    T sacc[G::EC];
#pragma unroll
    for (int q = 0; q < G::EC; ++q) sacc[q] = T(0);
    constexpr int ROUNDS = G::GR / RPR > 0 ? G::GR / RPR : 1;
    const int ntiles = (cnt + G::GR - 1) / G::GR;
    const bool direct = G::DIRW ^ ((p.dbg & 128) != 0);    // (see row_r2c_pair_pipe)
    const unsigned long long pfd = policy_evict_first();
    if (direct && dep != nullptr) {
      if (tid == 0) spin_wait(dep, dep_target);           // slot reuse: before the first write
      __syncthreads();
    }
#pragma unroll 1
    for (int ti = 0; ti < ntiles; ++ti) {
      const int rt0 = r0 + ti * G::GR;
#pragma unroll 1
      for (int rd = 0; rd < ROUNDS; ++rd) {
        const int ri = rd * RPR + 2 * line;              // first row of the pair inside the tile
        const bool act = ri < G::GR && ti * G::GR + ri < cnt;
        const int ra = act ? rt0 + ri : r0;
        const C* rowa = src_c + (size_t)ra * N;
        const C* rowb = rowa + N;
        C z[G::EC];
        T ta = T(0), tb = T(0);
        const T sa = (ra & 1) ? T(-1) : T(1);
        // float32: every load of the round in flight before any use (float64: registers too scarce)
        constexpr int PH = (REAL || sizeof(T) == 4) ? G::EC : 1;
        C va_[PH], vb_[PH];
        if constexpr (REAL) {          // compact rows: reals, row ra at src + ra N (T units)
          const T* ra_ = reinterpret_cast<const T*>(src_c) + (size_t)ra * N;
#pragma unroll
          for (int q = 0; q < G::EC; ++q) {
            const int m = t + q * G::THC;
            va_[q] = mk<T>(act ? __ldcs(ra_ + m) : T(0), T(0));
            vb_[q] = mk<T>(act ? __ldcs(ra_ + N + m) : T(0), T(0));
          }
        } else if constexpr (PH > 1) {
#pragma unroll
          for (int q = 0; q < G::EC; ++q) {
            const int m = t + q * G::THC;
            va_[q] = act ? __ldcs(rowa + m) : czero<T>();
            vb_[q] = act ? __ldcs(rowb + m) : czero<T>();
          }
        }
#pragma unroll
        for (int q = 0; q < G::EC; ++q) {
          const int m = t + q * G::THC;
          C va, vb;
          if constexpr (REAL || PH > 1) {
            va = va_[q];
            vb = vb_[q];
          } else {
            va = act ? __ldcs(rowa + m) : czero<T>();
            vb = act ? __ldcs(rowb + m) : czero<T>();
          }
          z[q] = mk<T>(va.x, vb.x);
          if (nyq) {
            const T sm = (m & 1) ? T(-1) : T(1);
            sacc[q] += sa * (va.y - vb.y);
            ta += sm * va.y;
            tb += sm * vb.y;
          }
        }
        if (ti == 0 && rd == 0) FFST_PROBE(p, 0);
        C* sl = scr + line * G::SMC;
        if (!(p.dbg & 1)) fft<N, false>(z, sl, t, tw);
        if (ti == 0 && rd == 0) FFST_PROBE(p, 1);
        if (nyq) {   // alternating row sums t(r) = sum_m1 (-1)^m1 Im c(r, m1): one partial per warp
#pragma unroll
          for (int o = (G::THC < 32 ? G::THC : 32) / 2; o > 0; o >>= 1) {
            ta += __shfl_xor_sync(0xffffffffu, ta, o);
            tb += __shfl_xor_sync(0xffffffffu, tb, o);
          }
          if ((t & 31) == 0 && act) {          // summed in warp order by nyq_inv_kernel
            T* tt = static_cast<T*>(p.nyq_T) + (((size_t)nyq_b * p.n_nyq + nyq_idx) * G::TPARTS + (t >> 5)) * N + ra;
            tt[0] = ta;
            tt[1] = tb;
          }
        }
        SyncOf<G::THC>::sync();
#pragma unroll
        for (int q = 0; q < G::EC; ++q) sl[Pad<T>::at(t + q * G::THC)] = z[q];
        SyncOf<G::THC>::sync();
        if (act && direct) {
#pragma unroll 2
          for (int kk = t; kk < ncols; kk += G::THC) {
            const int k = c_lo + kk;                         // 0..H
            const C zk = sl[Pad<T>::at(k)];
            const C zm = sl[Pad<T>::at(k == 0 ? 0 : N - k)];
            const C xa = cscale<T>(cadd_conj<T>(zk, zm), T(0.5));
            const C xb = cscale_mi<T>(csub_conj<T>(zk, zm), T(0.5));
            C* d = dst + G::iat(ra, kk, ncols);
            if (!(p.dbg & 2)) {
              if (p.ring_stream) store_pair_hint<T>(d, xa, xb, pfd);
              else store_pair_cg<T>(d, xa, xb);
            }
          }
        } else if (act) {
#pragma unroll 2
          for (int kk = t; kk < ncols; kk += G::THC) {
            const int k = c_lo + kk;                         // 0..H
            const C zk = sl[Pad<T>::at(k)];
            const C zm = sl[Pad<T>::at(k == 0 ? 0 : N - k)];
            tile[ri * G::TSTR + kk] = cscale<T>(cadd_conj<T>(zk, zm), T(0.5));
            tile[(ri + 1) * G::TSTR + kk] = cscale_mi<T>(csub_conj<T>(zk, zm), T(0.5));
          }
        }
        SyncOf<G::THC>::sync();
        if (ti == 0 && rd == 0) FFST_PROBE(p, 2);
      }
      if (direct) continue;          // (each line reuses only its own scratch: no CTA barrier per tile)
      if (dep != nullptr && ti == 0 && tid == 0) spin_wait(dep, dep_target);   // slot reuse: before the first write
      __syncthreads();
      const int rows_here = cnt - ti * G::GR < G::GR ? cnt - ti * G::GR : G::GR;
      const unsigned long long pf = policy_evict_first();
      // two rows of a column per thread: one 16-byte store (rows r, r + 1 are adjacent in W, r even)
      static_assert(!G::WBLK_INV && G::GR % 2 == 0, "pair stores need the plain column-major W");
#pragma unroll 1
      for (int e = tid; e < (p.dbg & 2 ? 0 : ncols * (G::GR / 2)); e += NT) {
        const int kk = e / (G::GR / 2), ri = 2 * (e - kk * (G::GR / 2));
        if (ri + 1 < rows_here) {
          C* d = dst + G::iat(rt0 + ri, kk, ncols);
          const C a = tile[ri * G::TSTR + kk], b = tile[(ri + 1) * G::TSTR + kk];
          if (p.ring_stream) store_pair_hint<T>(d, a, b, pf);
          else store_pair_cg<T>(d, a, b);
        } else if (ri < rows_here) {
          dst[G::iat(rt0 + ri, kk, ncols)] = tile[ri * G::TSTR + kk];
        }
      }
      __syncthreads();
      if (ti == 0) FFST_PROBE(p, 3);
    }
    if (nyq) {
      // partial alternating column sums s(m1) over this item's rows: lines summed in fixed order
      if (direct) __syncthreads();                          // (every line done with its scratch)
      T* rs = reinterpret_cast<T*>(scr);                    // [LPC][N] scalars (fits SCR_C)
#pragma unroll
      for (int q = 0; q < G::EC; ++q) rs[line * N + t + q * G::THC] = sacc[q];
      __syncthreads();
      T* outp = static_cast<T*>(p.nyq_S) + (((size_t)nyq_b * p.n_nyq + nyq_idx) * p.n_rowitems + nyq_group) * N;
#pragma unroll 1
      for (int m = tid; m < N; m += NT) {
        T v = T(0);
        for (int l = 0; l < G::LPC; ++l) v += rs[l * N + m];
        outp[m] = v;
      }
      __syncthreads();
    }
  }

  // Inverse pass 1, pipelined variant (float32, n >= 1024, planes without a Nyquist part -- their
  // imaginary parts are not needed -- and the compact rows): the real parts of the NEXT round's
  // two rows are loaded into registers (2 x EC floats) before the current round's FFT, so the
  // HBM fetch of the cube overlaps the arithmetic (the plain variant loads, then computes).
  // Same results as row_r2c_pair.
  template <bool REAL = false>
  static __device__ void row_r2c_pair_pipe(const KParams& p, const C* __restrict__ src_c, int c_lo, int ncols,
                                           int r0, int cnt, C* dst, C* smem, const int* dep, int dep_target) {
    C* scr = smem;
    C* tile = smem + G::SCRX;
    const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
    const C* tw = static_cast<const C*>(p.tw);
    constexpr int RPR = 2 * G::LPC;
    constexpr int STRIDE = REAL ? 1 : 2;                   // floats per element (real parts only)
    // rows per tile: as many as the tile region holds for this plane's columns (a power of two from
    // GR up to 16 dividing the item; row stride ncols | 1), so that each column segment of W is
    // 64-128 bytes instead of GR x 8 (fewer, fuller L2 writes, fewer store phases)
    int gr = G::GR, tstr = G::TSTR;
    if (G::GR < 16) {
      const int ts = ncols | 1;
      while (gr < 16 && 2 * gr * ts <= G::TILE_R && cnt % (2 * gr) == 0) gr *= 2;
      if (gr > G::GR) tstr = ts;
    }
    const int lg = 31 - __clz(gr);
    const int ROUNDS = gr / RPR > 0 ? gr / RPR : 1;
    const T* base = reinterpret_cast<const T*>(src_c);
    const int nrounds = (cnt + RPR - 1) / RPR;
    T ca[G::EC], cb[G::EC];
    {
      const int ri = 2 * line;
      const bool act = ri < cnt;
      const T* pa = base + (size_t)STRIDE * (act ? r0 + ri : r0) * N;
#pragma unroll
      for (int q = 0; q < G::EC; ++q) {
        const int m = STRIDE * (t + q * G::THC);
        ca[q] = act ? __ldcs(pa + m) : T(0);
        cb[q] = act ? __ldcs(pa + STRIDE * N + m) : T(0);
      }
    }
    const unsigned long long pf = policy_evict_first();
    // Direct stores (Geo::DIRW; FFST_DBG bit 128 flips it, measurement only): the pair extraction
    // stores each column's two rows straight to W (one 16-byte store per column and row pair,
    // column-major: rows ra, ra + 1 are adjacent), no shared tile and no CTA-wide store phase
    const bool direct = G::DIRW ^ ((p.dbg & 128) != 0);
    if (direct && dep != nullptr) {
      if (tid == 0) spin_wait(dep, dep_target);           // slot reuse: before the first write
      __syncthreads();
    }
#pragma unroll 1
    for (int i = 0; i < nrounds; ++i) {
      T na[G::EC], nb[G::EC];
      {
        const int ri = (i + 1) * RPR + 2 * line;
        const bool act = i + 1 < nrounds && ri < cnt;
        const T* pa = base + (size_t)STRIDE * (act ? r0 + ri : r0) * N;
#pragma unroll
        for (int q = 0; q < G::EC; ++q) {
          const int m = STRIDE * (t + q * G::THC);
          na[q] = act ? __ldcs(pa + m) : T(0);
          nb[q] = act ? __ldcs(pa + STRIDE * N + m) : T(0);
        }
      }
      const int rd = i % ROUNDS, ti = i / ROUNDS;
      const int ri = rd * RPR + 2 * line;                  // first row of the pair inside the tile
      const bool act = ti * gr + ri < cnt;
      C z[G::EC];
#pragma unroll
      for (int q = 0; q < G::EC; ++q) z[q] = mk<T>(ca[q], cb[q]);
      C* sl = scr + line * G::SMC;
      if (!(p.dbg & 1)) fft<N, false>(z, sl, t, tw);
      SyncOf<G::THC>::sync();
#pragma unroll
      for (int q = 0; q < G::EC; ++q) sl[Pad<T>::at(t + q * G::THC)] = z[q];
      SyncOf<G::THC>::sync();
      if (act && direct) {
        const int ra = r0 + ti * gr + ri;
#pragma unroll 2
        for (int kk = t; kk < ncols; kk += G::THC) {
          const int k = c_lo + kk;                         // 0..H
          const C zk = sl[Pad<T>::at(k)];
          const C zm = sl[Pad<T>::at(k == 0 ? 0 : N - k)];
          const C xa = cscale<T>(cadd_conj<T>(zk, zm), T(0.5));
          const C xb = cscale_mi<T>(csub_conj<T>(zk, zm), T(0.5));
          C* d = dst + G::iat(ra, kk, ncols);
          if (!(p.dbg & 2)) {
            if (p.ring_stream) {
              store_pair_hint<T>(d, xa, xb, pf);
            } else {
              store_pair_cg<T>(d, xa, xb);
            }
          }
        }
      } else if (act) {
#pragma unroll 2
        for (int kk = t; kk < ncols; kk += G::THC) {
          const int k = c_lo + kk;                         // 0..H
          const C zk = sl[Pad<T>::at(k)];
          const C zm = sl[Pad<T>::at(k == 0 ? 0 : N - k)];
          tile[ri * tstr + kk] = cscale<T>(cadd_conj<T>(zk, zm), T(0.5));
          tile[(ri + 1) * tstr + kk] = cscale_mi<T>(csub_conj<T>(zk, zm), T(0.5));
        }
      }
      SyncOf<G::THC>::sync();
      if (!direct && (rd == ROUNDS - 1 || i + 1 == nrounds)) {   // the tile is complete: -> W (column-major)
        if (dep != nullptr && ti == 0 && tid == 0) spin_wait(dep, dep_target);   // slot reuse
        __syncthreads();
        const int rt0 = r0 + ti * gr;
        const int rows_here = cnt - ti * gr < gr ? cnt - ti * gr : gr;
#pragma unroll 1
        for (int e = tid; e < (p.dbg & 2 ? 0 : ncols << (lg - 1)); e += NT) {   // (gr >= 4: row pairs, 16-byte stores)
          const int kk = e >> (lg - 1), r = 2 * (e & ((gr >> 1) - 1));
          if (r + 1 < rows_here) {
            C* d = dst + G::iat(rt0 + r, kk, ncols);
            const C a = tile[r * tstr + kk], b = tile[(r + 1) * tstr + kk];
            if (p.ring_stream) store_pair_hint<T>(d, a, b, pf);
            else store_pair_cg<T>(d, a, b);
          } else if (r < rows_here) {
            dst[G::iat(rt0 + r, kk, ncols)] = tile[r * tstr + kk];
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int q = 0; q < G::EC; ++q) {
        ca[q] = na[q];
        cb[q] = nb[q];
      }
    }
  }

  // ------------------------------------------------------------------ column FFT items
  // inverse pass 2: columns [g0, g0+LPC) of image b over the planes of one chunk:
  // FFT along r of W, * sym_i, summed over planes, written / accumulated into A[b].
  static __device__ void col_fft_acc(const KParams& p, const ItemDev& I, const PlaneDev* splanes, C* smem) {
    C* scr = smem;
    const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
    const C* tw = static_cast<const C*>(p.tw);
    const T delta = (T)p.delta;
    const Radial<T> R = radial_of<T, N>(p);
    const C* slot = static_cast<const C*>(p.W) + (size_t)I.slot * p.slot_elems;
    T* wbuf = reinterpret_cast<T*>(smem + G::SCR_C);
#pragma unroll 1
    for (int rd = 0; rd < G::IG; ++rd) {
      const int g0 = I.group * G::IGC + rd * G::LPC;
      if (g0 > H) break;                                             // CTA-uniform
      const int g1 = g0 + G::LPC < H + 1 ? g0 + G::LPC : H + 1;
      const int cb = g0 + line;
      const bool act = cb <= H;
      C acc[G::EC];
#pragma unroll
      for (int q = 0; q < G::EC; ++q) acc[q] = czero<T>();
      int woff = I.woff;
#pragma unroll 1
      for (int u = 0; u < I.np; ++u) {
        const PlaneDev& P = splanes[I.p + u];
        const int cur = woff;
        woff += N * P.ncols_pad;
        if (g1 <= P.c_lo || g0 >= P.c_lo + P.ncols) continue;          // CTA-uniform
        const bool in = act && cb >= P.c_lo && cb < P.c_lo + P.ncols;
        const C* ws = slot + cur;
        const int cc = in ? cb - P.c_lo : 0;
        C r[G::EC];
        if (p.ring_stream) {
          const unsigned long long pf = policy_evict_first();
#pragma unroll
          for (int q = 0; q < G::EC; ++q) r[q] = in ? ld_hint<T>(ws + G::iat(t + q * G::THC, cc, P.ncols), pf) : czero<T>();
        } else {
#pragma unroll
          for (int q = 0; q < G::EC; ++q) r[q] = in ? __ldcg(ws + G::iat(t + q * G::THC, cc, P.ncols)) : czero<T>();
        }
        window_lines(P, g0, in, wbuf, scr, R, delta, user_plane<T, N>(p, P), p.dbg & 4);
        if (!(p.dbg & 1)) fft<N, false>(r, scr + line * G::SMC, t, tw);
        if (in) {
#pragma unroll
          for (int q = 0; q < G::EC; ++q) {
            const T w = wbuf[q * NT + tid];
            acc[q] = cfma_real<T>(w, r[q], acc[q]);
          }
        }
        SyncOf<G::THC>::sync();
      }
      if (act && !(p.dbg & 64)) {            // (FFST_DBG bit 64, measurement only: no accumulation)
        C* a = static_cast<C*>(p.A) + (size_t)I.pad1 * p.a_lane_elems + ((size_t)I.b * (H + 1) + cb) * N;
        const unsigned long long pl = policy_evict_last();
#pragma unroll
        for (int q = 0; q < G::EC; ++q) {
          const int idx = t + q * G::THC;
          if (I.first) st_hint<T>(a + idx, acc[q], pl);
          else red_add<T>(a + idx, acc[q], pl);      // no read-modify-write latency
        }
      }
    }
  }

  // spectrum pass 2: columns of Fscr[b] (column-major) -> F[b] (plain FFT along r)
  static __device__ void col_fft_plain(const KParams& p, int b, int g, C* smem) {
    C* scr = smem;
    const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
    const C* tw = static_cast<const C*>(p.tw);
    const int cb = g * G::LPC + line;
    const bool act = cb <= H;
    const C* col = static_cast<const C*>(p.Fscr) + ((size_t)b * (H + 1) + cb) * N;
    C r[G::EC];
#pragma unroll
    for (int q = 0; q < G::EC; ++q) r[q] = act ? col[t + q * G::THC] : czero<T>();
    fft<N, false>(r, scr + line * G::SMC, t, tw);
    if (act) {
      C* f = static_cast<C*>(p.F) + ((size_t)b * (H + 1) + cb) * N;
#pragma unroll
      for (int q = 0; q < G::EC; ++q) f[t + q * G::THC] = r[q];
    }
  }

  // ------------------------------------------------------------------ persistent kernels
  static __device__ void fwd_item(const KParams& p, const ItemDev& I, const PlaneDev* splanes, C* smem) {
    const PlaneDev& P = splanes[I.p];
    C* w = static_cast<C*>(p.W) + (size_t)I.slot * p.slot_elems + I.woff;
    if (I.type == 0 && G::GC == G::LPC && I.pad0 >= 0) {   // paired images (planner: pad0 = second image)
      const int c0 = P.c_lo + I.group * G::GC;
      const int rem = P.c_lo + P.ncols - c0;
      const C* F0 = static_cast<const C*>(p.F) + (size_t)I.b * (H + 1) * N;
      const C* F1 = static_cast<const C*>(p.F) + (size_t)I.pad0 * (H + 1) * N;
      C* w1 = static_cast<C*>(p.W) + (size_t)I.pad1 * p.slot_elems + I.first;
      col_ifft_two(p, P, c0, rem < G::GC ? rem : G::GC, F0, F1, w, w1, P.ncols_pad, c0 - P.c_lo, smem,
                   I.wait_ctr >= 0 ? p.ctr + I.wait_ctr : nullptr, I.wait_tgt,
                   I.wait2_ctr >= 0 ? p.ctr + I.wait2_ctr : nullptr, I.np);
    } else if (I.type == 0) {
      const int c0 = P.c_lo + I.group * G::GC;
      const int rem = P.c_lo + P.ncols - c0;
      const C* Fb = static_cast<const C*>(p.F) + (size_t)I.b * (H + 1) * N;
      col_ifft<MODE_MAIN>(p, I.b, P, c0, rem < G::GC ? rem : G::GC, Fb, w, P.ncols_pad, c0 - P.c_lo, smem,
                          I.wait_ctr >= 0 ? p.ctr + I.wait_ctr : nullptr, I.wait_tgt);
    } else {
      const int r0 = I.group * G::RP2;
      const int cnt = N - r0 < G::RP2 ? N - r0 : G::RP2;
      const T* nyqG = nullptr;
      const T* nyqH = nullptr;
      if (P.nyq >= 0) {
        nyqG = static_cast<const T*>(p.nyq_fwd) + ((size_t)I.b * p.n_nyq + P.nyq) * 2 * N;
        nyqH = nyqG + N;
      }
      if (p.compact) {   // f1 format: real rows; the Nyquist term stays as (G, H) vectors
        T* outr = static_cast<T*>(p.coeff) + ((size_t)I.b * p.eta_l + I.p) * N * N;
        row_c2r<MODE_COMPACT>(p, w, P.ncols_pad, P.c_lo, P.ncols, r0, cnt, nullptr, outr, nullptr, nullptr, smem);
        return;
      }
      C* out = static_cast<C*>(p.coeff) + ((size_t)I.b * p.eta_l + I.p) * N * N;
      if constexpr (G::PAIR_FWD) row_c2r_pair(p, w, P.ncols_pad, P.c_lo, P.ncols, r0, cnt, out, nyqG, nyqH, smem);
      else row_c2r<MODE_MAIN>(p, w, P.ncols_pad, P.c_lo, P.ncols, r0, cnt, out, nullptr, nyqG, nyqH, smem);
    }
  }

  static constexpr bool PIPE_INV = sizeof(T) == 4 && N >= 1024;   // pipelined inverse pass 1
  static __device__ void inv_item(const KParams& p, const ItemDev& I, const PlaneDev* splanes, C* smem) {
    if (I.type == 0) {
      const PlaneDev& P = splanes[I.p];
      C* w = static_cast<C*>(p.W) + (size_t)I.slot * p.slot_elems + I.woff;
      const int r0 = I.group * p.rpi;
      const int cnt = N - r0 < p.rpi ? N - r0 : p.rpi;
      if (p.compact) {   // f1 format: real rows; the Nyquist sums come from (G, H) (nyq_compact_sums)
        const T* srcr = static_cast<const T*>(p.coeff) + ((size_t)I.b * p.eta_l + I.p) * N * N;
        if constexpr (G::PAIR_INV && PIPE_INV) {
          if (!(p.dbg & 32)) {
            row_r2c_pair_pipe<true>(p, reinterpret_cast<const C*>(srcr), P.c_lo, P.ncols, r0, cnt, w, smem,
                                    I.wait_ctr >= 0 ? p.ctr + I.wait_ctr : nullptr, I.wait_tgt);
            return;
          }
        }
        if constexpr (G::PAIR_INV)
          row_r2c_pair<true>(p, reinterpret_cast<const C*>(srcr), P.c_lo, P.ncols, r0, cnt, w, I.b, -1, I.group, smem,
                             I.wait_ctr >= 0 ? p.ctr + I.wait_ctr : nullptr, I.wait_tgt);
        else
          row_r2c<MODE_AUX>(p, nullptr, srcr, P.c_lo, P.ncols, r0, cnt, w, I.b, -1, I.group, smem,
                            I.wait_ctr >= 0 ? p.ctr + I.wait_ctr : nullptr, I.wait_tgt);
        return;
      }
      const C* src = static_cast<const C*>(p.coeff) + ((size_t)I.b * p.eta_l + I.p) * N * N;
      if constexpr (G::PAIR_INV && PIPE_INV) {
        if (P.nyq < 0 && !(p.dbg & 32)) {      // no Nyquist part: only the real parts are needed
          row_r2c_pair_pipe<false>(p, src, P.c_lo, P.ncols, r0, cnt, w, smem,
                                   I.wait_ctr >= 0 ? p.ctr + I.wait_ctr : nullptr, I.wait_tgt);
          return;
        }
      }
      if constexpr (G::PAIR_INV)
        row_r2c_pair(p, src, P.c_lo, P.ncols, r0, cnt, w, I.b, P.nyq, I.group, smem,
                     I.wait_ctr >= 0 ? p.ctr + I.wait_ctr : nullptr, I.wait_tgt);
      else
        row_r2c<MODE_MAIN>(p, src, nullptr, P.c_lo, P.ncols, r0, cnt, w, I.b, P.nyq, I.group, smem,
                         I.wait_ctr >= 0 ? p.ctr + I.wait_ctr : nullptr, I.wait_tgt);
    } else {
      col_fft_acc(p, I, splanes, smem);
    }
  }
};

// Persistent schedulers.  Thread 0 fetches the next item index one item ahead; pass-1 items
// wait for their ring slot only before writing it (inside the item); pass-2 items wait for the
// pass-1 items of their chunk (and, inverse, for the previous owner of their column group).
// Release fences are issued only by items whose writes another item reads (pass 1, and the
// inverse's accumulator chain); forward pass 2 writes only the cube, read by nobody in the kernel.
constexpr int MAX_PLANES_SMEM = 256;

__device__ __forceinline__ ItemDev load_item(const ItemDev* items, int it) {
  const int4* src = reinterpret_cast<const int4*>(items + it);
  ItemDev I;
  int4* dst = reinterpret_cast<int4*>(&I);
  dst[0] = __ldg(src);
  dst[1] = __ldg(src + 1);
  dst[2] = __ldg(src + 2);
  dst[3] = __ldg(src + 3);
  return I;
}

// Persistent scheduler shared by both directions.  Thread 0 fetches the next item index one item
// ahead.  Pass-1 items wait for their ring slot inside the item (just before writing it); pass-2
// items wait for the pass-1 items of their chunk (and, inverse, the previous owner of their column
// group).  Release fences only where another item reads what this item wrote (every item but the
// forward pass 2, whose output -- the cube -- nobody reads inside the kernel).
template <typename T, int N, bool FWD>
__device__ __forceinline__ void persistent_loop(const KParams& p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cpx<T>* smem = reinterpret_cast<cpx<T>*>(smem_raw);
  __shared__ int s_item[2];
  __shared__ PlaneDev s_planes[MAX_PLANES_SMEM];
  K<T, N>::tw2_fill(p);
  for (int i = threadIdx.x; i < p.eta_l; i += blockDim.x) s_planes[i] = p.planes[i];
  if (threadIdx.x == 0) {
    s_item[0] = atomicAdd(p.ctr, 1);
    s_probe[0] = s_probe[1] = s_probe[2] = s_probe[3] = 0;
  }
  int cur = 0;
  for (;;) {
    __syncthreads();
    const int it = s_item[cur];
    if (it >= p.n_items) break;
    if (threadIdx.x == 0) s_item[cur ^ 1] = atomicAdd(p.ctr, 1);
    const ItemDev I = load_item(p.items, it < p.n_items ? it : p.n_items - 1);   // (hoist-safe index)
    unsigned long long t_start = 0, t_ready = 0;
    if (p.trace != nullptr && threadIdx.x == 0) t_start = gtimer();
    if (I.type == 1) {
      if (threadIdx.x == 0) {
        spin_wait(p.ctr + I.wait_ctr, I.wait_tgt, p.sync_mode);
        if (I.wait2_ctr >= 0) spin_wait(p.ctr + I.wait2_ctr, 1, p.sync_mode);
      }
      __syncthreads();
    }
    if (p.trace != nullptr && threadIdx.x == 0) t_ready = gtimer();
    if constexpr (FWD) K<T, N>::fwd_item(p, I, s_planes, smem);
    else K<T, N>::inv_item(p, I, s_planes, smem);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (!FWD || I.type == 0 || (p.sync_mode & 2)) red_release(p.ctr + I.sig_ctr, 1);   // RAW or WAR
      else asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p.ctr + I.sig_ctr), "r"(1) : "memory");
      if (I.sig2_ctr >= 0) red_release(p.ctr + I.sig2_ctr, 1);
    }
    if (p.trace != nullptr && threadIdx.x == 0) {
      unsigned long long* tr = p.trace + 8 * (size_t)it;
      tr[0] = smid();
      tr[1] = t_start;
      tr[2] = t_ready;
      tr[3] = gtimer();
      tr[4] = s_probe[0]; tr[5] = s_probe[1]; tr[6] = s_probe[2]; tr[7] = s_probe[3];
    }
    cur ^= 1;
  }
}

template <typename T, int N>
__global__ void __launch_bounds__(256, 2) fwd_main_kernel(KParams p) {
  persistent_loop<T, N, true>(p);
}

template <typename T, int N>
__global__ void __launch_bounds__(256, 2) inv_main_kernel(KParams p) {
  persistent_loop<T, N, false>(p);
}

// ---------------------------------------------------------------------- auxiliary kernels

// spectrum pass 1: rows of img[b] -> Fscr[b] column-major (all bins 0..H); grid (N/RPS, B)
template <typename T, int N>
__global__ void __launch_bounds__(256) spec_rows_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K<T, N>::tw2_fill(p);
  using G = Geo<T, N>;
  const int b = blockIdx.y, g = blockIdx.x;
  const int r0 = g * G::RPS;
  const int cnt = N - r0 < G::RPS ? N - r0 : G::RPS;
  const T* src = static_cast<const T*>(p.img) + (size_t)b * N * N;
  cpx<T>* dst = static_cast<cpx<T>*>(p.Fscr) + (size_t)b * (N / 2 + 1) * N;
  K<T, N>::template row_r2c<MODE_AUX>(p, nullptr, src, 0, N / 2 + 1, r0, cnt, dst, b, -1, 0,
                                      reinterpret_cast<cpx<T>*>(smem_raw));
}

// spectrum pass 2: grid (ceil((H+1)/LPC), B)
template <typename T, int N>
__global__ void __launch_bounds__(256) spec_cols_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K<T, N>::tw2_fill(p);
  K<T, N>::col_fft_plain(p, blockIdx.y, blockIdx.x, reinterpret_cast<cpx<T>*>(smem_raw));
}

// final pass 1: columns of A[b] -> Fscr[b] row-major (stride NCPF); grid (ceil((H+1)/GC), B)
template <typename T, int N>
__global__ void __launch_bounds__(256) fin_cols_kernel(KParams p, int cpb) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K<T, N>::tw2_fill(p);
  using G = Geo<T, N>;
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * cpb;              // cpb <= GC columns per CTA (fewer for small problems)
  const int rem0 = N / 2 + 1 - c0;
  const int rem = rem0 < cpb ? rem0 : cpb;
  const cpx<T>* src = static_cast<const cpx<T>*>(p.A) + (size_t)b * (N / 2 + 1) * N;
  cpx<T>* dst = static_cast<cpx<T>*>(p.Fscr) + (size_t)b * N * G::NCPF;
  PlaneDev dummy{};
  K<T, N>::template col_ifft<MODE_AUX>(p, b, dummy, c0, rem < G::GC ? rem : G::GC, src, dst, G::NCPF, c0,
                                       reinterpret_cast<cpx<T>*>(smem_raw));
}

// final pass 2: rows of Fscr[b] -> img_out[b] minus the Nyquist correction; grid (N/RP2, B)
template <typename T, int N>
__global__ void __launch_bounds__(256) fin_rows_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K<T, N>::tw2_fill(p);
  using G = Geo<T, N>;
  const int b = blockIdx.y;
  const int r0 = blockIdx.x * G::RPF;
  const int cnt = N - r0 < G::RPF ? N - r0 : G::RPF;
  const cpx<T>* src = static_cast<const cpx<T>*>(p.Fscr) + (size_t)b * N * G::NCPF;
  T* out = static_cast<T*>(p.img_out) + (size_t)b * N * N;
  const T* cg = nullptr;
  const T* ch = nullptr;
  if (p.n_nyq > 0) {
    cg = static_cast<const T*>(p.corr) + (size_t)b * 2 * N;
    ch = cg + N;
  }
  K<T, N>::template row_c2r<MODE_AUX>(p, src, G::NCPF, 0, N / 2 + 1, r0, cnt, nullptr, out, cg, ch,
                                      reinterpret_cast<cpx<T>*>(smem_raw));
}

// forward Nyquist terms: grid (ceil(n_nyq / LPC), 2, B); line l of the CTA handles Nyquist
// plane blockIdx.x * LPC + l.  which = 0: G(m1) from the Nyquist row, which = 1: H(r) from the
// Nyquist column.
template <typename T, int N>
__global__ void __launch_bounds__(256) nyq_fwd_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using G = Geo<T, N>;
  using C = cpx<T>;
  constexpr int H = N / 2;
  const int which = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
  const int nq = blockIdx.x * G::LPC + line;
  const bool act = nq < p.n_nyq;
  PlaneDev P{};
  if (act) P = p.planes[p.nyq_planes[nq]];
  const C* F = static_cast<const C*>(p.F) + (size_t)b * (H + 1) * N;
  const T delta = (T)p.delta;
  const Radial<T> R = radial_of<T, N>(p);
  C r[G::EC];
#pragma unroll 1
  for (int q = 0; q < G::EC; ++q) {
    const int bin = t + q * G::THC;
    C v = czero<T>();
    if (act) {
      const int u = centred(bin, N);
      if (which == 0) {
        const T a = static_cast<const T*>(p.nyq_anti)[((size_t)nq * 2 + 0) * N + bin];
        if (a != T(0)) v = cscale<T>(bin <= H ? F[(size_t)bin * N + H] : conj_<T>(F[(size_t)(N - bin) * N + H]), a);
      } else {
        const T a = static_cast<const T*>(p.nyq_anti)[((size_t)nq * 2 + 1) * N + bin];
        if (a != T(0)) v = cscale<T>(F[(size_t)H * N + bin], a);
      }
    }
    reinterpret_cast<C*>(smem_raw)[G::SCR_C + q * G::NT + tid] = v;
  }
#pragma unroll
  for (int q = 0; q < G::EC; ++q) r[q] = reinterpret_cast<C*>(smem_raw)[G::SCR_C + q * G::NT + tid];
  LineFFT<T, N, true, N>::run(r, reinterpret_cast<C*>(smem_raw) + line * G::SMC, t, static_cast<const C*>(p.tw));
  if (act) {
    T* out = static_cast<T*>(p.nyq_fwd) + (((size_t)b * p.n_nyq + nq) * 2 + which) * N;
    const T s = T(1) / (T(N) * T(N));
#pragma unroll
    for (int q = 0; q < G::EC; ++q) out[t + q * G::THC] = r[q].y * s;
  }
}

// inverse Nyquist correction, stage 1: grid (2, B, G).  CTA g takes the rounds g, g + G, ... of
// LPC Nyquist planes (line l: plane round * LPC + l); its per-line sums are added in fixed line
// order and written as partial spectrum g; stage 2 (nyq_fin_kernel) adds the G partials in order
// and synthesises the correction (deterministic; G > 1 spreads the planes over the GPU at large n).
template <typename T, int N>
__global__ void __launch_bounds__(256) nyq_inv_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using G = Geo<T, N>;
  using C = cpx<T>;
  const int which = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
  const C* tw = static_cast<const C*>(p.tw);
  C* scr = reinterpret_cast<C*>(smem_raw) + line * G::SMC;
  C* stage = reinterpret_cast<C*>(smem_raw) + G::SCR_C;          // [EC][NT] (also the reduction buffer)
  const T delta = (T)p.delta;
  const Radial<T> R = radial_of<T, N>(p);
  C acc[G::EC];
#pragma unroll
  for (int q = 0; q < G::EC; ++q) acc[q] = czero<T>();
  const int rounds = (p.n_nyq + G::LPC - 1) / G::LPC;
#pragma unroll 1
  for (int rd = blockIdx.z; rd < rounds; rd += gridDim.z) {
    const int nq = rd * G::LPC + line;
    const bool act = nq < p.n_nyq;
    C r[G::EC];
#pragma unroll
    for (int q = 0; q < G::EC; ++q) {
      const int m = t + q * G::THC;
      T s = T(0);
      if (act) {
        if (which == 0) {
          const T* ps = static_cast<const T*>(p.nyq_S) + ((size_t)b * p.n_nyq + nq) * p.n_rowitems * N + m;
          for (int g = 0; g < p.n_rowitems; ++g) s += ps[(size_t)g * N];
        } else {
          const T* pt = static_cast<const T*>(p.nyq_T) + ((size_t)b * p.n_nyq + nq) * p.nyq_tparts * N + m;
          for (int w = 0; w < p.nyq_tparts; ++w) s += pt[(size_t)w * N];
        }
      }
      r[q] = mk<T>(s, T(0));
    }
    LineFFT<T, N, false, N>::run(r, scr, t, tw);
    if (act) {
      const T* anti = static_cast<const T*>(p.nyq_anti) + ((size_t)nq * 2 + which) * N;
#pragma unroll
      for (int q = 0; q < G::EC; ++q) {
        const T a = anti[t + q * G::THC];
        acc[q].x += a * r[q].x;
        acc[q].y += a * r[q].y;
      }
    }
    __syncthreads();
  }
  // sum the per-line accumulators (fixed order) into line 0
#pragma unroll
  for (int q = 0; q < G::EC; ++q) stage[q * G::NT + tid] = acc[q];
  __syncthreads();
  if (line == 0) {
#pragma unroll
    for (int q = 0; q < G::EC; ++q) {
      C s = czero<T>();
      for (int l = 0; l < G::LPC; ++l) s = cadd<T>(s, stage[q * G::NT + l * G::THC + t]);
      acc[q] = s;
    }
  }
  if (line == 0) {
    C* part = static_cast<C*>(p.nyq_part) + (((size_t)b * 2 + which) * gridDim.z + blockIdx.z) * N;
#pragma unroll
    for (int q = 0; q < G::EC; ++q) part[t + q * G::THC] = acc[q];
  }
}

// inverse Nyquist correction, stage 2: grid (2, B); the G partial spectra summed in order, inverse
// DFT, imaginary part scaled -> corr
template <typename T, int N>
__global__ void __launch_bounds__(256) nyq_fin_kernel(KParams p, int groups) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using G = Geo<T, N>;
  using C = cpx<T>;
  const int which = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, line = tid / G::THC, t = tid % G::THC;
  // every line computes the same result (a CTA is at least a warp); line 0 stores it
  const C* part = static_cast<const C*>(p.nyq_part) + ((size_t)b * 2 + which) * groups * N;
  C acc[G::EC];
#pragma unroll
  for (int q = 0; q < G::EC; ++q) acc[q] = czero<T>();
#pragma unroll 1
  for (int g = 0; g < groups; ++g)
#pragma unroll
    for (int q = 0; q < G::EC; ++q) acc[q] = cadd<T>(acc[q], part[(size_t)g * N + t + q * G::THC]);
  LineFFT<T, N, true, N>::run(acc, reinterpret_cast<C*>(smem_raw) + line * G::SMC, t, static_cast<const C*>(p.tw));
  if (line > 0) return;
  T* out = static_cast<T*>(p.corr) + ((size_t)b * 2 + which) * N;
  const T s = T(1) / (T(N) * T(N));
#pragma unroll
  for (int q = 0; q < G::EC; ++q) out[t + q * G::THC] = acc[q].y * s;
}

// Compact format (f1), inverse: the alternating sums of Im c from the forward's Nyquist vectors,
// Im c(r, m1) = (-1)^r G(m1) + (-1)^m1 H(r)  =>
//   s(m1) = sum_r (-1)^r Im c(r, m1) = n G(m1) + (-1)^m1 sum_r (-1)^r H(r)   -> nyq_S (one partial)
//   t(r)  = sum_m1 (-1)^m1 Im c(r, m1) = (-1)^r sum_m1 (-1)^m1 G(m1) + n H(r) -> nyq_T
// grid (n_nyq, B), 256 threads; fixed-order reductions (deterministic).
template <typename T, int N>
__global__ void __launch_bounds__(256) nyq_compact_sums_kernel(KParams p) {
  __shared__ T red[2][256];
  const int nq = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const T* g = static_cast<const T*>(p.nyq_fwd) + ((size_t)b * p.n_nyq + nq) * 2 * N;
  const T* h = g + N;
  T sg = T(0), sh = T(0);
  for (int m = tid; m < N; m += 256) {
    const T sgn = (m & 1) ? T(-1) : T(1);
    sg += sgn * g[m];
    sh += sgn * h[m];
  }
  red[0][tid] = sg;
  red[1][tid] = sh;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) {
      red[0][tid] += red[0][tid + o];
      red[1][tid] += red[1][tid + o];
    }
    __syncthreads();
  }
  const T SG = red[0][0], SH = red[1][0];
  T* s = static_cast<T*>(p.nyq_S) + ((size_t)b * p.n_nyq + nq) * N;       // n_rowitems = 1
  T* tt = static_cast<T*>(p.nyq_T) + ((size_t)b * p.n_nyq + nq) * N;
  for (int m = tid; m < N; m += 256) {
    const T sgn = (m & 1) ? T(-1) : T(1);
    s[m] = T(N) * g[m] + sgn * SH;
    tt[m] = sgn * SG + T(N) * h[m];
  }
}

// Compact format (f1) -> complex cube: c_i(r, m1) = x_i(r, m1) + i [(-1)^r G_i(m1) + (-1)^m1 H_i(r)] on
// the Nyquist planes, x_i + 0 i elsewhere.  Grid-stride over the cube, two
// elements per thread (16-byte stores).
template <typename T>
__global__ void __launch_bounds__(256) expand_compact_kernel(const PlaneDev* planes, int n, int eta_l, int n_nyq,
                                                             const T* re, const T* gh, cpx<T>* out, long long pairs) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < pairs; e += (long long)gridDim.x * blockDim.x) {
    const long long i0 = 2 * e;                      // element index (n even: a pair never spans rows)
    const int m = (int)(i0 % n);
    const long long row = i0 / n;
    const int r = (int)(row % n);
    const long long bp = row / n;                    // b * eta_l + local plane
    const int lp = (int)(bp % eta_l), b = (int)(bp / eta_l);
    const int q = planes[lp].nyq;
    T y0 = T(0), y1 = T(0);
    if (q >= 0) {
      const T* g = gh + ((size_t)b * n_nyq + q) * 2 * n;
      const T sr = (r & 1) ? T(-1) : T(1);
      const T h = g[n + r];
      y0 = sr * g[m] + h;                            // m even
      y1 = sr * g[m + 1] - h;                        // m + 1 odd
    }
    const cpx<T> a = mk<T>(re[i0], y0), c = mk<T>(re[i0 + 1], y1);
    store_pair_cs<T>(out + i0, a, c);
  }
}

// materialise spectra (tests only): psi[i][row][col], grid-stride
template <typename T, int N>
__global__ void spectra_kernel(KParams p, T* psi, int centred_layout) {
  const size_t total = (size_t)p.eta_l * N * N;
  const T delta = (T)p.delta;
  const Radial<T> R = radial_of<T, N>(p);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / ((size_t)N * N));
    const int rem = (int)(e - (size_t)i * N * N);
    const int row = rem / N, col = rem - row * N;
    int u1, u2;
    if (centred_layout) {
      u1 = col - N / 2;
      u2 = row - N / 2;
    } else {
      u1 = centred(col, N);
      u2 = centred(row, N);
    }
    const PlaneDev& P = p.planes[i];
    if (p.usym) {
      // user spectra: sym(u) = sym(-u mod n) from the Hermitian-half table, plus the anti part
      // on the Nyquist row / column
      constexpr int H = N / 2;
      int a1 = u1, a2 = u2;
      if (u1 < 0 && u1 != -H) { a1 = -u1; a2 = u2 == -H ? -H : -u2; }
      T v = user_plane<T, N>(p, P)[(size_t)(a1 == -H ? H : a1) * N + (a2 < 0 ? a2 + N : a2)];
      if (P.nyq >= 0) {
        const T* an = static_cast<const T*>(p.nyq_anti) + (size_t)P.nyq * 2 * N;
        if (u2 == -H) v += an[u1 < 0 ? u1 + N : u1];
        if (u1 == -H) v += an[N + (u2 < 0 ? u2 + N : u2)];
      }
      psi[e] = v;
    } else {
      psi[e] = window<T>(P, u1, u2, R);
    }
  }
}

}  // namespace ffst
