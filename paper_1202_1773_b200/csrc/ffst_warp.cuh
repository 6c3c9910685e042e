// ffst_warp.cuh — warp-granular persistent kernels of the two FFT passes (sm_100a), n <= 512.
//
// Every warp of the CTA is an independent worker (DESIGN.md 6.4 "Warp workers"):
//   * it takes work items from the global queue (one atomicAdd per item, lane 0);
//   * the item's input arrives in shared memory through 1-D TMA bulk copies
//     (cp.async.bulk, completion on an mbarrier) into a per-warp double buffer of
//     "stages": while the warp computes stage s, stage s+1 (or the first stage of its
//     next item) is in flight, so HBM / L2 latency is hidden without extra warps;
//   * each stage is a set of whole FFT lines held by the warp (LPR rows of length n/2
//     or LPC columns of length n, E = 16 elements per lane), so all exchanges are
//     __syncwarp-only: no CTA barrier anywhere in the loop;
//   * dependency waits (pass 2 on the pass-1 items of its chunk, ring-slot reuse,
//     the inverse's accumulation chain) spin in lane 0 of the waiting warp only.
//
// Item types (queue of the host planner, ffst_api.cu build_queue):
//   forward  0 FP1  column IFFT of sym_i * F over GC columns  -> W (row-major, L2)
//            1 FP2  row C2R of RP2 rows of W + Nyquist term  -> coefficient rows (HBM)
//   inverse  0 IP1  row R2C of Re c_i over RPI rows, pruned  -> W (column-major, L2)
//                   (+ alternating sums of Im c_i for Nyquist planes)
//            1 IP2  column FFT of W * sym_i over the chunk's planes, accumulated -> A
// The arithmetic of each item is the same as in ffst_kernels.cuh (the even-N
// decomposition of DESIGN.md 6.2, the window of 6.1); only the data movement differs.
#pragma once
#include "ffst_kernels.cuh"

namespace ffst {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// arm the barrier with the expected byte count and issue one bulk copy global -> shared
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

// Dependency counters.  Waiting side: relaxed (volatile) polls; the data behind a counter is read
// only through L2 (TMA bulk copies, ld.global.cg), so no L1 invalidation (ld.acquire / __threadfence
// emit CCTL.IVALL) is needed.  Publishing side: red.release (MEMBAR.ALL.GPU + RED, no CCTL).
__device__ __forceinline__ bool ctr_reached(const int* ctr, int target) {
  return *reinterpret_cast<const volatile int*>(ctr) >= target;
}
__device__ __forceinline__ void spin_until(const int* ctr, int target) {
  while (!ctr_reached(ctr, target)) __nanosleep(64);
}

// per-warp intra-item probes (trace mode, first stage of an item only)
__shared__ unsigned long long s_wprobe[32][4];
#define FFST_WPROBE(p, s, i)                                                              \
  do {                                                                                    \
    if ((p).trace != nullptr && (s) == 0 && (threadIdx.x & 31) == 0) s_wprobe[threadIdx.x >> 5][i] = gtimer(); \
  } while (0)

// ------------------------------------------------------------------ geometry
template <typename T, int N>
struct WGeo {
  static constexpr int H = N / 2;
  static constexpr int ESZ = (int)sizeof(cpx<T>);
  // Every pass works on lines of length N held by THC lanes, EC elements per lane: column lines
  // (FP1, IP2) and row PAIRS (FP2, IP1: two real rows r, r+1 as one complex line, "two-for-one").
  // 8 elements per lane (more resident warps), 16 where a line of 8 per lane would span two warps.
#ifndef FFST_EMIN
#define FFST_EMIN 16
#endif
  static constexpr int EMC = N / FFST_EMIN <= 32 ? FFST_EMIN : 16;
  static constexpr int EC = RadixPlan<N, EMC>::E, THC = N / EC, LPC_ = 32 / THC;   // lines per stage
  static constexpr int LPC = LPC_;
  static constexpr int LPR = 2 * LPC < N ? 2 * LPC : N;     // rows per row stage (2 per line)
  static constexpr int SMC = Pad<T, EMC>::len(N);
#ifndef FFST_NW8
#define FFST_NW8 12
#endif
  // work item sizes: stages per item
  static constexpr int S_FP1 = 8, S_FP2 = 8, S_IP1 = 8;
  static constexpr int GC = LPC * S_FP1;                   // FP1 columns per item
  static constexpr int RP2_ = LPR * S_FP2, RP2 = RP2_ < N ? RP2_ : N;   // FP2 rows per item
  static constexpr int RPI_ = LPR * S_IP1, RPI = RPI_ < N ? RPI_ : N;   // IP1 rows per item
  static constexpr int COLPAD = 4;                                      // W row stride multiple (fwd)
  static constexpr int NCP_MAX = ((H + 1 + COLPAD - 1) / COLPAD) * COLPAD;   // largest W row stride (fwd)
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  // per warp: two input stage buffers (TMA payloads) + one scratch area (FFT exchanges, the
  // inverse's post-processing, the IP2 window).  A stage buffer is released right after its data
  // has been read into registers, so two stage loads are in flight while the warp computes.
  static constexpr int WIN_C = (LPC * N * (int)sizeof(T) + ESZ - 1) / ESZ;   // IP2 window block (complex units)
#ifndef FFST_EARLY_RELEASE
#define FFST_EARLY_RELEASE 0
#endif
  // EARLY_RELEASE = 1: separate scratch, stage buffer refilled as soon as it is read (two loads in
  // flight, fewer warps fit); 0: the stage buffer is also the scratch and is refilled after the
  // stage's compute (one load in flight, more warps).  0 measured faster.
  static constexpr bool EARLY = FFST_EARLY_RELEASE != 0;
  static constexpr int SCR = WIN_C + LPC * SMC;
  static constexpr int STAGE = EARLY ? cmax(cmax(LPR * N, LPC * N), LPR * NCP_MAX)
                                     : cmax(cmax(cmax(LPR * N, LPC * N), LPR * NCP_MAX), SCR);
  static constexpr int STAGE_PAD = (STAGE * ESZ + 127) / 128 * 128 / ESZ;
  static constexpr int SCR_PAD = EARLY ? (SCR * ESZ + 127) / 128 * 128 / ESZ : 0;
  static constexpr int WARP_ELEMS = 2 * STAGE_PAD + SCR_PAD;
  // worker warps per CTA (1 CTA / SM): 12 at most (f32, E=16: 168 registers), fewer if the
  // per-warp buffers would not fit ~196 KB of shared memory
  static constexpr int NW_SMEM = (196 * 1024) / (WARP_ELEMS * ESZ);
  static constexpr int NW_ = sizeof(T) == 4 ? (EMC == 8 ? FFST_NW8 : 12) : 12;
  static constexpr int NW = NW_ < NW_SMEM ? NW_ : NW_SMEM;
  static constexpr int NT = NW * 32;
  static constexpr int RT_ROWS = (ilog2(N) + 2) / 2 + 1;   // radial table rows for j0 <= default + 1
  static constexpr size_t OFF_BARS = (size_t)NW * WARP_ELEMS * ESZ;
  static constexpr size_t OFF_TW = OFF_BARS + ((NW * 2 * 8 + 127) / 128) * 128;
  static constexpr size_t OFF_RT = OFF_TW + (size_t)N * ESZ;
  static constexpr size_t SMEM = OFF_RT + (((size_t)RT_ROWS * (H + 1) * sizeof(T) + 127) / 128) * 128;
  static_assert(THC <= 32, "warp kernels need lines of <= 32 lanes (n <= 512)");
  static_assert(RP2 % LPR == 0 && RPI % LPR == 0, "row items must be whole stages");
};

// shared-memory copies of the plan tables (twiddles exp(-2 pi i m / n), radial factors)
template <typename T>
struct Tabs {
  const cpx<T>* tw;
  const T* rt;
};

template <typename T, int N>
struct WK {
  using G = WGeo<T, N>;
  using C = cpx<T>;
  static constexpr int H = N / 2;

  // point-symmetric window sym_i along Hermitian-half column cb (bin 0..H), rows rb (bins):
  // window_sym() of ffst_math.cuh with the per-column work hoisted into the plan's column record
  // (ColRec: support hulls, radial factor, 1/|u1|).  Rows outside the hulls return 0 after three
  // integer range tests; only candidate rows evaluate the window.
  struct ColSym {
    ColWin<T> w0, w1;
    int lo0, hi0, lo1, hi1, lo2, hi2;
    bool nyqcol;
    __device__ ColSym(const PlaneDev& P, int cb, const T* rt, int j0, const ColRec<T>& R)
        : w0(P, cb == H ? -H : cb, rt, H + 1, j0, R.rh, R.inv_a1),
          w1(P, H, rt, H + 1, j0, R.rh, R.inv_a1),
          lo0(R.lo[0]), hi0(R.hi[0]), lo1(R.lo[1]), hi1(R.hi[1]), lo2(R.lo[2]), hi2(R.hi[2]), nyqcol(cb == H) {}
    __device__ bool cand(int u2) const {
      return (unsigned)(u2 - lo0) <= (unsigned)(hi0 - lo0) || (unsigned)(u2 - lo1) <= (unsigned)(hi1 - lo1) ||
             (unsigned)(u2 - lo2) <= (unsigned)(hi2 - lo2);
    }
    __device__ T at(int rb) const {
      const int u2 = centred(rb, N);
      if (!cand(u2)) return T(0);
      if (nyqcol) return T(0.5) * (w0.eval(u2) + w1.eval(rb == H ? H : u2));
      if (rb == H) return T(0.5) * (w0.eval(-H) + w0.eval(H));
      return w0.eval(u2);
    }
  };
  static __device__ __forceinline__ ColRec<T> col_rec(const KParams& p, const PlaneDev& P, int cb) {
    ColRec<T> r;
    // (clamped: callers may evaluate this for idle columns and the loads may be hoisted)
    const int cc = cb < P.c_lo ? 0 : (cb >= P.c_lo + P.ncols ? P.ncols - 1 : cb - P.c_lo);
    const ColRec<T>* src = static_cast<const ColRec<T>*>(p.colrec) + P.rec + cc;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      r.lo[i] = __ldg(&src->lo[i]);
      r.hi[i] = __ldg(&src->hi[i]);
    }
    r.rh = __ldg(&src->rh);
    r.inv_a1 = __ldg(&src->inv_a1);
    return r;
  }

  // ---------------------------------------------------------------- stage sources
  // Number of stages of an item and the (src, bytes) of stage s.  Pure functions of the item.
  struct Src { const void* src; unsigned bytes; };

  static __device__ __forceinline__ int fp1_cols(const PlaneDev& P, const ItemDev& I, int* c0) {
    *c0 = P.c_lo + I.group * G::GC;
    const int rem = P.c_lo + P.ncols - *c0;
    return rem < G::GC ? rem : G::GC;
  }
  static __device__ __forceinline__ int rows_of(int group, int per) {
    const int r0 = group * per;
    return N - r0 < per ? N - r0 : per;
  }

  template <bool FWD>
  static __device__ __forceinline__ int n_stages(const KParams& p, const ItemDev& I, const PlaneDev* sp) {
    if (FWD) {
      if (I.type == 0) {
        int c0;
        const int cnt = fp1_cols(sp[I.p], I, &c0);
        return (cnt + G::LPC - 1) / G::LPC;
      }
      return (rows_of(I.group, G::RP2) + G::LPR - 1) / G::LPR;
    }
    if (I.type == 0) return (rows_of(I.group, G::RPI) + G::LPR - 1) / G::LPR;
    return __popc((unsigned)I.pad0);
  }

  // IP2: plane (local index) and its W offset of the s-th touching plane of the chunk
  static __device__ __forceinline__ void ip2_plane(const ItemDev& I, const PlaneDev* sp, int s, int* pl, int* woff) {
    int w = I.woff, seen = 0;
    for (int u = 0; u < I.np; ++u) {
      const PlaneDev& P = sp[I.p + u];
      if ((I.pad0 >> u) & 1) {
        if (seen == s) { *pl = I.p + u; *woff = w; return; }
        ++seen;
      }
      w += N * P.ncols_pad;
    }
    *pl = I.p; *woff = I.woff;
  }

  template <bool FWD>
  static __device__ __forceinline__ Src stage_src(const KParams& p, const ItemDev& I, const PlaneDev* sp, int s) {
    const C* slot = static_cast<const C*>(p.W) + (size_t)I.slot * p.slot_elems;
    if (FWD) {
      const PlaneDev& P = sp[I.p];
      if (I.type == 0) {   // F columns [c0 + s*LPC, ...), column-major, contiguous
        int c0;
        const int cnt = fp1_cols(P, I, &c0);
        const int cs = c0 + s * G::LPC;
        const int nc = cnt - s * G::LPC < G::LPC ? cnt - s * G::LPC : G::LPC;
        const C* F = static_cast<const C*>(p.F) + ((size_t)I.b * (H + 1) + cs) * N;
        return {F, (unsigned)(nc * N * G::ESZ)};
      }
      const int r0 = I.group * G::RP2 + s * G::LPR;   // W rows (row-major, stride ncols_pad)
      const int nr = N - r0 < G::LPR ? N - r0 : G::LPR;
      return {slot + I.woff + (size_t)r0 * P.ncols_pad, (unsigned)(nr * P.ncols_pad * G::ESZ)};
    }
    if (I.type == 0) {     // cube rows
      const int r0 = I.group * G::RPI + s * G::LPR;
      const int nr = N - r0 < G::LPR ? N - r0 : G::LPR;
      const C* src = static_cast<const C*>(p.coeff) + (((size_t)I.b * p.eta_l + I.p) * N + r0) * N;
      return {src, (unsigned)(nr * N * G::ESZ)};
    }
    int pl, woff;          // IP2: W columns of the s-th touching plane, intersected with the group
    ip2_plane(I, sp, s, &pl, &woff);
    const PlaneDev& P = sp[pl];
    const int g0 = I.group * G::LPC;
    const int lo = g0 > P.c_lo ? g0 : P.c_lo;
    const int hi_g = g0 + G::LPC < H + 1 ? g0 + G::LPC : H + 1;
    const int hi = hi_g < P.c_lo + P.ncols ? hi_g : P.c_lo + P.ncols;
    return {slot + woff + (size_t)(lo - P.c_lo) * N, (unsigned)((hi - lo) * N * G::ESZ)};
  }

  // ---------------------------------------------------------------- FP1: column IFFT
  template <typename Rel>
  static __device__ __forceinline__ void fp1_stage(const KParams& p, const Tabs<T>& tb, const ItemDev& I, const PlaneDev& P, int s,
                                   C* st, C* sc, Rel&& rel, bool& waited) {
    const int lane = threadIdx.x & 31, line = lane / G::THC, t = lane % G::THC;
    int c0;
    const int cnt = fp1_cols(P, I, &c0);
    const int cs = c0 + s * G::LPC;
    const int ci = s * G::LPC + line;
    const bool act = ci < cnt;
    const int cb = cs + line;
    C* col = st + line * N;
    // window at the lane's own rows: the (rolled) candidate loop scales the staged F values in
    // place, the (unrolled) register load masks the non-candidate rows to zero.  The forward's
    // 1/N^2 (a power of two: exact) is folded into the window.
    const T scale = T(1) / (T(N) * T(N));
    C r[G::EC];
    if (act && (p.dbg & 4)) {
#pragma unroll
      for (int q = 0; q < G::EC; ++q) r[q] = col[t + q * G::THC];
    } else if (act) {
      const ColSym cw(P, cb, tb.rt, p.j0, col_rec(p, P, cb));
#pragma unroll 1
      for (int q = 0; q < G::EC; ++q) {
        const int rb = t + q * G::THC;
        if (cw.cand(centred(rb, N))) col[rb] = cscale<T>(col[rb], cw.at(rb) * scale);
      }
#pragma unroll
      for (int q = 0; q < G::EC; ++q) {
        const int rb = t + q * G::THC;
        r[q] = cw.cand(centred(rb, N)) ? col[rb] : czero<T>();
      }
    } else {
#pragma unroll
      for (int q = 0; q < G::EC; ++q) r[q] = czero<T>();
    }
    FFST_WPROBE(p, s, 0);
    rel();
    if (!(p.dbg & 1)) LineFFT<T, N, true, N, true, G::EMC>::run(r, sc + line * G::SMC, t, tb.tw);
    FFST_WPROBE(p, s, 1);
    if (!waited) {                 // ring slot reuse: wait only before the first write
      if (I.wait_ctr >= 0 && lane == 0) spin_until(p.ctr + I.wait_ctr, I.wait_tgt);
      __syncwarp();
      waited = true;
    }
    FFST_WPROBE(p, s, 2);
    if (act && !(p.dbg & 2)) {
      C* w = static_cast<C*>(p.W) + (size_t)I.slot * p.slot_elems + I.woff + (cb - P.c_lo);
#pragma unroll
      for (int q = 0; q < G::EC; ++q) __stcg(w + (size_t)(t + q * G::THC) * P.ncols_pad, r[q]);
    }
    FFST_WPROBE(p, s, 3);
  }

  // ---------------------------------------------------------------- FP2: row C2R, two rows per line
  // Rows ra = r and rb = r + 1 of the plane are real (sym part) with Hermitian spectra Ta, Tb
  // (bins 0..H in W).  One complex inverse FFT of Z = Ta + i Tb over all N bins (bins above H from
  // the Hermitian mirror) gives x_ra + i x_rb.  The 1/N^2 is already in W (fp1_stage).
  template <typename Rel>
  static __device__ __forceinline__ void fp2_stage(const KParams& p, const Tabs<T>& tb, const ItemDev& I,
                                                   const PlaneDev& P, int s, const C* st, C* sc, Rel&& rel,
                                                   const T* gN, T (&gv)[G::EC]) {
    const int lane = threadIdx.x & 31, line = lane / G::THC, t = lane % G::THC;
    const int ra = I.group * G::RP2 + s * G::LPR + 2 * line;
    const bool act = 2 * line < G::LPR && ra < N;
    const C* wa = st + (2 * line) * P.ncols_pad - P.c_lo;
    const C* wb = wa + P.ncols_pad;
    const unsigned c_lo = (unsigned)P.c_lo, nc = (unsigned)P.ncols;
    C z[G::EC];
#pragma unroll
    for (int q = 0; q < G::EC; ++q) {
      const int c = t + q * G::THC;
      const bool up = c > H;
      const int k = up ? N - c : c;
      C a = czero<T>(), b = czero<T>();
      if (act && (unsigned)(k - (int)c_lo) < nc) {
        a = wa[k];
        b = wb[k];
      }
      // c <= H: Ta[c] + i Tb[c];  c > H: conj(Ta[N-c]) + i conj(Tb[N-c])
      z[q] = up ? mk<T>(a.x + b.y, b.x - a.y) : mk<T>(a.x - b.y, a.y + b.x);
    }
    rel();
    FFST_WPROBE(p, s, 0);
    if (!(p.dbg & 1)) LineFFT<T, N, true, N, true, G::EMC>::run(z, sc + line * G::SMC, t, tb.tw);
    FFST_WPROBE(p, s, 1);
    if (act && !(p.dbg & 2)) {
      C* outa = static_cast<C*>(p.coeff) + (((size_t)I.b * p.eta_l + I.p) * N + ra) * N;
      C* outb = outa + N;
      if (gN != nullptr) {   // rank-2 imaginary Nyquist term (-1)^r G(m1) + (-1)^m1 H(r)
        const T ha = gN[N + ra], hb = gN[N + ra + 1];
        const T sa = (ra & 1) ? T(-1) : T(1);
#pragma unroll
        for (int q = 0; q < G::EC; ++q) {
          const int m1 = t + q * G::THC;
          const T sm = (m1 & 1) ? T(-1) : T(1);
          __stcs(outa + m1, mk<T>(z[q].x, sa * gv[q] + sm * ha));
          __stcs(outb + m1, mk<T>(z[q].y, -sa * gv[q] + sm * hb));
        }
      } else {
#pragma unroll
        for (int q = 0; q < G::EC; ++q) {
          const int m1 = t + q * G::THC;
          __stcs(outa + m1, mk<T>(z[q].x, T(0)));
          __stcs(outb + m1, mk<T>(z[q].y, T(0)));
        }
      }
    }
    FFST_WPROBE(p, s, 2);
  }

  // ---------------------------------------------------------------- IP1: row R2C, two rows per line
  // Z = Re c(ra, .) + i Re c(rb, .), one forward FFT; the two real rows' spectra are
  // Xa[k] = (Z[k] + conj Z[N-k]) / 2 and Xb[k] = (Z[k] - conj Z[N-k]) / (2i), kept for the plane's
  // bins k in [c_lo, c_lo + ncols) -> W (column-major, the two rows adjacent: one 16-byte store).
  // Nyquist planes also accumulate the alternating sums of Im c.
  template <typename Rel>
  static __device__ __forceinline__ void ip1_stage(const KParams& p, const Tabs<T>& tb, const ItemDev& I,
                                                   const PlaneDev& P, int s, const C* st, C* sc, Rel&& rel,
                                                   T (&sacc)[G::EC], bool& waited) {
    const int lane = threadIdx.x & 31, line = lane / G::THC, t = lane % G::THC;
    const int ra = I.group * G::RPI + s * G::LPR + 2 * line;
    const bool act = 2 * line < G::LPR && ra < N;
    const bool nyq = P.nyq >= 0;
    const C* rowa = st + (2 * line) * N;
    const C* rowb = rowa + N;
    C z[G::EC];
    T ta = T(0), tb_ = T(0);
    const T sa = (ra & 1) ? T(-1) : T(1);
#pragma unroll
    for (int q = 0; q < G::EC; ++q) {
      C va = czero<T>(), vb = czero<T>();
      if (act) {
        va = rowa[t + q * G::THC];
        vb = rowb[t + q * G::THC];
      }
      z[q] = mk<T>(va.x, vb.x);
      if (nyq) {
        sacc[q] += sa * (va.y - vb.y);          // rows ra, ra+1 carry opposite signs
        const T sm = ((t + q * G::THC) & 1) ? T(-1) : T(1);
        ta += sm * va.y;
        tb_ += sm * vb.y;
      }
    }
    rel();
    FFST_WPROBE(p, s, 0);
    C* sl = sc + line * G::SMC;
    if (!(p.dbg & 1)) LineFFT<T, N, false, N, true, G::EMC>::run(z, sl, t, tb.tw);
    FFST_WPROBE(p, s, 1);
    if (nyq) {   // alternating row sums t(r) = sum_m1 (-1)^m1 Im c(r, m1), reduced over the line's lanes
      T va = ta, vb = tb_;
#pragma unroll
      for (int o = G::THC / 2; o > 0; o >>= 1) {
        va += __shfl_xor_sync(0xffffffffu, va, o);
        vb += __shfl_xor_sync(0xffffffffu, vb, o);
      }
      if (t == 0 && act) {
        T* tt = static_cast<T*>(p.nyq_T) + ((size_t)I.b * p.n_nyq + P.nyq) * N + ra;
        tt[0] = va;
        tt[1] = vb;
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < G::EC; ++q) sl[Pad<T, G::EMC>::at(t + q * G::THC)] = z[q];
    __syncwarp();
    if (!waited) {
      if (I.wait_ctr >= 0 && lane == 0) spin_until(p.ctr + I.wait_ctr, I.wait_tgt);
      __syncwarp();
      waited = true;
    }
    FFST_WPROBE(p, s, 2);
    if (act && !(p.dbg & 2)) {
      C* w = static_cast<C*>(p.W) + (size_t)I.slot * p.slot_elems + I.woff + ra;
#pragma unroll 4
      for (int kk = t; kk < P.ncols; kk += G::THC) {
        const int k = P.c_lo + kk;                       // 0..H
        const C zk = sl[Pad<T, G::EMC>::at(k)];
        const C zm = sl[Pad<T, G::EMC>::at(k == 0 ? 0 : N - k)];
        const C xa = mk<T>(T(0.5) * (zk.x + zm.x), T(0.5) * (zk.y - zm.y));
        const C xb = mk<T>(T(0.5) * (zk.y + zm.y), T(0.5) * (zm.x - zk.x));
        store_pair_cg<T>(w + (size_t)kk * N, xa, xb);
      }
    }
    FFST_WPROBE(p, s, 3);
  }

  // partial alternating column sums s(m1) over the item's rows: reduce over the warp's lines
  // (fixed order: deterministic), lanes of line 0 write
  static __device__ __forceinline__ void ip1_finish(const KParams& p, const ItemDev& I, const PlaneDev& P,
                                                    T (&sacc)[G::EC]) {
    const int lane = threadIdx.x & 31, line = lane / G::THC, t = lane % G::THC;
#pragma unroll
    for (int q = 0; q < G::EC; ++q) {
      T v = sacc[q];
#pragma unroll
      for (int o = G::THC; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      sacc[q] = v;
    }
    if (line == 0) {
      T* outp = static_cast<T*>(p.nyq_S) + (((size_t)I.b * p.n_nyq + P.nyq) * p.n_rowitems + I.group) * N;
#pragma unroll
      for (int q = 0; q < G::EC; ++q) outp[t + q * G::THC] = sacc[q];
    }
  }

  // ---------------------------------------------------------------- IP2: column FFT * window, accumulate
  template <typename Rel>
  static __device__ __forceinline__ void ip2_stage(const KParams& p, const Tabs<T>& tb, const ItemDev& I, const PlaneDev* sp, int s,
                                   const C* st, C* sc, Rel&& rel, C (&acc)[G::EC]) {
    const int lane = threadIdx.x & 31, line = lane / G::THC, t = lane % G::THC;
    int pl, woff;
    ip2_plane(I, sp, s, &pl, &woff);
    const PlaneDev& P = sp[pl];
    const int g0 = I.group * G::LPC;
    const int lo = g0 > P.c_lo ? g0 : P.c_lo;
    const int cb = g0 + line;
    const bool in = cb <= H && cb >= P.c_lo && cb < P.c_lo + P.ncols;
    const C* col = st + (cb - lo) * N;
    C r[G::EC];
#pragma unroll
    for (int q = 0; q < G::EC; ++q) r[q] = in ? col[t + q * G::THC] : czero<T>();
    rel();
    // window of this column at the lane's rows: candidate rows evaluated in a rolled loop into the
    // (already consumed) stage buffer, loaded back masked (non-candidates are zero)
    T wv[G::EC];
    T* wb = reinterpret_cast<T*>(sc) + line * N;
    if (in && (p.dbg & 4)) {
#pragma unroll
      for (int q = 0; q < G::EC; ++q) wv[q] = T(1);
    } else if (in) {
      const ColSym cw(P, cb, tb.rt, p.j0, col_rec(p, P, cb));
#pragma unroll 1
      for (int q = 0; q < G::EC; ++q) {
        const int rb = t + q * G::THC;
        if (cw.cand(centred(rb, N))) wb[rb] = cw.at(rb);
      }
#pragma unroll
      for (int q = 0; q < G::EC; ++q) {
        const int rb = t + q * G::THC;
        wv[q] = cw.cand(centred(rb, N)) ? wb[rb] : T(0);
      }
    } else {
#pragma unroll
      for (int q = 0; q < G::EC; ++q) wv[q] = T(0);
    }
    __syncwarp();
    constexpr int WOFF = G::WIN_C;   // FFT scratch after the window reals
    FFST_WPROBE(p, s, 0);
    if (!(p.dbg & 1)) LineFFT<T, N, false, N, true, G::EMC>::run(r, sc + WOFF + line * G::SMC, t, tb.tw);
    FFST_WPROBE(p, s, 1);
#pragma unroll
    for (int q = 0; q < G::EC; ++q) {
      acc[q].x += wv[q] * r[q].x;
      acc[q].y += wv[q] * r[q].y;
    }
  }

  static __device__ __forceinline__ void ip2_finish(const KParams& p, const ItemDev& I, C (&acc)[G::EC]) {
    const int lane = threadIdx.x & 31, line = lane / G::THC, t = lane % G::THC;
    if (I.wait2_ctr >= 0) {        // previous owner of this column group (accumulation chain)
      if (lane == 0) spin_until(p.ctr + I.wait2_ctr, 1);
      __syncwarp();
    }
    const int cb = I.group * G::LPC + line;
    if (cb <= H) {
      const int cbc = cb <= H ? cb : H;          // in range even if the loads below are hoisted
      C* a = static_cast<C*>(p.A) + (size_t)I.pad1 * p.a_lane_elems + ((size_t)I.b * (H + 1) + cbc) * N;
#pragma unroll
      for (int q = 0; q < G::EC; ++q) {
        const int idx = t + q * G::THC;
        if (I.first) {
          __stcg(a + idx, acc[q]);
        } else {
          const C o = __ldcg(a + idx);
          __stcg(a + idx, mk<T>(o.x + acc[q].x, o.y + acc[q].y));
        }
      }
    }
  }
};

// ------------------------------------------------------------------ the persistent warp loop
// Per-warp pipeline: two stage buffers (b = 0, 1) with one mbarrier each; `phase` holds the
// parity bit of each barrier.  No runtime-indexed arrays (they would live in local memory).
template <typename T, int N, bool FWD>
struct WarpLoop {
  using G = WGeo<T, N>;
  using W = WK<T, N>;
  using C = cpx<T>;

  const KParams& p;
  const PlaneDev* sp;
  Tabs<T> tb;
  C* buf0;
  unsigned long long* bar0;
  unsigned phase = 0;
  int cur = 0;
  int lane;

  __device__ C* buf(int b) const { return buf0 + b * G::STAGE_PAD; }
  __device__ unsigned long long* bar(int b) const { return bar0 + b; }

  // Item fetch through a per-CTA batch of `p.fetch_batch` consecutive queue items (one global
  // atomic per batch): the CTA's warps run neighbouring items -- the same item type, the same code
  // -- which keeps the instruction cache warm.  The host planner checks that no item depends on
  // an item less than fetch_batch positions before it (no deadlock inside a batch).
  unsigned long long* q;    // shared: (batch base << 32) | taken
  __device__ int fetch() const {
    int it = 0;
    if (lane == 0) {
      const unsigned B = (unsigned)p.fetch_batch;
      for (;;) {
        const unsigned long long old = atomicAdd(q, 1ull);
        const unsigned k = (unsigned)old, base = (unsigned)(old >> 32);
        if (k < B) { it = (int)(base + k); break; }
        if (k == B) {            // this warp refills the batch
          const unsigned nb = (unsigned)atomicAdd(p.ctr, (int)B);
          atomicExch(q, ((unsigned long long)nb << 32) | 1ull);
          it = (int)nb;
          break;
        }
        while ((unsigned)(*reinterpret_cast<volatile unsigned long long*>(q) >> 32) == base) __nanosleep(20);
      }
    }
    return __shfl_sync(0xffffffffu, it, 0);
  }
  // read dependency of an item: pass 2 reads what pass 1 of its chunk wrote
  __device__ bool read_ready(const ItemDev& I) const {
    if (I.type == 0) return true;
    int ok = 0;
    if (lane == 0) ok = ctr_reached(p.ctr + I.wait_ctr, I.wait_tgt) ? 1 : 0;
    return __shfl_sync(0xffffffffu, ok, 0) != 0;
  }
  __device__ void read_wait(const ItemDev& I) const {
    if (I.type == 0) return;
    if (lane == 0) spin_until(p.ctr + I.wait_ctr, I.wait_tgt);
    __syncwarp();
  }
  // issue stage s of item I into buffer b (lane 0).  Pass-2 items read data other SMs wrote with
  // generic stores through the async proxy: a proxy fence orders the copy after the counter poll.
  __device__ void issue(const ItemDev& I, int s, int b) const {
    const typename W::Src sc = W::template stage_src<FWD>(p, I, sp, s);
    if (lane == 0) {
      if (I.type == 1 && s == 0) fence_async_global();
      fence_async_smem();         // prior generic accesses of this buffer before the async write
      bulk_load(buf(b), sc.src, sc.bytes, bar(b));
    }
  }
  unsigned long long t_ready = 0;   // trace: first stage of the current item landed
  __device__ C* wait_stage(int b) {
    mbar_wait(bar(b), (phase >> b) & 1u);
    phase ^= 1u << b;
    if (p.trace != nullptr && t_ready == 0) t_ready = gtimer();
    return buf(b);
  }

  // Next-item bookkeeping shared by the item bodies.
  // The item descriptors live in shared memory (two slots per warp: current and next), not in
  // registers: the fields are re-read where used, which keeps the FFT register budget free.
  ItemDev* islot;   // shared [2]
  C* scr;           // per-warp scratch
  struct Next {
    int it;         // next item (valid if < n_items), fetched
    int slot;       // islot[slot] holds it
    int ns;
    int issued;     // its stages already issued (in order, from the buffer after the current item's)
    bool fetched;
  };
  __device__ void load_item_to(int slot, int it) const {
    if (lane < 4)
      reinterpret_cast<int4*>(islot + slot)[lane] =
          __ldg(reinterpret_cast<const int4*>(p.items + (it < p.n_items ? it : p.n_items - 1)) + lane);
    __syncwarp();
  }
  __device__ void fetch_next(Next& nx) const {
    nx.it = fetch();
    nx.ns = 0;
    nx.issued = 0;
    nx.fetched = true;
    nx.slot ^= 1;
    if (nx.it < p.n_items) {
      load_item_to(nx.slot, nx.it);
      nx.ns = W::template n_stages<FWD>(p, islot[nx.slot], sp);
    }
  }
  // Buffer b was just released after stage s of item I (ns stages): refill it with the stage two
  // ahead in this warp's sequence -- stage s+2 of I, or stage x = s+2-ns of the next item (stages
  // of the next item are issued in order; its first one only once its input is ready).
  __device__ void refill(const ItemDev& I, int s, int ns, Next& nx, int b) const {
    const int x = s + 2 - ns;
    if (x < 0) {
      issue(I, s + 2, b);
      return;
    }
    if (!nx.fetched) fetch_next(nx);
    if (nx.it >= p.n_items || nx.issued != x || x >= nx.ns) return;
    const ItemDev& J = islot[nx.slot];
    if (x == 0 && !read_ready(J)) return;
    issue(J, x, b);
    ++nx.issued;
  }

  // Stage loop of one item: body(s, stage, scratch, rel) reads stage s, calls rel() once it no
  // longer needs the stage buffer (the buffer is then refilled), and computes in the scratch.
  template <typename Body>
  __device__ void stages(const ItemDev& I, int ns, Next& nx, Body&& body) {
    nx.fetched = false;
    for (int s = 0; s < ns; ++s) {
      const int b = cur;
      C* st = wait_stage(b);
      if constexpr (G::EARLY) {
        auto rel = [&]() {
          __syncwarp();           // every lane done reading buffer b
          refill(I, s, ns, nx, b);
        };
        body(s, st, scr, rel);
        __syncwarp();             // scratch reuse by the next stage
      } else {
        auto rel = [&]() { __syncwarp(); };   // stage buffer is the scratch: refill after compute
        body(s, st, st, rel);
        __syncwarp();
        refill(I, s, ns, nx, b);
      }
      cur ^= 1;
    }
    if (!nx.fetched) fetch_next(nx);
  }

  __device__ void signal(const ItemDev& I, bool publishes) const {
    if (publishes) fence_async_global();   // generic writes before async-proxy readers
    __syncwarp();
    if (lane == 0) {
      if (publishes) red_release(p.ctr + I.sig_ctr, 1);
      else red_relaxed(p.ctr + I.sig_ctr, 1);       // reads only (TMA, completed): WAR release
      if (I.sig2_ctr >= 0) red_release(p.ctr + I.sig2_ctr, 1);
    }
  }

  __device__ void item_fp1(const ItemDev& I, int ns, Next& nx) {
    bool waited = false;
    const PlaneDev& P = sp[I.p];
    stages(I, ns, nx, [&](int s, C* st, C* sc, auto& rel) { W::fp1_stage(p, tb, I, P, s, st, sc, rel, waited); });
    signal(I, true);
  }
  __device__ void item_fp2(const ItemDev& I, int ns, Next& nx) {
    const PlaneDev& P = sp[I.p];
    T gv[G::EC];
    const T* gN = nullptr;
    if (P.nyq >= 0) {
      gN = static_cast<const T*>(p.nyq_fwd) + ((size_t)I.b * p.n_nyq + P.nyq) * 2 * N;
      const int t = lane % G::THC;
#pragma unroll
      for (int q = 0; q < G::EC; ++q) gv[q] = gN[t + q * G::THC];
    }
    stages(I, ns, nx, [&](int s, C* st, C* sc, auto& rel) { W::fp2_stage(p, tb, I, P, s, st, sc, rel, gN, gv); });
    signal(I, false);
  }
  __device__ void item_ip1(const ItemDev& I, int ns, Next& nx) {
    bool waited = false;
    const PlaneDev& P = sp[I.p];
    T sacc[G::EC];
#pragma unroll
    for (int q = 0; q < G::EC; ++q) sacc[q] = T(0);
    stages(I, ns, nx, [&](int s, C* st, C* sc, auto& rel) { W::ip1_stage(p, tb, I, P, s, st, sc, rel, sacc, waited); });
    if (P.nyq >= 0) W::ip1_finish(p, I, P, sacc);
    signal(I, true);
  }
  __device__ void item_ip2(const ItemDev& I, int ns, Next& nx) {
    C acc[G::EC];
#pragma unroll
    for (int q = 0; q < G::EC; ++q) acc[q] = czero<T>();
    stages(I, ns, nx, [&](int s, C* st, C* sc, auto& rel) { W::ip2_stage(p, tb, I, sp, s, st, sc, rel, acc); });
    W::ip2_finish(p, I, acc);
    signal(I, true);
  }

  __device__ void run() {
    Next nx;
    nx.slot = 1;
    fetch_next(nx);                // -> slot 0
    while (nx.it < p.n_items) {
      const ItemDev& I = islot[nx.slot];
      const int ns = nx.ns;
      const int it = nx.it;
      unsigned long long t_start = 0;
      if (p.trace != nullptr) {
        t_start = gtimer();
        t_ready = 0;
      }
      // prologue: the first two stages (those not already issued by the previous item)
      if (nx.issued == 0 && ns > 0) read_wait(I);
      for (int x = nx.issued; x < 2 && x < ns; ++x) issue(I, x, cur ^ (x & 1));
      if (FWD) {
        if (I.type == 0) item_fp1(I, ns, nx);
        else item_fp2(I, ns, nx);
      } else {
        if (I.type == 0) item_ip1(I, ns, nx);
        else item_ip2(I, ns, nx);
      }
      if (p.trace != nullptr && lane == 0) {
        unsigned long long* tr = p.trace + 8 * (size_t)it;
        tr[0] = (smid() << 8) | (threadIdx.x >> 5);
        tr[1] = t_start;
        tr[2] = t_ready ? t_ready : t_start;
        tr[3] = gtimer();
        const int w = threadIdx.x >> 5;
        tr[4] = s_wprobe[w][0]; tr[5] = s_wprobe[w][1]; tr[6] = s_wprobe[w][2]; tr[7] = s_wprobe[w][3];
        s_wprobe[w][0] = s_wprobe[w][1] = s_wprobe[w][2] = s_wprobe[w][3] = 0;
      }
    }
  }
};

template <typename T, int N, bool FWD>
__device__ __forceinline__ void warp_loop(const KParams& p) {
  using G = WGeo<T, N>;
  using C = cpx<T>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ PlaneDev s_planes[MAX_PLANES_SMEM];
  __shared__ unsigned long long s_q;
  __shared__ ItemDev s_items[G::NW][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_q = (unsigned long long)(unsigned)p.fetch_batch;   // empty batch: first taker refills
  C* stages = reinterpret_cast<C*>(smem_raw);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw + G::OFF_BARS);
  C* s_tw = reinterpret_cast<C*>(smem_raw + G::OFF_TW);
  T* s_rt = reinterpret_cast<T*>(smem_raw + G::OFF_RT);
  for (int i = threadIdx.x; i < p.eta_l; i += blockDim.x) s_planes[i] = p.planes[i];
  for (int i = threadIdx.x; i < N; i += blockDim.x) s_tw[i] = static_cast<const C*>(p.tw)[i];
  for (int i = threadIdx.x; i < (p.j0 + 1) * (N / 2 + 1); i += blockDim.x) s_rt[i] = static_cast<const T*>(p.rtab)[i];
  if (lane == 0) {
    mbar_init(bars + 2 * warp, 1);
    mbar_init(bars + 2 * warp + 1, 1);
  }
  fence_async_smem();
  __syncthreads();   // the only CTA barrier: plane table + barrier init
  C* wbase = stages + (size_t)warp * G::WARP_ELEMS;
  WarpLoop<T, N, FWD> L{p, s_planes, Tabs<T>{s_tw, s_rt}, wbase, bars + 2 * warp};
  L.scr = G::EARLY ? wbase + 2 * G::STAGE_PAD : nullptr;
  L.lane = lane;
  L.q = &s_q;
  L.islot = s_items[warp];
  L.run();
}

template <typename T, int N>
__global__ void __launch_bounds__(WGeo<T, N>::NT, 1) fwd_warp_kernel(KParams p) {
  warp_loop<T, N, true>(p);
}

template <typename T, int N>
__global__ void __launch_bounds__(WGeo<T, N>::NT, 1) inv_warp_kernel(KParams p) {
  warp_loop<T, N, false>(p);
}

}  // namespace ffst
