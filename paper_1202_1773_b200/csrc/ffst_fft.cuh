// ffst_fft.cuh — register/shared-memory Stockham FFT of one line per thread group.
//
// A line of length L is held by TH = L/E threads, thread t owning the elements
// x[t + q*TH], q = 0..E-1 (E = min(L, 16)) in registers, both on input and on
// output (natural order, no bit reversal).  Passes are radix-16 in registers with
// the remainder radix (2/4/8) in the middle:  L = 16 * r * 16 for L in 512..4096,
// 16 * r for 32..256, single pass for L <= 16.  Between passes the line goes
// through shared memory once (Stockham autosort: read x[v + q L/R], write
// y[(v-k)R + k + q Ns], v = butterfly index, k = v mod Ns), so an L = 4096 line
// takes two exchanges.  Shared addresses are padded by one element per 16
// (float2) / 8 (double2) to break the power-of-two bank strides.
//
// Twiddles come from a plan-owned table tw[m] = exp(-2 pi i m / TWN) (read-only
// path); the inverse uses conj.  Transforms are unnormalised.
#pragma once
#include "ffst_math.cuh"

namespace ffst {

// --------------------------------------------------------------- in-register DFTs

template <typename T, bool INV> FFST_HD cpx<T> mul_mi(cpx<T> a) {   // * exp(-+ i pi/2)
  return INV ? mk<T>(-a.y, a.x) : mk<T>(a.y, -a.x);
}

// multiply by exp(-+ 2 pi i m / 16), m in 0..15 (compile time)
template <typename T, int M, bool INV> FFST_HD cpx<T> mul_w16(cpx<T> a) {
  constexpr int m = M & 15;
  if constexpr (m == 0) return a;
  else if constexpr (m == 4) return mul_mi<T, INV>(a);
  else if constexpr (m == 8) return mk<T>(-a.x, -a.y);
  else if constexpr (m == 12) return mul_mi<T, !INV>(a);
  else {
    constexpr double C[16] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                              0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
                              -1.0, -0.92387953251128675613, -0.70710678118654752440, -0.38268343236508977173,
                              0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613};
    constexpr double S[16] = {0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613,
                              1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                              0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
                              -1.0, -0.92387953251128675613, -0.70710678118654752440, -0.38268343236508977173};
    const T c = T(C[m]);
    const T s = INV ? T(S[m]) : T(-S[m]);      // exp(-+ i theta) = cos -+ i sin
#ifdef FFST_HAVE_F2
    if constexpr (sizeof(T) == 4) return cmul<T>(a, mk<T>(c, s));
#endif
    return mk<T>(a.x * c - a.y * s, a.x * s + a.y * c);
  }
}

template <typename T, bool INV> FFST_HD void dft2(cpx<T>& a0, cpx<T>& a1) {
  const cpx<T> s = cadd<T>(a0, a1), d = csub<T>(a0, a1);
  a0 = s; a1 = d;
}

template <typename T, bool INV> FFST_HD void dft4(cpx<T>& a0, cpx<T>& a1, cpx<T>& a2, cpx<T>& a3) {
  const cpx<T> s0 = cadd<T>(a0, a2), d0 = csub<T>(a0, a2);
#ifdef FFST_HAVE_F2
  if constexpr (sizeof(T) == 4) {   // d0 +- (-+ i) e as fused multiply-adds on the swapped pair
    const float2 s1 = f2_add(a1, a3), e = f2_sub(a1, a3);
    const float2 es = make_float2(e.y, e.x);
    const float sg = INV ? -1.f : 1.f;                  // * (-+ i): (e.y, -e.x) / (-e.y, e.x)
    a0 = f2_add(s0, s1); a2 = f2_sub(s0, s1);
    a1 = f2_fma(es, make_float2(sg, -sg), d0);
    a3 = f2_fma(es, make_float2(-sg, sg), d0);
    return;
  }
#endif
  const cpx<T> s1 = cadd<T>(a1, a3), d1 = mul_mi<T, INV>(csub<T>(a1, a3));
  a0 = cadd<T>(s0, s1); a2 = csub<T>(s0, s1);
  a1 = cadd<T>(d0, d1); a3 = csub<T>(d0, d1);
}

// natural order in, natural order out, R in {1,2,4,8,16}
template <typename T, int R, bool INV> struct DFT;
template <typename T, bool INV> struct DFT<T, 1, INV> {
  static FFST_HD void run(cpx<T>*) {}
};
template <typename T, bool INV> struct DFT<T, 2, INV> {
  static FFST_HD void run(cpx<T>* a) { dft2<T, INV>(a[0], a[1]); }
};
template <typename T, bool INV> struct DFT<T, 4, INV> {
  static FFST_HD void run(cpx<T>* a) { dft4<T, INV>(a[0], a[1], a[2], a[3]); }
};
template <typename T, bool INV> struct DFT<T, 8, INV> {
  static FFST_HD void run(cpx<T>* a) {
    cpx<T> e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
    cpx<T> o0 = a[1], o1 = a[3], o2 = a[5], o3 = a[7];
    dft4<T, INV>(e0, e1, e2, e3);
    dft4<T, INV>(o0, o1, o2, o3);
    o1 = mul_w16<T, 2, INV>(o1);
    o2 = mul_w16<T, 4, INV>(o2);
    o3 = mul_w16<T, 6, INV>(o3);
    a[0] = cadd<T>(e0, o0); a[4] = csub<T>(e0, o0);
    a[1] = cadd<T>(e1, o1); a[5] = csub<T>(e1, o1);
    a[2] = cadd<T>(e2, o2); a[6] = csub<T>(e2, o2);
    a[3] = cadd<T>(e3, o3); a[7] = csub<T>(e3, o3);
  }
};
template <typename T, bool INV> struct DFT<T, 16, INV> {
  // x[4 n1 + n2] -> X[q1 + 4 q2]: DFT4 over n1, twiddle W16^(n2 q1), DFT4 over n2
  static FFST_HD void run(cpx<T>* a) {
    dft4<T, INV>(a[0], a[4], a[8], a[12]);
    dft4<T, INV>(a[1], a[5], a[9], a[13]);
    dft4<T, INV>(a[2], a[6], a[10], a[14]);
    dft4<T, INV>(a[3], a[7], a[11], a[15]);
    // now a[4 q1 + n2] = Y[n2][q1]
    a[5] = mul_w16<T, 1, INV>(a[5]);
    a[6] = mul_w16<T, 2, INV>(a[6]);
    a[7] = mul_w16<T, 3, INV>(a[7]);
    a[9] = mul_w16<T, 2, INV>(a[9]);
    a[10] = mul_w16<T, 4, INV>(a[10]);
    a[11] = mul_w16<T, 6, INV>(a[11]);
    a[13] = mul_w16<T, 3, INV>(a[13]);
    a[14] = mul_w16<T, 6, INV>(a[14]);
    a[15] = mul_w16<T, 9, INV>(a[15]);
    dft4<T, INV>(a[0], a[1], a[2], a[3]);
    dft4<T, INV>(a[4], a[5], a[6], a[7]);
    dft4<T, INV>(a[8], a[9], a[10], a[11]);
    dft4<T, INV>(a[12], a[13], a[14], a[15]);
    // now a[4 q1 + q2] = X[q1 + 4 q2]: transpose the 4x4 index
    cpx<T> t;
#define FFST_SW(i, j) t = a[i]; a[i] = a[j]; a[j] = t;
    FFST_SW(1, 4) FFST_SW(2, 8) FFST_SW(3, 12) FFST_SW(6, 9) FFST_SW(7, 13) FFST_SW(11, 14)
#undef FFST_SW
  }
};

// --------------------------------------------------------------- line FFT

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// Padded shared-memory index of a line: one pad element per 2^SH elements.  The Stockham write of
// the first pass has lane stride R = EM: padding every EM (float2) elements makes it conflict-free.
template <typename T, int EM = 16> struct Pad {
  static constexpr int SH = sizeof(cpx<T>) == 8 ? (EM == 8 ? 3 : 4) : 3;
  static FFST_HD int at(int i) { return i + (i >> SH); }
  static constexpr int len(int L) { return L + (L >> SH) + 1; }
  // at(i0 + q S) = at(i0) + q step(S) for i0 >= 0 when S is a multiple of the pad period (or S = 1 and
  // i0 a multiple of it, q below it): strided accesses become base + immediate offsets
  static constexpr bool linear(int S, int Q) { return S % (1 << SH) == 0 || (S == 1 && Q <= (1 << SH)); }
  static constexpr int step(int S) { return S % (1 << SH) == 0 ? S + (S >> SH) : 1; }
};

// Pass plan of a length-L line with EM (8 or 16) elements per thread: radix-EM passes with the
// remainder radix in the middle pass.
template <int L, int EM = 16> struct RadixPlan {
  static constexpr int M = ilog2(L);
  static constexpr int LE = ilog2(EM);
  static constexpr int E = L < EM ? L : EM;
  static constexpr int P = M <= LE ? 1 : (M <= 2 * LE ? 2 : 3);
  static_assert(M <= 3 * LE, "line too long for three passes");
  static constexpr int rad(int s) {
    return P == 1 ? L : (P == 2 ? (s == 0 ? EM : (1 << (M - LE))) : (s == 1 ? (1 << (M - 2 * LE)) : EM));
  }
};

// Barrier of one line's TH threads: a warp barrier (TH <= 32), else the CTA barrier, or with NAMED
// the line's own named barrier (id 1 + threadIdx.x / TH, TH threads) -- the lines of a CTA then
// run out of step with each other (their barrier waits overlap the other lines' work).  NAMED
// requires every use of the line's scratch to be ordered by the line's own threads only.
template <int TH, bool NAMED = false> struct SyncOf {
  static __device__ __forceinline__ void sync() {
    if constexpr (TH <= 32) __syncwarp();
    else if constexpr (NAMED) asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / TH)), "n"(TH) : "memory");
    else __syncthreads();
  }
};

// TWS: the twiddle table is in shared memory (plain loads) instead of global (read-only path).
template <typename T, int L, bool INV, int TWN, bool TWS = false, int EM = 16, bool TW2 = false, bool NAMED = false>
struct LineFFT {
  using RP = RadixPlan<L, EM>;
  static constexpr int E = RP::E;
  static constexpr int TH = L / E;
  static constexpr int SMLEN = Pad<T, EM>::len(L);   // shared elements per line

  template <int S, int NS>
  static __device__ __forceinline__ void pass(cpx<T> (&r)[E], cpx<T>* sm, int t, const cpx<T>* __restrict__ tw) {
    constexpr int R = RP::rad(S);
    constexpr int NB = E / R;          // butterflies per thread
    constexpr bool FIRST = (S == 0), LAST = (S == RP::P - 1);
    cpx<T> x[E];
    if constexpr (FIRST) {
      // register layout: butterfly b, input q is r[b + q * NB]; regroup to x[b*R+q]
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int q = 0; q < R; ++q) x[b * R + q] = r[b + q * NB];
    } else {
      using PD = Pad<T, EM>;
      static_assert(PD::linear(L / R, R), "strided reads: linear padded addresses");
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const cpx<T>* s0 = sm + PD::at(t + b * TH);
#pragma unroll
        for (int q = 0; q < R; ++q) x[b * R + q] = s0[q * PD::step(L / R)];
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      cpx<T>* xb = x + b * R;
      if constexpr (NS > 1) {
        const int v = t + b * TH;
        const int k = v & (NS - 1);
        if constexpr (TWS) {
          // one table read per butterfly, w^q by products (w^2q = (w^q)^2, w^(q+1) = w^q w):
          // shared-memory bandwidth is the scarce resource on this path, the FMA pipe is not.
          // TW2 (two-level table in shared memory, TWN/64 + 64 entries): w^m = hi[m / 64] lo[m % 64]
          cpx<T> wp[R];
          if constexpr (TW2) {
            const int m = k * (TWN / (NS * R));
            wp[1] = cmul<T>(tw[m >> 6], tw[TWN / 64 + (m & 63)]);
          } else {
            wp[1] = tw[k * (TWN / (NS * R))];
          }
#pragma unroll
          for (int q = 2; q < R; ++q) wp[q] = (q & 1) ? cmul<T>(wp[q - 1], wp[1]) : cmul<T>(wp[q / 2], wp[q / 2]);
#pragma unroll
          for (int q = 1; q < R; ++q) xb[q] = INV ? cmulc<T>(xb[q], wp[q]) : cmul<T>(xb[q], wp[q]);
        } else {
#pragma unroll
          for (int q = 1; q < R; ++q) {
            const cpx<T> w = __ldg(tw + (q * k) * (TWN / (NS * R)));
            xb[q] = INV ? cmulc<T>(xb[q], w) : cmul<T>(xb[q], w);
          }
        }
      }
      DFT<T, R, INV>::run(xb);
    }
    if constexpr (LAST) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int q = 0; q < R; ++q) r[b + q * NB] = x[b * R + q];
    } else {
      if constexpr (!FIRST) SyncOf<TH, NAMED>::sync();   // all reads of this pass done
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int v = t + b * TH;
        const int k = v & (NS - 1);
        const int base = (v - k) * R + k;
        using PD = Pad<T, EM>;
        if constexpr (PD::linear(NS, R) && (NS > 1 || R % (1 << PD::SH) == 0)) {
          cpx<T>* d0 = sm + PD::at(base);
#pragma unroll
          for (int q = 0; q < R; ++q) d0[q * PD::step(NS)] = x[b * R + q];
        } else {
#pragma unroll
          for (int q = 0; q < R; ++q) sm[PD::at(base + q * NS)] = x[b * R + q];
        }
      }
      SyncOf<TH, NAMED>::sync();                     // writes visible to the next pass
      pass<S + 1, NS * R>(r, sm, t, tw);
    }
  }

  // In: thread t holds x[t + q*TH] in r[q].  Out: X[t + q*TH] in r[q].
  // sm: this line's scratch (SMLEN elements); callers must not touch it concurrently.
  // All threads of the CTA (TH > 32) or warp (TH <= 32) must call run() together.
  static __device__ __forceinline__ void run(cpx<T> (&r)[E], cpx<T>* sm, int t, const cpx<T>* __restrict__ tw) {
    if constexpr (RP::P == 1) {
      DFT<T, L, INV>::run(r);
    } else {
      pass<0, 1>(r, sm, t, tw);
    }
  }
};

}  // namespace ffst
