// ffst_math.cuh — complex helpers and the shearlet window psi_hat_i evaluated on
// the fly from integer frequencies (product code; shares nothing with oracle/).
//
// The window is the paper's cone-adapted Meyer shearlet system (Sec. 2-3.5):
//   v        eq:v
//   psi1     eq:Psi1     closed form of Sec. 3.4
//   psi2     eq:Psi2
//   varphi   P:L696-703 and the cone low-pass eq:phi P:L705-711
//   cones    P:L547-594; horizontal / vertical / glued seam P:L603-688
//   sampling psi_hat(Delta * u) on the centred integer grid u.
//
// Integer formulation: with u = (u1, u2) integers
// and Delta a power of two, the shear argument of a horizontal shearlet is
//   2^j * w2/w1 + k = (k*u1 + 2^j*u2) / u1
// so |arg| < 1  <=>  |k*u1 + 2^j*u2| < |u1|  is decided exactly in integers and
// 1 - |arg| = (|u1| - |num|)/|u1| is a single rounded division.  The radial
// argument 4^-j * Delta * |u1| is exact (powers of two).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#define FFST_HD __host__ __device__ __forceinline__

namespace ffst {

template <typename T> struct Cpx;
template <> struct Cpx<float> { using type = float2; };
template <> struct Cpx<double> { using type = double2; };
template <typename T> using cpx = typename Cpx<T>::type;

template <typename T> FFST_HD cpx<T> mk(T x, T y) { cpx<T> r; r.x = x; r.y = y; return r; }
template <typename T> FFST_HD cpx<T> cadd(cpx<T> a, cpx<T> b) { return mk<T>(a.x + b.x, a.y + b.y); }
template <typename T> FFST_HD cpx<T> csub(cpx<T> a, cpx<T> b) { return mk<T>(a.x - b.x, a.y - b.y); }
template <typename T> FFST_HD cpx<T> cmul(cpx<T> a, cpx<T> b) {
  return mk<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename T> FFST_HD cpx<T> cmulc(cpx<T> a, cpx<T> b) {
  return mk<T>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename T> FFST_HD cpx<T> conj_(cpx<T> a) { return mk<T>(a.x, -a.y); }
template <typename T> FFST_HD cpx<T> cscale(cpx<T> a, T s) { return mk<T>(a.x * s, a.y * s); }
template <typename T> FFST_HD cpx<T> czero() { return mk<T>(T(0), T(0)); }
// a + conj(b), a - conj(b), a + i b, -i s a, acc + w r (w real): the Hermitian split / merge steps of the
// real-data row passes and the window accumulation
template <typename T> FFST_HD cpx<T> cadd_conj(cpx<T> a, cpx<T> b) { return mk<T>(a.x + b.x, a.y - b.y); }
template <typename T> FFST_HD cpx<T> csub_conj(cpx<T> a, cpx<T> b) { return mk<T>(a.x - b.x, a.y + b.y); }
template <typename T> FFST_HD cpx<T> cadd_i(cpx<T> a, cpx<T> b) { return mk<T>(a.x - b.y, a.y + b.x); }
template <typename T> FFST_HD cpx<T> cscale_mi(cpx<T> a, T s) { return mk<T>(s * a.y, -s * a.x); }
template <typename T> FFST_HD cpx<T> cfma_real(T w, cpx<T> r, cpx<T> acc) { return mk<T>(acc.x + w * r.x, acc.y + w * r.y); }

// Packed float32 pairs (sm_100a FADD2 / FMUL2 / FFMA2: one instruction for both halves of a complex
// value; ptxas folds the half swaps, broadcasts and per-half signs into operand modifiers).  Same
// IEEE operations as the scalar forms (a product rounded, then one fused multiply-add).
// (-DFFST_NO_F32X2 builds the scalar forms: A/B measurements.)
#if defined(__CUDA_ARCH__) && !defined(FFST_NO_F32X2)
#define FFST_HAVE_F2 1
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; add.rn.f32x2 rc, ra, rb; mov.b64 {%0,%1}, rc;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; sub.rn.f32x2 rc, ra, rb; mov.b64 {%0,%1}, rc;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; mul.rn.f32x2 rc, ra, rb; mov.b64 {%0,%1}, rc;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc, rd; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; mov.b64 rc, {%6,%7}; "
      "fma.rn.f32x2 rd, ra, rb, rc; mov.b64 {%0,%1}, rd;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
template <> __device__ __forceinline__ float2 cadd<float>(float2 a, float2 b) { return f2_add(a, b); }
template <> __device__ __forceinline__ float2 csub<float>(float2 a, float2 b) { return f2_sub(a, b); }
template <> __device__ __forceinline__ float2 cmul<float>(float2 a, float2 b) {
  const float2 t = f2_mul(make_float2(a.y, a.y), make_float2(b.y, b.x));
  return f2_fma(make_float2(a.x, a.x), b, make_float2(-t.x, t.y));
}
template <> __device__ __forceinline__ float2 cmulc<float>(float2 a, float2 b) {
  const float2 t = f2_mul(make_float2(a.y, a.y), make_float2(b.y, b.x));
  return f2_fma(make_float2(a.x, a.x), make_float2(b.x, -b.y), t);
}
template <> __device__ __forceinline__ float2 cscale<float>(float2 a, float s) { return f2_mul(a, make_float2(s, s)); }
template <> __device__ __forceinline__ float2 cadd_conj<float>(float2 a, float2 b) { return f2_fma(b, make_float2(1.f, -1.f), a); }
template <> __device__ __forceinline__ float2 csub_conj<float>(float2 a, float2 b) { return f2_fma(b, make_float2(-1.f, 1.f), a); }
template <> __device__ __forceinline__ float2 cadd_i<float>(float2 a, float2 b) {
  return f2_fma(make_float2(b.y, b.x), make_float2(-1.f, 1.f), a);
}
template <> __device__ __forceinline__ float2 cscale_mi<float>(float2 a, float s) {
  return f2_mul(make_float2(a.y, a.x), make_float2(s, -s));
}
template <> __device__ __forceinline__ float2 cfma_real<float>(float w, float2 r, float2 acc) {
  return f2_fma(make_float2(w, w), r, acc);
}
#endif

// ---------------------------------------------------------------- window math

template <typename T> FFST_HD T sinpi_(T x);
template <typename T> FFST_HD T cospi_(T x);
#ifdef __CUDA_ARCH__
template <> FFST_HD float sinpi_<float>(float x) { return sinpif(x); }
template <> FFST_HD float cospi_<float>(float x) { return cospif(x); }
template <> FFST_HD double sinpi_<double>(double x) { return sinpi(x); }
template <> FFST_HD double cospi_<double>(double x) { return cospi(x); }
#else   // host planner (support / Nyquist classification only)
template <> FFST_HD float sinpi_<float>(float x) { return (float)sin(3.14159265358979323846 * x); }
template <> FFST_HD float cospi_<float>(float x) { return (float)cos(3.14159265358979323846 * x); }
template <> FFST_HD double sinpi_<double>(double x) { return sin(3.14159265358979323846 * x); }
template <> FFST_HD double cospi_<double>(double x) { return cos(3.14159265358979323846 * x); }
#endif

// Meyer's v on [0,1] (eq:v), reflected through v(x) = 1 - v(1-x) (Lemma P:L321-348)
// for x > 1/2 so the polynomial is always evaluated where it is small.
template <typename T> FFST_HD T meyer_v(T x) {
  if (x <= T(0)) return T(0);
  if (x >= T(1)) return T(1);
  const bool refl = x > T(0.5);
  const T y = refl ? T(1) - x : x;
  const T y2 = y * y;
  const T p = y2 * y2 * (T(35) + y * (T(-84) + y * (T(70) + y * T(-20))));
  return refl ? T(1) - p : p;
}

// psi1_hat(a), a >= 0, closed form P:L1824-1835; sin(pi/2 v) = sinpi(v/2).
template <typename T> FFST_HD T psi1_w(T a) {
  if (a <= T(0.5) || a >= T(4)) return T(0);
  if (a < T(1)) return sinpi_<T>(T(0.5) * meyer_v<T>(T(2) * a - T(1)));
  if (a <= T(2)) return T(1);
  return cospi_<T>(T(0.5) * meyer_v<T>(T(0.5) * a - T(1)));
}

// varphi(a), a >= 0
template <typename T> FFST_HD T varphi_w(T a) {
  if (a <= T(0.5)) return T(1);
  if (a >= T(1)) return T(0);
  return cospi_<T>(T(0.5) * meyer_v<T>(T(2) * a - T(1)));
}

// Plane descriptor shared by host planner and kernels.
struct PlaneDev {
  int gi;            // global 0-based flat index
  int kind;          // 0 low-pass, 1 h, 2 v, 3 x (ffst_kind)
  int j, k;          // scale, shear
  int c_lo, ncols;   // Hermitian-half column range [c_lo, c_lo + ncols), columns 0..n/2
  int ncols_pad;     // row stride of the forward intermediate
  int nyq;           // index among the plan's Nyquist planes, or -1
  int rec;           // user spectra: local plane index (block of the table)
};

// Radial factors.  psi1_hat(4^-j Delta a) and varphi(Delta a) depend only on the integer
// radius a = |u| (0 <= a <= n/2) and the scale: a per-plan (j0+1) x (n/2+1) table holds them
// (computed once in float64 from the closed forms above).  The 2-D window --
// cones, seam glue and the shear factor psi2 -- is still evaluated on the fly per element.
template <typename T> struct Radial {
  const T* tab;   // rows j < j0: psi1(4^-j Delta a); row j0: varphi(Delta a)
  int stride;     // n/2 + 1
  int j0;
  FFST_HD T ld(const T* a) const {
#ifdef __CUDA_ARCH__
    return __ldg(a);
#else
    return *a;
#endif
  }
  FFST_HD T psi1(int j, int a) const { return ld(tab + j * stride + a); }
  FFST_HD T phi(int a) const { return ld(tab + j0 * stride + a); }
  // smooth variant (Sec. smoothShearlets): rows of B_j(a) = varphi^2(4^-j Delta a),
  // j = 0..j0+1, then of D_j(a) = B_(j+1)(a) - B_j(a), j = 0..j0 (computed stably by the planner);
  // nullptr for the classic system.  Psi1(4^-j Delta u)^2 = B_(j+1)(a1) D_j(a2) + B_j(a2) D_j(a1):
  // eq:newPsi1 with the tensor scaling function eq:Phi, a sum of non-negative terms (no cancellation).
  const T* smooth = nullptr;
  FFST_HD T corona(int j, int a1, int a2) const {
    const T* B = smooth;
    const T* D = smooth + (j0 + 2) * stride;
    const T s = ld(B + (j + 1) * stride + a1) * ld(D + j * stride + a2) +
                ld(B + j * stride + a2) * ld(D + j * stride + a1);
    return s > T(0) ? sqrt(s) : T(0);
  }
};

// psi1_hat(4^-j Delta |ua|) psi2_hat((k ua + 2^j ub)/ua) for |ub| <= |ua| (cone shearlet,
// P:L845-848).
template <typename T> FFST_HD T cone_shearlet(int j, int k, int ua, int ub, const Radial<T>& R) {
  const int aa = ua < 0 ? -ua : ua;
  if (aa == 0) return T(0);                              // reading A5: 0 on w_a = 0
  const int num = k * ua + ub * (1 << j);                // exact (|num| < 2^24)
  const int anum = num < 0 ? -num : num;
  if (anum >= aa) return T(0);                           // |shear argument| >= 1 -> psi2 = 0
  const int ab = ub < 0 ? -ub : ub;
  const T r = R.smooth != nullptr ? R.corona(j, aa, ab) : R.psi1(j, aa);   // eq:Psi1 or eq:newPsi1
  if (r == T(0)) return T(0);
  const T t = T(aa - anum) / T(aa);                      // 1 - |argument|, one rounding
  return r * sqrt(meyer_v<T>(t));                        // psi2 = sqrt(v(1 - |x|))
}

// psi_hat_i(Delta u1, Delta u2) for integer u (u may be +n/2: the mirrored point).
template <typename T> FFST_HD T window(const PlaneDev& P, int u1, int u2, const Radial<T>& R) {
  const int a1 = u1 < 0 ? -u1 : u1, a2 = u2 < 0 ? -u2 : u2;
  if (P.kind == 0)                                        // eq:phi (classic) / eq:Phi (smooth)
    return R.smooth != nullptr ? R.phi(a1) * R.phi(a2) : R.phi(a2 <= a1 ? a1 : a2);
  if (P.kind == 1) {                                     // horizontal cone |u2| < |u1|
    return a2 < a1 ? cone_shearlet<T>(P.j, P.k, u1, u2, R) : T(0);
  }
  if (P.kind == 2) {                                     // vertical cone |u1| < |u2|
    return a1 < a2 ? cone_shearlet<T>(P.j, P.k, u2, u1, R) : T(0);
  }
  // glued seam shearlet: h on C^h, v on C^v, horizontal formula on the seam |u1| = |u2|
  if (a1 < a2) return cone_shearlet<T>(P.j, P.k, u2, u1, R);
  return cone_shearlet<T>(P.j, P.k, u1, u2, R);
}

// Point-symmetric part of the sampled window on the even grid:
// sym(u) = (w(u) + w(mirror u)) / 2 with w(mirror u) = psi(Delta u^), u^ = u with any
// -n/2 component replaced by +n/2 (psi is even).  anti = (w(u) - w(u^)) / 2 lives on the
// Nyquist row / column only.
template <typename T> FFST_HD T window_sym(const PlaneDev& P, int u1, int u2, int half, const Radial<T>& R) {
  const T w = window<T>(P, u1, u2, R);
  if (u1 != -half && u2 != -half) return w;
  const int e1 = u1 == -half ? half : u1, e2 = u2 == -half ? half : u2;
  return T(0.5) * (w + window<T>(P, e1, e2, R));
}
template <typename T> FFST_HD T window_anti(const PlaneDev& P, int u1, int u2, int half, const Radial<T>& R) {
  if (u1 != -half && u2 != -half) return T(0);
  const int e1 = u1 == -half ? half : u1, e2 = u2 == -half ? half : u2;
  return T(0.5) * (window<T>(P, u1, u2, R) - window<T>(P, e1, e2, R));
}

// Candidate rows of plane P in column u1 (a prefilter for the window evaluation; a superset of
// the rows where window_sym can be non-zero, from the same integer tests):
//   h part: the wedge |k u1 + 2^j u2| < |u1| is the open interval of u2 strictly between
//           (-|u1| - k u1)/2^j and (|u1| - k u1)/2^j;
//   v part: |u1| < |u2| and the radial band 1/2 < 4^-j Delta |u2| < 4;
//   low-pass: max(|u1|, |u2|) < 1/Delta.
struct ColBounds {
  int hlo, hhi;   // u2 interval (inclusive), empty if hlo > hhi
  int alo, ahi;   // |u2| interval (inclusive), empty if alo > ahi
};

FFST_HD int floordiv_(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

template <typename T> FFST_HD ColBounds col_bounds(const PlaneDev& P, int u1, int half, T delta) {
  ColBounds b{1, 0, 1, 0};
  const int a1 = u1 < 0 ? -u1 : u1;
  if (P.kind == 0) {
    const int A = (int)(T(1) / delta) + 1;
    if (a1 <= A) { b.hlo = -A; b.hhi = A; }
    return b;
  }
  const T s = delta * (T(1) / T(1 << (2 * P.j)));
  const int band_lo = (int)(T(0.5) / s), band_hi = (int)(T(4) / s) + 1;
  if ((P.kind == 1 || P.kind == 3) && a1 > 0 && a1 >= band_lo && a1 <= band_hi) {
    const int K = 1 << P.j, c = P.k * u1;
    b.hlo = floordiv_(-a1 - c, K);
    b.hhi = floordiv_(a1 - c, K) + 1;
    if (b.hlo < -a1) b.hlo = -a1;
    if (b.hhi > a1) b.hhi = a1;
  }
  if (P.kind == 2 || P.kind == 3) {
    b.alo = a1 > band_lo ? a1 : band_lo;
    b.ahi = band_hi < half ? band_hi : half;
  }
  return b;
}

FFST_HD bool col_candidate(const ColBounds& b, int u2) {
  const int a2 = u2 < 0 ? -u2 : u2;
  return (u2 >= b.hlo && u2 <= b.hhi) || (a2 >= b.alo && a2 <= b.ahi);
}

// natural FFT bin -> centred frequency in [-n/2, n/2)
FFST_HD int centred(int bin, int n) { return bin < (n >> 1) ? bin : bin - n; }

}  // namespace ffst
