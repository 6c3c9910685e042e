// ffst_api.cu — host planner and the C ABI of include/ffst.h.
//
// The planner turns (n, j0, batch, shard) into:
//  * the local plane table (flat index order of Sec. 3.5.1), each plane's
//    Hermitian-half column range (pruning of the first FFT pass) and Nyquist flag;
//  * the work queues of the persistent kernels: units (image, plane) grouped into
//    single-image chunks whose intermediates fit one ring slot (L2-resident), items
//    ordered P1(0), P1(1), P2(0), P1(2), P2(1), ... so that every dependency of an
//    item is an earlier item (deadlock-free dynamic scheduling);
//  * all device workspace, allocated once here (no allocation per call).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/ffst.h"
#include "ffst_generic.cuh"
#include "ffst_internal.h"

using namespace ffst;

namespace {

thread_local std::string g_detail;

ffst_status fail(ffst_status s, const std::string& why) {
  g_detail = why;
  return s;
}

ffst_status cuda_fail(cudaError_t e, const char* where) {
  g_detail = std::string(where) + ": " + cudaGetErrorString(e);
  return FFST_ERR_CUDA;
}

#define API_NCCL(x, where)                                                        \
  do {                                                                            \
    ncclResult_t r_ = (x);                                                        \
    if (r_ != ncclSuccess) {                                                      \
      g_detail = std::string(where) + ": " + ncclGetErrorString(r_);              \
      return FFST_ERR_NCCL;                                                       \
    }                                                                             \
  } while (0)

#define API_CUDA(x, where)                       \
  do {                                           \
    cudaError_t e_ = (x);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

int default_j0(int n) {
  int bits = 0;
  while ((1 << (bits + 1)) <= n) ++bits;   // floor(log2 n)
  return bits / 2;
}

struct Triple { int kind, j, k; };

std::vector<Triple> index_table(int j0) {
  std::vector<Triple> t;
  t.push_back({0, 0, 0});
  for (int j = 0; j < j0; ++j) {
    const int K = 1 << j;
    t.push_back({1, j, 0});
    for (int k = -1; k > -K; --k) t.push_back({1, j, k});
    t.push_back({3, j, -K});
    for (int k = -K + 1; k < K; ++k) t.push_back({2, j, k});
    t.push_back({3, j, K});
    for (int k = K - 1; k > 0; --k) t.push_back({1, j, k});
  }
  return t;
}

// Delta = 2^(2 j0) / (N_odd - 1) with N_odd = n (odd n) or n + 1 (even n)
double grid_delta(int n, int j0) { return std::ldexp(1.0, 2 * j0) / (double)(n % 2 ? n - 1 : n); }

// Superset of the columns c = |u1| (0..n/2) where the plane can be non-zero.
void plane_columns(int n, int j0, const Triple& tr, int* lo, int* hi) {
  const int H = n / 2;
  const double delta = grid_delta(n, j0);
  auto clampi = [&](long v) { return (int)std::max(0L, std::min((long)H, v)); };
  if (tr.kind == 0) {
    *lo = 0;
    *hi = clampi((long)std::ceil(1.0 / delta));
    return;
  }
  const double s = delta / std::ldexp(1.0, 2 * tr.j);      // 4^-j Delta
  const long band_lo = (long)std::floor(0.5 / s);           // psi1(s a) > 0  <=>  1/2 < s a < 4
  const long band_hi = (long)std::ceil(4.0 / s);
  const int K = 1 << tr.j;
  const int ak = std::abs(tr.k);
  int hlo = H + 1, hhi = -1, vlo = H + 1, vhi = -1;
  if (tr.kind == 1 || tr.kind == 3) {
    hlo = clampi(band_lo);
    hhi = clampi(band_hi);
  }
  if (tr.kind == 2 || tr.kind == 3) {
    const long u2max = std::min((long)H, band_hi);
    const double frac_hi = std::min(1.0, (double)(1 + ak) / K);
    vhi = clampi((long)std::ceil(u2max * frac_hi) + 1);
    vlo = ak >= 2 ? clampi((long)std::floor(band_lo * (double)(ak - 1) / K) - 1) : 0;
  }
  *lo = std::min(hlo, vlo);
  *hi = std::max(hhi, vhi);
}

// Plane-to-rank map.  LPT: planes by decreasing cost n/2 + (pruned column count)
// -- the row pass plus the pruned column pass of a direction, in line FFTs -- each dealt to the
// least-loaded rank (lowest rank on ties); round robin: plane i on rank i mod G.
std::vector<int> shard_owner(int n, int j0, int eta, int count, int policy) {
  std::vector<int> owner(eta);
  if (policy == FFST_SHARD_ROUND_ROBIN || count <= 1) {
    for (int i = 0; i < eta; ++i) owner[i] = i % std::max(1, count);
    return owner;
  }
  const auto table = index_table(j0);
  std::vector<std::pair<long, int>> order;
  for (int i = 0; i < eta; ++i) {
    int lo, hi;
    plane_columns(n, j0, table[i], &lo, &hi);
    order.push_back({-(long)(n / 2 + (hi - lo + 1)), i});
  }
  std::sort(order.begin(), order.end());
  std::vector<long> load(count, 0);
  for (auto& o : order) {
    int r = 0;
    for (int q = 1; q < count; ++q)
      if (load[q] < load[r]) r = q;
    owner[o.second] = r;
    load[r] += -o.first;
  }
  return owner;
}

// Radial factor table (float64): rows j < j0: psi1_hat(4^-j Delta a) by the closed form of
// P:L1824-1835; row j0: varphi(Delta a); a = 0 .. n/2.
std::vector<double> radial_table(int n, int j0) {
  const int H = n / 2;
  const double delta = grid_delta(n, j0);
  const double pi = 3.14159265358979323846;
  auto v = [](double x) {
    if (x <= 0) return 0.0;
    if (x >= 1) return 1.0;
    const bool refl = x > 0.5;
    const double y = refl ? 1 - x : x, y2 = y * y;
    const double p = y2 * y2 * (35 + y * (-84 + y * (70 - 20 * y)));
    return refl ? 1 - p : p;
  };
  std::vector<double> t((size_t)(j0 + 1) * (H + 1));
  for (int j = 0; j <= j0; ++j)
    for (int a = 0; a <= H; ++a) {
      double val;
      if (j < j0) {
        const double x = std::ldexp(delta * a, -2 * j);
        if (x <= 0.5 || x >= 4) val = 0;
        else if (x < 1) val = std::sin(pi / 2 * v(2 * x - 1));
        else if (x <= 2) val = 1;
        else val = std::cos(pi / 2 * v(x / 2 - 1));
      } else {
        const double x = delta * a;
        if (x <= 0.5) val = 1;
        else if (x >= 1) val = 0;
        else val = std::cos(pi / 2 * v(2 * x - 1));
      }
      t[(size_t)j * (H + 1) + a] = val;
    }
  return t;
}

// Smooth-variant rows appended to the radial table (Sec. smoothShearlets):
// B_j(a) = varphi^2(4^-j Delta a), j = 0..j0+1, then D_j(a) = varphi^2(4^-(j+1) Delta a) -
// varphi^2(4^-j Delta a), j = 0..j0, each written piecewise from eq:varphi so that
// no difference of nearly equal numbers is formed: with x = 4^-j Delta a, D = 0 (x <= 1/2),
// sin^2(pi/2 v(2x-1)) (1/2 < x < 1), 1 (1 <= x <= 2), cos^2(pi/2 v(x/2-1)) (2 < x < 4), 0 (x >= 4).
std::vector<double> smooth_rows(int n, int j0) {
  const int H = n / 2;
  const double delta = grid_delta(n, j0);
  const double pi = 3.14159265358979323846;
  auto v = [](double x) {
    if (x <= 0) return 0.0;
    if (x >= 1) return 1.0;
    const bool refl = x > 0.5;
    const double y = refl ? 1 - x : x, y2 = y * y;
    const double p = y2 * y2 * (35 + y * (-84 + y * (70 - 20 * y)));
    return refl ? 1 - p : p;
  };
  auto phi2 = [&](double x) {
    if (x <= 0.5) return 1.0;
    if (x >= 1) return 0.0;
    const double c = std::cos(pi / 2 * v(2 * x - 1));
    return c * c;
  };
  auto dif = [&](double x) {
    if (x <= 0.5 || x >= 4) return 0.0;
    if (x < 1) { const double s = std::sin(pi / 2 * v(2 * x - 1)); return s * s; }
    if (x <= 2) return 1.0;
    const double c = std::cos(pi / 2 * v(x / 2 - 1));
    return c * c;
  };
  std::vector<double> t((size_t)(2 * j0 + 3) * (H + 1));
  for (int j = 0; j <= j0 + 1; ++j)
    for (int a = 0; a <= H; ++a) t[(size_t)j * (H + 1) + a] = phi2(std::ldexp(delta * a, -2 * j));
  for (int j = 0; j <= j0; ++j)
    for (int a = 0; a <= H; ++a) t[(size_t)(j0 + 2 + j) * (H + 1) + a] = dif(std::ldexp(delta * a, -2 * j));
  return t;
}

// The plan's whole radial table: classic rows, then the smooth rows when variant == FFST_SMOOTH.
std::vector<double> radial_all(int n, int j0, int variant) {
  std::vector<double> t = radial_table(n, j0);
  if (variant == FFST_SMOOTH) {
    const std::vector<double> s = smooth_rows(n, j0);
    t.insert(t.end(), s.begin(), s.end());
  }
  return t;
}

Radial<double> host_radial(const std::vector<double>& tab, int n, int j0, int variant) {
  Radial<double> R{tab.data(), n / 2 + 1, j0};
  if (variant == FFST_SMOOTH) R.smooth = tab.data() + (size_t)(j0 + 1) * (n / 2 + 1);
  return R;
}

bool plane_nyquist(int n, int j0, const Triple& tr, int variant) {
  PlaneDev P{};
  P.kind = tr.kind; P.j = tr.j; P.k = tr.k;
  const int H = n / 2;
  const std::vector<double> tab = radial_all(n, j0, variant);
  const Radial<double> R = host_radial(tab, n, j0, variant);
  for (int u = -H; u < H; ++u) {
    if (window_anti<double>(P, u, -H, H, R) != 0.0) return true;
    if (window_anti<double>(P, -H, u, H, R) != 0.0) return true;
  }
  return false;
}

struct Queue {
  int batch = 0;
  int n_chunks = 0, n_fwd = 0, n_inv = 0, n_g = 0;
  int a_lanes = 1;                    // accumulator lanes of the inverse (copies of A summed at the end)
  long long slot_elems = 0;
  int nslots = 0;
  UnitDev* d_units = nullptr;
  ChunkDev* d_chunks = nullptr;
  ItemDev* d_fwd = nullptr;
  ItemDev* d_inv = nullptr;
};

}  // namespace

struct ffst_plan {
  ffst_plan_desc d{};
  int n = 0, j0 = 0, eta = 0, eta_l = 0, H = 0;
  size_t rsz = 0;       // bytes per real
  double delta = 0;
  std::vector<PlaneDev> planes;
  std::vector<int> nyq;
  Geometry geo{};
  int sm_count = 0, grid_fwd = 0, grid_inv = 0;
  int workers = 0;                // concurrent item consumers (CTAs) of the persistent kernels
  long long slot_budget = 0;
  int chunk_planes = 4;           // max planes per chunk (pipelining granularity of the passes)
  int acc_lanes = 4;              // max accumulator lanes of the inverse (FFST_ACC_LANES)
  // device memory
  PlaneDev* d_planes = nullptr;
  int* d_nyq = nullptr;
  void* d_tw = nullptr;
  void* d_rtab = nullptr;
  void *F = nullptr, *Fscr = nullptr, *A = nullptr, *W = nullptr;
  long long W_elems = 0;
  void *nyq_fwd = nullptr, *nyq_S = nullptr, *nyq_T = nullptr, *corr = nullptr, *nyq_anti = nullptr;
  void* nyq_part = nullptr;
  void* stage = nullptr;          // host-variant image staging [batch][n][n]
  int* d_ctr = nullptr;
  size_t ctr_cap = 0;
  int n_rowitems = 0;
  int rpi = 0;                    // inverse pass 1: rows per item
  std::map<int, Queue> queues;
  size_t ws_bytes = 0;
  bool timing = false;
  unsigned long long* d_trace[2] = {nullptr, nullptr};   // per-item traces (fwd, inv), optional
  int trace_items[2] = {0, 0};
  bool tracing = false;
  cudaEvent_t ev[8] = {};
  cudaStream_t aux = nullptr;     // side stream of the inverse (Nyquist correction beside the final column pass)
  ncclComm_t comm = nullptr;      // desc.nccl_comm (not owned): the library's exchange steps
  cudaStream_t cs = nullptr;      // comm stream (broadcast / reduce, chunked by image groups)
  cudaEvent_t cev[6] = {};        // [0] start, [1..4] image groups, [5] adjoint spectra final
  cudaEvent_t fork[2] = {};
  int launches[2] = {0, 0};
  std::vector<void*> allocs;
  // small-n fused path (ffst_tiny.cuh): one CTA per (plane, image), n <= 64
  bool tiny = false;
  void* part = nullptr;           // [batch][eta_l][n][n] T partial images of its inverse
  // arbitrary-n path (ffst_generic.cuh): full complex 2-D transforms, Bluestein line DFTs
  bool generic = false;
  int gen_M = 0, gen_np = 0;      // Bluestein FFT length, planes per chunk
  void *g_chirp = nullptr, *g_bhat = nullptr, *g_twm = nullptr, *g_usr = nullptr;
  void *Ft = nullptr, *S = nullptr, *At = nullptr, *Wt = nullptr, *W2 = nullptr;
  int* g_gidx = nullptr;
  // user spectra (f4, ffst_plan_create_user)
  void* d_usym = nullptr;         // [eta_l][n/2+1][n] T symmetric parts
  double tightness = -1, asymmetry = -1;   // admission check; -1: not computed yet
};

namespace {

template <typename T>
void fill_twiddles(std::vector<unsigned char>& buf, int n) {
  buf.resize((size_t)n * sizeof(cpx<T>));
  cpx<T>* tw = reinterpret_cast<cpx<T>*>(buf.data());
  for (int m = 0; m < n; ++m) {
    // exp(-2 pi i m / n) from the angle reduced to [0, pi/4] for accuracy
    const long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)m / (long double)n;
    tw[m].x = (T)cosl(a);
    tw[m].y = (T)(-sinl(a));
  }
}

ffst_status dalloc(ffst_plan* p, void** ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FFST_ERR_OOM, std::string("cudaMalloc ") + std::to_string(bytes) + " bytes: " + cudaGetErrorString(e));
  }
  p->allocs.push_back(*ptr);
  p->ws_bytes += bytes;
  return FFST_OK;
}

#define TRY(x) do { ffst_status s_ = (x); if (s_ != FFST_OK) return s_; } while (0)

// Work queues of the persistent kernels for `batch` images.
//
// 1. Chunks: consecutive planes of ONE image, at most chunk_planes planes and
//    slot_budget elements of intermediates.
// 2. Chunk order S: images in groups of Wg, round-robin over the chunk index inside
//    a group, so two chunks of the same image are Wg apart (the inverse chains the
//    accumulation of one image's chunks per column group).
// 3. Lookahead D: P2(S_c) is queued after P1(S_{c+D}); D is the smallest number of
//    chunks whose items cover ~3 waves of the grid, so the pass-1 items a pass-2 item
//    depends on have normally finished by the time it is dispatched.  The ring has
//    R = D + 2 slots; P1(S_c) reuses the slot of S_{c-R}, whose P2 items are queued
//    earlier.  Every dependency of an item is an earlier item: deadlock-free.
ffst_status build_queue(ffst_plan* p, int batch, Queue** out) {
  auto it = p->queues.find(batch);
  if (it != p->queues.end()) { *out = &it->second; return FFST_OK; }
  if (batch < 1 || batch > p->d.batch) return fail(FFST_ERR_INVALID_ARG, "batch outside 1..plan batch");
  const int N = p->n, H = p->H;
  const Geometry& g = p->geo;
  // ---- 1. chunks per image (in image order)
  struct Proto { int b, lp0, np; long long elems; };
  std::vector<Proto> protos;
  for (int b = 0; b < batch; ++b) {
    int lp0 = 0;
    long long used = 0;
    for (int lp = 0; lp < p->eta_l; ++lp) {
      const long long need = (long long)N * p->planes[lp].ncols_pad;
      const int in_chunk = lp - lp0;
      if (in_chunk > 0 && (used + need > p->slot_budget || in_chunk >= p->chunk_planes)) {
        protos.push_back({b, lp0, in_chunk, used});
        lp0 = lp;
        used = 0;
      }
      used += need;
    }
    protos.push_back({b, lp0, p->eta_l - lp0, used});
  }
  const int chunks_per_image = (int)protos.size() / batch;   // identical for every image
  auto items_fwd = [&](const Proto& c) {
    int n1 = 0;
    for (int lp = c.lp0; lp < c.lp0 + c.np; ++lp) n1 += (p->planes[lp].ncols + g.gc - 1) / g.gc;
    return n1 + c.np * ((N + g.rp2 - 1) / g.rp2);
  };
  double avg_items = 0;
  long long slot = 0;
  for (auto& c : protos) {
    avg_items += items_fwd(c);
    slot = std::max(slot, c.elems);
  }
  avg_items /= (double)protos.size();
  const int grid = p->workers;
  // Lookahead: at least ~3 waves of items, and as far as the ring allows (item counts
  // under-estimate the lookahead when pass-1 items are few and long, e.g. n = 4096).
  int D = (int)std::ceil(3.0 * grid / std::max(1.0, avg_items));
  const long long slot_elems = (slot + 63) / 64 * 64;
  // slot reuse distance R - D = D + 2: a pass-1 item reuses the slot of a chunk whose
  // pass-2 items were queued ~D chunks earlier
  const int max_slots = (int)std::max(2LL, p->W_elems / slot_elems);
  D = std::max(D, (max_slots - 2) / 2);
  D = std::max(1, std::min(D, std::min((int)protos.size(), std::max(1, (max_slots - 2) / 2))));
  int R = std::min((int)protos.size(), std::min(max_slots, 2 * D + 2));
  if ((long long)R * slot_elems > p->W_elems) return fail(FFST_ERR_INVALID_ARG, "intermediate ring exceeds workspace");
  // ---- 2. interleaved chunk order
  const int Wg = std::max(1, std::min(batch, D));
  std::vector<int> order;   // indices into protos
  for (int b0 = 0; b0 < batch; b0 += Wg) {
    const int b1 = std::min(batch, b0 + Wg);
    for (int ci = 0; ci < chunks_per_image; ++ci)
      for (int b = b0; b < b1; ++b) order.push_back(b * chunks_per_image + ci);
  }
  const int C = (int)order.size();
  // accumulator lanes: consecutive chunks of an image accumulate into different copies of A
  // (chunk index mod K), summed in lane order by the final pass -- the inverse's accumulation
  // chain then links chunks K apart instead of neighbours (deterministic, no atomics)
  const int K = std::max(1, std::min(p->acc_lanes, chunks_per_image));
  std::vector<UnitDev> units;
  std::vector<ChunkDev> chunks(C);
  std::vector<int> chunk_lane(C, 0);
  std::vector<int> last_chunk_of_lane((size_t)batch * K, -1);
  for (int c = 0; c < C; ++c) {
    const Proto& pr = protos[order[c]];
    ChunkDev& ch = chunks[c];
    ch.b = pr.b;
    ch.unit0 = (int)units.size();
    ch.nunits = pr.np;
    ch.slot = c % R;
    ch.prev_slot_chunk = c - R >= 0 ? c - R : -1;
    const int lane = (order[c] % chunks_per_image) % K;
    chunk_lane[c] = lane;
    ch.first_of_image = last_chunk_of_lane[(size_t)pr.b * K + lane] < 0 ? 1 : 0;   // first of its lane
    last_chunk_of_lane[(size_t)pr.b * K + lane] = c;
    long long used = 0;
    for (int lp = pr.lp0; lp < pr.lp0 + pr.np; ++lp) {
      UnitDev u{};
      u.b = pr.b; u.p = lp; u.chunk = c; u.woff = (int)used;
      units.push_back(u);
      used += (long long)N * p->planes[lp].ncols_pad;
    }
  }
  // ---- 3. items (self-contained; counters: [0] dispatch, [1 + c] pass-1 done, [1 + C + c] pass-2 done,
  //      [1 + 2C + g] inverse column-group flags)
  std::vector<std::vector<ItemDev>> f1(C), f2(C), i1(C), i2(C);
  const int ngroups = (H + 1 + g.igc - 1) / g.igc;
  std::vector<int> last_self((size_t)batch * K * ngroups, -1);
  int n_self = 0;
  auto mk_item = [](int type, int c, int group, int b, int pl, int np, int woff, int slot) {
    ItemDev it{};
    it.type = type; it.chunk = c; it.group = group; it.b = b; it.p = pl; it.np = np; it.woff = woff; it.slot = slot;
    it.wait_ctr = -1; it.wait_tgt = 0; it.wait2_ctr = -1; it.first = 0; it.sig_ctr = -1; it.sig2_ctr = -1;
    return it;
  };
  for (int c = 0; c < C; ++c) {
    const ChunkDev& ch = chunks[c];
    for (int u = ch.unit0; u < ch.unit0 + ch.nunits; ++u) {
      const PlaneDev& P = p->planes[units[u].p];
      const int ng1 = (P.ncols + g.gc - 1) / g.gc;
      for (int gi = 0; gi < ng1; ++gi) f1[c].push_back(mk_item(0, c, gi, ch.b, units[u].p, 1, units[u].woff, ch.slot));
      const int ng2 = (N + g.rp2 - 1) / g.rp2;
      for (int gi = 0; gi < ng2; ++gi) f2[c].push_back(mk_item(1, c, gi, ch.b, units[u].p, 1, units[u].woff, ch.slot));
      const int ni1 = (N + p->rpi - 1) / p->rpi;
      for (int gi = 0; gi < ni1; ++gi) i1[c].push_back(mk_item(0, c, gi, ch.b, units[u].p, 1, units[u].woff, ch.slot));
    }
    for (int gg = 0; gg < ngroups; ++gg) {
      bool touched = ch.first_of_image != 0;
      const int g0 = gg * g.igc, g1 = std::min(g0 + g.igc, H + 1);
      for (int u = ch.unit0; u < ch.unit0 + ch.nunits && !touched; ++u) {
        const PlaneDev& P = p->planes[units[u].p];
        if (g1 > P.c_lo && g0 < P.c_lo + P.ncols) touched = true;
      }
      if (!touched) continue;
      int& last = last_self[((size_t)ch.b * K + chunk_lane[c]) * ngroups + gg];
      ItemDev it = mk_item(1, c, gg, ch.b, units[ch.unit0].p, ch.nunits, units[ch.unit0].woff, ch.slot);
      it.first = ch.first_of_image;
      it.pad1 = chunk_lane[c];
      it.wait2_ctr = last >= 0 ? 1 + 2 * C + last : -1;
      it.sig2_ctr = 1 + 2 * C + n_self;
      i2[c].push_back(it);
      last = n_self++;
    }
  }
  // dependency / signal counters
  for (int c = 0; c < C; ++c) {
    const int prev = chunks[c].prev_slot_chunk;
    for (auto* vec : {&f1[c], &i1[c]}) {
      const bool fw = vec == &f1[c];
      for (auto& it : *vec) {
        it.sig_ctr = 1 + c;
        if (prev >= 0) {
          it.wait_ctr = 1 + C + prev;
          it.wait_tgt = (int)(fw ? f2[prev].size() : i2[prev].size());
        }
      }
    }
    for (auto* vec : {&f2[c], &i2[c]}) {
      const bool fw = vec == &f2[c];
      for (auto& it : *vec) {
        it.sig_ctr = 1 + C + c;
        it.wait_ctr = 1 + c;
        it.wait_tgt = (int)(fw ? f1[c].size() : i1[c].size());
      }
    }
  }
  // Forward pass 1, paired images (CTA kernels, one round per column group): chunks c and c+1
  // of two images holding the same planes share their pass-1 items -- the window of a column group
  // is evaluated once for both images (K::col_ifft_two).  The shared item signals both chunks
  // and waits for both ring slots.
  for (int c = 0; c < C; ++c)
    for (auto& it : f1[c]) it.pad0 = -1;
  const char* envp = std::getenv("FFST_PAIR");
  const bool pair_ok = g.gc == g.lpc && batch >= 2 && !(envp && std::atoi(envp) == 0);
  if (pair_ok) {
    for (int c = 0; c + 1 < C; ++c) {
      const Proto& a = protos[order[c]];
      const Proto& b = protos[order[c + 1]];
      if (a.b == b.b || a.lp0 != b.lp0 || a.np != b.np || f1[c].empty() || f1[c].size() != f1[c + 1].size())
        continue;
      for (size_t k = 0; k < f1[c].size(); ++k) {
        ItemDev& it = f1[c][k];
        const ItemDev& jt = f1[c + 1][k];
        it.pad0 = jt.b;
        it.pad1 = jt.slot;
        it.first = jt.woff;
        it.sig2_ctr = jt.sig_ctr;
        it.wait2_ctr = jt.wait_ctr;
        it.np = jt.wait_tgt;
      }
      f1[c + 1].clear();
      ++c;                                           // c+1 is consumed
    }
  }
  auto emit = [&](std::vector<std::vector<ItemDev>>& a, std::vector<std::vector<ItemDev>>& b,
                  std::vector<ItemDev>& dst) {
    for (int c = 0; c < std::min(D, C); ++c) dst.insert(dst.end(), a[c].begin(), a[c].end());
    for (int c = 0; c < C; ++c) {
      if (c + D < C) dst.insert(dst.end(), a[c + D].begin(), a[c + D].end());
      dst.insert(dst.end(), b[c].begin(), b[c].end());
    }
  };
  std::vector<ItemDev> fwd, inv;
  emit(f1, f2, fwd);
  emit(i1, i2, inv);
  // FFST_QUEUE_ONLY=1 / 2 (measurement only; results are wrong): keep only the pass-1 / pass-2
  // items, dependencies removed, to time each pass type alone
  if (const char* only = std::getenv("FFST_QUEUE_ONLY")) {
    const int keep = std::atoi(only) - 1;
    for (auto* q : {&fwd, &inv}) {
      std::vector<ItemDev> k;
      for (auto it : *q)
        if (it.type == keep) {
          it.wait_ctr = 0; it.wait_tgt = 0; it.wait2_ctr = -1;
          k.push_back(it);
        }
      *q = k;
    }
  }
  std::vector<ChunkDev> chunks_inv = chunks;
  for (int c = 0; c < C; ++c) {
    chunks[c].p1_items = (int)f1[c].size();
    chunks[c].p2_items = (int)f2[c].size();
    chunks_inv[c].p1_items = (int)i1[c].size();
    chunks_inv[c].p2_items = (int)i2[c].size();
  }
  Queue q;
  q.batch = batch;
  q.n_chunks = C;
  q.slot_elems = slot_elems;
  q.nslots = R;
  q.n_fwd = (int)fwd.size();
  q.n_inv = (int)inv.size();
  q.n_g = n_self;
  q.a_lanes = K;
  const size_t need_ctr = 1 + 2 * (size_t)C + (size_t)n_self;
  if (need_ctr > p->ctr_cap) {
    void* c = nullptr;
    TRY(dalloc(p, &c, need_ctr * sizeof(int)));
    p->d_ctr = static_cast<int*>(c);
    p->ctr_cap = need_ctr;
  }
  void* ptr = nullptr;
  TRY(dalloc(p, &ptr, units.size() * sizeof(UnitDev)));
  q.d_units = static_cast<UnitDev*>(ptr);
  TRY(dalloc(p, &ptr, 2 * chunks.size() * sizeof(ChunkDev)));
  q.d_chunks = static_cast<ChunkDev*>(ptr);
  TRY(dalloc(p, &ptr, fwd.size() * sizeof(ItemDev)));
  q.d_fwd = static_cast<ItemDev*>(ptr);
  TRY(dalloc(p, &ptr, inv.size() * sizeof(ItemDev)));
  q.d_inv = static_cast<ItemDev*>(ptr);
  // (plan creation / ffst_plan_reserve only: transforms never reach this upload)
  API_CUDA(cudaMemcpy(q.d_units, units.data(), units.size() * sizeof(UnitDev), cudaMemcpyHostToDevice), "queue upload");
  API_CUDA(cudaMemcpy(q.d_chunks, chunks.data(), chunks.size() * sizeof(ChunkDev), cudaMemcpyHostToDevice), "queue upload");
  API_CUDA(cudaMemcpy(q.d_chunks + chunks.size(), chunks_inv.data(), chunks.size() * sizeof(ChunkDev),
                      cudaMemcpyHostToDevice), "queue upload");
  API_CUDA(cudaMemcpy(q.d_fwd, fwd.data(), fwd.size() * sizeof(ItemDev), cudaMemcpyHostToDevice), "queue upload");
  API_CUDA(cudaMemcpy(q.d_inv, inv.data(), inv.size() * sizeof(ItemDev), cudaMemcpyHostToDevice), "queue upload");
  if (std::getenv("FFST_VERBOSE"))
    std::fprintf(stderr, "[ffst] batch=%d chunks=%d (per image %d) D=%d R=%d Wg=%d slot=%.1f MB items fwd=%d inv=%d\n",
                 batch, C, chunks_per_image, D, R, Wg, slot_elems * 2.0 * p->rsz / 1048576.0, q.n_fwd, q.n_inv);
  auto res = p->queues.emplace(batch, q);
  *out = &res.first->second;
  return FFST_OK;
}

// The queue of a reserved batch size (ffst_plan_create reserves the plan batch; other sizes
// through ffst_plan_reserve): transforms never allocate or upload.
ffst_status find_queue(ffst_plan* p, int batch, Queue** out) {
  auto it = p->queues.find(batch);
  if (it == p->queues.end())
    return fail(FFST_ERR_INVALID_ARG, "batch " + std::to_string(batch) + " not reserved (ffst_plan_reserve)");
  *out = &it->second;
  return FFST_OK;
}

KParams base_params(ffst_plan* p) {
  KParams k{};
  k.n = p->n; k.j0 = p->j0; k.batch = p->d.batch; k.eta_l = p->eta_l; k.n_nyq = (int)p->nyq.size();
  k.delta = p->delta;
  k.variant = (int)p->d.variant;
  k.usym = p->d_usym;
  k.planes = p->d_planes;
  k.nyq_planes = p->d_nyq;
  k.tw = p->d_tw;
  k.rtab = p->d_rtab;
  k.F = p->F; k.Fscr = p->Fscr; k.A = p->A; k.W = p->W;
  k.part = p->part;
  k.nyq_fwd = p->nyq_fwd; k.nyq_S = p->nyq_S; k.nyq_T = p->nyq_T; k.corr = p->corr; k.nyq_anti = p->nyq_anti; k.nyq_part = p->nyq_part;
  k.n_rowitems = p->n_rowitems;
  k.nyq_tparts = p->geo.tparts;
  k.rpi = p->rpi;
  k.a_lane_elems = (long long)p->d.batch * (p->n / 2 + 1) * p->n;
  if (const char* d = std::getenv("FFST_DBG")) k.dbg = std::atoi(d);
  k.ring_stream = (long long)p->W_elems * 2 * (long long)p->rsz > (96LL << 20) ? 1 : 0;
  if (const char* rs = std::getenv("FFST_RING_STREAM")) k.ring_stream = std::atoi(rs) != 0;   // tuning only
  k.sync_mode = 3;
  if (const char* sm = std::getenv("FFST_SYNC")) k.sync_mode = std::atoi(sm) & 3;   // measurement only
  return k;
}

template <typename T>
struct Ops {
  static Geometry geo(int n) { return geometry<T>(n); }
};

cudaError_t L_spectrum(ffst_plan* p, const KParams& k, int b, cudaStream_t s) {
  return p->d.dtype == FFST_F32 ? launch_spectrum<float>(k, b, s) : launch_spectrum<double>(k, b, s);
}
cudaError_t L_nyq_fwd(ffst_plan* p, const KParams& k, int b, cudaStream_t s) {
  return p->d.dtype == FFST_F32 ? launch_nyq_fwd<float>(k, b, s) : launch_nyq_fwd<double>(k, b, s);
}
cudaError_t L_fwd_main(ffst_plan* p, const KParams& k, int g, cudaStream_t s) {
  return p->d.dtype == FFST_F32 ? launch_fwd_main<float>(k, g, s) : launch_fwd_main<double>(k, g, s);
}
cudaError_t L_inv_main(ffst_plan* p, const KParams& k, int g, cudaStream_t s) {
  return p->d.dtype == FFST_F32 ? launch_inv_main<float>(k, g, s) : launch_inv_main<double>(k, g, s);
}
cudaError_t L_nyq_inv(ffst_plan* p, const KParams& k, int b, cudaStream_t s) {
  return p->d.dtype == FFST_F32 ? launch_nyq_inv<float>(k, b, s) : launch_nyq_inv<double>(k, b, s);
}
cudaError_t L_final(ffst_plan* p, const KParams& k, int b, int which, cudaStream_t s) {
  return p->d.dtype == FFST_F32 ? launch_final<float>(k, b, which, s) : launch_final<double>(k, b, which, s);
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

ffst_status set_device(ffst_plan* p) {
  API_CUDA(cudaSetDevice(p->d.device), "cudaSetDevice");
  return FFST_OK;
}

ffst_status trace_buffer(ffst_plan* p, int which, int n_items, KParams* k) {
  k->trace = nullptr;
  if (!p->tracing) return FFST_OK;
  if (p->trace_items[which] < n_items) {
    void* ptr = nullptr;
    TRY(dalloc(p, &ptr, (size_t)n_items * 8 * sizeof(unsigned long long)));
    p->d_trace[which] = static_cast<unsigned long long*>(ptr);
    p->trace_items[which] = n_items;
  }
  k->trace = p->d_trace[which];
  return FFST_OK;
}

// nyq_gh != nullptr: compact (f1) format -- coeff holds the real parts, nyq_gh the Nyquist vectors
// Argument checks of a transform call, all before anything is launched or copied.
ffst_status validate_call(ffst_plan* p, const void* a, const void* b, int batch, Queue** q) {
  if (!a || !b) return fail(FFST_ERR_INVALID_ARG, "null buffer");
  if (batch < 1 || batch > p->d.batch) return fail(FFST_ERR_INVALID_ARG, "batch outside 1..plan batch");
  if (!aligned16(a) || !aligned16(b)) return fail(FFST_ERR_ALIGNMENT, "buffers must be 16-byte aligned");
  if (p->generic) {                 // the arbitrary-n path has no work queues
    *q = nullptr;
    return FFST_OK;
  }
  return find_queue(p, batch, q);
}

// Image groups of the library's collectives (sharded plans with an NCCL communicator): the
// exchange of group g overlaps the kernels of the other groups.
constexpr int COMM_GROUPS = 4;
int comm_groups(int batch) { return std::min(batch, COMM_GROUPS); }
void group_range(int batch, int G, int g, int* g0, int* g1) {
  *g0 = (int)((long long)batch * g / G);
  *g1 = (int)((long long)batch * (g + 1) / G);
}
ncclDataType_t nccl_type(const ffst_plan* p) { return p->d.dtype == FFST_F32 ? ncclFloat32 : ncclFloat64; }

ffst_status forward_generic(ffst_plan* p, const void* img, void* coeff, int batch, cudaStream_t s);
ffst_status inverse_generic(ffst_plan* p, const void* coeff, void* img_out, int batch, int root_rank, cudaStream_t s);

// nyq_gh != nullptr: compact (f1) format -- coeff holds the real parts, nyq_gh the Nyquist vectors.
// With a communicator: img is read on rank 0 and broadcast (image groups on the comm stream, each
// group's spectrum kernels start as soon as its images have arrived); other ranks receive into the
// plan's staging buffer (img may be NULL there).
ffst_status forward_impl(ffst_plan* p, const void* img, void* coeff, int batch, cudaStream_t s,
                         void* nyq_gh = nullptr) {
  if (p->generic) {
    if (nyq_gh) return fail(FFST_ERR_UNSUPPORTED, "compact format: power-of-two n (fast path) only");
    return forward_generic(p, img, coeff, batch, s);
  }
  const bool coll = p->comm != nullptr;
  const bool root = p->d.shard_rank == 0;
  const void* src = coll && !root ? p->stage : img;
  Queue* q = nullptr;
  TRY(validate_call(p, src, coeff, batch, &q));
  TRY(set_device(p));
  KParams k = base_params(p);
  k.batch = batch;
  k.img = src;
  k.coeff = coeff;
  if (nyq_gh != nullptr) {
    k.compact = 1;
    k.nyq_fwd = nyq_gh;          // nyq_fwd writes G, H straight into the caller's buffer
  }
  k.units = q->d_units;
  k.chunks = q->d_chunks;
  k.items = q->d_fwd;
  k.n_items = q->n_fwd;
  k.slot_elems = q->slot_elems;
  k.ctr = p->d_ctr;
  k.ctr_p1 = 1;
  k.ctr_p2 = 1 + q->n_chunks;
  k.ctr_g = 1 + 2 * q->n_chunks;
  TRY(trace_buffer(p, 0, q->n_fwd, &k));
  int nl = 0;
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[0], s), "event");
  if (p->tiny && nyq_gh == nullptr) {   // fused small-n path: one launch
    if (coll) {
      API_CUDA(cudaEventRecord(p->cev[0], s), "event");
      API_CUDA(cudaStreamWaitEvent(p->cs, p->cev[0], 0), "stream wait");
      API_NCCL(ncclBroadcast(src, const_cast<void*>(src), (size_t)batch * p->n * p->n, nccl_type(p), 0, p->comm, p->cs),
               "ncclBroadcast (images)");
      API_CUDA(cudaEventRecord(p->cev[1], p->cs), "event");
      API_CUDA(cudaStreamWaitEvent(s, p->cev[1], 0), "stream wait");
    }
    if (p->timing) API_CUDA(cudaEventRecord(p->ev[1], s), "event");
    API_CUDA(p->d.dtype == FFST_F32 ? launch_tiny<float>(k, batch, 0, s) : launch_tiny<double>(k, batch, 0, s),
             "tiny forward kernel");
    if (p->timing) API_CUDA(cudaEventRecord(p->ev[2], s), "event");
    p->launches[0] = 1;
    return FFST_OK;
  }
  if (coll) {
    const size_t img_elems = (size_t)p->n * p->n;
    const size_t h1n = (size_t)(p->n / 2 + 1) * p->n;
    const int G = comm_groups(batch);
    API_CUDA(cudaEventRecord(p->cev[0], s), "event");
    API_CUDA(cudaStreamWaitEvent(p->cs, p->cev[0], 0), "stream wait");
    for (int g = 0; g < G; ++g) {
      int g0, g1;
      group_range(batch, G, g, &g0, &g1);
      const char* sb = static_cast<const char*>(src) + g0 * img_elems * p->rsz;
      API_NCCL(ncclBroadcast(sb, const_cast<char*>(sb), (g1 - g0) * img_elems, nccl_type(p), 0, p->comm, p->cs),
               "ncclBroadcast (images)");
      API_CUDA(cudaEventRecord(p->cev[1 + g], p->cs), "event");
    }
    for (int g = 0; g < G; ++g) {
      int g0, g1;
      group_range(batch, G, g, &g0, &g1);
      API_CUDA(cudaStreamWaitEvent(s, p->cev[1 + g], 0), "stream wait");
      KParams kg = k;
      kg.img = static_cast<const char*>(src) + g0 * img_elems * p->rsz;
      kg.F = static_cast<char*>(p->F) + g0 * h1n * 2 * p->rsz;
      kg.Fscr = static_cast<char*>(p->Fscr) + g0 * h1n * 2 * p->rsz;
      API_CUDA(L_spectrum(p, kg, g1 - g0, s), "spectrum kernels");
      nl += 2;
    }
  } else {
    API_CUDA(L_spectrum(p, k, batch, s), "spectrum kernels");
    nl += 2;
  }
  if (!p->nyq.empty()) {
    API_CUDA(L_nyq_fwd(p, k, batch, s), "nyq_fwd kernel");
    ++nl;
  }
  API_CUDA(cudaMemsetAsync(p->d_ctr, 0, (1 + 2 * (size_t)q->n_chunks) * sizeof(int), s), "counter reset");
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[1], s), "event");
  API_CUDA(L_fwd_main(p, k, p->grid_fwd, s), "fwd_main kernel");
  ++nl;
  if (p->timing) {
    API_CUDA(cudaEventRecord(p->ev[2], s), "event");
  }
  p->launches[0] = nl;
  return FFST_OK;
}

// With a communicator: every rank forms its partial adjoint spectrum A_r (all accumulator lanes)
// and Nyquist correction; the comm stream sums them onto `root` image group by image group
// (ncclReduce, in place), and the root runs the final synthesis of group g while group g + 1 is
// being reduced.  img_out is written on the root only (it may be NULL elsewhere).
ffst_status inverse_impl(ffst_plan* p, const void* coeff, void* img_out, int batch, int root_rank, cudaStream_t s,
                         const void* nyq_gh = nullptr) {
  if (p->generic) {
    if (nyq_gh) return fail(FFST_ERR_UNSUPPORTED, "compact format: power-of-two n (fast path) only");
    return inverse_generic(p, coeff, img_out, batch, root_rank, s);
  }
  const bool coll = p->comm != nullptr;
  if (coll && (root_rank < 0 || root_rank >= p->d.shard_count)) return fail(FFST_ERR_INVALID_ARG, "root outside 0..shard_count-1");
  const bool root = !coll || p->d.shard_rank == root_rank;
  Queue* q = nullptr;
  TRY(validate_call(p, coeff, root ? img_out : p->stage, batch, &q));
  TRY(set_device(p));
  KParams k = base_params(p);
  k.batch = batch;
  k.coeff = const_cast<void*>(coeff);
  k.img_out = img_out;
  if (nyq_gh != nullptr) {
    k.compact = 1;
    k.nyq_fwd = const_cast<void*>(nyq_gh);
    k.n_rowitems = 1;            // the alternating sums come whole from (G, H)
    k.nyq_tparts = 1;
  }
  k.units = q->d_units;
  k.chunks = q->d_chunks + q->n_chunks;
  k.items = q->d_inv;
  k.n_items = q->n_inv;
  k.a_lanes = q->a_lanes;
  k.slot_elems = q->slot_elems;
  k.ctr = p->d_ctr;
  k.ctr_p1 = 1;
  k.ctr_p2 = 1 + q->n_chunks;
  k.ctr_g = 1 + 2 * q->n_chunks;
  TRY(trace_buffer(p, 1, q->n_inv, &k));
  int nl = 0;
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[3], s), "event");
  if (p->tiny && nyq_gh == nullptr) {   // fused small-n path: partial images, summed in plane order
    k.img_out = root ? img_out : p->stage;
    if (p->timing) API_CUDA(cudaEventRecord(p->ev[4], s), "event");
    API_CUDA(p->d.dtype == FFST_F32 ? launch_tiny<float>(k, batch, 1, s) : launch_tiny<double>(k, batch, 1, s),
             "tiny inverse kernels");
    if (p->timing) API_CUDA(cudaEventRecord(p->ev[5], s), "event");
    if (coll) {   // the partial image sums of the ranks onto root (the inverse is linear in the planes)
      API_CUDA(cudaEventRecord(p->cev[5], s), "event");
      API_CUDA(cudaStreamWaitEvent(p->cs, p->cev[5], 0), "stream wait");
      API_NCCL(ncclReduce(k.img_out, k.img_out, (size_t)batch * p->n * p->n, nccl_type(p), ncclSum, root_rank, p->comm,
                          p->cs), "ncclReduce (images)");
      API_CUDA(cudaEventRecord(p->cev[1], p->cs), "event");
      API_CUDA(cudaStreamWaitEvent(s, p->cev[1], 0), "stream wait");
    }
    if (p->timing) API_CUDA(cudaEventRecord(p->ev[6], s), "event");
    p->launches[1] = 2;
    return FFST_OK;
  }
  API_CUDA(cudaMemsetAsync(p->d_ctr, 0, (1 + 2 * (size_t)q->n_chunks + q->n_g) * sizeof(int), s), "counter reset");
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[4], s), "event");
  API_CUDA(L_inv_main(p, k, p->grid_inv, s), "inv_main kernel");
  ++nl;
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[5], s), "event");
  if (!p->nyq.empty()) {
    // fork: the Nyquist correction (needed only by the final row pass) beside the column pass
    API_CUDA(cudaEventRecord(p->fork[0], s), "event");
    API_CUDA(cudaStreamWaitEvent(p->aux, p->fork[0], 0), "stream wait");
    if (k.compact)
      API_CUDA(p->d.dtype == FFST_F32 ? launch_nyq_compact_sums<float>(k, batch, p->aux)
                                      : launch_nyq_compact_sums<double>(k, batch, p->aux), "nyq_compact_sums kernel");
    API_CUDA(L_nyq_inv(p, k, batch, p->aux), "nyq_inv kernels");
    API_CUDA(cudaEventRecord(p->fork[1], p->aux), "event");
    nl += 2;
  }
  if (!coll) {
    API_CUDA(L_final(p, k, batch, 0, s), "final column pass");
    if (!p->nyq.empty()) API_CUDA(cudaStreamWaitEvent(s, p->fork[1], 0), "stream wait");
    API_CUDA(L_final(p, k, batch, 1, s), "final row pass");
    nl += 2;
  } else {
    const size_t n = (size_t)p->n, h1n = (n / 2 + 1) * n;
    if (!p->nyq.empty()) API_CUDA(cudaStreamWaitEvent(s, p->fork[1], 0), "stream wait");
    API_CUDA(cudaEventRecord(p->cev[5], s), "event");              // A lanes and corr final
    API_CUDA(cudaStreamWaitEvent(p->cs, p->cev[5], 0), "stream wait");
    const int G = comm_groups(batch);
    for (int g = 0; g < G; ++g) {
      int g0, g1;
      group_range(batch, G, g, &g0, &g1);
      API_NCCL(ncclGroupStart(), "ncclGroupStart");
      for (int l = 0; l < k.a_lanes; ++l) {
        char* a = static_cast<char*>(p->A) + ((size_t)l * k.a_lane_elems + g0 * h1n) * 2 * p->rsz;
        API_NCCL(ncclReduce(a, a, (g1 - g0) * h1n * 2, nccl_type(p), ncclSum, root_rank, p->comm, p->cs),
                 "ncclReduce (adjoint spectra)");
      }
      if (!p->nyq.empty()) {
        char* c = static_cast<char*>(p->corr) + g0 * 2 * n * p->rsz;
        API_NCCL(ncclReduce(c, c, (g1 - g0) * 2 * n, nccl_type(p), ncclSum, root_rank, p->comm, p->cs),
                 "ncclReduce (Nyquist correction)");
      }
      API_NCCL(ncclGroupEnd(), "ncclGroupEnd");
      API_CUDA(cudaEventRecord(p->cev[1 + g], p->cs), "event");
    }
    for (int g = 0; g < G; ++g) {
      API_CUDA(cudaStreamWaitEvent(s, p->cev[1 + g], 0), "stream wait");
      if (!root) continue;
      int g0, g1;
      group_range(batch, G, g, &g0, &g1);
      KParams kg = k;
      kg.A = static_cast<char*>(p->A) + g0 * h1n * 2 * p->rsz;
      kg.Fscr = static_cast<char*>(p->Fscr) + g0 * n * (size_t)p->geo.ncpf * 2 * p->rsz;
      kg.img_out = static_cast<char*>(img_out) + g0 * n * n * p->rsz;
      kg.corr = static_cast<char*>(p->corr) + g0 * 2 * n * p->rsz;
      API_CUDA(L_final(p, kg, g1 - g0, 0, s), "final column pass");
      API_CUDA(L_final(p, kg, g1 - g0, 1, s), "final row pass");
      nl += 2;
    }
  }
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[6], s), "event");
  p->launches[1] = nl;
  return FFST_OK;
}

struct UserSpectra {
  int eta;
  const void* psi;
  int centred;
};

// ============================================================ arbitrary-n path (ffst_generic.cuh)

// Host FFT (float64, radix 2, forward sign): the Bluestein kernel's spectrum FFT_M(b) (a plan table).
void host_fft(std::vector<std::complex<double>>& a) {
  const size_t M = a.size();
  for (size_t i = 1, j = 0; i < M; ++i) {
    size_t bit = M >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  const long double pi = 3.14159265358979323846264338327950288L;
  for (size_t len = 2; len <= M; len <<= 1)
    for (size_t i = 0; i < M; i += len)
      for (size_t k = 0; k < len / 2; ++k) {
        const long double ang = -2.0L * pi * (long double)k / (long double)len;
        const std::complex<double> w((double)cosl(ang), (double)sinl(ang));
        const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
}

GenParams gen_params(const ffst_plan* p, int batch) {
  GenParams g{};
  g.n = p->n; g.M = p->gen_M; g.eta_l = p->eta_l; g.batch = batch;
  g.planes = p->d_planes; g.rtab = p->d_rtab; g.j0 = p->j0;
  g.variant = p->d.variant == FFST_SMOOTH ? 1 : 0;
  g.usr = p->g_usr;
  g.chirp = p->g_chirp; g.bhat = p->g_bhat; g.twm = p->g_twm;
  return g;
}

cudaError_t G_rows(const ffst_plan* p, int op, const GenParams& g, const void* src, void* dst, int np, int p0, int first,
                   double scale, int cube_side, int mats, cudaStream_t s) {
  return p->d.dtype == FFST_F32
             ? launch_gen_rows<float>(op, g, src, dst, np, p0, first, scale, cube_side, cube_side ? p->eta_l : 0, mats, s)
             : launch_gen_rows<double>(op, g, src, dst, np, p0, first, scale, cube_side, cube_side ? p->eta_l : 0, mats, s);
}
cudaError_t G_transpose(const ffst_plan* p, const void* src, void* dst, int mats, cudaStream_t s) {
  return p->d.dtype == FFST_F32 ? launch_gen_transpose<float>(src, dst, p->n, mats, s)
                                : launch_gen_transpose<double>(src, dst, p->n, mats, s);
}

// Generic-path tables (chirp, FFT_M(b), twiddles) and workspace; user spectra copied to a
// natural-order table of the local planes.
ffst_status generic_setup(ffst_plan* p, const UserSpectra* us) {
  const int n = p->n;
  int M = 16;
  while (M < 2 * n - 1) M *= 2;
  if (M > 4096) return fail(FFST_ERR_UNSUPPORTED, "this n needs the arbitrary-n path, built up to n = 2048");
  p->gen_M = M;
  const size_t B = (size_t)p->d.batch, nn = (size_t)n * n, csz = 2 * p->rsz;
  const size_t budget = (size_t)512 << 20;
  p->gen_np = (int)std::max<size_t>(1, std::min<size_t>(p->eta_l, budget / (2 * B * nn * csz)));
  void* ptr = nullptr;
#define GALLOC(dst, bytes) do { TRY(dalloc(p, &ptr, (bytes))); dst = static_cast<decltype(dst)>(ptr); } while (0)
  GALLOC(p->d_planes, p->planes.size() * sizeof(PlaneDev));
  GALLOC(p->d_rtab, (size_t)(p->d.variant == FFST_SMOOTH ? 3 * p->j0 + 4 : p->j0 + 1) * (n / 2 + 1) * p->rsz);
  GALLOC(p->g_chirp, (size_t)n * csz);
  GALLOC(p->g_bhat, (size_t)M * csz);
  GALLOC(p->g_twm, (size_t)M * csz);
  GALLOC(p->Ft, B * nn * csz);
  GALLOC(p->S, B * nn * csz);
  GALLOC(p->At, B * nn * csz);
  GALLOC(p->Wt, B * p->gen_np * nn * csz);
  GALLOC(p->W2, B * p->gen_np * nn * csz);
  GALLOC(p->stage, B * nn * p->rsz);
  GALLOC(p->g_gidx, p->planes.size() * sizeof(int));
  if (us) GALLOC(p->g_usr, (size_t)p->eta_l * nn * p->rsz);
#undef GALLOC
  // chirp c_m = exp(-i pi m^2 / n) (angle reduced through m^2 mod 2n), b_t = conj(c_|t|), FFT_M(b)
  const long double pi = 3.14159265358979323846264338327950288L;
  std::vector<std::complex<double>> ch(n), b(M, 0.0);
  for (int m = 0; m < n; ++m) {
    const long long q = ((long long)m * m) % (2LL * n);
    const long double ang = -pi * (long double)q / (long double)n;
    ch[m] = std::complex<double>((double)cosl(ang), (double)sinl(ang));
  }
  for (int t = 0; t < n; ++t) {
    b[t] = std::conj(ch[t]);
    if (t > 0) b[M - t] = std::conj(ch[t]);
  }
  host_fft(b);
  std::vector<unsigned char> tw;
  if (p->d.dtype == FFST_F32) fill_twiddles<float>(tw, M); else fill_twiddles<double>(tw, M);
  auto upload_c = [&](void* dst, const std::vector<std::complex<double>>& v) {
    if (p->d.dtype == FFST_F32) {
      std::vector<float> f(2 * v.size());
      for (size_t i = 0; i < v.size(); ++i) { f[2 * i] = (float)v[i].real(); f[2 * i + 1] = (float)v[i].imag(); }
      return cudaMemcpy(dst, f.data(), f.size() * sizeof(float), cudaMemcpyHostToDevice);
    }
    return cudaMemcpy(dst, v.data(), v.size() * sizeof(std::complex<double>), cudaMemcpyHostToDevice);
  };
  cudaError_t e = upload_c(p->g_chirp, ch);
  if (e == cudaSuccess) e = upload_c(p->g_bhat, b);
  if (e == cudaSuccess) e = cudaMemcpy(p->g_twm, tw.data(), tw.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const std::vector<double> rt = radial_all(n, p->j0, p->d.variant);
    if (p->d.dtype == FFST_F32) {
      std::vector<float> rf(rt.begin(), rt.end());
      e = cudaMemcpy(p->d_rtab, rf.data(), rf.size() * sizeof(float), cudaMemcpyHostToDevice);
    } else {
      e = cudaMemcpy(p->d_rtab, rt.data(), rt.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
  }
  std::vector<int> gidx;
  for (auto& P : p->planes) gidx.push_back(P.gi);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_planes, p->planes.data(), p->planes.size() * sizeof(PlaneDev), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->g_gidx, gidx.data(), gidx.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "arbitrary-n plan upload");
  if (us) {
    void* st = nullptr;
    e = cudaMalloc(&st, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(st, 0, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess)
      e = p->d.dtype == FFST_F32
              ? launch_gen_user<float>(us->psi, p->g_usr, n, p->g_gidx, p->eta_l, us->eta, us->centred,
                                       static_cast<unsigned long long*>(st), 0)
              : launch_gen_user<double>(us->psi, p->g_usr, n, p->g_gidx, p->eta_l, us->eta, us->centred,
                                        static_cast<unsigned long long*>(st), 0);
    unsigned long long h[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(st);
    if (e != cudaSuccess) return cuda_fail(e, "user spectra copy");
    std::memcpy(&p->tightness, &h[0], sizeof(double));
    std::memcpy(&p->asymmetry, &h[1], sizeof(double));
  }
  return FFST_OK;
}

// Forward, arbitrary n: F = DFT2(f) (rows, transpose, rows: Ft = F^T); per chunk of planes the
// windowed first pass along omega_2 (lines of Ft) -> transpose -> second pass along omega_1
// straight into the cube (1/n^2).  With a communicator: images broadcast from rank 0 first.
ffst_status forward_generic(ffst_plan* p, const void* img, void* coeff, int batch, cudaStream_t s) {
  const bool coll = p->comm != nullptr;
  const void* src = coll && p->d.shard_rank != 0 ? p->stage : img;
  if (!src || !coeff) return fail(FFST_ERR_INVALID_ARG, "null buffer");
  if (batch < 1 || batch > p->d.batch) return fail(FFST_ERR_INVALID_ARG, "batch outside 1..plan batch");
  if (!aligned16(src) || !aligned16(coeff)) return fail(FFST_ERR_ALIGNMENT, "buffers must be 16-byte aligned");
  TRY(set_device(p));
  const GenParams g = gen_params(p, batch);
  const double inv_nn = 1.0 / ((double)p->n * p->n);
  int nl = 0;
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[0], s), "event");
  if (coll) {
    API_CUDA(cudaEventRecord(p->cev[0], s), "event");
    API_CUDA(cudaStreamWaitEvent(p->cs, p->cev[0], 0), "stream wait");
    API_NCCL(ncclBroadcast(src, const_cast<void*>(src), (size_t)batch * p->n * p->n, nccl_type(p), 0, p->comm, p->cs),
             "ncclBroadcast (images)");
    API_CUDA(cudaEventRecord(p->cev[1], p->cs), "event");
    API_CUDA(cudaStreamWaitEvent(s, p->cev[1], 0), "stream wait");
  }
  API_CUDA(G_rows(p, GEN_OP_SPEC, g, src, p->S, 1, 0, 0, 1.0, 0, batch, s), "arbitrary-n spectrum rows");
  API_CUDA(G_transpose(p, p->S, p->Ft, batch, s), "transpose");
  API_CUDA(G_rows(p, GEN_OP_DFT, g, p->Ft, p->Ft, 1, 0, 0, 1.0, 0, batch, s), "arbitrary-n spectrum columns");
  nl += 3;
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[1], s), "event");
  for (int p0 = 0; p0 < p->eta_l; p0 += p->gen_np) {
    const int np = std::min(p->gen_np, p->eta_l - p0);
    API_CUDA(G_rows(p, GEN_OP_FWD_COL, g, p->Ft, p->Wt, np, p0, 0, 1.0, 0, batch * np, s), "arbitrary-n forward pass 1");
    API_CUDA(G_transpose(p, p->Wt, p->W2, batch * np, s), "transpose");
    API_CUDA(G_rows(p, GEN_OP_IDFT, g, p->W2, coeff, np, p0, 0, inv_nn, 2, batch * np, s), "arbitrary-n forward pass 2");
    nl += 3;
  }
  if (p->timing) {
    API_CUDA(cudaEventRecord(p->ev[2], s), "event");
  }
  p->launches[0] = nl;
  return FFST_OK;
}

// Inverse, arbitrary n: per chunk, DFT of the cube rows -> transpose -> per line of At the sum over
// the chunk's planes of psi_i * DFT (eq:inverseShearletTransform); then f = Re IDFT2(A).  With a
// communicator: At summed onto root (ncclReduce), the final synthesis on the root only.
ffst_status inverse_generic(ffst_plan* p, const void* coeff, void* img_out, int batch, int root_rank, cudaStream_t s) {
  const bool coll = p->comm != nullptr;
  if (coll && (root_rank < 0 || root_rank >= p->d.shard_count)) return fail(FFST_ERR_INVALID_ARG, "root outside 0..shard_count-1");
  const bool root = !coll || p->d.shard_rank == root_rank;
  if (!coeff || (root && !img_out)) return fail(FFST_ERR_INVALID_ARG, "null buffer");
  if (batch < 1 || batch > p->d.batch) return fail(FFST_ERR_INVALID_ARG, "batch outside 1..plan batch");
  if (!aligned16(coeff) || (root && !aligned16(img_out))) return fail(FFST_ERR_ALIGNMENT, "buffers must be 16-byte aligned");
  TRY(set_device(p));
  const GenParams g = gen_params(p, batch);
  const double inv_nn = 1.0 / ((double)p->n * p->n);
  int nl = 0;
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[3], s), "event");
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[4], s), "event");
  for (int p0 = 0; p0 < p->eta_l; p0 += p->gen_np) {
    const int np = std::min(p->gen_np, p->eta_l - p0);
    API_CUDA(G_rows(p, GEN_OP_DFT, g, coeff, p->W2, np, p0, 0, 1.0, 1, batch * np, s), "arbitrary-n inverse pass 1");
    API_CUDA(G_transpose(p, p->W2, p->Wt, batch * np, s), "transpose");
    API_CUDA(G_rows(p, GEN_OP_INV_COL, g, p->Wt, p->At, np, p0, p0 == 0, 1.0, 0, batch, s), "arbitrary-n inverse pass 2");
    nl += 3;
  }
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[5], s), "event");
  if (coll) {
    API_CUDA(cudaEventRecord(p->cev[5], s), "event");
    API_CUDA(cudaStreamWaitEvent(p->cs, p->cev[5], 0), "stream wait");
    API_NCCL(ncclReduce(p->At, p->At, (size_t)batch * p->n * p->n * 2, nccl_type(p), ncclSum, root_rank, p->comm, p->cs),
             "ncclReduce (adjoint spectra)");
    API_CUDA(cudaEventRecord(p->cev[1], p->cs), "event");
    API_CUDA(cudaStreamWaitEvent(s, p->cev[1], 0), "stream wait");
  }
  if (root) {
    API_CUDA(G_rows(p, GEN_OP_IDFT, g, p->At, p->S, 1, 0, 0, 1.0, 0, batch, s), "arbitrary-n final pass 1");
    API_CUDA(G_transpose(p, p->S, p->Ft, batch, s), "transpose");
    API_CUDA(G_rows(p, GEN_OP_FINAL, g, p->Ft, img_out, 1, 0, 0, inv_nn, 0, batch, s), "arbitrary-n final pass 2");
    nl += 3;
  }
  if (p->timing) API_CUDA(cudaEventRecord(p->ev[6], s), "event");
  p->launches[1] = nl;
  return FFST_OK;
}

// User spectra (f4): run the prepare kernels (ffst_user.cuh) on the caller's eta planes, keep the
// admission numbers, and replace each local plane's provisional geometry by its column hull and
// Nyquist flag.  `anti` receives the anti parts of every local plane ([eta_l][2][n], float64).

ffst_status user_prepare(ffst_plan* p, const UserSpectra& us, std::vector<double>& anti) {
  const int n = p->n, H = n / 2, L = p->eta_l;
  const size_t rsz = p->rsz;
  void* ptr = nullptr;
  TRY(dalloc(p, &ptr, (size_t)L * (H + 1) * n * rsz));
  p->d_usym = ptr;
  void *d_hull = nullptr, *d_anti = nullptr, *d_stats = nullptr;
  cudaError_t e = cudaMalloc(&d_hull, (size_t)L * 2 * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&d_anti, (size_t)L * 2 * n * rsz);
  if (e == cudaSuccess) e = cudaMalloc(&d_stats, 2 * sizeof(unsigned long long));
  std::vector<int> hull((size_t)L * 2);
  for (int l = 0; l < L; ++l) { hull[2 * l] = H + 1; hull[2 * l + 1] = -1; }
  if (e == cudaSuccess) e = cudaMemcpy(d_hull, hull.data(), hull.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(d_stats, 0, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) {
    UserPrep u{};
    u.psi = us.psi; u.n = n; u.eta = us.eta; u.centred = us.centred;
    u.shard_rank = p->d.shard_rank; u.shard_count = p->d.shard_count; u.eta_l = L;
    u.usym = p->d_usym; u.hull = static_cast<int*>(d_hull); u.anti = d_anti;
    u.stats = static_cast<unsigned long long*>(d_stats);
    const int grid = p->sm_count * 8;
    e = p->d.dtype == FFST_F32 ? launch_user_prepare<float>(u, grid, 0) : launch_user_prepare<double>(u, grid, 0);
  }
  std::vector<unsigned char> an((size_t)L * 2 * n * rsz);
  unsigned long long st[2] = {0, 0};
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(hull.data(), d_hull, hull.size() * sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(an.data(), d_anti, an.size(), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(st, d_stats, sizeof(st), cudaMemcpyDeviceToHost);
  cudaFree(d_hull); cudaFree(d_anti); cudaFree(d_stats);
  if (e != cudaSuccess) return cuda_fail(e, "user spectra prepare");
  std::memcpy(&p->tightness, &st[0], sizeof(double));
  std::memcpy(&p->asymmetry, &st[1], sizeof(double));
  // psi_i(u) = psi_i(-u) off the Nyquist lines is what the even-n decomposition relies on (real
  // shearlets); an asymmetric part there would be dropped silently, so it is refused
  const double tol = p->d.dtype == FFST_F32 ? 1e-5 : 1e-12;
  if (!(p->asymmetry <= tol))
    return fail(FFST_ERR_INVALID_ARG, "user spectra not point-symmetric off the Nyquist lines (max |psi(u) - psi(-u)| = " +
                                          std::to_string(p->asymmetry) + ")");
  anti.assign((size_t)L * 2 * n, 0.0);
  for (size_t i = 0; i < anti.size(); ++i)
    anti[i] = p->d.dtype == FFST_F32 ? (double)reinterpret_cast<const float*>(an.data())[i]
                                      : reinterpret_cast<const double*>(an.data())[i];
  p->nyq.clear();
  for (int l = 0; l < L; ++l) {
    PlaneDev& P = p->planes[l];
    if (hull[2 * l] > hull[2 * l + 1]) { hull[2 * l] = 0; hull[2 * l + 1] = 0; }   // an all-zero plane
    P.c_lo = hull[2 * l];
    P.ncols = hull[2 * l + 1] - hull[2 * l] + 1;
    P.ncols_pad = (P.ncols + p->geo.colpad - 1) / p->geo.colpad * p->geo.colpad;
    bool nyq = false;
    for (int m = 0; m < 2 * n && !nyq; ++m) nyq = anti[(size_t)l * 2 * n + m] != 0.0;
    P.nyq = nyq ? (int)p->nyq.size() : -1;
    if (nyq) p->nyq.push_back(l);
  }
  return FFST_OK;
}

}  // namespace

// ============================================================================ C ABI

extern "C" {

ffst_status ffst_scales_for_size(int n, int* j0) {
  if (!j0) return fail(FFST_ERR_INVALID_ARG, "null j0");
  if (n < 4) return fail(FFST_ERR_INVALID_SIZE, "n < 4: no scale fits (P:L2163-2168)");
  *j0 = default_j0(n);
  return FFST_OK;
}

int ffst_num_shearlets(int j0) { return j0 < 1 || j0 > 12 ? -1 : (1 << (j0 + 2)) - 3; }

ffst_status ffst_index_to_params(int j0, int index, int* kind, int* j, int* k) {
  if (!kind || !j || !k) return fail(FFST_ERR_INVALID_ARG, "null output");
  if (j0 < 1 || j0 > 12) return fail(FFST_ERR_INVALID_ARG, "j0 outside 1..12");
  if (index < 0 || index >= ffst_num_shearlets(j0)) return fail(FFST_ERR_INDEX, "index outside 0..eta-1");
  const Triple t = index_table(j0)[index];
  *kind = t.kind; *j = t.j; *k = t.k;
  return FFST_OK;
}

ffst_status ffst_params_to_index(int j0, int kind, int j, int k, int* index) {
  if (!index) return fail(FFST_ERR_INVALID_ARG, "null output");
  if (j0 < 1 || j0 > 12) return fail(FFST_ERR_INVALID_ARG, "j0 outside 1..12");
  const auto t = index_table(j0);
  for (size_t i = 0; i < t.size(); ++i)
    if (t[i].kind == kind && t[i].j == j && t[i].k == k && (kind != 0 || (j == 0 && k == 0))) {
      *index = (int)i;
      return FFST_OK;
    }
  return fail(FFST_ERR_INDEX, "no shearlet with these parameters");
}

ffst_status ffst_plane_support(int n, int j0, int index, int* col_lo, int* col_hi) {
  if (!col_lo || !col_hi) return fail(FFST_ERR_INVALID_ARG, "null output");
  if (n < 4) return fail(FFST_ERR_INVALID_SIZE, "n < 4");
  if (j0 == 0) j0 = default_j0(n);
  if (j0 < 1 || j0 > 12) return fail(FFST_ERR_INVALID_ARG, "j0 outside 1..12");
  if (index < 0 || index >= ffst_num_shearlets(j0)) return fail(FFST_ERR_INDEX, "index outside 0..eta-1");
  plane_columns(n, j0, index_table(j0)[index], col_lo, col_hi);
  return FFST_OK;
}

ffst_status ffst_plane_is_nyquist(int n, int j0, int index, int* is_nyquist) {
  if (!is_nyquist) return fail(FFST_ERR_INVALID_ARG, "null output");
  if (n < 4) return fail(FFST_ERR_INVALID_SIZE, "n < 4");
  if (j0 == 0) j0 = default_j0(n);
  if (j0 < 1 || j0 > 12) return fail(FFST_ERR_INVALID_ARG, "j0 outside 1..12");
  if (index < 0 || index >= ffst_num_shearlets(j0)) return fail(FFST_ERR_INDEX, "index outside 0..eta-1");
  // odd n: the grid is point-symmetric (no -n/2 bin), every plane is symmetric
  *is_nyquist = n % 2 == 0 && plane_nyquist(n, j0, index_table(j0)[index], FFST_CLASSIC) ? 1 : 0;
  return FFST_OK;
}

ffst_status ffst_shard_planes(int n, int j0, int shard_count, int shard_rank, ffst_shard_policy policy, int* count,
                              int* global_indices) {
  if (!count) return fail(FFST_ERR_INVALID_ARG, "null output");
  if (n < 4) return fail(FFST_ERR_INVALID_SIZE, "n < 4");
  if (j0 == 0) j0 = default_j0(n);
  if (j0 < 1 || j0 > 12) return fail(FFST_ERR_INVALID_ARG, "j0 outside 1..12");
  if (policy != FFST_SHARD_LPT && policy != FFST_SHARD_ROUND_ROBIN) return fail(FFST_ERR_INVALID_ARG, "unknown policy");
  const int eta = ffst_num_shearlets(j0);
  if (shard_count < 1 || shard_count > eta || shard_rank < 0 || shard_rank >= shard_count)
    return fail(FFST_ERR_INVALID_ARG, "bad shard_rank / shard_count");
  const std::vector<int> owner = shard_owner(n, j0, eta, shard_count, policy);
  int c = 0;
  for (int i = 0; i < eta; ++i)
    if (owner[i] == shard_rank) {
      if (global_indices) global_indices[c] = i;
      ++c;
    }
  *count = c;
  return FFST_OK;
}

ffst_status ffst_nccl_unique_id(ffst_nccl_id* id) {
  static_assert(sizeof(ffst_nccl_id) == sizeof(ncclUniqueId), "ffst_nccl_id must hold an ncclUniqueId");
  if (!id) return fail(FFST_ERR_INVALID_ARG, "null id");
  ncclUniqueId u;
  API_NCCL(ncclGetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  return FFST_OK;
}

ffst_status ffst_nccl_comm_create(void** comm, int nranks, int rank, const ffst_nccl_id* id, int device) {
  if (!comm || !id) return fail(FFST_ERR_INVALID_ARG, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FFST_ERR_INVALID_ARG, "bad rank / nranks");
  API_CUDA(cudaSetDevice(device), "cudaSetDevice");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  API_NCCL(ncclCommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
  *comm = c;
  return FFST_OK;
}

ffst_status ffst_nccl_comm_destroy(void* comm) {
  if (!comm) return FFST_OK;
  API_NCCL(ncclCommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  return FFST_OK;
}

ffst_status ffst_plan_destroy(ffst_plan* p) {
  if (!p) return FFST_OK;
  int cur = -1;
  cudaGetDevice(&cur);
  cudaSetDevice(p->d.device);
  for (void* a : p->allocs) cudaFree(a);
  for (auto& e : p->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : p->fork)
    if (e) cudaEventDestroy(e);
  if (p->aux) cudaStreamDestroy(p->aux);
  for (auto& e : p->cev)
    if (e) cudaEventDestroy(e);
  if (p->cs) cudaStreamDestroy(p->cs);
  if (cur >= 0) cudaSetDevice(cur);
  delete p;
  return FFST_OK;
}

static ffst_status plan_create_impl(ffst_plan** out, const ffst_plan_desc* d, const UserSpectra* us);

ffst_status ffst_plan_create(ffst_plan** out, const ffst_plan_desc* d) {
  if (!out || !d) return fail(FFST_ERR_INVALID_ARG, "null argument");
  if (d->variant == FFST_USER) return fail(FFST_ERR_INVALID_ARG, "FFST_USER plans come from ffst_plan_create_user");
  return plan_create_impl(out, d, nullptr);
}

ffst_status ffst_plan_create_user(ffst_plan** out, const ffst_plan_desc* d, int eta, const void* psi,
                                  int centred_layout) {
  if (!out || !d || !psi) return fail(FFST_ERR_INVALID_ARG, "null argument");
  if (eta < 1) return fail(FFST_ERR_INVALID_ARG, "eta < 1");
  const UserSpectra us{eta, psi, centred_layout ? 1 : 0};
  return plan_create_impl(out, d, &us);
}

// The library's exchange steps (desc.nccl_comm): the communicator must be the shard_count ranks,
// rank = shard_rank; a comm stream and its events.
static ffst_status setup_comm(ffst_plan* p, const ffst_plan_desc* d) {
  if (d->nccl_comm == nullptr) return FFST_OK;
  p->comm = static_cast<ncclComm_t>(d->nccl_comm);
  int cn = 0, cr = -1;
  if (ncclCommCount(p->comm, &cn) != ncclSuccess || ncclCommUserRank(p->comm, &cr) != ncclSuccess)
    return fail(FFST_ERR_NCCL, "nccl_comm is not a valid communicator");
  if (cn != d->shard_count || cr != d->shard_rank)
    return fail(FFST_ERR_INVALID_ARG, "nccl_comm size / rank differ from shard_count / shard_rank");
  cudaError_t e = cudaStreamCreateWithFlags(&p->cs, cudaStreamNonBlocking);
  for (auto& ev : p->cev)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(e, "comm stream / events");
  return FFST_OK;
}

static ffst_status plan_create_impl(ffst_plan** out, const ffst_plan_desc* d_in, const UserSpectra* us) {
  *out = nullptr;
  ffst_plan_desc desc = *d_in;
  if (us) { desc.variant = FFST_USER; desc.j0 = 0; }
  const ffst_plan_desc* d = &desc;
  if (d->n < 4) return fail(FFST_ERR_INVALID_SIZE, "n < 4: no scale fits (P:L2163-2168)");
  if (d->dtype != FFST_F32 && d->dtype != FFST_F64) return fail(FFST_ERR_DTYPE, "dtype must be FFST_F32 or FFST_F64");
  const int maxn = d->dtype == FFST_F32 ? 4096 : 2048;
  if (d->n > maxn) return fail(FFST_ERR_INVALID_SIZE, "n above the largest built size (4096 f32, 2048 f64)");
  // arbitrary n (odd, or even but not a power of two): the full complex path
  bool generic = !is_pow2(d->n);
  if (generic && d->n > 2048) return fail(FFST_ERR_UNSUPPORTED, "n not a power of two: built up to n = 2048");
  if (d->shard_policy != FFST_SHARD_LPT && d->shard_policy != FFST_SHARD_ROUND_ROBIN)
    return fail(FFST_ERR_INVALID_ARG, "unknown shard policy");
  if (d->variant != FFST_CLASSIC && d->variant != FFST_SMOOTH && d->variant != FFST_USER)
    return fail(FFST_ERR_INVALID_ARG, "unknown variant");
  if (d->batch < 1) return fail(FFST_ERR_INVALID_ARG, "batch < 1");
  if (d->shard_count < 1 || d->shard_rank < 0 || d->shard_rank >= d->shard_count)
    return fail(FFST_ERR_INVALID_ARG, "bad shard_rank / shard_count");
  const int j0 = d->j0 == 0 ? default_j0(d->n) : d->j0;
  if (j0 < 1 || j0 > 12 || (1 << (2 * j0)) > 4 * d->n)
    return fail(FFST_ERR_INVALID_ARG, "j0 outside 1..(floor(log2 n)/2 + 1)");
  const int eta = us ? us->eta : ffst_num_shearlets(j0);
  if (d->shard_count > eta) return fail(FFST_ERR_INVALID_ARG, "more shards than shearlets");

  ffst_plan* p = new ffst_plan();
  p->d = *d;
  p->n = d->n; p->j0 = j0; p->eta = eta; p->H = d->n / 2;
  p->rsz = d->dtype == FFST_F32 ? 4 : 8;
  p->delta = grid_delta(d->n, j0);
  if (!generic) p->geo = d->dtype == FFST_F32 ? geometry<float>(d->n) : geometry<double>(d->n);
  const auto table = index_table(j0);
  // plane-to-rank map: LPT by default (user spectra: round robin, the order ffst_user.cuh reads)
  const std::vector<int> owner = us ? shard_owner(d->n, j0, eta, d->shard_count, FFST_SHARD_ROUND_ROBIN)
                                    : shard_owner(d->n, j0, eta, d->shard_count, d->shard_policy);
  for (int i = 0; i < eta; ++i) {
    if (owner[i] != d->shard_rank) continue;
    PlaneDev P{};
    P.gi = i;
    P.rec = (int)p->planes.size();
    P.nyq = -1;
    if (us) {   // user spectra: the whole half plane until the prepare pass has found the hulls
      P.c_lo = 0; P.ncols = d->n / 2 + 1;
    } else {
      P.kind = table[i].kind; P.j = table[i].j; P.k = table[i].k;
      int lo, hi;
      plane_columns(d->n, j0, table[i], &lo, &hi);
      P.c_lo = lo; P.ncols = hi - lo + 1;
      if (!generic && plane_nyquist(d->n, j0, table[i], d->variant)) {
        P.nyq = (int)p->nyq.size();
        p->nyq.push_back((int)p->planes.size());
      }
    }
    P.ncols_pad = generic ? P.ncols : (P.ncols + p->geo.colpad - 1) / p->geo.colpad * p->geo.colpad;
    p->planes.push_back(P);
  }
  p->eta_l = (int)p->planes.size();
  if (p->eta_l > 256) {
    delete p;
    return fail(FFST_ERR_UNSUPPORTED, "more than 256 local planes: shard the plan (shard_count > 1)");
  }

  auto cleanup = [&](ffst_status s) { ffst_plan_destroy(p); return s; };
  cudaError_t e = cudaSetDevice(d->device);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaSetDevice"));
  int dev = d->device;
  e = cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "device query"));
  if (us && !generic && d->n <= 2048) {
    // user spectra that are not point-symmetric off the Nyquist lines cannot use the Hermitian
    // fast path: they run on the full complex (arbitrary-n) path, which takes any Psi
    void* st = nullptr;
    e = cudaMalloc(&st, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(st, 0, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess)
      e = d->dtype == FFST_F32 ? launch_gen_user<float>(us->psi, nullptr, d->n, nullptr, 0, us->eta, us->centred,
                                                         static_cast<unsigned long long*>(st), 0)
                               : launch_gen_user<double>(us->psi, nullptr, d->n, nullptr, 0, us->eta, us->centred,
                                                          static_cast<unsigned long long*>(st), 0);
    unsigned long long h[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(st);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "user spectra symmetry probe"));
    double asym = 0.0;
    std::memcpy(&asym, &h[1], sizeof(double));
    if (!(asym <= (d->dtype == FFST_F32 ? 1e-5 : 1e-12))) generic = true;
  }
  if (generic) {
    p->generic = true;
    p->geo = Geometry{};
    ffst_status sg = generic_setup(p, us);
    if (sg != FFST_OK) return cleanup(sg);
    for (auto& ev : p->ev) {
      e = cudaEventCreate(&ev);
      if (e != cudaSuccess) return cleanup(cuda_fail(e, "event create"));
    }
    sg = setup_comm(p, d);
    if (sg != FFST_OK) return cleanup(sg);
    *out = p;
    return FFST_OK;
  }
  {
    const int af = d->dtype == FFST_F32 ? max_active_main<float>(d->n, dev, 0) : max_active_main<double>(d->n, dev, 0);
    const int ai = d->dtype == FFST_F32 ? max_active_main<float>(d->n, dev, 1) : max_active_main<double>(d->n, dev, 1);
    if (af < 1 || ai < 1) return cleanup(fail(FFST_ERR_CUDA, "persistent kernels cannot be made resident"));
    p->grid_fwd = p->sm_count * af;
    p->grid_inv = p->sm_count * ai;
    if (const char* cs = std::getenv("FFST_CTAS_PER_SM")) {   // measurement / debugging only
      p->grid_fwd = p->sm_count * std::max(1, std::min(af, std::atoi(cs)));
      p->grid_inv = p->sm_count * std::max(1, std::min(ai, std::atoi(cs)));
    }
    if (std::getenv("FFST_VERBOSE"))
      std::fprintf(stderr, "[ffst] CTAs/SM fwd %d inv %d (grid %d / %d)\n", af, ai, p->grid_fwd, p->grid_inv);
    p->workers = std::max(p->grid_fwd, p->grid_inv);
  }

  const size_t B = (size_t)d->batch, N = (size_t)d->n, H1 = N / 2 + 1;
  const size_t csz = 2 * p->rsz;
  std::vector<double> user_anti;      // user spectra: anti parts of every local plane [eta_l][2][n]
  if (us) {
    ffst_status st_u = user_prepare(p, *us, user_anti);
    if (st_u != FFST_OK) return cleanup(st_u);
  }
  const size_t ncpf = (size_t)p->geo.ncpf;          // row stride of the final column pass (aux kernels)
  // ring of intermediates: slot budget ~ L2 share, at least the largest plane
  long long maxplane = 0, image_total = 0;
  for (auto& P : p->planes) {
    maxplane = std::max(maxplane, (long long)N * P.ncols_pad);
    image_total += (long long)N * P.ncols_pad;
  }
  const char* env = std::getenv("FFST_SLOT_KB");
  // chunk byte budget: 4 MB; 16 MB from n = 1024 (planes of ~1.6 MB: longer chunks shorten the
  // inverse's accumulation chains; measured config 4: 868 -> 943 images/s at 12 MB, 1173 -> 1202 at
  // 16 MB (24-128 MB no further gain), config 3 no gain); 256 MB from n = 2048, where the ring is in
  // HBM anyway (config 5: chunks of ~9 planes instead of one, the adjoint accumulating them in
  // registers: 31.5 -> 30.1 ms per step; 64 / 128 / 512 MB: 31.1 / 30.4 / 30.5 ms)
  const long long budget_kb = d->n >= 2048 ? 262144 : (d->n >= 1024 ? 16384 : 4096);
  const long long budget_bytes = (env ? std::atoll(env) : budget_kb) * 1024LL;
  p->slot_budget = std::max(maxplane, budget_bytes / (long long)csz);
  {
    // accumulator lanes: as many as keep the lanes of A L2-sized (<= 32 MB), at most 4 (16 for
    // batch <= 4, where the inverse's pass 2 has few column groups to spread); above 32 MB the
    // final pass's extra reads would go to HBM (configs 3-5: one lane)
    const long long a_bytes = (long long)d->batch * (d->n / 2 + 1) * d->n * 2 * (long long)p->rsz;
    const long long cap = d->batch <= 4 ? 16 : 4;
    p->acc_lanes = (int)std::max(1LL, std::min(cap, (32LL << 20) / std::max(1LL, a_bytes)));
    if (const char* el = std::getenv("FFST_ACC_LANES")) p->acc_lanes = std::max(1, std::min(16, std::atoi(el)));
  }
  // planes per chunk: 4 (pipelining granularity).  Small batches: one chunk per accumulator lane
  // (the lanes' pass-2 items then run side by side instead of one item walking every plane:
  // config 1 inverse 0.166 -> 0.037 ms); with a single lane, long chunks keep the accumulation
  // chain (one link per chunk) short.
  const char* envc = std::getenv("FFST_CHUNK_PLANES");
  const int small_chunk = p->acc_lanes >= 2 ? std::max(2, (p->eta_l + p->acc_lanes - 1) / p->acc_lanes) : 32;
  p->chunk_planes = std::max(1, envc ? std::atoi(envc) : (d->batch <= 4 ? small_chunk : 4));
  const long long slot_max = std::min(image_total, std::max(maxplane, p->slot_budget)) + 64;
  const char* envr = std::getenv("FFST_RING_MB");
  const long long ring_bytes = (envr ? std::atoll(envr) : 80) * 1024LL * 1024LL;
  // ring: the budget (L2-sized) or at least 12 slots when single planes are large (n >= 2048:
  // the intermediates then live in HBM; a short ring would serialise the two passes)
  const char* envs = std::getenv("FFST_MIN_SLOTS");
  const long long min_slots = envs ? std::max(2, std::atoi(envs)) : 12;
  p->W_elems = std::max(min_slots * ((slot_max + 63) / 64 * 64), ring_bytes / (long long)csz);
  // inverse pass-1 rows per item (FFST_RPI: tuning only; a multiple of the row tile)
  p->rpi = p->geo.rpi;
  if (const char* er = std::getenv("FFST_RPI")) {
    const int v = std::atoi(er);
    if (v >= p->geo.gr && v % p->geo.gr == 0 && v <= d->n) p->rpi = v;
  }
  p->n_rowitems = (int)((N + p->rpi - 1) / p->rpi);
  const size_t nn = std::max<size_t>(1, p->nyq.size());

  void* ptr = nullptr;
  ffst_status st;
#define ALLOC(dst, bytes) do { st = dalloc(p, &ptr, (bytes)); if (st != FFST_OK) return cleanup(st); dst = static_cast<decltype(dst)>(ptr); } while (0)
  ALLOC(p->d_planes, p->planes.size() * sizeof(PlaneDev));
  ALLOC(p->d_nyq, nn * sizeof(int));
  ALLOC(p->d_tw, N * csz);
  ALLOC(p->d_rtab, (size_t)(d->variant == FFST_SMOOTH ? 3 * j0 + 4 : j0 + 1) * H1 * p->rsz);
  ALLOC(p->F, B * H1 * N * csz);
  ALLOC(p->Fscr, B * std::max(H1 * N, N * ncpf) * csz);
  ALLOC(p->A, (size_t)p->acc_lanes * B * H1 * N * csz);
  ALLOC(p->W, (size_t)p->W_elems * csz);
  ALLOC(p->nyq_fwd, B * nn * 2 * N * p->rsz);
  ALLOC(p->nyq_S, B * nn * p->n_rowitems * N * p->rsz);
  ALLOC(p->nyq_T, B * nn * p->geo.tparts * N * p->rsz);
  ALLOC(p->corr, B * 2 * N * p->rsz);
  ALLOC(p->nyq_anti, nn * 2 * N * p->rsz);
  ALLOC(p->nyq_part, B * 2 * std::min<size_t>(nn, 64) * N * csz);
  ALLOC(p->stage, B * N * N * p->rsz);
  {
    // the fused small-n path (FFST_TINY=0 keeps the persistent kernels; tuning / tests only)
    const char* et = std::getenv("FFST_TINY");
    p->tiny = d->n <= 64 && d->variant != FFST_USER && B * p->eta_l * N * N <= (64u << 20) && !(et && std::atoi(et) == 0);
    if (p->tiny) ALLOC(p->part, B * p->eta_l * N * N * p->rsz);
  }
#undef ALLOC
  std::vector<unsigned char> tw;
  if (d->dtype == FFST_F32) fill_twiddles<float>(tw, d->n); else fill_twiddles<double>(tw, d->n);
  e = cudaMemcpy(p->d_tw, tw.data(), tw.size(), cudaMemcpyHostToDevice);
  {
    const std::vector<double> rt = radial_all(d->n, j0, d->variant);
    if (d->dtype == FFST_F32) {
      std::vector<float> rf(rt.begin(), rt.end());
      if (e == cudaSuccess) e = cudaMemcpy(p->d_rtab, rf.data(), rf.size() * sizeof(float), cudaMemcpyHostToDevice);
    } else if (e == cudaSuccess) {
      e = cudaMemcpy(p->d_rtab, rt.data(), rt.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
  }
  if (e == cudaSuccess && !p->nyq.empty() && us) {
    std::vector<double> anti(p->nyq.size() * 2 * N);
    for (size_t q = 0; q < p->nyq.size(); ++q)
      std::copy_n(user_anti.begin() + (size_t)p->nyq[q] * 2 * N, 2 * N, anti.begin() + q * 2 * N);
    if (d->dtype == FFST_F32) {
      std::vector<float> af(anti.begin(), anti.end());
      e = cudaMemcpy(p->nyq_anti, af.data(), af.size() * sizeof(float), cudaMemcpyHostToDevice);
    } else {
      e = cudaMemcpy(p->nyq_anti, anti.data(), anti.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
  } else if (e == cudaSuccess && !p->nyq.empty()) {
    // anti part of each Nyquist plane on the Nyquist row / column (2n values per plane)
    const std::vector<double> tab = radial_all(d->n, j0, d->variant);
    const Radial<double> R = host_radial(tab, d->n, j0, d->variant);
    const int Hh = d->n / 2;
    std::vector<double> anti(p->nyq.size() * 2 * N);
    for (size_t q = 0; q < p->nyq.size(); ++q) {
      const PlaneDev& P = p->planes[p->nyq[q]];
      for (int bin = 0; bin < d->n; ++bin) {
        const int u = bin < Hh ? bin : bin - d->n;
        anti[(q * 2 + 0) * N + bin] = window_anti<double>(P, u, -Hh, Hh, R);
        anti[(q * 2 + 1) * N + bin] = window_anti<double>(P, -Hh, u, Hh, R);
      }
    }
    if (d->dtype == FFST_F32) {
      std::vector<float> af(anti.begin(), anti.end());
      e = cudaMemcpy(p->nyq_anti, af.data(), af.size() * sizeof(float), cudaMemcpyHostToDevice);
    } else {
      e = cudaMemcpy(p->nyq_anti, anti.data(), anti.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
  }
  if (e == cudaSuccess) e = cudaMemcpy(p->d_planes, p->planes.data(), p->planes.size() * sizeof(PlaneDev), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p->nyq.empty()) e = cudaMemcpy(p->d_nyq, p->nyq.data(), p->nyq.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(p->nyq_S, 0, B * nn * p->n_rowitems * N * p->rsz);
  if (e == cudaSuccess) e = cudaMemset(p->corr, 0, B * 2 * N * p->rsz);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "plan upload"));
  for (auto& ev : p->ev) {
    e = cudaEventCreate(&ev);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "event create"));
  }
  for (auto& ev : p->fork) {
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "event create"));
  }
  e = cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "stream create"));
  {
    ffst_status sc = setup_comm(p, d);
    if (sc != FFST_OK) return cleanup(sc);
  }
  Queue* q = nullptr;
  st = build_queue(p, d->batch, &q);
  if (st != FFST_OK) return cleanup(st);
  *out = p;
  return FFST_OK;
}

ffst_status ffst_plan_reserve(ffst_plan* p, int batch) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  if (batch < 1 || batch > p->d.batch) return fail(FFST_ERR_INVALID_ARG, "batch outside 1..plan batch");
  if (p->generic) return FFST_OK;          // the arbitrary-n path has no work queues
  TRY(set_device(p));
  Queue* q = nullptr;
  return build_queue(p, batch, &q);
}

ffst_status ffst_plan_local_planes(const ffst_plan* p, int* count, int* global_indices) {
  if (!p || !count) return fail(FFST_ERR_INVALID_ARG, "null argument");
  *count = p->eta_l;
  if (global_indices)
    for (int i = 0; i < p->eta_l; ++i) global_indices[i] = p->planes[i].gi;
  return FFST_OK;
}

ffst_status ffst_plan_workspace_bytes(const ffst_plan* p, size_t* bytes) {
  if (!p || !bytes) return fail(FFST_ERR_INVALID_ARG, "null argument");
  *bytes = p->ws_bytes;
  return FFST_OK;
}

ffst_status ffst_plan_info(const ffst_plan* p, int* n, int* j0, int* eta, int* eta_local, int* batch) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  if (n) *n = p->n;
  if (j0) *j0 = p->j0;
  if (eta) *eta = p->eta;
  if (eta_local) *eta_local = p->eta_l;
  if (batch) *batch = p->d.batch;
  return FFST_OK;
}

ffst_status ffst_plan_path(const ffst_plan* p, int* path) {
  if (!p || !path) return fail(FFST_ERR_INVALID_ARG, "null argument");
  *path = p->generic ? FFST_PATH_ARBITRARY_N : p->tiny ? FFST_PATH_FUSED_SMALL : FFST_PATH_PERSISTENT;
  return FFST_OK;
}

ffst_status ffst_plan_spectra_check(ffst_plan* p, double* tightness, double* asymmetry) {
  if (!p || !tightness || !asymmetry) return fail(FFST_ERR_INVALID_ARG, "null argument");
  if (p->tightness < 0) {
    // built-in systems: materialise the spectra once and reduce the same admission numbers
    if (p->d.shard_count != 1) return fail(FFST_ERR_UNSUPPORTED, "spectra check of a sharded built-in plan");
    TRY(set_device(p));
    if (p->generic) {   // materialise the local (= all) spectra, reduce the admission numbers
      const size_t bytes_g = (size_t)p->eta * p->n * p->n * p->rsz;
      void *psi_g = nullptr, *st_g = nullptr;
      cudaError_t eg = cudaMalloc(&psi_g, bytes_g);
      if (eg == cudaSuccess) eg = cudaMalloc(&st_g, 2 * sizeof(unsigned long long));
      if (eg == cudaSuccess) eg = cudaMemset(st_g, 0, 2 * sizeof(unsigned long long));
      const GenParams g = gen_params(p, 1);
      if (eg == cudaSuccess)
        eg = p->d.dtype == FFST_F32 ? launch_gen_spectra<float>(g, psi_g, 0, 0) : launch_gen_spectra<double>(g, psi_g, 0, 0);
      if (eg == cudaSuccess)
        eg = p->d.dtype == FFST_F32
                 ? launch_gen_user<float>(psi_g, nullptr, p->n, nullptr, 0, p->eta, 0, static_cast<unsigned long long*>(st_g), 0)
                 : launch_gen_user<double>(psi_g, nullptr, p->n, nullptr, 0, p->eta, 0, static_cast<unsigned long long*>(st_g), 0);
      unsigned long long hg[2] = {0, 0};
      if (eg == cudaSuccess) eg = cudaMemcpy(hg, st_g, sizeof(hg), cudaMemcpyDeviceToHost);
      cudaFree(psi_g);
      cudaFree(st_g);
      if (eg != cudaSuccess) { cudaGetLastError(); return cuda_fail(eg, "spectra check"); }
      std::memcpy(&p->tightness, &hg[0], sizeof(double));
      std::memcpy(&p->asymmetry, &hg[1], sizeof(double));
      *tightness = p->tightness;
      *asymmetry = p->asymmetry;
      return FFST_OK;
    }
    const size_t bytes = (size_t)p->eta * p->n * p->n * p->rsz;
    void *psi = nullptr, *st = nullptr;
    cudaError_t e = cudaMalloc(&psi, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&st, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(st, 0, 2 * sizeof(unsigned long long));
    KParams k = base_params(p);
    if (e == cudaSuccess)
      e = p->d.dtype == FFST_F32 ? launch_spectra_export<float>(k, psi, 0, 0) : launch_spectra_export<double>(k, psi, 0, 0);
    if (e == cudaSuccess) {
      UserPrep u{};
      u.psi = psi; u.n = p->n; u.eta = p->eta; u.centred = 0;
      u.shard_rank = 0; u.shard_count = 1; u.eta_l = p->eta_l;
      u.stats = static_cast<unsigned long long*>(st);
      e = p->d.dtype == FFST_F32 ? launch_user_prepare<float>(u, p->sm_count * 8, 0)
                                 : launch_user_prepare<double>(u, p->sm_count * 8, 0);
    }
    unsigned long long h[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(psi);
    cudaFree(st);
    if (e != cudaSuccess) { cudaGetLastError(); return cuda_fail(e, "spectra check"); }
    std::memcpy(&p->tightness, &h[0], sizeof(double));
    std::memcpy(&p->asymmetry, &h[1], sizeof(double));
  }
  *tightness = p->tightness;
  *asymmetry = p->asymmetry;
  return FFST_OK;
}

ffst_status ffst_shearlet_spectra(ffst_plan* p, void* psi, int centred, void* stream) {
  if (!p || !psi) return fail(FFST_ERR_INVALID_ARG, "null argument");
  TRY(set_device(p));
  if (p->generic) {
    const cudaError_t eg = p->d.dtype == FFST_F32
        ? launch_gen_spectra<float>(gen_params(p, 1), psi, centred, static_cast<cudaStream_t>(stream))
        : launch_gen_spectra<double>(gen_params(p, 1), psi, centred, static_cast<cudaStream_t>(stream));
    if (eg != cudaSuccess) return cuda_fail(eg, "spectra kernel");
    return FFST_OK;
  }
  KParams k = base_params(p);
  cudaError_t e = p->d.dtype == FFST_F32
                      ? launch_spectra_export<float>(k, psi, centred, static_cast<cudaStream_t>(stream))
                      : launch_spectra_export<double>(k, psi, centred, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "spectra kernel");
  return FFST_OK;
}

ffst_status ffst_sheartrans_batch(ffst_plan* p, const void* img, void* coeff, int batch, void* stream) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  return forward_impl(p, img, coeff, batch, static_cast<cudaStream_t>(stream));
}

ffst_status ffst_sheartrans(ffst_plan* p, const void* img, void* coeff, void* stream) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  return forward_impl(p, img, coeff, p->d.batch, static_cast<cudaStream_t>(stream));
}

ffst_status ffst_inversesheartrans_batch(ffst_plan* p, const void* coeff, void* img, int batch, int root,
                                         void* stream) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  return inverse_impl(p, coeff, img, batch, root, static_cast<cudaStream_t>(stream));
}

ffst_status ffst_inversesheartrans(ffst_plan* p, const void* coeff, void* img, int root, void* stream) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  return inverse_impl(p, coeff, img, p->d.batch, root, static_cast<cudaStream_t>(stream));
}

// Host-buffer variants: sharded plans with a communicator read / write the host images on rank 0.
ffst_status ffst_sheartrans_host(ffst_plan* p, const void* img_host, void* coeff, int batch, void* stream) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  const bool reads = p->comm == nullptr || p->d.shard_rank == 0;
  if (reads && !img_host) return fail(FFST_ERR_INVALID_ARG, "null argument");
  Queue* q = nullptr;
  TRY(validate_call(p, p->stage, coeff, batch, &q));          // everything checked before the copy
  TRY(set_device(p));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t bytes = (size_t)batch * p->n * p->n * p->rsz;
  if (reads) API_CUDA(cudaMemcpyAsync(p->stage, img_host, bytes, cudaMemcpyHostToDevice, s), "H2D image copy");
  return forward_impl(p, p->stage, coeff, batch, s);
}

ffst_status ffst_inversesheartrans_host(ffst_plan* p, const void* coeff, void* img_host, int batch, void* stream) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  const bool writes = p->comm == nullptr || p->d.shard_rank == 0;
  if (writes && !img_host) return fail(FFST_ERR_INVALID_ARG, "null argument");
  Queue* q = nullptr;
  TRY(validate_call(p, coeff, p->stage, batch, &q));
  TRY(set_device(p));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TRY(inverse_impl(p, coeff, p->stage, batch, 0, s));
  const size_t bytes = (size_t)batch * p->n * p->n * p->rsz;
  if (writes) API_CUDA(cudaMemcpyAsync(img_host, p->stage, bytes, cudaMemcpyDeviceToHost, s), "D2H image copy");
  return FFST_OK;
}

ffst_status ffst_sheartrans_compact(ffst_plan* p, const void* img, void* coeff_re, void* nyq_gh, int batch,
                                    void* stream) {
  if (!p || !nyq_gh) return fail(FFST_ERR_INVALID_ARG, "null argument");
  if (!aligned16(nyq_gh)) return fail(FFST_ERR_ALIGNMENT, "buffers must be 16-byte aligned");
  return forward_impl(p, img, coeff_re, batch, static_cast<cudaStream_t>(stream), nyq_gh);
}

ffst_status ffst_inversesheartrans_compact(ffst_plan* p, const void* coeff_re, const void* nyq_gh, void* img,
                                           int batch, void* stream) {
  if (!p || !nyq_gh) return fail(FFST_ERR_INVALID_ARG, "null argument");
  if (!aligned16(nyq_gh)) return fail(FFST_ERR_ALIGNMENT, "buffers must be 16-byte aligned");
  return inverse_impl(p, coeff_re, img, batch, 0, static_cast<cudaStream_t>(stream), nyq_gh);
}

ffst_status ffst_expand_compact(ffst_plan* p, const void* coeff_re, const void* nyq_gh, void* coeff, int batch,
                                void* stream) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  if (!coeff_re || !nyq_gh || !coeff) return fail(FFST_ERR_INVALID_ARG, "null buffer");
  if (batch < 1 || batch > p->d.batch) return fail(FFST_ERR_INVALID_ARG, "batch outside 1..plan batch");
  if (!aligned16(coeff_re) || !aligned16(nyq_gh) || !aligned16(coeff))
    return fail(FFST_ERR_ALIGNMENT, "buffers must be 16-byte aligned");
  if (p->generic) return fail(FFST_ERR_UNSUPPORTED, "compact format: power-of-two n (fast path) only");
  TRY(set_device(p));
  KParams k = base_params(p);
  const cudaError_t e = p->d.dtype == FFST_F32
      ? launch_expand_compact<float>(k, coeff_re, nyq_gh, coeff, batch, static_cast<cudaStream_t>(stream))
      : launch_expand_compact<double>(k, coeff_re, nyq_gh, coeff, batch, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "expand_compact kernel");
  return FFST_OK;
}

ffst_status ffst_plan_nyquist_planes(const ffst_plan* p, int* count, int* local_indices) {
  if (!p || !count) return fail(FFST_ERR_INVALID_ARG, "null argument");
  *count = (int)p->nyq.size();
  if (local_indices)
    for (size_t i = 0; i < p->nyq.size(); ++i) local_indices[i] = p->nyq[i];
  return FFST_OK;
}

ffst_status ffst_plan_set_timing(ffst_plan* p, int enable) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  p->timing = enable != 0;
  return FFST_OK;
}

ffst_status ffst_plan_phase_times(ffst_plan* p, float* times, int* launches) {
  if (!p || !times) return fail(FFST_ERR_INVALID_ARG, "null argument");
  if (!p->timing) return fail(FFST_ERR_INVALID_ARG, "timing not enabled");
  TRY(set_device(p));
  API_CUDA(cudaEventSynchronize(p->ev[6]), "event sync");
  API_CUDA(cudaEventSynchronize(p->ev[2]), "event sync");
  API_CUDA(cudaEventElapsedTime(&times[0], p->ev[1], p->ev[2]), "event time");
  API_CUDA(cudaEventElapsedTime(&times[1], p->ev[4], p->ev[5]), "event time");
  API_CUDA(cudaEventElapsedTime(&times[2], p->ev[0], p->ev[2]), "event time");
  API_CUDA(cudaEventElapsedTime(&times[3], p->ev[3], p->ev[6]), "event time");
  if (launches) {
    launches[0] = p->launches[0];
    launches[1] = p->launches[1];
  }
  return FFST_OK;
}

ffst_status ffst_plan_set_trace(ffst_plan* p, int enable) {
  if (!p) return fail(FFST_ERR_INVALID_ARG, "null plan");
  p->tracing = enable != 0;
  return FFST_OK;
}

ffst_status ffst_plan_trace(ffst_plan* p, int which, int batch, unsigned long long* host_out, int max_records,
                            int* n_records) {
  if (!p || !host_out || !n_records || (which != 0 && which != 1)) return fail(FFST_ERR_INVALID_ARG, "bad argument");
  if (!p->tracing || !p->d_trace[which]) return fail(FFST_ERR_INVALID_ARG, "tracing not enabled / no call yet");
  Queue* q = nullptr;
  TRY(set_device(p));
  TRY(find_queue(p, batch, &q));
  const int n = std::min(std::min(max_records, which == 0 ? q->n_fwd : q->n_inv), p->trace_items[which]);
  if (n < 0) return fail(FFST_ERR_INVALID_ARG, "max_records < 0");
  API_CUDA(cudaDeviceSynchronize(), "trace sync");
  API_CUDA(cudaMemcpy(host_out, p->d_trace[which], (size_t)n * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost),
           "trace copy");
  std::vector<ItemDev> items(n);
  API_CUDA(cudaMemcpy(items.data(), which == 0 ? q->d_fwd : q->d_inv, (size_t)n * sizeof(ItemDev),
                      cudaMemcpyDeviceToHost), "trace copy");
  // record = {smid, t_start, t_ready, t_end} -> append type/chunk in the high bits of smid
  for (int i = 0; i < n; ++i) host_out[8 * i] |= ((unsigned long long)items[i].type << 32) | ((unsigned long long)items[i].chunk << 40);
  *n_records = n;
  return FFST_OK;
}

const char* ffst_status_string(ffst_status s) {
  switch (s) {
    case FFST_OK: return "ok";
    case FFST_ERR_INVALID_SIZE: return "invalid size";
    case FFST_ERR_INVALID_ARG: return "invalid argument";
    case FFST_ERR_INDEX: return "index out of range";
    case FFST_ERR_DTYPE: return "invalid dtype";
    case FFST_ERR_ALIGNMENT: return "misaligned buffer";
    case FFST_ERR_OOM: return "out of device memory";
    case FFST_ERR_CUDA: return "CUDA error";
    case FFST_ERR_NCCL: return "NCCL error";
    case FFST_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* ffst_last_error_detail(void) { return g_detail.c_str(); }

}  // extern "C"
