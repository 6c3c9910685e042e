// ffst_internal.h — structures shared by the host planner (ffst_api.cu) and the
// kernels (ffst_kernels.cuh).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "ffst_math.cuh"

namespace ffst {

// One (image, local plane) of a batch call.
struct UnitDev {
  int b, p;        // image in the batch, local plane index
  int chunk;       // chunk this unit belongs to
  int woff;        // element (complex) offset of its intermediate inside the ring slot
};

// A self-contained work item of the persistent kernels (64 bytes, read with 4 vector loads;
// no dependent table lookups at item start).
//   type 0 = first pass (fwd: window * F -> column IFFT; inv: row R2C of a coefficient plane)
//   type 1 = second pass (fwd: row C2R -> coefficients; inv: column FFT * window, accumulate)
struct __align__(16) ItemDev {
  int type, chunk, group, b;
  int p;           // local plane (inverse pass 2: first plane of the chunk)
  int np;          // inverse pass 2: planes of the chunk (else 1)
  int woff;        // element offset of the (first) plane's intermediate in the ring slot
  int slot;        // ring slot
  int wait_ctr;    // counter to wait for (-1: none); pass 1 waits only before writing its slot
  int wait_tgt;    // value it must reach
  int wait2_ctr;   // inverse pass 2: previous owner of the column group (-1: none), target 1
  int first;       // inverse pass 2: first chunk of the image (initialise A)
  int sig_ctr;     // counter incremented when done
  int sig2_ctr;    // second counter (inverse pass 2: own column-group flag), or -1
  int pad0;        // forward pass 1 (paired images): the second image, or -1
  int pad1;        // inverse pass 2: accumulator lane of the chunk (copy of A it accumulates into)
};

struct ChunkDev {
  int slot;            // ring slot of the chunk's intermediates
  int b;               // image (chunks never span images)
  int unit0, nunits;   // units [unit0, unit0 + nunits)
  int p1_items, p2_items;
  int first_of_image;  // inverse: this chunk initialises the image's accumulator
  int prev_slot_chunk; // chunk that used the same slot before (or -1)
};

struct KParams {
  int n, j0, batch, eta_l, n_nyq;
  double delta;                 // grid spacing Delta = 2^(2 j0) / n
  const PlaneDev* planes;       // [eta_l]
  const int* nyq_planes;        // [n_nyq] local plane index of each Nyquist plane
  const void* tw;               // cpx<T>[n]: exp(-2 pi i m / n)
  const void* rtab;             // T[(j0+1)][n/2+1]: radial factors psi1(4^-j Delta a), varphi(Delta a)
  const void* img;              // [batch][n][n] T
  void* coeff;                  // [batch][eta_l][n][n] cpx<T>
  void* img_out;                // [batch][n][n] T
  void* F;                      // [batch][n/2+1][n] cpx<T>: image spectrum, column-major half (F[b][u1][u2])
  void* Fscr;                   // [batch][n/2+1][n] cpx<T>: scratch (row-pass output)
  void* A;                      // [lanes][batch][n/2+1][n] cpx<T>: adjoint accumulators, same layout as F
  long long a_lane_elems;       // elements per accumulator lane
  int a_lanes;                  // lanes in use (the final pass sums them in lane order)
  void* W;                      // ring of intermediates, slot s at W + s * slot_elems
  long long slot_elems;
  void* nyq_fwd;                // [batch][n_nyq][2][n] T: forward Nyquist terms G(m1), H(r)
  void* nyq_S;                  // [batch][n_nyq][n_rowitems][n] T: partial alternating column sums
  void* nyq_T;                  // [batch][n_nyq][nyq_tparts][n] T: alternating row sums (partials summed in order)
  void* corr;                   // [batch][2][n] T: inverse Nyquist corrections
  void* nyq_part;               // [batch][2][<=64][n] cpx<T>: partial Nyquist spectra (stage 1 -> 2)
  void* part;                   // small-n fused path: [batch][eta_l][n][n] T partial images of the inverse
  const void* nyq_anti;         // [n_nyq][2][n] T: anti part of each Nyquist plane on the Nyquist row (0) /
                                //   column (1), natural bin order (plan table)
  int n_rowitems;               // inverse pass-1 items per plane (row groups)
  int nyq_tparts;               // partial row sums per row in nyq_T (the pair row pass: one per warp of a line)
  int rpi;                      // inverse pass 1: rows per item (a multiple of Geo::GR)
  const ItemDev* items;
  int n_items;
  const ChunkDev* chunks;
  const UnitDev* units;
  int* ctr;                     // [0] dispatch; [ctr_p1 + c]; [ctr_p2 + c]; [ctr_g + item]
  int ctr_p1, ctr_p2, ctr_g;
  int variant;                  // 0 classic (meyerShearletSpect), 1 smooth (meyerNewShearletSpect), 2 user
  const void* usym;             // user spectra: [eta_l][n/2+1][n] T symmetric parts (ffst_user.cuh), else nullptr
  int compact;                  // f1 compact format: cube of reals + Nyquist vectors (G, H) in nyq_fwd
  int dbg;                      // measurement only (FFST_DBG): bit 0 skip FFTs, bit 1 skip output stores
  int ring_stream;              // the intermediate ring is larger than L2: stream it (evict_first)
  int sync_mode;                // dependency ordering: bit 0 acquire fence after waits, bit 1 release on WAR-only signals
  unsigned long long* trace;    // optional: per item {smid, t_start, t_ready, t_end} (globaltimer ns)
};

// Plan-time preparation of user-supplied spectra (ffst_user.cuh).
struct UserPrep {
  const void* psi;          // [eta][n][n] T, device (the caller's; read only here)
  int n, eta, centred;
  int shard_rank, shard_count, eta_l;
  void* usym;               // [eta_l][n/2+1][n] T (out)
  int* hull;                // [eta_l][2] column lo / hi where sym != 0 (in: n/2+1 / -1)
  void* anti;               // [eta_l][2][n] T (out): anti part on the Nyquist row (0) / column (1)
  unsigned long long* stats;   // [2] bit patterns of two non-negative doubles (in: 0): tightness, asymmetry
};

// Launch geometry of one (T, N) instantiation (host + device visible).
struct Geometry {
  int nt;            // threads per CTA
  int gc;            // fwd pass 1: columns per item
  int rp2;           // fwd pass 2: rows per item
  int rpi;           // inv pass 1: rows per item
  int gr;            // inv pass 1: rows per tile
  int lpc;           // columns per round of the column kernels
  int igc;           // inv pass 2: columns per item (column group of the accumulation chain)
  size_t smem_fwd, smem_inv, smem_aux;   // dynamic shared bytes of the kernels
  int colpad;        // forward intermediate: row stride = ncols rounded up to a multiple of colpad
  int ncpf;          // final column pass (aux kernels, Geo): padded row stride of its output
  int tparts;        // inv pass 1: partial alternating row sums per row (nyq_T)
};

// Launchers (defined per dtype in ffst_kern_f32.cu / ffst_kern_f64.cu).
template <typename T> Geometry geometry(int n);
template <typename T> cudaError_t launch_spectrum(const KParams& p, int batch, cudaStream_t s);
template <typename T> cudaError_t launch_nyq_fwd(const KParams& p, int batch, cudaStream_t s);
template <typename T> cudaError_t launch_fwd_main(const KParams& p, int grid, cudaStream_t s);
template <typename T> cudaError_t launch_inv_main(const KParams& p, int grid, cudaStream_t s);
template <typename T> cudaError_t launch_nyq_inv(const KParams& p, int batch, cudaStream_t s);
template <typename T> cudaError_t launch_nyq_compact_sums(const KParams& p, int batch, cudaStream_t s);
template <typename T> cudaError_t launch_final(const KParams& p, int batch, int which, cudaStream_t s);
template <typename T> cudaError_t launch_user_prepare(const UserPrep& u, int grid, cudaStream_t s);
template <typename T> cudaError_t launch_spectra_export(const KParams& p, void* psi, int centred, cudaStream_t s);
template <typename T> cudaError_t launch_expand_compact(const KParams& p, const void* re, const void* gh, void* out,
                                                        int batch, cudaStream_t s);
template <typename T> int max_active_main(int n, int device, int which);   // CTAs/SM of fwd (0) / inv (1)
template <typename T> cudaError_t launch_tiny(const KParams& p, int batch, int which, cudaStream_t s);   // n <= 64

// Arbitrary-n path (ffst_generic.cuh, ffst_gen_launch.cuh).
struct GenParams;
enum { GEN_OP_SPEC = 0, GEN_OP_DFT = 1, GEN_OP_IDFT = 2, GEN_OP_FWD_COL = 3, GEN_OP_INV_COL = 4, GEN_OP_FINAL = 5 };
template <typename T> cudaError_t launch_gen_rows(int op, const GenParams& g, const void* src, void* dst, int np,
                                                  int p0, int first, double scale, int cube_side, int cube_eta,
                                                  int mats, cudaStream_t s);
template <typename T> cudaError_t launch_gen_transpose(const void* src, void* dst, int n, int mats, cudaStream_t s);
template <typename T> cudaError_t launch_gen_spectra(const GenParams& g, void* psi, int centred, cudaStream_t s);
template <typename T> cudaError_t launch_gen_user(const void* psi, void* out, int n, const int* gidx, int eta_l,
                                                  int eta, int centred, unsigned long long* stats, cudaStream_t s);

}  // namespace ffst
