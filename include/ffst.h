/*
 * ffst.h — C ABI of the B200-native Fast Finite Shearlet Transform (FFST,
 * arxiv 1202.1773; citations "P:Lnnn" are lines of the paper's PAPER.md).
 *
 * The library computes, on one CUDA device (sm_100a), the data-parallel hot
 * path of the paper: the forward transform
 *     SH(f)(i) = ifft2( psi_hat_i * fft2(f) ),  i = 1..eta          (eq:shearletTransform)
 * and its adjoint / inverse
 *     f = Re ifft2( sum_i psi_hat_i * fft2(c_i) )                  (eq:inverseShearletTransform)
 * with the cone-adapted Meyer shearlet spectra psi_hat_i of Sec. 2-3.5
 * evaluated on the fly inside the kernels (never stored).
 *
 * Conventions (all functions):
 *  - Images are real, square, row-major [batch][n][n]: element (r, c) is the
 *    sample at m2 = r (row), m1 = c (column).
 *  - Coefficient cubes are complex, interleaved (re, im), row-major
 *    [batch][eta_local][n][n], planes in the flat-index order of Sec. 3.5.1
 *    (P:L2076-2097).  Coefficients are complex: for even n the finest-scale
 *    planes carry an imaginary part (reading A8).
 *  - Element precision is the plan's dtype (float or double) for images and
 *    for each of re/im of coefficients.
 *  - Flat indices in this ABI are 0-based (the paper's i = index + 1).
 *  - Ownership: the caller owns every image / coefficient / spectra buffer it
 *    passes (device memory unless the function name ends in _host).  The plan
 *    owns its tables and workspace, allocated in ffst_plan_create (and, for the
 *    work queue of another batch size, ffst_plan_reserve); no transform call
 *    allocates, uploads or synchronises, and the library never frees caller memory.
 *  - Streams: `stream` is a cudaStream_t (0 = legacy default stream).  All
 *    device-buffer calls are asynchronous on that stream; a plan serves one
 *    stream at a time (calls on one plan must not overlap).
 *  - Errors: every function returns an ffst_status (never aborts, never throws).
 *    Arguments are validated before anything is launched.  CUDA failures map to
 *    FFST_ERR_CUDA with a detail string (ffst_last_error_detail, thread-local);
 *    asynchronous kernel faults surface at a later call or synchronisation.
 *  - Buffers must be 16-byte aligned and contiguous.
 *  - Multi-GPU (eta-sharding): a plan created with shard_count = G > 1
 *    owns a subset of the planes (ffst_shard_planes: a cost-balanced LPT map by
 *    default, or round robin i mod G); its cube holds only those planes.  With an
 *    NCCL communicator in the descriptor (nccl_comm, the G ranks, rank = shard_rank)
 *    the library runs the two exchange steps itself on a plan-owned stream, chunked
 *    by image groups so that they overlap the kernels: the forward broadcasts the
 *    images from rank 0, the inverse sums the ranks' partial adjoint spectra onto
 *    `root` (the inverse is linear in the planes, eq:inverseShearletTransform,
 *    P:L1730-1764) and only the root runs the final synthesis.  Without a
 *    communicator the inverse returns the partial image of the local planes (the
 *    caller reduces).
 */
#ifndef FFST_H
#define FFST_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FFST_OK = 0,
  FFST_ERR_INVALID_SIZE = 1,   /* n < 4 (no scale fits) or n > 4096 */
  FFST_ERR_INVALID_ARG = 2,    /* null pointer, bad batch / shard / option */
  FFST_ERR_INDEX = 3,          /* flat index or (kind, j, k) outside the system */
  FFST_ERR_DTYPE = 4,          /* unknown dtype */
  FFST_ERR_ALIGNMENT = 5,      /* buffer not 16-byte aligned */
  FFST_ERR_OOM = 6,            /* workspace allocation failed at plan creation */
  FFST_ERR_CUDA = 7,           /* CUDA runtime error (see ffst_last_error_detail) */
  FFST_ERR_NCCL = 8,           /* NCCL failure (see ffst_last_error_detail) */
  FFST_ERR_UNSUPPORTED = 9     /* size or option outside the build (see each call), or more local planes than built */
} ffst_status;

typedef enum { FFST_F32 = 0, FFST_F64 = 1 } ffst_dtype;

/* FFST_CLASSIC: meyerShearletSpect, eq:Psi1/eq:Psi2.
 * FFST_SMOOTH: meyerNewShearletSpect, the smooth system of Sec. smoothShearlets
 * (P:L1766-1820): low-pass Phi(w) = varphi(w1) varphi(w2) (eq:Phi), cone shearlets
 * Psi1(4^-j w) psi2(2^j w_b/w_a + k) with Psi1 = sqrt(Phi^2(w/4) - Phi^2(w)) (eq:newPsi1,
 * eq:smoothPsi), same cones, seams and index order; isotropic dilation (reading A18). */
typedef enum { FFST_CLASSIC = 0, FFST_SMOOTH = 1, FFST_USER = 2 } ffst_variant;   /* USER: see ffst_plan_create_user */

/* Shearlet kinds of the flat index (Sec. 3.5.1): low-pass, horizontal cone,
 * vertical cone, glued seam ("h x v", |k| = 2^j). */
typedef enum { FFST_KIND_LOWPASS = 0, FFST_KIND_H = 1, FFST_KIND_V = 2, FFST_KIND_X = 3 } ffst_kind;

typedef struct ffst_plan ffst_plan;   /* opaque */

/* Plane-to-rank map of a sharded plan.  LPT: planes sorted by their cost
 * n/2 + (pruned column count) (the row pass plus the pruned column pass of each direction, in
 * line FFTs) and dealt greedily to the least-loaded rank; ROUND_ROBIN: plane i on rank i mod G. */
typedef enum { FFST_SHARD_LPT = 0, FFST_SHARD_ROUND_ROBIN = 1 } ffst_shard_policy;

typedef struct {
  int n;              /* image side: a power of two 4..4096 (float64: ..2048), or any other n in 5..2048
                         (the arbitrary-n path, full complex transforms with Bluestein
                         line DFTs; no compact format) */
  int j0;             /* number of scales; 0 = default floor(log2(n)/2) */
  int batch;          /* maximum images per call, >= 1 */
  ffst_dtype dtype;   /* FFST_F32 or FFST_F64 */
  ffst_variant variant;
  int device;         /* CUDA device ordinal */
  int shard_rank;     /* 0 <= shard_rank < shard_count */
  int shard_count;    /* >= 1: the planes of ffst_shard_planes(n, j0, shard_count, shard_rank, policy) are local */
  ffst_shard_policy shard_policy;   /* FFST_SHARD_LPT (0, default) or FFST_SHARD_ROUND_ROBIN; user-spectra
                                       plans always use round robin */
  void* nccl_comm;    /* ncclComm_t over the shard_count ranks (NCCL rank = shard_rank) from
                         ffst_nccl_comm_create, or NULL (no library collectives); not owned by the plan */
} ffst_plan_desc;

/* ---- host-only queries (no device needed) ------------------------------ */

/* j0 = floor(1/2 log2 n).  n < 4 -> FFST_ERR_INVALID_SIZE. */
ffst_status ffst_scales_for_size(int n, int* j0);

/* eta = 2^(j0+2) - 3 (eq:numberOfScalesAndShears); -1 if j0 < 1. */
int ffst_num_shearlets(int j0);

/* Flat index (0-based) <-> (kind, j, k), order of Sec. 3.5.1:
 * per band j: (h,0), (h,-1..-(2^j-1)), (x,-2^j), (v,-2^j+1..2^j-1), (x,2^j), (h,2^j-1..1).
 * The low-pass (index 0) reports kind 0, j = 0, k = 0. */
ffst_status ffst_index_to_params(int j0, int index, int* kind, int* j, int* k);
ffst_status ffst_params_to_index(int j0, int kind, int j, int k, int* index);

/* Column range [*col_lo, *col_hi] (0 <= col <= n/2, column c <-> |omega_1| = c on the
 * Delta-scaled grid) outside which plane `index` is identically zero
 * (used for pruning the first FFT pass; a superset of the true support). */
ffst_status ffst_plane_support(int n, int j0, int index, int* col_lo, int* col_hi);

/* 1 if plane `index` of the CLASSIC system is not point-symmetric on the even grid (non-zero
 * anti-symmetric part on the Nyquist row/column), else 0.  A plan's own list, for either
 * variant: ffst_plan_nyquist_planes. */
ffst_status ffst_plane_is_nyquist(int n, int j0, int index, int* is_nyquist);

/* Global 0-based indices of the planes rank `shard_rank` of `shard_count` owns (ascending), for the
 * built-in systems; j0 = 0: default.  global_indices may be NULL (count only).
 * Errors: INVALID_SIZE, INVALID_ARG (bad shard / policy), UNSUPPORTED (n not supported). */
ffst_status ffst_shard_planes(int n, int j0, int shard_count, int shard_rank, ffst_shard_policy policy, int* count,
                              int* global_indices);

/* ---- NCCL communicators for sharded plans -------------------------------- */

/* 128 opaque bytes (an ncclUniqueId): created on one rank, shared with the others out of band
 * (e.g. a torch.distributed broadcast), then passed to ffst_nccl_comm_create on every rank. */
typedef struct { char bytes[128]; } ffst_nccl_id;
ffst_status ffst_nccl_unique_id(ffst_nccl_id* id);
/* Collective over the nranks ranks (each calls it with its rank and device).  *comm receives an
 * ncclComm_t for ffst_plan_desc.nccl_comm.  Errors: INVALID_ARG, CUDA, NCCL. */
ffst_status ffst_nccl_comm_create(void** comm, int nranks, int rank, const ffst_nccl_id* id, int device);
ffst_status ffst_nccl_comm_destroy(void* comm);

/* ---- plans ------------------------------------------------------------- */

/* Create a plan: all tables (index order, pruning ranges, radial factors, Nyquist anti-window
 * edges, work queues) and all device workspace are built here; transforms allocate nothing.
 * Errors: INVALID_SIZE (n < 4 or above the built sizes), UNSUPPORTED (n not a power of two above 2048,
 * more than 256 local planes), INVALID_ARG (incl. an unknown variant), OOM, CUDA.
 * Environment (read here, tuning only; results are identical up to rounding order):
 *   FFST_RING_MB        intermediate ring budget (default 80; at least 12 slots)
 *   FFST_CHUNK_PLANES   planes per chunk (default 4; batch <= 4: eta / lanes, or 32 with one lane)
 *   FFST_SLOT_KB        chunk byte budget (default 4096; 12288 for n >= 1024)
 *   FFST_ACC_LANES      accumulator lanes of the inverse (default: up to 4, 16 for batch <= 4, while <= 32 MB)
 *   FFST_VERBOSE        print the queue geometry and the persistent grids
 *   FFST_CTAS_PER_SM    cap on resident CTAs per SM of the persistent kernels (default: occupancy)
 * Measurement only (results are WRONG): FFST_QUEUE_ONLY=1|2 (one pass type), FFST_DBG bits (1 skip the
 * FFTs, 2 skip the item output stores, 4 window = 1 on the support columns, 8 skip the Nyquist sums,
 * 32 the plain (not pipelined) inverse pass 1),
 * FFST_SYNC (0..3: drop the acquire fences / the WAR releases). */
ffst_status ffst_plan_create(ffst_plan** out, const ffst_plan_desc* desc);
ffst_status ffst_plan_destroy(ffst_plan* plan);

/* User-supplied spectra: "precomputed shearlet spectra which are then used for
 * the computation of the transform" (the inverse with the same Psi,
 * P:L2221-2224).  psi: DEVICE pointer (on desc->device) to eta real spectra [eta][n][n] of the
 * plan's dtype, rows omega_2, columns omega_1; centred_layout != 0: omega = 0 at (n/2, n/2) (the
 * paper's Psi), else natural FFT bin order.  Read during this call only (the plan
 * keeps its own Hermitian-half copy of the symmetric parts, eta_local x (n/2+1) x n reals, and
 * prunes each plane to its non-zero column range).  desc->variant and desc->j0 are ignored;
 * eta may be any count >= 1 (the plan's eta).  Sharding as for ffst_plan_create (all eta
 * planes are passed on every rank).  Any real spectra are accepted: point-symmetric ones off the
 * Nyquist lines (psi(u) = psi(-u) for u1, u2 != -n/2 to within 1e-5 (float32) / 1e-12 (float64),
 * the spectra of real shearlets; every built-in system is) run on the Hermitian fast path (the
 * Nyquist row and column may be asymmetric, handled exactly); any other set runs on
 * the full complex path of arbitrary n (n <= 2048; above: INVALID_ARG).  The Parseval admission
 * check of P:L2219-2220 is computed but not enforced: ffst_plan_spectra_check.
 * Errors: as ffst_plan_create, plus INVALID_ARG (null psi, eta < 1, asymmetric spectra at n = 4096). */
ffst_status ffst_plan_create_user(ffst_plan** out, const ffst_plan_desc* desc, int eta, const void* psi,
                                  int centred_layout);

/* Admission numbers of the plan's system: *tightness = max over the grid of
 * |sum_i psi_i^2 - 1| (0 for a Parseval frame, "close to zero" in the paper), *asymmetry = max
 * |psi_i(u) - psi_i(-u)| off the Nyquist lines.  User plans: computed at creation.  Built-in
 * plans: computed on the first call from the materialised spectra (needs shard_count == 1,
 * else UNSUPPORTED; allocates eta n^2 reals temporarily). */
ffst_status ffst_plan_spectra_check(ffst_plan* plan, double* tightness, double* asymmetry);

/* Reserve the work queues of the persistent kernels for calls with `batch` images (1 <= batch <=
 * the plan's batch; ffst_plan_create reserves the plan's batch).  Builds and uploads the queue
 * (plan-owned device memory, synchronous); a no-op if already reserved.  Transforms with a batch
 * that was not reserved fail with INVALID_ARG before launching anything (so a transform never
 * allocates, uploads or synchronises, and can be captured in a CUDA graph).
 * Errors: INVALID_ARG (null plan, batch out of range), OOM, CUDA. */
ffst_status ffst_plan_reserve(ffst_plan* plan, int batch);

/* Number of local planes and (if global_indices != NULL) their 0-based global indices. */
ffst_status ffst_plan_local_planes(const ffst_plan* plan, int* count, int* global_indices);
ffst_status ffst_plan_workspace_bytes(const ffst_plan* plan, size_t* bytes);
ffst_status ffst_plan_info(const ffst_plan* plan, int* n, int* j0, int* eta, int* eta_local, int* batch);

/* The schedule the plan's complex transforms run on:
 * PERSISTENT   power-of-two n >= 128 (and n <= 64 with FFST_TINY=0, or user spectra): the two
 *              persistent work-queue kernels per direction (Hermitian halving, pruning);
 * FUSED_SMALL  power-of-two n <= 64: one CTA per (plane, image) in shared memory (the compact
 *              format still uses the persistent kernels);
 * ARBITRARY_N  any other n (or asymmetric user spectra): full complex transforms, Bluestein DFTs. */
typedef enum { FFST_PATH_PERSISTENT = 0, FFST_PATH_FUSED_SMALL = 1, FFST_PATH_ARBITRARY_N = 2 } ffst_path;
ffst_status ffst_plan_path(const ffst_plan* plan, int* path);

/* ---- transforms (device buffers) ---------------------------------------- */

/* Materialise the local spectra psi_hat_i (tests / diagnostics only; the
 * transforms never store them): psi is [eta_local][n][n] real; centred != 0 puts
 * omega = 0 at (n/2, n/2) (the paper's Psi layout), else natural
 * FFT bin order. */
ffst_status ffst_shearlet_spectra(ffst_plan* plan, void* psi, int centred, void* stream);

/* Forward: img [batch][n][n] real -> coeff [batch][eta_local][n][n] complex.
 * With an NCCL communicator: img is read on rank 0 only (it may be NULL elsewhere) and broadcast
 * to the other ranks inside the call (into the plan's staging buffer). */
ffst_status ffst_sheartrans(ffst_plan* plan, const void* img, void* coeff, void* stream);
ffst_status ffst_sheartrans_batch(ffst_plan* plan, const void* img, void* coeff, int batch, void* stream);

/* Inverse / adjoint: coeff [batch][eta_local][n][n] complex -> img_out [batch][n][n] real
 * = Re ifft2(sum_i psi_hat_i fft2(c_i)).  shard_count == 1: the full image (root ignored).
 * Sharded with an NCCL communicator: the ranks' partial adjoint spectra are summed onto rank
 * `root`, which alone writes img_out (the full image; img_out may be NULL on other ranks).
 * Sharded without one: img_out is the partial image of the local planes (root ignored). */
ffst_status ffst_inversesheartrans(ffst_plan* plan, const void* coeff, void* img_out, int root, void* stream);
ffst_status ffst_inversesheartrans_batch(ffst_plan* plan, const void* coeff, void* img_out, int batch, int root,
                                         void* stream);

/* ---- host-buffer variants (end-to-end path) ----------------------------- */

/* Same as the _batch calls, with the image in HOST memory (pinned for full speed):
 * the host<->device copy of the image is issued on `stream` inside the call
 * (through a plan-owned device staging buffer).  The cube stays on the device.
 * Sharded plans with a communicator: root 0 (the images are read / written on rank 0). */
ffst_status ffst_sheartrans_host(ffst_plan* plan, const void* img_host, void* coeff, int batch, void* stream);
ffst_status ffst_inversesheartrans_host(ffst_plan* plan, const void* coeff, void* img_host, int batch, void* stream);

/* ---- instrumentation ----------------------------------------------------- */

/* ---- compact coefficient format ---------------------------
 * For even n the forward's complex cube is c_i = x_i + i y_i with x_i real and y_i of rank <= 2,
 * y_i(r, m1) = (-1)^r G_i(m1) + (-1)^m1 H_i(r), non-zero only for the plan's Nyquist planes
 * (DESIGN.md 6.2).  The compact format stores x as [batch][eta_local][n][n] reals and (G_i, H_i)
 * as nyq_gh [batch][n_nyq][2][n] reals (Nyquist planes in the order of
 * ffst_plan_nyquist_planes): half the bytes of the complex cube, lossless for every cube the
 * forward produces (an arbitrary complex cube, e.g. after thresholding, is not representable:
 * use the complex entry points).  Same validation, streams, errors and sharding (root 0) as the
 * complex calls. */
ffst_status ffst_sheartrans_compact(ffst_plan* plan, const void* img, void* coeff_re, void* nyq_gh, int batch,
                                    void* stream);
ffst_status ffst_inversesheartrans_compact(ffst_plan* plan, const void* coeff_re, const void* nyq_gh, void* img_out,
                                           int batch, void* stream);
/* The complex cube of a compact one (format conversion, one kernel): coeff [batch][eta_local][n][n]
 * complex = coeff_re + i (-1)^r G_i(m1) + i (-1)^m1 H_i(r) on the Nyquist planes, coeff_re + 0 i
 * elsewhere.  Errors: INVALID_ARG, ALIGNMENT, CUDA. */
ffst_status ffst_expand_compact(ffst_plan* plan, const void* coeff_re, const void* nyq_gh, void* coeff, int batch,
                                void* stream);
/* The local Nyquist planes: count and (if local_indices != NULL) their local plane indices. */
ffst_status ffst_plan_nyquist_planes(const ffst_plan* plan, int* count, int* local_indices);

/* enable != 0: record CUDA events around each internal kernel phase (on the
 * call's stream).  ffst_plan_phase_times returns the durations (ms) of the last
 * call of each direction: times[0] = forward main kernel, [1] = inverse main
 * kernel, [2] = forward total, [3] = inverse total; launches[0..1] = number of
 * kernels the last forward / inverse call launched.  Synchronises the events. */
ffst_status ffst_plan_set_timing(ffst_plan* plan, int enable);
ffst_status ffst_plan_phase_times(ffst_plan* plan, float* times, int* launches);

/* Per-item trace of the persistent kernels (diagnostics): enable, run a call, then read
 * which = 0 (forward) / 1 (inverse) records of the queue for `batch` images:
 * 8 x u64 per item in queue order = {smid | type << 32 | chunk << 40, t_start, t_ready, t_end,
 * probe0..probe3} (%globaltimer ns; t_ready = after the item's dependency wait; probes = intra-item
 * phase marks, 0 if unused).  Synchronises the device. */
ffst_status ffst_plan_set_trace(ffst_plan* plan, int enable);
ffst_status ffst_plan_trace(ffst_plan* plan, int which, int batch, unsigned long long* host_out, int max_records,
                            int* n_records);

const char* ffst_status_string(ffst_status status);
const char* ffst_last_error_detail(void);

#ifdef __cplusplus
}
#endif
#endif /* FFST_H */
