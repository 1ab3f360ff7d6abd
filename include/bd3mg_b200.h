/*
 * bd3mg_b200.h -- C ABI of the B200-native BD3MG hot path.
 *
 * Drop-in boundary for the reference package `bd3mg` (arXiv 2002.02328 CPU
 * reference, /root/reference/pkg).  The reference binds its native core at
 * import time in pkg/src/bd3mg/kernels.py:16-28 (`_core` or `_kernels_np`);
 * a ctypes binding of this library replaces that module (see
 * INTEGRATION.md).  Every entry point:
 *   - takes plain pointers and sizes (no framework types),
 *   - returns an int status (BD3MG_OK = 0); the message of the last failure on
 *     the calling thread is available from bd3mg_last_error(),
 *   - device-pointer variants are asynchronous on `stream` (a cudaStream_t
 *     passed as void*, NULL = legacy default stream),
 *   - *_host variants take host buffers and are synchronous (they stage
 *     through device memory and return after the result is on the host).
 * Volumes are C-contiguous (nz, ny, nx), x fastest; kernel stacks are
 * (nz, kz, ky, kx) indexed by the OUTPUT depth (reference blur.py:5-12).
 * Depth coordinates are global: fragment plane 0 is depth frag_z0.
 */
#ifndef BD3MG_B200_H
#define BD3MG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BD3MG_OK = 0,
  BD3MG_EINVAL = 1,      /* bad shape / range / coverage (reference: ValueError) */
  BD3MG_ECUDA = 2,       /* CUDA runtime failure */
  BD3MG_EWORKSPACE = 3,  /* workspace smaller than *_ws_bytes reported */
  BD3MG_ENONFINITE = 4,  /* non-finite gradient (directions.py:64-65) */
  BD3MG_EFORMAT = 5,     /* container payload violates the format (volume.py:31 FormatError) */
  BD3MG_EIO = 6          /* file open / read / write failure (reference: OSError) */
};

enum { BD3MG_F64 = 0, BD3MG_F32 = 1 };

/* Problem geometry: volume (nz, ny, nx) and kernel extents (kz, ky, kx), odd. */
typedef struct {
  int64_t nx, ny, nz;
  int32_t kx, ky, kz;
  int32_t dtype; /* BD3MG_F64 or BD3MG_F32: element type of every array */
} bd3mg_geom_t;

/* Regulariser weights: reference objective.py:46-62 (RegParams). */
typedef struct {
  double lam, eta, kappa, delta, x_min, x_max;
} bd3mg_reg_t;

/* One block step of the memory-gradient solver (reference
 * directions.py:89-94 mg_direction + scheduler.py:151-153 receive_update).
 * `frag` is the anchor slab; it must cover [z_lo-kz, z_hi+kz] clamped to the
 * volume (blur.py:190-198 slab_support).  Pointers are device pointers of
 * the geometry's dtype. */
typedef struct {
  const void* frag;
  int64_t frag_z0, nzf;
  int64_t z_lo, z_hi;
  const void* d_mem;  /* block rows of the memory direction, or NULL (= 0) */
  void* inc_out;      /* block rows receiving the increment, or NULL */
  void* x_rows;       /* block rows of an iterate updated in place, or NULL */
  void* dmem_rows;    /* block rows of the memory store overwritten, or NULL */
} bd3mg_task_t;

/* Per-task StepInfo record (reference directions.py:29-40), 16 doubles:
 * [0..2] gram (00,01,11 over the kept columns; one column -> [0]),
 * [3..4] rhs, [5..6] coeffs, [7] ncols, [8] status (1 = non-finite g, 2 = non-finite
 * increment: the 2x2 solve overflowed; in both cases nothing is applied),
 * [9] |g|, [10] coefficient of -g, [11] coefficient of d_mem,
 * [12] kept-column mask (1 = -g, 2 = d_mem). */
#define BD3MG_INFO_DOUBLES 16

/* Objective terms written by bd3mg_eval_f (device, 7 doubles):
 * [0] data, [1] box, [2] tv, [3] axial, [4] f, [5] |x-snap|^2, [6] |snap|^2 */
#define BD3MG_EVAL_DOUBLES 7

const char* bd3mg_last_error(void);
const char* bd3mg_version(void);
/* Number of kernels this library has launched in the process (eager calls;
 * a captured CUDA graph's replays are not counted). */
long long bd3mg_launch_count(void);
/* The library's own CUDA runtime is bound to the device of the caller's
 * streams with bd3mg_set_device (cudaSetDevice); the Python layer does it
 * whenever the device of the stream it passes changes. */
int bd3mg_set_device(int device);
int bd3mg_get_device(int* device);

/* ---- drop-in native core: replaces bd3mg._core (src/_core.pyx:17-96) ---- */
/* H rows: out[i] = sum_{a,b,c} K[zo,a,b,c] frag[zo+a-rz-frag_z0, y+b-ry, x+c-rx],
 * zo = out_lo + i, zero outside the fragment.  Replaces
 * _core.depthvar_correlate (src/_core.pyx:17-53).  out: (out_hi-out_lo+1, ny, nx). */
int bd3mg_depthvar_correlate_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx,
                                 const double* kernels, int64_t nzk, int64_t kz, int64_t ky, int64_t kx,
                                 int64_t frag_z0, int64_t out_lo, int64_t out_hi, double* out, void* stream);
/* H^T rows.  Replaces _core.depthvar_correlate_adjoint (src/_core.pyx:56-96). */
int bd3mg_depthvar_correlate_adjoint_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx,
                                         const double* kernels, int64_t nzk, int64_t kz, int64_t ky,
                                         int64_t kx, int64_t frag_z0, int64_t out_lo, int64_t out_hi,
                                         double* out, void* stream);
int bd3mg_depthvar_correlate_f32(const float* frag, int64_t nzf, int64_t ny, int64_t nx, const float* kernels,
                                 int64_t nzk, int64_t kz, int64_t ky, int64_t kx, int64_t frag_z0,
                                 int64_t out_lo, int64_t out_hi, float* out, void* stream);
int bd3mg_depthvar_correlate_adjoint_f32(const float* frag, int64_t nzf, int64_t ny, int64_t nx,
                                         const float* kernels, int64_t nzk, int64_t kz, int64_t ky, int64_t kx,
                                         int64_t frag_z0, int64_t out_lo, int64_t out_hi, float* out,
                                         void* stream);
/* Host-buffer twins with the exact contract of the Cython functions: the
 * callee computes into `out` (caller-allocated, zero-initialised semantics
 * not required).  Synchronous. */
int bd3mg_depthvar_correlate_host_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx,
                                      const double* kernels, int64_t nzk, int64_t kz, int64_t ky, int64_t kx,
                                      int64_t frag_z0, int64_t out_lo, int64_t out_hi, double* out);
int bd3mg_depthvar_correlate_adjoint_host_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx,
                                              const double* kernels, int64_t nzk, int64_t kz, int64_t ky,
                                              int64_t kx, int64_t frag_z0, int64_t out_lo, int64_t out_hi,
                                              double* out);

/* ---- fused objective operators (device pointers, async) ---------------- */
/* Gradient rows [lo, hi] from a fragment: reference objective.py:159-187
 * (_grad_rows).  frag must cover [lo-1, hi+1] (clamped); rows of H are
 * read with zero padding outside it.  Also writes the half-quadratic
 * weights omega of rows [lo, hi] (objective.py:130-132). */
size_t bd3mg_grad_rows_ws_bytes(const bd3mg_geom_t* g, int64_t lo, int64_t hi);
int bd3mg_grad_rows(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                    const void* frag, int64_t frag_z0, int64_t nzf, int64_t lo, int64_t hi, void* g_out,
                    void* omega_out, void* ws, size_t ws_bytes, void* stream);

/* Full objective value and stop-rule norms: objective.py:140-156 (eval_f),
 * scheduler.py:218-219.  snap may be NULL.  terms_out: device, 7 doubles. */
size_t bd3mg_eval_f_ws_bytes(const bd3mg_geom_t* g);
int bd3mg_eval_f(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                 const void* x, const void* snap, double* terms_out, void* ws, size_t ws_bytes, void* stream);

/* Objective terms restricted to rows [lo, hi] (a rank's owned planes in the
 * multi-GPU layout): data term over H rows [lo, hi] of `frag` minus y_rows
 * (row lo of y), box / TV / axial terms of rows [lo, hi]; frag must cover
 * [lo, hi+1] and, for exact data terms, [lo-2rz, hi+2rz].  snap_rows (row lo
 * of the sweep snapshot) may be NULL.  Terms as bd3mg_eval_f (sums over the
 * rows; add across ranks for the global value). */
size_t bd3mg_eval_rows_ws_bytes(const bd3mg_geom_t* g, int64_t lo, int64_t hi);
int bd3mg_eval_rows(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y_rows,
                    const void* frag, int64_t frag_z0, int64_t nzf, int64_t lo, int64_t hi, const void* snap_rows,
                    double* terms_out, void* ws, size_t ws_bytes, void* stream);

/* Half-quadratic weights 1/sqrt(dx^2+dy^2+delta^2) of rows [lo, hi] of a
 * fragment: objective.py:130-132 (_omega), as cached by MajorantOperator
 * (objective.py:233-235).  omega_out: (hi-lo+1, ny, nx). */
int bd3mg_omega_rows(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* frag, int64_t frag_z0, int64_t nzf,
                     int64_t lo, int64_t hi, void* omega_out, void* stream);

/* A_S(x~) v for block [lo, hi]: objective.py:245-275 (MajorantOperator.apply),
 * omega = block rows of the anchor's weights. */
size_t bd3mg_majorant_apply_ws_bytes(const bd3mg_geom_t* g, int64_t lo, int64_t hi);
int bd3mg_majorant_apply(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* omega,
                         const void* v, int64_t lo, int64_t hi, void* out, void* ws, size_t ws_bytes,
                         void* stream);

/* Conjugate gradients for A_S(x~) w = b on block [lo, hi] (reference
 * directions.py:117-149, the inner solve of mm_direction :152-168), entirely
 * on the device: the recursion's scalars stay in device memory and the call
 * never waits on an iteration (it only keeps at most 3 iterations queued
 * ahead of the device).  x_out: x if converged, else the best iterate (as
 * the reference).  state_out (device, 16 doubles, may be NULL):
 * [0] |b|, [1] r.r, [2] best residual norm, [5] status (1 converged, 2
 * stopped: breakdown p.Ap <= 0 or budget; 0 only when maxit == 0),
 * [6] iterations, [7] relative residual of x_out. */
size_t bd3mg_cg_solve_ws_bytes(const bd3mg_geom_t* g, int64_t lo, int64_t hi);
int bd3mg_cg_solve(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* omega, const void* b,
                   int64_t lo, int64_t hi, double tol, int32_t maxit, void* x_out, double* state_out, void* ws,
                   size_t ws_bytes, void* stream);

/* Diagnostics of the persistent sweep: with BD3MG_PK_TRACE=1 set, every
 * persistent bd3mg_jacobi_sweep records per item 4 u64: dequeue, dependencies
 * met and completion times (ns, %globaltimer) and (sm << 48 | type << 40 |
 * block << 32 | z << 16 | aux).  Copies the last sweep's records (after a
 * device synchronise); *n_out = items of that sweep. */
int bd3mg_pk_trace(void* host, int64_t max_items, int64_t* n_out);
/* Persistent sweeps launched in this process (BD3MG_PK=1 selects them where
 * they apply; otherwise the multi-kernel sweep runs, with the same results). */
long long bd3mg_pk_launches(void);

/* `iters` power-iteration steps on H^T H over the full volume (reference
 * objective.py:358-366): v <- H^T H v / |H^T H v| in place; norms_out
 * (device, iters doubles) receives every |H^T H v|.  state_out (device, 2
 * doubles, may be NULL): [0] = 1 if a norm was 0 (the remaining steps were
 * skipped; the caller restarts from its RNG as the reference does). */
size_t bd3mg_power_hth_ws_bytes(const bd3mg_geom_t* g);
int bd3mg_power_hth(const bd3mg_geom_t* g, const void* kernels, void* v, int32_t iters, double* norms_out,
                    double* state_out, void* ws, size_t ws_bytes, void* stream);

/* Batched memory-gradient block steps (mg_direction + receive_update) with
 * the forward-only Gram.  `y` must satisfy: y + z*ny*nx is observation row z
 * for every row the tasks touch (a shard may pass its local rows shifted).  Tasks sharing one anchor fragment compute the
 * residual H x - y once over the union of their rows (block-Jacobi cycle of
 * run_bp3mg_barrier, runtime.py:244-292).  info_out: device, ntasks*16.
 * Tasks run in launches of 32; calls with in-place updates (x_rows) are
 * limited to 32 tasks (BD3MG_EINVAL otherwise) so that no launch moves the
 * anchor of the next -- pass inc_out and apply with bd3mg_apply_increment. */
size_t bd3mg_mg_steps_ws_bytes(const bd3mg_geom_t* g, const bd3mg_task_t* tasks, int ntasks);
int bd3mg_mg_steps(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                   const bd3mg_task_t* tasks, int ntasks, double* info_out, void* ws, size_t ws_bytes,
                   void* stream);

/* receive_update's block write (scheduler.py:151-153): x_rows += inc and,
 * when dmem_rows is not NULL, dmem_rows = inc; n elements of `dtype`. */
int bd3mg_apply_increment(int32_t dtype, void* x_rows, void* dmem_rows, const void* inc, int64_t n, void* stream);

/* One block-Jacobi sweep on a device-resident fragment (reference
 * run_bp3mg_barrier with every block of the fragment as a worker,
 * runtime.py:244-292, plus the per-sweep recorder of runtime.py:108-141).
 * Order: (1) recorder terms of the ANCHOR x over rows [rec_lo, rec_hi]
 * (data term taken from the step's own residual, box / TV / axial and the
 * stop norms against `snap`), (2) snap <- anchor rows, (3) every block's
 * fused step at the anchor, x and dmem updated in place.  With hd_cache
 * (variant "hd-cache", bd3mg_jacobi_cache_elems elements, zero-initialised)
 * the Gram reuses H E_S d_mem cached from the block's previous visit
 * (linearity of H) instead of recomputing it. */
typedef struct {
  void* x;              /* iterate fragment, plane 0 = depth frag_z0 */
  void* dmem;           /* memory-direction store, same layout as x */
  int64_t frag_z0, nzf;
  const int64_t* blocks; /* host: nblocks (z_lo, z_hi) pairs inside the fragment, <= 32 */
  int nblocks;
  int64_t rec_lo, rec_hi; /* recorder rows; rec_hi < rec_lo disables it */
  void* snap;           /* rows rec_lo..rec_hi of the sweep snapshot, or NULL */
  void* hd_cache;       /* NULL, or the hd-cache buffer */
} bd3mg_sweep_t;
size_t bd3mg_jacobi_sweep_ws_bytes(const bd3mg_geom_t* g, const bd3mg_sweep_t* sw);
int64_t bd3mg_jacobi_cache_elems(const bd3mg_geom_t* g, const bd3mg_sweep_t* sw);
int bd3mg_jacobi_sweep(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                       const bd3mg_sweep_t* sw, double* terms_out, double* info_out, void* ws, size_t ws_bytes,
                       void* stream);

/* Variant "hd-incremental" of the sweep (cached H d_mem +
 * incremental residual).  `resid` (device, nz*ny*nx elements of the dtype)
 * holds r = H x - y of the current anchor; the call keeps it current by
 * linearity, r += sum_b H E_b inc_b, from the hd-cache rows it updates, so no
 * residual correlation runs.  refresh != 0 recomputes r exactly (required on
 * the first call; periodic refreshes bound the rounding drift).  Needs
 * sw->hd_cache and blocks tiling the whole volume on this device; same
 * workspace as bd3mg_jacobi_sweep. */
int bd3mg_jacobi_sweep_incremental(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                                   const bd3mg_sweep_t* sw, void* resid, int refresh, double* terms_out,
                                   double* info_out, void* ws, size_t ws_bytes, void* stream);

/* The same variant for block steps (the deterministic cyclic schedule):
 * bd3mg_mg_steps with every task in place on one whole-volume anchor, hd[t]
 * the task's hd-cache rows (H E_S d_mem over rows [z_lo-rz, z_hi+rz] clamped,
 * zero-initialised), and `resid` the kept r = H x - y of the anchor (the
 * caller computes it exactly once, e.g. H x then minus y); each call updates
 * both by linearity.  bd3mg_eval_f_resid is bd3mg_eval_f with the data term
 * taken from `resid` (workspace: bd3mg_eval_f_ws_bytes). */
size_t bd3mg_mg_steps_incremental_ws_bytes(const bd3mg_geom_t* g, const bd3mg_task_t* tasks, int ntasks);
int bd3mg_mg_steps_incremental(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                               const bd3mg_task_t* tasks, int ntasks, void* const* hd, void* resid,
                               double* info_out, void* ws, size_t ws_bytes, void* stream);
int bd3mg_eval_f_resid(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* resid, const void* x,
                       const void* snap, double* terms_out, void* ws, size_t ws_bytes, void* stream);

/* Sharded sweep with the halo exchange fused into the in-place update: the
 * updated iterate rows [z_lo, z_hi] (global depths, each inside one of the
 * sweep's blocks) are ALSO stored to dst (plane z_lo first), typically a
 * peer GPU's halo inbox opened with bd3mg_peer_open -- the NVLink stores
 * replace the per-sweep ncclSend/Recv of the kz halo planes (
 * the reference's slab copy of make_task, scheduler.py:186-194).  Same
 * workspace as bd3mg_jacobi_sweep.  Ordering is the caller's: a peer may read
 * its inbox only after this call's stream work completed (the sharded driver
 * double-buffers the inboxes across the per-sweep all-reduce). */
typedef struct {
  int64_t z_lo, z_hi;
  void* dst;
} bd3mg_mirror_t;
int bd3mg_jacobi_sweep_mirrored(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                                const bd3mg_sweep_t* sw, const bd3mg_mirror_t* mirrors, int nmirrors,
                                double* terms_out, double* info_out, void* ws, size_t ws_bytes, void* stream);

/* bd3mg_mg_steps with the in-place update's rows also stored to mirrors (the
 * asynchronous mode's halo rings); one launch (<= 32 tasks). */
int bd3mg_mg_steps_mirrored(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                            const bd3mg_task_t* tasks, int ntasks, const bd3mg_mirror_t* mirrors, int nmirrors,
                            double* info_out, void* ws, size_t ws_bytes, void* stream);

/* Version flags of the asynchronous halo rings: host memory (e.g. a shared
 * mapping every rank's process maps) registered for device access, and a
 * stream-ordered publish that stores each value after a system-scope fence
 * (a reader that sees flag i sees the stream's earlier stores, ring data
 * included). */
#define BD3MG_MAX_FLAGS 16
typedef struct {
  int64_t* word;  /* device-visible address (bd3mg_host_register) */
  int64_t value;
} bd3mg_flag_t;
int bd3mg_host_register(void* host, size_t bytes, void** dev_out);
int bd3mg_host_unregister(void* host);
int bd3mg_publish(const bd3mg_flag_t* flags, int nflags, void* stream);

/* Peer memory for the halo inboxes: a zeroed device allocation plus its
 * 64-byte cudaIpc handle; bd3mg_peer_open maps another process's allocation
 * (NVLink peer access enabled lazily); close unmaps, free releases own. */
int bd3mg_peer_alloc(size_t bytes, void** dev_out, void* ipc_handle_out);
int bd3mg_peer_open(const void* ipc_handle, void** dev_out);
int bd3mg_peer_close(void* dev);
int bd3mg_peer_free(void* dev);

/* ---- host-buffer problem handle (worker-task boundary of the reference:
 * TaskMessage -> UpdateMessage, scheduler.py:36-57, runtime.py:92-105) ---- */
typedef struct bd3mg_problem bd3mg_problem;
/* kernels/y are host float64 arrays; dtype selects the device arithmetic.
 * Thread safety: calls on one handle are serialised by a per-handle mutex
 * (they share its stream and buffers).  Threads that must run concurrently
 * (the reference's live engine, runtime.py:188-241) use one handle each. */
int bd3mg_problem_create(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const double* kernels_host,
                         const double* y_host, int device, bd3mg_problem** out);
int bd3mg_problem_destroy(bd3mg_problem* p);
/* mg_direction(obj, x_slab, slab_z0, block, d_mem) with host float64 buffers:
 * x_slab (nzs, ny, nx), d_mem block rows or NULL, inc_out block rows,
 * info_out 16 doubles (may be NULL).  Returns BD3MG_ENONFINITE on a
 * non-finite gradient. */
int bd3mg_problem_mg_direction_host(bd3mg_problem* p, const double* x_slab, int64_t slab_z0, int64_t nzs,
                                    int64_t z_lo, int64_t z_hi, const double* d_mem, double* inc_out,
                                    double* info_out);

/* ---- measurement probe ------------------------------------------------- */
/* Dense FMA throughput probe (fp64 or fp32): `blocks` x 256 threads, 8
 * independent chains each, 128*iters FMAs per thread; *flops_out receives
 * the flop count of the launch.  out: blocks*256 elements of dtype.  Used by
 * bench.py to measure the FMA-pipe peak of the roofline. */
int bd3mg_fma_probe(int32_t dtype, int32_t blocks, int32_t iters, void* out, double* flops_out, void* stream);

/* One block-Jacobi sweep with HOST buffers (the sweep-level drop-in for the
 * reference's bp3mg barrier cycle, runtime.py:244-292): the fragment of x
 * (nzf planes from depth frag_z0; the whole volume or a rank's slab with
 * its halos) and the memory store dmem (same shape) are read from host
 * memory, the sweep of bd3mg_jacobi_sweep runs on the device (recorder over
 * the blocks' rows, no stop norms), and the updated x and dmem (= the
 * increments) are written back in place.  blocks: host (z_lo, z_hi) pairs,
 * <= 32.  terms_out (7) / info_out (nblocks*16) may be NULL.  Use pinned
 * host memory for full PCIe rate.  dmem == NULL selects session mode: the
 * memory store lives on the device inside the handle (zeroed on the first
 * call for a fragment), so only x crosses PCIe. */
int bd3mg_problem_jacobi_sweep_host(bd3mg_problem* p, double* x, double* dmem, int64_t frag_z0, int64_t nzf,
                                    const int64_t* blocks, int nblocks, double* terms_out, double* info_out);

/* ---- BD3MGVOL / BD3MGPSF payloads straight to / from device memory ----
 * The containers (reference volume.py:104-145 write_volume/read_volume,
 * blur.py:201-236 write_psf/read_psf) are a little-endian header and a
 * float64 payload; the host parses the header, these move the payload
 * through two alternating pinned 16 MiB chunks (file read overlapped with the
 * H2D copy).  dtype selects the device element type (fp32: narrowed on the
 * device after the float64 finiteness check). */
/* Read n float64 values at byte `offset` of `path` into dev_out.  Synchronous.
 * BD3MG_EFORMAT: "truncated payload ..." (file too short) or "non-finite
 * payload" (volume.py:142-143); BD3MG_EIO: open/read failure. */
int bd3mg_payload_read_device(const char* path, int64_t offset, int64_t n, void* dev_out, int32_t dtype,
                              void* stream);
/* Append n values of dev_in to `path` as float64 (the caller wrote the header).
 * Synchronous. */
int bd3mg_payload_write_device(const char* path, const void* dev_in, int64_t n, int32_t dtype, void* stream);
/* *bad_out = 1 if any of the n device values is NaN/Inf (check_volume,
 * volume.py:87-94).  Synchronous. */
int bd3mg_field_nonfinite(const void* dev, int64_t n, int32_t dtype, int32_t* bad_out, void* stream);

/* ---- separable-PSF fast path ----
 * For stacks whose every plane is rank one, K[zo] = u[zo] (x) v[zo] (x) w[zo]
 * (u: (nzk, kz) depth factors, v: (nzk, ky), w: (nzk, kx); ky == kx in
 * {3,5,7,9}): H rows (adjoint = 0) or H^T rows (adjoint = 1) with the
 * contract of bd3mg_depthvar_correlate[_adjoint] (_core.pyx:17-96), in
 * kz + ky + kx FMAs per voxel.  Results agree with the dense path to
 * rounding (different summation order); the dense kernels stay the default.
 * Memory-bound: report against HBM, not the FMA roofline. */
int bd3mg_sep_correlate_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx, const double* u,
                            const double* v, const double* w, int64_t nzk, int64_t kz, int64_t ky, int64_t kx,
                            int64_t frag_z0, int64_t out_lo, int64_t out_hi, double* out, int32_t adjoint,
                            void* stream);
int bd3mg_sep_correlate_f32(const float* frag, int64_t nzf, int64_t ny, int64_t nx, const float* u, const float* v,
                            const float* w, int64_t nzk, int64_t kz, int64_t ky, int64_t kx, int64_t frag_z0,
                            int64_t out_lo, int64_t out_hi, float* out, int32_t adjoint, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BD3MG_B200_H */
