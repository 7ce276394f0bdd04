/*
 * dvm.h -- C ABI of libdvm: B200-native (sm_100a, fp64) evaluation of the fast
 * periodized discrete-velocity Boltzmann collision operator D^{Ñ,N̄}(f,f) of
 * Mouhot, Pareschi & Rey, arXiv 1201.3986.
 *
 * Operation (identical, up to fp64 rounding order, to oracle/dvm_oracle.c):
 *
 *   Q_i = sum_{e in A^{d-1}_{N̄}} a_e [ S_e(i) T_e(i) - f_i U_e(i) ]        eq:decD
 *   S_e(i) = sum_{1<=|m|<=M_e} f_{i+me}              (k-line factor alpha_p)
 *   T_e(i) = sum_{l in e^⊥, |l|_inf<=Ñ} f_{i+l}       (perp factor alpha'_p)
 *   U_e(i) = sum_{l in e^⊥, |l|_inf<=Ñ} S_e(i+l)
 *   a_e = h^{d+1}|e|_2  (= a(me) for every m, a(k) = h^{d+1}|k|/gcd(k))
 *   M_e = floor(Ñ / |e|_inf),  h = 2L/N,  indices periodic mod N
 *
 * A^{d-1}_{N̄} is the set of canonical primitive directions e (gcd 1, first
 * nonzero component > 0) with |e|_inf <= N̄ -- the "primal representants" of
 * lines of order N̄.  The sum equals the
 * direct pair sum of eq:DR restricted to k on those lines; with N̄ = Ñ it is
 * eq:DR exactly.
 *
 * Grid and layout: N points per axis (reading R1), node j <-> v = (j - N/2) h,
 * N a power of two.  Fields are fp64, row-major [cells][N]...[N] (d axes, last
 * axis fastest); a cell is N^d contiguous doubles (cell_stride elements apart).
 *
 * Conventions for every entry point:
 *   - Ownership: the plan owns its device direction table and workspace;
 *     dvm_plan_destroy frees them.  f and Q are caller-owned DEVICE pointers
 *     (except the *_host variants), 8-byte aligned (16 B recommended).
 *   - Streams: calls are asynchronous and stream-ordered on the plan's stream
 *     (params.stream, a cudaStream_t passed as void*; NULL = legacy default
 *     stream); the *_host variants synchronise before returning.
 *   - Errors: status codes only -- no exceptions cross the ABI, nothing aborts.
 *     Asynchronous device faults surface as DVM_E_CUDA at the next call that
 *     synchronises (or dvm_sync).  dvm_last_error() returns a human-readable
 *     message for the last failure on the calling thread.
 *   - Threading: one host thread per plan at a time; distinct plans are
 *     independent.
 *   - Determinism: for a fixed plan, input (batch) and device the result is
 *     bitwise reproducible (no floating-point atomics on the accumulation path).
 */
#ifndef DVM_H
#define DVM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DVM_ABI_VERSION 1

#if defined(__GNUC__)
#define DVM_API __attribute__((visibility("default")))
#else
#define DVM_API
#endif

typedef struct dvm_plan_s *dvm_plan_t;

/* Collision kernels with decoupled Heintz-Panferov weights a(k) b(l), b = 1
 * (PAPER.md:579-587): 2D Maxwell molecules a = h^3|k|/gcd(k1,k2); 3D hard
 * spheres a = h^5|k|/gcd(k1,k2,k3). */
typedef enum { DVM_MAXWELL_2D = 0, DVM_HARD_SPHERES_3D = 1 } dvm_kernel_t;

typedef enum {
    DVM_OK = 0,
    DVM_E_NULL = 1,        /* a required pointer argument is NULL */
    DVM_E_DIM = 2,         /* d not in {2,3} */
    DVM_E_KERNEL = 3,      /* kernel does not match d (Maxwell<->2D, hard spheres<->3D) */
    DVM_E_ORDER = 4,       /* not 1 <= N̄ <= Ñ, or 2Ñ+1 > N */
    DVM_E_UNSUPPORTED = 5, /* N not a power of two in [4, 1024] (2D) / [4, 256] (3D); bad L */
    DVM_E_SHAPE = 6,       /* ncells < 0, cell_stride < N^d, size overflow, bad shard */
    DVM_E_ALIAS = 7,       /* Q overlaps f */
    DVM_E_NOMEM = 8,       /* device or host allocation failed */
    DVM_E_CUDA = 9,        /* CUDA runtime error (incl. asynchronous faults) */
    DVM_E_STATE = 10       /* call not valid for this plan (e.g. wrong d for dvm_euler moments) */
} dvm_status_t;

typedef struct {
    int d;               /* velocity dimension, 2 or 3 */
    int N;               /* points per axis (power of two) */
    int Nbar;            /* direction order N̄ >= 1 */
    int Ntilde;          /* kernel truncation Ñ; 0 -> max(floor(N/(3+sqrt 2)), N̄) (reading R2) */
    double L;            /* box half-width, h = 2L/N; 0 -> 8.0 (reading R3) */
    dvm_kernel_t kernel; /* must match d */
    int device;          /* CUDA device ordinal; -1 -> current device */
    void *stream;        /* cudaStream_t for all launches; NULL -> default stream */
    int shard_rank;      /* direction sharding: this plan evaluates only its LPT share */
    int shard_world;     /*   of the directions (partial Q); 1 -> all directions */
} dvm_plan_params_t;

typedef struct {
    int d, N, Nbar, Ntilde, kernel;
    int A;               /* number of directions in A^{d-1}_{N̄} */
    int A_local;         /* directions evaluated by this plan (== A unless sharded) */
    int rows_total;      /* sum over directions of the perp-polygon rows (3D), A (2D) */
    int64_t nodes;       /* N^d */
    double L, h;
    size_t workspace_bytes; /* device bytes currently held by the plan */
    uint64_t launches;   /* device kernel launches issued by this plan so far */
} dvm_plan_info_t;

/* Build a plan with Ñ from the rule, L = 8, current device, default stream,
 * no sharding.  Builds the direction table on the device (K1) and its
 * per-direction metadata (K2), synchronously.  *out is set only on DVM_OK. */
DVM_API dvm_status_t dvm_plan(int d, int N, int Nbar, dvm_kernel_t kernel, dvm_plan_t *out);

/* Same with every parameter explicit (see dvm_plan_params_t). */
DVM_API dvm_status_t dvm_plan_ex(const dvm_plan_params_t *params, dvm_plan_t *out);

DVM_API dvm_status_t dvm_plan_info(dvm_plan_t plan, dvm_plan_info_t *info);

/* Copy the plan's direction table to host arrays (each may be NULL):
 * dirs[A*d] (canonical e, lexicographic), M[A] (M_e), a[A] (a_e), local[A]
 * (1 if the direction belongs to this plan's shard). Synchronous. */
DVM_API dvm_status_t dvm_plan_directions(dvm_plan_t plan, int *dirs, int *M, double *a, int *local);

/* Geometry of direction idx (0 <= idx < A), for inspection and tests: the
 * row vector u and second basis vector w of e^⊥ ∩ Z^d (3D; 2D: u = e^⊥,
 * w = 0) and the rows {α u + β w : lo <= α <= hi} of P_e.
 * u, w receive d ints; b, lo, hi receive up to cap rows; *nrows the count.
 * Synchronous. */
DVM_API dvm_status_t dvm_plan_geometry(dvm_plan_t plan, int idx, int *u, int *w, int *nrows, int *b, int *lo,
                               int *hi, int cap);

/* Change the stream used by subsequent calls (cudaStream_t as void*). */
DVM_API dvm_status_t dvm_set_stream(dvm_plan_t plan, void *stream);

/* Q = D^{Ñ,N̄}(f,f) for one cell (eq:decD: the gain
 * a_e S_e T_e and loss a_e f U_e summed over the lines e of order <= N̄,
 * PAPER.md:796-827; equal to the direct pair sum of eq:DR, PAPER.md:386-390,
 * restricted to those lines).  f, Q: caller-owned DEVICE arrays of N^d doubles
 * (layout above), Q must not overlap f.  For a sharded plan Q is the partial
 * sum over this shard's directions; the caller sums the
 * shards.  Asynchronous on the plan's stream.  Errors: DVM_E_NULL (plan, f or
 * Q NULL), DVM_E_ALIAS (overlap), DVM_E_NOMEM (workspace), DVM_E_CUDA. */
DVM_API dvm_status_t dvm_collide(dvm_plan_t plan, const double *f, double *Q);

/* The same operator for ncells independent spatial cells (the
 * space-inhomogeneous setting: the collision step is local
 * in space, one evaluation per cell); cell c occupies [c*cell_stride,
 * c*cell_stride + N^d) of f and of Q (cell_stride 0 -> N^d; f and Q DEVICE,
 * caller-owned, non-overlapping).  ncells = 0 is a no-op.  Errors as
 * dvm_collide plus DVM_E_SHAPE (ncells < 0, cell_stride < N^d, overflow).
 * The plan grows a device workspace on first use of a batch size (3D: ~3 × 16 B
 * per node per cell pair plus a 256 MiB FFT batch; 2D: <= 512 MiB of per-pair
 * partials); DVM_E_NOMEM if it cannot.  Small batches (ncells N^d <= 2^22)
 * are host-launch bound: the second call with the same (f, Q, ncells,
 * cell_stride) is captured as one CUDA graph on a plan-owned stream and every
 * later identical call replays it on the plan's stream (the same kernels, so
 * the same bits; f is read at replay time; not for the persistent 3D N = 64
 * and batched N = 32 kernels, whose CTA groups need a cooperative launch).
 * Any dvm_set_* call on the plan and
 * any workspace reallocation invalidate the graph; dvm_set_graphs(plan, 0)
 * turns capture off. */
DVM_API dvm_status_t dvm_collide_batched(dvm_plan_t plan, const double *f, double *Q, int64_t ncells,
                                 int64_t cell_stride);

/* Space-dependent N̄ ("the parameter N̄ can be made space
 * dependent ... some regions in space deserve less accuracy than others, being
 * close to equilibrium"): cell c of the batch is evaluated with
 * plans[level[c]], i.e. Q_c = D^{Ñ,N̄_l}(f_c, f_c) with N̄_l the order of that
 * plan (eq:decD, with the direction truncation of order N̄_l).
 *   plans:  nlevels (1..64) plans that differ only in N̄ (same d, N, Ñ, L,
 *           kernel, device, stream and shard; DVM_E_STATE otherwise).
 *   f, Q:   DEVICE arrays as in dvm_collide_batched (cell_stride 0 -> N^d).
 *   level:  DEVICE array of ncells int32, level[c] in [0, nlevels).
 * The cells are bucketed by level on the device (stable, ascending cell index
 * within a bucket), each bucket is gathered into the workspace of plans[0],
 * evaluated as one batch with its plan and scattered back; a bucket holding
 * the whole batch is evaluated in place.  Synchronises once (the bucket sizes
 * are read back to size the launches).  Each cell's Q equals a batched
 * evaluation of that cell with its plan to rounding (the 3D FFT paths pair
 * cells within a bucket).  Errors: DVM_E_NULL, DVM_E_SHAPE (bad nlevels,
 * ncells, stride, or a level out of range: Q unspecified), DVM_E_ALIAS,
 * DVM_E_STATE, DVM_E_NOMEM, DVM_E_CUDA. */
DVM_API dvm_status_t dvm_collide_batched_levels(const dvm_plan_t *plans, int nlevels, const double *f, double *Q,
                                                int64_t ncells, int64_t cell_stride, const int *level);

/* End-to-end variant with HOST buffers: copies f to the device, evaluates and
 * copies Q back; synchronous.  Batches of >= 256 cells are pipelined in 4
 * chunks of whole cell pairs (host->device copies on one plan-owned copy
 * stream, device->host on another, evaluation on the plan's stream), so with
 * pinned host memory the copies overlap the evaluation.  The plan holds a
 * device staging copy of f and Q (2 × ncells × N^d doubles). */
DVM_API dvm_status_t dvm_collide_batched_host(dvm_plan_t plan, const double *f_host, double *Q_host,
                                      int64_t ncells, int64_t cell_stride);

/* ---- Direction-shard reduction over peer memory (one GPU per rank) ----------
 * Q is a sum over the directions (eq:decD; "completely
 * parallelizable"): rank r of a direction-sharded set of
 * plans (dvm_plan_ex shard_rank = r, shard_world = W) evaluates the partial
 * Q_r of its LPT share, and Q = Σ_r Q_r.  Instead of a separate all-reduce,
 * the evaluation pushes Q_r straight into every rank's PEER WINDOW over
 * NVLink (P2P stores), and each rank then adds the W slots of its own window
 * in rank order (one-shot reduction, identical bits on every rank).
 *
 * A peer window (one per rank, same ncells everywhere) is a device buffer of
 * dvm_peer_window_bytes(plan, ncells, W) bytes: W slots of ncells × N^d
 * doubles (slot r holds rank r's partial) followed by W uint32 arrival
 * counters.  dvm_peer_window_alloc allocates it (cudaMalloc on the plan's
 * device, counters zeroed; free with dvm_peer_window_free).  Other ranks map
 * it through CUDA IPC: dvm_ipc_handle writes the 64-byte handle of a device
 * allocation, dvm_ipc_open maps a peer's handle into this process (peer access
 * enabled lazily), dvm_ipc_close unmaps it.
 *
 * dvm_collide_push(plan, f, ncells, windows, rank, world, epoch)
 *   f:       DEVICE, ncells cells of N^d doubles (contiguous), the same f on
 *            every rank.
 *   windows: HOST array of `world` DEVICE pointers, windows[r] = rank r's
 *            window as mapped in this process (windows[rank] = the local one).
 *   rank, world: must equal the plan's shard_rank / shard_world.
 *   epoch:   1 for the first push into these windows, +1 per later call.
 *   Evaluates Q_rank into slot `rank` of the local window, copies it into slot
 *   `rank` of every other window, then (after a system-scope fence) adds the
 *   arrival of every push CTA to counter `rank` of every window.  Never waits
 *   for other ranks; stream-ordered on the plan's stream.  A repeated call with
 *   the same f and windows on a small batch replays the evaluation and the
 *   push as one CUDA graph (as dvm_collide_batched does).
 * dvm_peer_reduce(plan, window, Q, ncells, world, epoch)
 *   Waits on the device until every counter of the LOCAL window shows the
 *   pushes of `epoch`, then Q = Σ_{r=0}^{world-1} slot r (in r order).  Every
 *   rank must have called dvm_collide_push for this epoch (on its own GPU),
 *   or this call never completes.
 * Errors: DVM_E_NULL, DVM_E_SHAPE (ncells, world), DVM_E_STATE (rank/world
 * differ from the plan's shard, epoch 0), DVM_E_NOMEM, DVM_E_CUDA. */
DVM_API size_t dvm_peer_window_bytes(dvm_plan_t plan, int64_t ncells, int world);
DVM_API dvm_status_t dvm_peer_window_alloc(dvm_plan_t plan, int64_t ncells, int world, void **out);
DVM_API dvm_status_t dvm_peer_window_free(void *window);
DVM_API dvm_status_t dvm_ipc_handle(const void *dptr, unsigned char handle[64]);
DVM_API dvm_status_t dvm_ipc_open(const unsigned char handle[64], void **out);
DVM_API dvm_status_t dvm_ipc_close(void *dptr);
DVM_API dvm_status_t dvm_collide_push(dvm_plan_t plan, const double *f, int64_t ncells, void *const *windows,
                                      int rank, int world, unsigned int epoch);
DVM_API dvm_status_t dvm_peer_reduce(dvm_plan_t plan, const void *window, double *Q, int64_t ncells, int world,
                                     unsigned int epoch);

/* Moments of one cell (device f): out_host[0] = h^d sum f, out_host[1..d] =
 * h^d sum v f, out_host[d+1] = h^d sum |v|^2 f (reading R16).  Synchronous,
 * deterministic. */
DVM_API dvm_status_t dvm_moments(dvm_plan_t plan, const double *f, double *out_host);

/* dst cell dst_idx[c] = src cell src_idx[c] for c < ncells (cells of N^d
 * doubles, device arrays; device int64 index arrays, NULL = identity; no range
 * checks on the indices).  Stream-ordered, asynchronous.  Used to bucket the
 * cells of a batch by N̄ (space-dependent N̄). */
DVM_API dvm_status_t dvm_copy_cells(dvm_plan_t plan, const double *src, const int64_t *src_idx, double *dst,
                                    const int64_t *dst_idx, int64_t ncells);

/* Explicit Euler f <- f + dt D(f,f), nsteps times, in place on the device
 * array f (one cell).  If moments_host != NULL it receives (nsteps+1) rows of
 * d+2 moments (before the first step and after every step).  Synchronous. */
DVM_API dvm_status_t dvm_euler(dvm_plan_t plan, double *f, double dt, int nsteps, double *moments_host);

/* Second-order TVD Runge-Kutta (Heun) f1 = f + dt D(f,f), f <- (f + f1 +
 * dt D(f1,f1)) / 2, the time discretisation of PAPER.md:946-947; otherwise as
 * dvm_euler.  Both steppers run step 1 directly and replay steps 2..nsteps as
 * one captured CUDA graph on a plan-owned stream (ordered after and before the
 * plan's stream); results are identical to direct launches. */
DVM_API dvm_status_t dvm_rk2(dvm_plan_t plan, double *f, double dt, int nsteps, double *moments_host);

/* Enable (default) or disable the CUDA-graph replay of the time steppers and of
 * repeated small dvm_collide_batched calls. */
DVM_API dvm_status_t dvm_set_graphs(dvm_plan_t plan, int enable);

/* Per-kernel timing with CUDA events recorded on the plan's stream around
 * every launch (for bench.py's roofline; adds one event pair per launch).
 * enable != 0 clears previous records and starts recording; 0 stops. */
DVM_API dvm_status_t dvm_profile_enable(dvm_plan_t plan, int enable);

/* Synchronises the plan's stream, then writes, for kernel class k < n, the
 * summed device time in ms and the launch count of the recorded launches.
 * Class names: dvm_profile_name(k) (NULL past the last class). */
DVM_API dvm_status_t dvm_profile_read(dvm_plan_t plan, double *ms, uint64_t *count, int n);
DVM_API const char *dvm_profile_name(int k);

/* Evaluation path: 0 = auto (default), 1 = v1 orbit sweeps only, 2 = the
 * FFT-loss paths whenever the plan built them, 4 = 3D N = 64: the gain by
 * per-direction FFT filtering (T_e of two cells from one inverse transform of
 * f̂ t̂_e, S_e as line taps; auto for 3D N = 64; like 2, used whenever the
 * plan supports it: the 3D kernels hold 2 M_e <= 32 taps, so plans with
 * Ñ > 16 evaluate by the v1 sweeps), 5 = 2D with N <= 64 (auto there): one
 * CTA per direction pair {e, e⊥} and cell holds f in shared memory and
 * evaluates gain and loss of the pair with direct line windows (the loss as
 * f [a (Box − W_e⊥) + a (Box − W_e)], Box the 2D window), partials summed in
 * pair order (two launches, no FFT), 6 = 3D N = 32: two directions of one
 * cell per complex transform, T_a + i T_b = IFFT(f̂ (t̂_a + i t̂_b)), all
 * direction pairs in one batch plus the loss array f̂ λ̂ (auto for batches of
 * <= 2 cells at N = 32), 7 = 2D tiles: one CTA per 16 x 32 node tile with a
 * halo of Ñ in shared memory evaluates every pair unit's windows per node,
 * Q = −fΛ + G (auto for 2D batches with >= 96 tiles when the tile fits shared
 * memory, e.g. c3), 3 = the spectral reference
 * path (per direction one inverse transform gives
 * S_e + i T_e from the real filter spectra; a second cross-check, slow:
 * A inverse FFTs per cell; its tables need 16 A N^d bytes, <= 4 GB).  The FFT-loss paths evaluate
 * the loss as one FFT convolution f (λ ⊛ f) (reading R21): 3D with N in
 * {32, 64}: gain by the frame-plane kernel (two cells per node,
 * warp-specialised, TMEM accumulators); 2D with 16 <= N <= 256: gain by
 * direction pairs {e, e⊥}.  Auto picks them for 3D, for 2D N >= 256 and for
 * N = 128 with >= 100 directions, path 5
 * for 2D 16 <= N <= 64, v1 otherwise.  All paths compute the same
 * operator; results agree to rounding (the FFT loss pairs cells in one complex
 * transform, so a cell's last bits may depend on its batch partner; a repeated
 * identical call is bitwise reproducible). */
DVM_API dvm_status_t dvm_set_path(dvm_plan_t plan, int path);

/* General decoupled collision weights (eq:decoup):
 * Γ̃_{k,l} = B̃(|k|,|l|) w_{k,l} = a(k) b(l) on the same truncated pair set
 * (k on the lines of order <= N̄, l ∈ e^⊥ ∩ [-Ñ,Ñ]^d), replacing the built-in
 * a(k) = h^{d+1}|k|/gcd(k), b = 1 of PAPER.md:582-587.
 *   a_box, b_box: HOST arrays of (2Ñ+1)^d doubles, row-major over
 *     [-Ñ,Ñ]^d with index k + Ñ per axis (last axis fastest); copied, the
 *     caller keeps ownership.  NULL for one table keeps its built-in values;
 *     both NULL restores the built-in operator (and the fast paths).
 *   Requirements: finite and even (a(-k) = a(k), b(-l) = b(l): then both
 *     filter spectra and the loss-kernel spectrum are real); a(0) is unused.
 *   Evaluation: the spectral path (dvm_set_path 0 or 3; 1 and 2 then return
 *     DVM_E_STATE at collide time), N in [16, 256], filter tables
 *     16 A_local N^d bytes <= 4 GB, built on the first collide.
 *   Errors: DVM_E_NULL (plan), DVM_E_UNSUPPORTED (odd / non-finite weights,
 *     N out of range; the plan keeps the built-in weights), DVM_E_NOMEM. */
DVM_API dvm_status_t dvm_set_weights(dvm_plan_t plan, const double *a_box, const double *b_box);

/* Tuning and timing switches of a plan (never read from the environment):
 *   "max_groups" cap on concurrent cell groups of the persistent 3D kernels
 *                (0 = every group that fits, the default)
 *   "ring_slots" 3D N = 64 kernel: T_e ring slots per cell group, 2 (default) to 4
 *   "fg_chunks"  3D N = 64 kernel: direction chunks per cell pair, 1 to 64
 *                (0 = automatic, the default)
 *   "g3_cl"      frame-plane kernel CTAs per cell group at N = 32: 4, 8
 *                (default) or 16
 *   "verbose"    1 = print launch geometry on stderr
 *   "timing_dbg" skip work inside the 3D N = 64 kernel for phase timing (bits:
 *                1 phase B, 2 phase A, 4 line taps).  Q IS WRONG while nonzero;
 *                for profiling experiments only.
 * None of the others changes Q beyond fp64 summation order.  Errors:
 * DVM_E_NULL, DVM_E_STATE (unknown key or out-of-range value; the plan is
 * unchanged). */
DVM_API dvm_status_t dvm_set_tuning(dvm_plan_t plan, const char *key, int value);

/* Wait for all work issued on the plan's stream; reports asynchronous faults. */
DVM_API dvm_status_t dvm_sync(dvm_plan_t plan);

DVM_API dvm_status_t dvm_plan_destroy(dvm_plan_t plan);

DVM_API const char *dvm_status_str(dvm_status_t status);
DVM_API const char *dvm_last_error(void);
DVM_API int dvm_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DVM_H */
