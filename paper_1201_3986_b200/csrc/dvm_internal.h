// dvm_internal.h -- private declarations of libdvm (product code; never shared with oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/dvm.h"

namespace dvm {

constexpr int kMaxD = 3;

// Packed node index: the row-major linear index of a node, viewed as d fields
// of p = log2(N) bits (axis 0 most significant).  Adding two packed vectors
// component-wise modulo N is a carry-less SWAR add (swar_add); this is how the
// periodic wrap of PAPER.md:383-385 is applied to every stencil offset.
struct Packing {
    int d, p, N;
    uint32_t H;     // top bit of every field
    uint32_t mask;  // all fields
};

__host__ __device__ inline uint32_t swar_add(uint32_t a, uint32_t b, uint32_t H)
{
    return ((a & ~H) + (b & ~H)) ^ ((a ^ b) & H);
}

// Perp-basis change for the T2D_e table lookups of the 3D FFT gain kernels:
// u' = c[0] u + c[1] w, w' = c[2] u + c[3] w with c[0] c[3] − c[1] c[2] = 1,
// u'.z = 0 and w'.z = g = gcd(u.z, w.z) (extended Euclid; u.z = w.z = 0 keeps
// the basis, g = 0).  Lanes that step ξ_z then read one table row at columns
// q0 + g·lane: distinct banks for odd g; the column swizzle t2d_col below with
// mask (g odd ? 0 : 15) spreads even g.  Returns false if the result fails its
// own check.
inline bool perp_basis_zfree(const int *u, const int *w, int c[4], int up[3], int wp[3], int *g)
{
    const int uz = u[2], wz = w[2];
    c[0] = 1, c[1] = 0, c[2] = 0, c[3] = 1;
    *g = 0;
    if (uz != 0 || wz != 0) {
        long long r0 = uz, r1 = wz, s0 = 1, s1 = 0, t0 = 0, t1 = 1;  // s uz + t wz = r
        while (r1 != 0) {
            const long long q = r0 / r1;
            long long x = r0 - q * r1;
            r0 = r1, r1 = x;
            x = s0 - q * s1;
            s0 = s1, s1 = x;
            x = t0 - q * t1;
            t0 = t1, t1 = x;
        }
        if (r0 < 0) r0 = -r0, s0 = -s0, t0 = -t0;
        *g = (int)r0;
        c[0] = wz / *g, c[1] = -uz / *g, c[2] = (int)s0, c[3] = (int)t0;
    }
    for (int j = 0; j < 3; ++j) {
        up[j] = c[0] * u[j] + c[1] * w[j];
        wp[j] = c[2] * u[j] + c[3] * w[j];
    }
    return up[2] == 0 && wp[2] == *g && c[0] * c[3] - c[1] * c[2] == 1;
}
// column of T2D'(p, q) in its table row (see perp_basis_zfree)
__host__ __device__ __forceinline__ int t2d_col(int q, int m) { return q ^ ((q >> 4) & m); }

__host__ __device__ inline uint32_t pack_vec(const int *c, int d, int p, int N)
{
    uint32_t r = 0;
    for (int j = 0; j < d; ++j) {
        int m = c[j] % N;
        if (m < 0) m += N;
        r = (r << p) | (uint32_t)m;
    }
    return r;
}

// Device-resident direction table (struct of arrays, A directions, R rows).
struct DirTable {
    int *e = nullptr;        // [A*3] canonical primitive direction (unused comps 0)
    int *M = nullptr;        // [A] M_e = floor(Ñ/|e|_inf)
    double *a = nullptr;     // [A] a_e = h^{d+1} |e|_2
    int *u = nullptr;        // [A*3] row vector of the perp polygon (2D: e^⊥)
    int *w = nullptr;        // [A*3] second basis vector of e^⊥ ∩ Z^3 (2D: 0)
    int *z = nullptr;        // [A*3] transverse vector, z.e = 1: (u, w, z) is unimodular (3D)
    int *nrows = nullptr;    // [A]
    int *row_off = nullptr;  // [A+1] CSR offsets into rows
    int *cost = nullptr;     // [A] work estimate (LPT sharding)
    int *row_b = nullptr;    // [R]
    int *row_lo = nullptr;   // [R]
    int *row_hi = nullptr;   // [R]
    uint32_t *off_in = nullptr;     // [R] packed (hi_b+1) u + b w
    uint32_t *off_out = nullptr;    // [R] packed lo_b u + b w (also the row start)
    int *local = nullptr;           // [A_local] direction indices of this plan's shard
};

struct Workspace {
    double *S = nullptr;     // [slots][cells][nodes] line sums S_e
    double *part = nullptr;  // [slots][cells][nodes] per-direction contributions
    size_t slot_elems = 0;   // cells*nodes capacity per slot
    int slots = 0;
    double *f_stage = nullptr, *q_stage = nullptr;  // host e2e staging
    size_t stage_elems = 0;
    double *mom_partial = nullptr;  // [kMomBlocks][kMaxD+2]
    double *mom_dev = nullptr;      // [(steps+1)][kMaxD+2]
    size_t mom_rows = 0;
    double *qtmp = nullptr;         // time stepping scratch: Q (nodes)
    double *f1tmp = nullptr;        // time stepping scratch: RK2 first stage (nodes)
    int *mom_ctr = nullptr;         // time stepping: device row counter of the moments table
    double2 *fft_z = nullptr;       // 3D loss: complex FFT workspace [pairs][nodes]
    double2 *g3_f = nullptr;        // 3D gain: cell pairs of f, interleaved [pairs][nodes]
    double2 *g3_t = nullptr;        // 3D gain: per-group ring of T_e buffers [groups][slots][nodes]
    double2 *g3_q = nullptr;        // 3D gain: interleaved Q accumulators [chunks][pairs][nodes]
    unsigned int *g3_ctr = nullptr; // 3D gain: group barrier counters
    size_t fft_z_elems = 0, g3_f_elems = 0, g3_t_elems = 0, g3_q_elems = 0, g3_ctr_elems = 0;
    double *p2_scr = nullptr;       // 2D pair path: line windows of the first direction [units][cells][nodes]
    double *p2_part = nullptr;      // 2D pair path: partial gains [units][cells][nodes]
    size_t p2_scr_elems = 0, p2_part_elems = 0;
    double2 *sp_z = nullptr;        // spectral path: f̂ and the per-direction transform
    size_t sp_z_elems = 0;
    double2 *f32_z = nullptr;       // N = 32 spectral gain: one complex array per direction pair
    double *f32_part = nullptr;     // N = 32 spectral gain: per-chunk partial gains
    size_t f32_z_elems = 0, f32_part_elems = 0;
    double2 *fg_fhat = nullptr;     // FFT gain: f̂ of the cell pairs [pairs][nodes]
    size_t fg_fhat_elems = 0;
    double *lv_f = nullptr, *lv_q = nullptr;  // per-cell N̄: gathered cells of one level and their Q
    int64_t *lv_idx = nullptr;                // per-cell N̄: cells bucketed by level
    int *lv_cnt = nullptr;                    // per-cell N̄: bucket sizes (+ invalid count)
    size_t lv_f_elems = 0, lv_q_elems = 0, lv_idx_elems = 0, lv_cnt_elems = 0;
};

}  // namespace dvm

namespace dvm {
enum KernelClass { KC_LINESUM = 0, KC_ROWSUM, KC_REDUCE, KC_ZERO, KC_MOMENTS, KC_AXPY, KC_PLAN, KC_GAIN3D, KC_FFT, KC_FGAIN3D,
                   KC_SMALL2D, KC_WLINE2D, KC_PAIR2D, KC_FG32, KC_COUNT };
struct ProfRec {
    int cls;
    cudaEvent_t a, b;
};
}  // namespace dvm

namespace dvm {
// Plan tables of the 3D gain/loss path (dvm_gain3d.cu, dvm_frame.h).
struct GainTables {
    bool ready = false;
    int4 *rec = nullptr;      // [A_local][recw] frame metadata (6 int4) + sliding-program entries
    int recw = 0;
    double *aw = nullptr;     // [A_local] a_e
    double2 *tw = nullptr;    // FFT twiddles exp(-2πik/N), k < N/2
    double *lamhat = nullptr; // [N^d] spectrum of the loss kernel λ (real)
    void *units = nullptr;    // 2D: direction-pair units (dvm_pair2d.cu)
    std::vector<char> h_units2d;  // host copy of the units (kernel-parameter path of k_tile2d)
    int nunits = 0;
    int maxitems2d = 0;       // 2D: work items of the longest line walk
    double *shat = nullptr;   // spectral path: [A_local][N^d] line-filter spectra (real)
    double *that = nullptr;   // spectral path: [A_local][N^d] perp-filter spectra (real)
    int4 *fg_rec = nullptr;   // FFT gain: [A_local][3] (e, M), (u, 0), (w, 0)
    double *fg_aw = nullptr;  // FFT gain: [A_local] a_e / N^3
    double *fg_t2d = nullptr; // FFT gain: [A_local][N][N] plane-filter spectra T2D_e(p, q)
    int4 *f32_rec = nullptr;  // N = 32 spectral gain: [A_local] (u, M), [A_local] (w, 0) (see dvm_fg32.cu)
    uint32_t *f32_off = nullptr; // N = 32 spectral gain: [A_local][2 M_max] packed tap offsets ±m e
    double *f32_aw = nullptr; // N = 32 spectral gain: [A_local] a_e / N^3
    double *f32_t2d = nullptr; // N = 32 spectral gain: [A_local][N][N]
    int f32_mmax = 0;
    size_t bytes = 0;
};

// Caller weights of the decoupled kernel Γ̃_{k,l} = a(k) b(l) (eq:decoup,
// PAPER.md:575-579), evaluated by the spectral path only (dvm_set_weights).
struct WeightTables {
    bool on = false;
    double *a_box = nullptr;  // [(2Ñ+1)^d] a(k), index k + Ñ (row-major)
    double *b_box = nullptr;  // [(2Ñ+1)^d] b(l)
    double2 *tw = nullptr;    // FFT twiddles
    double *lamhat = nullptr; // [N^d] spectrum of the weighted loss kernel λ_w (real)
    double *shat = nullptr;   // [A_local][N^d] weighted line-filter spectra (lazy)
    double *that = nullptr;   // [A_local][N^d] weighted perp-filter spectra (lazy)
};
}  // namespace dvm

namespace dvm {
// Tuning and timing switches (dvm_set_tuning; never read from the environment).
// None changes Q beyond fp64 summation order except fg_dbg / g3_dbg, which
// skip work for timing experiments and are rejected unless set explicitly.
struct Tuning {
    int fg_dbg = 0;      // k_fg2 timing bits: 1 skip B work, 2 skip A work, 4 skip taps (results wrong)
    int max_groups = 0;  // cap on concurrent cell groups of the persistent 3D kernels (0: all that fit)
    int ring_slots = 0;  // c5 kernel ring depth per group (0: 2)
    int fg_chunks = 0;   // c5 kernel direction chunks per cell pair (0: automatic)
    int g3_cl = 0;       // frame-plane kernel CTAs per group at N = 32 (0: 8)
    int verbose = 0;     // launch geometry on stderr
};
}  // namespace dvm

struct dvm_plan_s {
    int d, N, p, Nbar, Ntilde, kernel, device;
    double L, h;
    cudaStream_t stream;
    int A = 0, R = 0;
    int shard_rank = 0, shard_world = 1;
    dvm::Packing pk;
    dvm::DirTable t;
    // host mirrors (small)
    std::vector<int> h_e, h_M, h_nrows, h_row_off, h_cost;
    std::vector<double> h_a;
    std::vector<int> local;      // direction indices evaluated by this plan, ascending
    std::vector<uint8_t> is_local;
    dvm::Workspace ws;
    dvm::GainTables g;
    dvm::WeightTables wt;
    uint64_t launches = 0;
    size_t table_bytes = 0;
    bool profiling = false;
    dvm::Tuning tune;
    int path_mode = 0;      // evaluation path: 0 auto, 1 v1 orbit sweeps, 2 gain3d/pair2d when built, 3 spectral, 4 FFT gain (3D N = 64)
    bool use_graphs = true; // time steppers replay one captured step (CUDA graph)
    cudaStream_t gstream = nullptr;      // plan-owned stream for graph capture/replay
    cudaStream_t cstream[2] = {nullptr, nullptr};  // host variant: host->device / device->host copy streams
    cudaEvent_t gev[2] = {nullptr, nullptr};
    std::vector<dvm::ProfRec> prof;
    // Repeated dvm_collide_batched calls with the same arguments on small batches
    // replay one captured CUDA graph (captured at the second identical call):
    // `version` changes with every plan setting, dvm::ws_epoch() with every
    // workspace reallocation; either invalidates the graph.
    uint64_t version = 0;
    uint64_t peer_key = 0;  // hash of the last dvm_collide_push window set (a new set bumps `version`)
    struct CollideGraph {
        cudaGraphExec_t exec = nullptr;
        const void *f = nullptr, *Q = nullptr;
        int64_t n = -1, stride = 0;
        uint64_t version = 0, epoch = 0, launches = 0;
        int kind = -1;  // 0 device buffers, 1 host buffers (copies captured too), 2 peer push
        int state = 0;  // 0 first call seen, 1 graph ready, 2 capture failed (no retry for this key)
    } cg;
};

namespace dvm {

// Launch bookkeeping: counts every launch; with profiling on, brackets it
// with CUDA events on the plan's stream.
struct LaunchScope {
    dvm_plan_s *P;
    ProfRec rec;
    bool on;
    LaunchScope(dvm_plan_s *p, int cls) : P(p), on(p->profiling)
    {
        ++P->launches;
        if (on) {
            rec.cls = cls;
            cudaEventCreate(&rec.a);
            cudaEventCreate(&rec.b);
            cudaEventRecord(rec.a, P->stream);
        }
    }
    ~LaunchScope()
    {
        if (on) {
            cudaEventRecord(rec.b, P->stream);
            P->prof.push_back(rec);
        }
    }
};
void clear_profile(dvm_plan_s *P);



// error reporting (thread-local message)
void set_error(const std::string &msg);
dvm_status_t cuda_fail(cudaError_t err, const char *what);

#define DVM_CUDA(call)                                                   \
    do {                                                                 \
        cudaError_t _e = (call);                                         \
        if (_e != cudaSuccess) return ::dvm::cuda_fail(_e, #call);       \
    } while (0)

// Grow-only device workspace buffer (stream-synchronised before a reallocation).
// process-wide workspace epoch: bumped by every workspace reallocation (any plan)
uint64_t ws_epoch();
void ws_epoch_bump();

template <typename T>
dvm_status_t grow(T **ptr, size_t *cap, size_t need, cudaStream_t s)
{
    if (*cap >= need) return DVM_OK;
    ws_epoch_bump();
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    // a regrowth takes at least 1.5x the old capacity (batches that creep up, e.g.
    // the level buckets of space-dependent N̄, reallocate O(log) times)
    if (*cap > 0 && need < *cap + *cap / 2) need = *cap + *cap / 2;
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    *cap = 0;
    if (cudaMalloc(ptr, sizeof(T) * need) != cudaSuccess) {
        *ptr = nullptr;
        cudaGetLastError();
        set_error("workspace allocation failed");
        return DVM_E_NOMEM;
    }
    *cap = need;
    return DVM_OK;
}

// plan construction (dvm_plan.cu)
dvm_status_t build_table(dvm_plan_s *P);
void free_table(dvm_plan_s *P);

// evaluation (dvm_collide.cu)
dvm_status_t collide_batched(dvm_plan_s *P, const double *f, double *Q, int64_t ncells, int64_t stride);
dvm_status_t moments(dvm_plan_s *P, const double *f, double *dev_out_row);
dvm_status_t axpy(dvm_plan_s *P, double *f, const double *q, double dt);
dvm_status_t moments_ctr(dvm_plan_s *P, const double *f, double *dev_base, int *dev_ctr);
dvm_status_t rk2_stage(dvm_plan_s *P, int stage, double *f, double *f1, const double *q, double dt);
// peer-memory shard reduction (dvm_peer.cu): argument checks of dvm_collide_push
// (sets *mine = slot `rank` of the local window) and the push launch
dvm_status_t peer_push_check(dvm_plan_s *P, const double *f, int64_t ncells, void *const *windows, int rank,
                             int world, unsigned int epoch, double **mine);
dvm_status_t peer_push_launch(dvm_plan_s *P, const double *mine, int64_t n, void *const *windows, int rank,
                              int world);
dvm_status_t collide_levels(dvm_plan_s *const *plans, int nlevels, const double *f, double *Q, int64_t ncells,
                            int64_t stride, const int *level);
dvm_status_t copy_cells(dvm_plan_s *P, const double *src, const int64_t *si, double *dst, const int64_t *di,
                        int64_t ncells);
dvm_status_t zero_cells(dvm_plan_s *P, double *Q, int64_t q_stride, int64_t ncells, int64_t nodes);
dvm_status_t reduce_slots(dvm_plan_s *P, double *Q, int64_t q_stride, const double *part, int64_t slot_elems,
                          int nslots, int64_t ncells, int64_t nodes);
// 3D gain (dvm_gain3d.cu), loss as one FFT convolution (dvm_loss.cu)
dvm_status_t build_loss(dvm_plan_s *P);
dvm_status_t set_weights(dvm_plan_s *P, const double *a_box, const double *b_box);
void free_weights(dvm_plan_s *P);
dvm_status_t fft_forward_pairs(dvm_plan_s *P, const double *f, int64_t f_stride, int64_t ncells, double2 *out);
dvm_status_t ifft_batch(dvm_plan_s *P, double2 *z, int64_t narrays);
dvm_status_t loss_init(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride, int64_t ncells,
                       double2 *QI);
dvm_status_t collide_spectral(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                              int64_t ncells);
dvm_status_t build_gain3d(dvm_plan_s *P);
dvm_status_t build_pair2d(dvm_plan_s *P);
dvm_status_t collide_small2d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                             int64_t ncells, bool *handled);
// one explicit Euler step of one small 2D cell with the unit sum, f += dt Q and
// the moments partials fused (handled = false: use the general path)
dvm_status_t euler_small2d(dvm_plan_s *P, double *f, double *Q, double dt, double *mpart, int *nblocks,
                           bool *handled);
dvm_status_t moments_final_ctr(dvm_plan_s *P, int nblocks, double *dev_base, int *dev_ctr);
dvm_status_t collide_pair2d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                            int64_t ncells, bool *handled);
void free_gain3d(dvm_plan_s *P);
dvm_status_t interleave_pairs(dvm_plan_s *P, const double *f, int64_t f_stride, int64_t ncells, int64_t nodes,
                              double2 *fI);
dvm_status_t deinterleave_pairs(dvm_plan_s *P, const double2 *QI, int nchunks, int64_t npairs, int64_t ncells,
                                int64_t nodes, double *Q, int64_t q_stride);
// 3D gain by per-direction FFT filtering (dvm_fgain3d.cu)
dvm_status_t collide_fgain3d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                             int64_t ncells, bool *handled);
dvm_status_t collide_gain3d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                            int64_t ncells, bool *handled);
// 3D N = 32 gain by batched direction-pair spectral filtering (dvm_fg32.cu)
dvm_status_t collide_fg32(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                          int64_t ncells, bool *handled);
void free_workspace(dvm_plan_s *P);

}  // namespace dvm
