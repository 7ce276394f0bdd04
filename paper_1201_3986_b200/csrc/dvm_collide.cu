// dvm_collide.cu -- evaluation of Q = D^{Ñ,N̄}(f,f) (eq:decD).
//
// Per direction e the operator is (dvm.h):
//   q_e(i) = a_e [ S_e(i) T_e(i) - f_i U_e(i) ]
//   S_e = sum_{1<=|m|<=M_e} f(.+me)    (alpha_p factor)
//   T_e = sum_{l in P_e} f(.+l)        (alpha'_p factor)
//   U_e = sum_{l in P_e} S_e(.+l)      (= sum_{m != 0} T_e(.+me): loss of eq:decD)
// and Q = sum_e q_e, accumulated in direction order (deterministic, no atomics).
//
// Kernels (v1, "orbit sweeps"):
//   k_linesum  thread per (cell, e-orbit segment): sliding window along the
//              periodic lattice line {x + t e} -> S_e          (2 loads / node)
//   k_rowsum   thread per (cell, u-orbit segment): sliding window of the perp
//              polygon along its row vector u; each step adds the entering and
//              subtracts the leaving node of every row -> T_e, U_e and q_e
//              (4 loads per row per node)
//   k_reduce   ordered sum of per-direction partials into Q (chunked mode)
// For N = 2^p every primitive lattice vector has orbits of length exactly N,
// and {x : x_j = 0} (v_j odd) is a transversal (one start per orbit).  Warp
// lanes walk adjacent orbits so that every load is 32 consecutive doubles of
// the fastest axis whenever the orbit vector has an odd non-fastest component.
#include <algorithm>

#include <vector>

#include "dvm_internal.h"

namespace dvm {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxRowsSmem = 512;
constexpr int kMomBlocks = 128;

struct Geo {
    int d, p, N;
    uint32_t H;
    int64_t nodes;
};

__device__ inline void unpack(uint32_t x, const Geo &g, int *c)
{
    for (int j = g.d - 1; j >= 0; --j) {
        c[j] = (int)(x & (uint32_t)(g.N - 1));
        x >>= g.p;
    }
}

// transversal axis of vector v: first non-fastest odd component, else the fastest.
__device__ inline int transversal_axis(const int *v, int d)
{
    for (int j = 0; j < d - 1; ++j)
        if (v[j] & 1) return j;
    return d - 1;
}

// Start node of segment `seg` (length seg_len) of orbit r of vector v.
__device__ inline uint32_t orbit_start(uint32_t r, int seg, int seg_len, const int *v, const Geo &g)
{
    int j = transversal_axis(v, g.d);
    int shift = g.p * (g.d - 1 - j);
    uint32_t low = r & ((1u << shift) - 1u);
    uint32_t high = r >> shift;
    uint32_t s = (high << (shift + g.p)) | low;  // insert x_j = 0
    int c[kMaxD];
    unpack(s, g, c);
    long long t = (long long)seg * seg_len;
    for (int k = 0; k < g.d; ++k) c[k] = (int)(((long long)c[k] + t * v[k]) % g.N + g.N) % g.N;
    return pack_vec(c, g.d, g.p, g.N);
}

__device__ inline uint32_t pack_scaled(const int *v, int m, const Geo &g)
{
    int c[kMaxD];
    for (int k = 0; k < g.d; ++k) c[k] = m * v[k];
    return pack_vec(c, g.d, g.p, g.N);
}

// S_e for the directions dir_list[blockIdx.z] of every cell.
__global__ void __launch_bounds__(kThreads) k_linesum(const double *__restrict__ f, int64_t f_stride,
                                                      double *__restrict__ S, int64_t slot_elems,
                                                      int64_t ncells, Geo g, const int *__restrict__ dir_list,
                                                      const int *__restrict__ E, const int *__restrict__ Mtab,
                                                      int seg_len, int nseg)
{
    const int slot = blockIdx.z;
    const int dir = dir_list[slot];
    const int e[3] = {E[3 * dir], E[3 * dir + 1], E[3 * dir + 2]};
    const int M = Mtab[dir];
    const int64_t norbits = g.nodes / g.N;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= norbits * nseg) return;
    const uint32_t r = (uint32_t)(tid % norbits);
    const int seg = (int)(tid / norbits);
    const uint32_t Ev = pack_scaled(e, 1, g);
    const uint32_t Pin = pack_scaled(e, M + 1, g);
    const uint32_t Pout = pack_scaled(e, -M, g);
    const uint32_t H = g.H;
    const uint32_t x0 = orbit_start(r, seg, seg_len, e, g);
    for (int64_t cell = blockIdx.y; cell < ncells; cell += gridDim.y) {
        const double *fc = f + cell * f_stride;
        double *Sc = S + (int64_t)slot * slot_elems + cell * g.nodes;
        uint32_t x = x0;
        uint32_t y = swar_add(x, Pout, H);
        double W = 0.0;
        for (int m = -M; m <= M; ++m) {
            W += fc[y];
            y = swar_add(y, Ev, H);
        }
        for (int s = 0; s < seg_len; ++s) {
            double fx = fc[x];
            Sc[x] = W - fx;
            W += fc[swar_add(x, Pin, H)] - fc[swar_add(x, Pout, H)];
            x = swar_add(x, Ev, H);
        }
    }
}

// T_e, U_e and q_e along u-orbits; mode 0: Q += q_e, mode 1: part[slot] = q_e.
__global__ void __launch_bounds__(kThreads) k_rowsum(const double *__restrict__ f, int64_t f_stride,
                                                     const double *__restrict__ S, int64_t slot_elems,
                                                     double *__restrict__ Q, int64_t q_stride,
                                                     double *__restrict__ part, int mode, int64_t ncells, Geo g,
                                                     const int *__restrict__ dir_list, const int *__restrict__ U,
                                                     const double *__restrict__ aw,
                                                     const int *__restrict__ row_off,
                                                     const int *__restrict__ row_lo, const int *__restrict__ row_hi,
                                                     const uint32_t *__restrict__ off_in,
                                                     const uint32_t *__restrict__ off_out, int seg_len, int nseg)
{
    __shared__ uint32_t s_in[kMaxRowsSmem], s_out[kMaxRowsSmem];
    __shared__ int s_len[kMaxRowsSmem];
    const int slot = blockIdx.z;
    const int dir = dir_list[slot];
    const int r0 = row_off[dir], nr = row_off[dir + 1] - r0;
    for (int k = threadIdx.x; k < nr && k < kMaxRowsSmem; k += blockDim.x) {
        s_in[k] = off_in[r0 + k];
        s_out[k] = off_out[r0 + k];
        s_len[k] = row_hi[r0 + k] - row_lo[r0 + k] + 1;
    }
    __syncthreads();
    const int u[3] = {U[3 * dir], U[3 * dir + 1], U[3 * dir + 2]};
    const double a = aw[dir];
    const int64_t norbits = g.nodes / g.N;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= norbits * nseg) return;
    const uint32_t r = (uint32_t)(tid % norbits);
    const int seg = (int)(tid / norbits);
    const uint32_t Uv = pack_scaled(u, 1, g);
    const uint32_t H = g.H;
    const uint32_t x0 = orbit_start(r, seg, seg_len, u, g);
    for (int64_t cell = blockIdx.y; cell < ncells; cell += gridDim.y) {
        const double *fc = f + cell * f_stride;
        const double *Sc = S + (int64_t)slot * slot_elems + cell * g.nodes;
        uint32_t x = x0;
        double T = 0.0, Uu = 0.0;
        for (int k = 0; k < nr; ++k) {  // direct sum over the polygon at the segment start
            uint32_t y = swar_add(x, s_out[k], H);
            for (int q = 0; q < s_len[k]; ++q) {
                T += fc[y];
                Uu += Sc[y];
                y = swar_add(y, Uv, H);
            }
        }
        double *Qc = mode == 0 ? Q + cell * q_stride : part + (int64_t)slot * slot_elems + cell * g.nodes;
        for (int s = 0; s < seg_len; ++s) {
            const double qv = a * (Sc[x] * T - fc[x] * Uu);
            if (mode == 0)
                Qc[x] += qv;
            else
                Qc[x] = qv;
            double dT = 0.0, dU = 0.0;
            for (int k = 0; k < nr; ++k) {
                const uint32_t yi = swar_add(x, s_in[k], H), yo = swar_add(x, s_out[k], H);
                dT += fc[yi] - fc[yo];
                dU += Sc[yi] - Sc[yo];
            }
            T += dT;
            Uu += dU;
            x = swar_add(x, Uv, H);
        }
    }
}

// Q += part[0] + part[1] + ... in slot (= direction) order.
__global__ void k_reduce(double *__restrict__ Q, int64_t q_stride, const double *__restrict__ part,
                         int64_t slot_elems, int nslots, int64_t ncells, int64_t nodes)
{
    const int64_t total = ncells * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cell = i / nodes, x = i % nodes;
        double acc = Q[cell * q_stride + x];
        for (int s = 0; s < nslots; ++s) acc += part[(int64_t)s * slot_elems + i];
        Q[cell * q_stride + x] = acc;
    }
}

__global__ void k_zero(double *Q, int64_t q_stride, int64_t ncells, int64_t nodes)
{
    const int64_t total = ncells * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        Q[(i / nodes) * q_stride + i % nodes] = 0.0;
}

// Moments (reading R16): fixed-grid block partials, fixed-order trees.
__global__ void k_moments_partial(const double *__restrict__ f, Geo g, double h, double *partial)
{
    constexpr int K = kMaxD + 2;
    __shared__ double sm[K][kThreads];
    double acc[K] = {0, 0, 0, 0, 0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.nodes;
         i += (int64_t)gridDim.x * blockDim.x) {
        int c[kMaxD];
        unpack((uint32_t)i, g, c);
        double fv = f[i], v2 = 0.0;
        acc[0] += fv;
        for (int j = 0; j < g.d; ++j) {
            double v = (c[j] - g.N / 2) * h;
            acc[1 + j] += v * fv;
            v2 += v * v;
        }
        acc[g.d + 1] += v2 * fv;
    }
    for (int k = 0; k < K; ++k) sm[k][threadIdx.x] = acc[k];
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
            for (int k = 0; k < K; ++k) sm[k][threadIdx.x] += sm[k][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) partial[blockIdx.x * K + k] = sm[k][0];
}

// The kMomBlocks block partials of each moment added by a fixed-order tree in
// shared memory (one thread per partial; kMomBlocks = 128 threads).
__device__ __forceinline__ void moments_tree(const double *partial, int nblocks, double scale, double *out)
{
    constexpr int K = kMaxD + 2;
    __shared__ double sm[K][kMomBlocks];
    const int t = threadIdx.x;
    for (int k = 0; k < K; ++k) sm[k][t] = t < nblocks ? partial[t * K + k] : 0.0;
    __syncthreads();
    for (int s = kMomBlocks / 2; s > 0; s >>= 1) {
        if (t < s)
            for (int k = 0; k < K; ++k) sm[k][t] += sm[k][t + s];
        __syncthreads();
    }
    if (t < K) out[t] = sm[t][0] * scale;
}

__global__ void __launch_bounds__(kMomBlocks) k_moments_final(const double *partial, int nblocks, double scale,
                                                              double *out)
{
    moments_tree(partial, nblocks, scale, out);
}

// moments row selected by a device counter (graph-replayable): out[ctr] = ..., ctr++
__global__ void __launch_bounds__(kMomBlocks) k_moments_final_ctr(const double *partial, int nblocks, double scale,
                                                                  double *base, int *ctr)
{
    constexpr int K = kMaxD + 2;
    const int row = *ctr;
    moments_tree(partial, nblocks, scale, base + (size_t)row * K);
    __syncthreads();
    if (threadIdx.x == 0) *ctr = row + 1;
}

// dst[dst_idx[c]] = src[src_idx[c]] for c < ncells (NULL index = identity), one cell = nodes doubles
__global__ void k_copy_cells(const double *__restrict__ src, const int64_t *__restrict__ si, double *__restrict__ dst,
                             const int64_t *__restrict__ di, int64_t ncells, int64_t nodes)
{
    const int64_t total = ncells * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / nodes, x = i % nodes;
        const int64_t a = si ? si[c] : c, b = di ? di[c] : c;
        dst[b * nodes + x] = src[a * nodes + x];
    }
}

// strided variant: dst cell di[c] (stride dst_stride) = src cell si[c] (stride src_stride)
__global__ void k_copy_cells_strided(const double *__restrict__ src, int64_t src_stride, const int64_t *__restrict__ si,
                                     double *__restrict__ dst, int64_t dst_stride, const int64_t *__restrict__ di,
                                     int64_t ncells, int64_t nodes)
{
    const int64_t total = ncells * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / nodes, x = i % nodes;
        const int64_t a = si ? si[c] : c, b = di ? di[c] : c;
        dst[b * dst_stride + x] = src[a * src_stride + x];
    }
}

// Space-dependent N̄: stable bucketing of the cells by level on the device.
// idx[] receives the cells of level 0 in ascending order, then level 1, ...;
// cnt[lv] the bucket sizes and cnt[nlevels] the number of cells whose level is
// out of [0, nlevels).  One block; every count is an exact integer.
__global__ void k_level_bucket(const int *__restrict__ level, int64_t ncells, int nlevels, int64_t *__restrict__ idx,
                               int *__restrict__ cnt)
{
    __shared__ int warp_tot[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
    int64_t base = 0;
    for (int lv = -1; lv < nlevels; ++lv) {  // lv = -1: cells with an invalid level (counted only)
        int64_t n = 0;
        for (int64_t c0 = 0; c0 < ncells; c0 += blockDim.x) {
            const int64_t c = c0 + t;
            bool flag = false;
            if (c < ncells) {
                const int v = level[c];
                flag = lv < 0 ? (v < 0 || v >= nlevels) : v == lv;
            }
            const unsigned m = __ballot_sync(0xffffffffu, flag);
            if (lane == 0) warp_tot[w] = __popc(m);
            __syncthreads();
            int off = 0, tot = 0;
            for (int k = 0; k < nw; ++k) {
                off += k < w ? warp_tot[k] : 0;
                tot += warp_tot[k];
            }
            if (flag && lv >= 0) idx[base + n + off + __popc(m & ((1u << lane) - 1u))] = c;
            n += tot;
            __syncthreads();
        }
        if (t == 0) cnt[lv < 0 ? nlevels : lv] = (int)n;
        if (lv >= 0) base += n;
    }
}

// TVD-RK2 (Heun) stages: f1 = f + dt q ; f = (f + f1 + dt q1) / 2
__global__ void k_rk2_stage1(const double *f, const double *q, double dt, double *f1, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        f1[i] = f[i] + dt * q[i];
}
__global__ void k_rk2_stage2(double *f, const double *f1, const double *q1, double dt, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        f[i] = 0.5 * (f[i] + (f1[i] + dt * q1[i]));
}

__global__ void k_axpy(double *f, const double *q, double dt, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        f[i] += dt * q[i];
}

Geo geo_of(const dvm_plan_s *P)
{
    Geo g;
    g.d = P->d;
    g.p = P->p;
    g.N = P->N;
    g.H = P->pk.H;
    g.nodes = 1;
    for (int j = 0; j < P->d; ++j) g.nodes *= P->N;
    return g;
}

dvm_status_t ensure_ws(dvm_plan_s *P, int slots, size_t slot_elems, bool need_part)
{
    Workspace &w = P->ws;
    if (w.S && w.slots >= slots && w.slot_elems >= slot_elems && (!need_part || w.part)) return DVM_OK;
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    if (w.S) cudaFree(w.S);
    if (w.part) cudaFree(w.part);
    w.S = w.part = nullptr;
    w.slots = 0;
    w.slot_elems = 0;
    cudaError_t e1 = cudaMalloc(&w.S, sizeof(double) * slots * slot_elems);
    if (e1 != cudaSuccess) {
        w.S = nullptr;
        set_error("workspace allocation (S) failed");
        return DVM_E_NOMEM;
    }
    if (need_part) {
        cudaError_t e2 = cudaMalloc(&w.part, sizeof(double) * slots * slot_elems);
        if (e2 != cudaSuccess) {
            cudaFree(w.S);
            w.S = w.part = nullptr;
            set_error("workspace allocation (part) failed");
            return DVM_E_NOMEM;
        }
    }
    w.slots = slots;
    w.slot_elems = slot_elems;
    return DVM_OK;
}

}  // namespace

dvm_status_t zero_cells(dvm_plan_s *P, double *Q, int64_t q_stride, int64_t ncells, int64_t nodes)
{
    LaunchScope ls(P, KC_ZERO);
    k_zero<<<592, kThreads, 0, P->stream>>>(Q, q_stride, ncells, nodes);
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t reduce_slots(dvm_plan_s *P, double *Q, int64_t q_stride, const double *part, int64_t slot_elems,
                          int nslots, int64_t ncells, int64_t nodes)
{
    LaunchScope ls(P, KC_REDUCE);
    k_reduce<<<592, kThreads, 0, P->stream>>>(Q, q_stride, part, slot_elems, nslots, ncells, nodes);
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

#ifndef FG32_AUTO_CELLS
#define FG32_AUTO_CELLS 2
#endif
constexpr int64_t kFg32AutoCells = FG32_AUTO_CELLS;

dvm_status_t collide_batched(dvm_plan_s *P, const double *f, double *Q, int64_t ncells, int64_t stride)
{
    const Geo g = geo_of(P);
    if (ncells == 0) return DVM_OK;
    // auto: 3D N = 64 the FFT-filter gain, other 3D the frame-plane kernel when
    // built; 2D N <= 64 the small-grid pair kernel, the 2D pair kernels from
    // N = 256 and at N = 128 with >= 100 directions of this plan's shard, the
    // v1 sweeps otherwise (fewer, latency-bound launches)
    if (P->wt.on) {  // caller weights a(k) b(l): the spectral path evaluates them
        if (P->path_mode == 1 || P->path_mode == 2 || P->path_mode == 4 || P->path_mode == 6 || P->path_mode == 7) {
            set_error("custom weights (dvm_set_weights) are evaluated by the spectral path: dvm_set_path 0 or 3");
            return DVM_E_STATE;
        }
        return collide_spectral(P, f, stride, Q, stride, ncells);
    }
    if (P->path_mode == 3) return collide_spectral(P, f, stride, Q, stride, ncells);
    // auto for 3D N = 64: the FFT-filter gain (faster than the frame-plane kernel)
    if (P->path_mode == 4 || (P->path_mode == 0 && P->d == 3 && P->N == 64)) {
        bool handled = false;
        dvm_status_t st = collide_fgain3d(P, f, stride, Q, stride, ncells, &handled);
        if (st || handled) return st;
    }
    // 3D N = 32 (c4): direction pairs through one batched spectral filter (dvm_fg32.cu);
    // auto for single cells, batches go to the frame-plane kernel (two cells per node)
    if (P->path_mode == 6 || (P->path_mode == 0 && P->d == 3 && P->N == 32 && ncells <= kFg32AutoCells)) {
        bool handled = false;
        dvm_status_t st = collide_fg32(P, f, stride, Q, stride, ncells, &handled);
        if (st || handled) return st;
    }
    // auto for 2D N <= 64: pair units with the loss per pair, f in shared memory (two launches)
    if (P->path_mode == 5 || (P->path_mode == 0 && P->d == 2 && P->N <= 64)) {
        bool handled = false;
        dvm_status_t st = collide_small2d(P, f, stride, Q, stride, ncells, &handled);
        if (st || handled) return st;
    }
    // auto: the 2D pair kernels from N = 256, and at N = 128 once there are >= 100 directions
    // (tools/path128.py: N = 128 with N̄ = 7 (A = 72) v1 96 us vs 117, N̄ = 10 (A = 128) 131 vs 120)
    const bool pair_auto = P->N >= 256 || (P->N >= 128 && (int)P->local.size() >= 100);
    const bool use_new = P->path_mode == 2 || P->path_mode == 4 || P->path_mode == 7 ||
                         (P->path_mode == 0 && (P->d == 3 || pair_auto));
    if (use_new) {
        bool handled = false;
        dvm_status_t st = P->d == 3 ? collide_gain3d(P, f, stride, Q, stride, ncells, &handled)
                                    : collide_pair2d(P, f, stride, Q, stride, ncells, &handled);
        if (st || handled) return st;
    }
    const int zero_blocks = 592;
    {
        LaunchScope ls(P, KC_ZERO);
        k_zero<<<zero_blocks, kThreads, 0, P->stream>>>(Q, stride, ncells, g.nodes);
    }
    DVM_CUDA(cudaGetLastError());
    const int nloc = (int)P->local.size();
    if (nloc == 0) return DVM_OK;
    // chunk of directions evaluated per launch: one slot of S (+ partial) per direction
    const size_t cell_bytes = sizeof(double) * (size_t)g.nodes * (size_t)ncells;
    const size_t budget = (size_t)768 << 20;
    int D = (int)std::min<size_t>((size_t)nloc, std::max<size_t>(1, budget / (2 * cell_bytes)));
    D = std::min(D, 65535);
    const bool chunked = D > 1;
    dvm_status_t st = ensure_ws(P, D, (size_t)g.nodes * ncells, chunked);
    if (st) return st;
    const int *dlist = P->t.local;
    const int64_t norbits = g.nodes / g.N;
    // segments per orbit: enough threads to fill the GPU, segments >= 16 nodes (3D) / 4 (2D)
    const int64_t want = 148LL * 2048;
    int min_seg = P->d == 3 ? 16 : 4;
    int nseg = 1;
    while (nseg * 2 <= P->N / min_seg && norbits * nseg * ncells * D < want) nseg *= 2;
    const int seg_len = P->N / nseg;
    const int64_t threads = norbits * nseg;
    const unsigned bx = (unsigned)((threads + kThreads - 1) / kThreads);
    const unsigned by = (unsigned)std::min<int64_t>(ncells, 65535);
    for (int c0 = 0; c0 < nloc; c0 += D) {
        const int nd = std::min(D, nloc - c0);
        dim3 grid(bx, by, nd);
        {
            LaunchScope ls(P, KC_LINESUM);
            k_linesum<<<grid, kThreads, 0, P->stream>>>(f, stride, P->ws.S, (int64_t)P->ws.slot_elems, ncells, g,
                                                        dlist + c0, P->t.e, P->t.M, seg_len, nseg);
        }
        {
        LaunchScope ls(P, KC_ROWSUM);
        k_rowsum<<<grid, kThreads, 0, P->stream>>>(f, stride, P->ws.S, (int64_t)P->ws.slot_elems, Q, stride,
                                                   P->ws.part, chunked ? 1 : 0, ncells, g, dlist + c0, P->t.u,
                                                   P->t.a, P->t.row_off, P->t.row_lo, P->t.row_hi, P->t.off_in,
                                                   P->t.off_out, seg_len, nseg);
        }
        if (chunked) {
            LaunchScope ls(P, KC_REDUCE);
            k_reduce<<<zero_blocks, kThreads, 0, P->stream>>>(Q, stride, P->ws.part, (int64_t)P->ws.slot_elems, nd,
                                                              ncells, g.nodes);
        }
        DVM_CUDA(cudaGetLastError());
    }
    return DVM_OK;
}

dvm_status_t moments(dvm_plan_s *P, const double *f, double *dev_out_row)
{
    const Geo g = geo_of(P);
    if (!P->ws.mom_partial) DVM_CUDA(cudaMalloc(&P->ws.mom_partial, sizeof(double) * kMomBlocks * (kMaxD + 2)));
    double scale = 1.0;
    for (int j = 0; j < P->d; ++j) scale *= P->h;
    {
        LaunchScope ls(P, KC_MOMENTS);
        k_moments_partial<<<kMomBlocks, kThreads, 0, P->stream>>>(f, g, P->h, P->ws.mom_partial);
    }
    {
        LaunchScope ls(P, KC_MOMENTS);
        k_moments_final<<<1, kMomBlocks, 0, P->stream>>>(P->ws.mom_partial, kMomBlocks, scale, dev_out_row);
    }
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

// the final fixed-order tree over `nblocks` (<= kMomBlocks) partials already in ws.mom_partial
dvm_status_t moments_final_ctr(dvm_plan_s *P, int nblocks, double *dev_base, int *dev_ctr)
{
    double scale = 1.0;
    for (int j = 0; j < P->d; ++j) scale *= P->h;
    {
        LaunchScope ls(P, KC_MOMENTS);
        k_moments_final_ctr<<<1, kMomBlocks, 0, P->stream>>>(P->ws.mom_partial, nblocks, scale, dev_base, dev_ctr);
    }
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t moments_ctr(dvm_plan_s *P, const double *f, double *dev_base, int *dev_ctr)
{
    const Geo g = geo_of(P);
    if (!P->ws.mom_partial) DVM_CUDA(cudaMalloc(&P->ws.mom_partial, sizeof(double) * kMomBlocks * (kMaxD + 2)));
    double scale = 1.0;
    for (int j = 0; j < P->d; ++j) scale *= P->h;
    {
        LaunchScope ls(P, KC_MOMENTS);
        k_moments_partial<<<kMomBlocks, kThreads, 0, P->stream>>>(f, g, P->h, P->ws.mom_partial);
    }
    {
        LaunchScope ls(P, KC_MOMENTS);
        k_moments_final_ctr<<<1, kMomBlocks, 0, P->stream>>>(P->ws.mom_partial, kMomBlocks, scale, dev_base,
                                                             dev_ctr);
    }
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t copy_cells(dvm_plan_s *P, const double *src, const int64_t *si, double *dst, const int64_t *di,
                        int64_t ncells)
{
    const Geo g = geo_of(P);
    if (ncells <= 0) return DVM_OK;
    {
        LaunchScope ls(P, KC_ZERO);
        k_copy_cells<<<592, kThreads, 0, P->stream>>>(src, si, dst, di, ncells, g.nodes);
    }
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t collide_levels(dvm_plan_s *const *plans, int nlevels, const double *f, double *Q, int64_t ncells,
                            int64_t stride, const int *level)
{
    dvm_plan_s *P0 = plans[0];
    const Geo g = geo_of(P0);
    if (ncells == 0) return DVM_OK;
    Workspace &w = P0->ws;
    dvm_status_t st;
    if ((st = grow(&w.lv_idx, &w.lv_idx_elems, (size_t)ncells, P0->stream))) return st;
    if ((st = grow(&w.lv_cnt, &w.lv_cnt_elems, (size_t)nlevels + 1, P0->stream))) return st;
    {
        LaunchScope ls(P0, KC_ZERO);
        k_level_bucket<<<1, 1024, 0, P0->stream>>>(level, ncells, nlevels, w.lv_idx, w.lv_cnt);
        DVM_CUDA(cudaGetLastError());
    }
    std::vector<int> cnt(nlevels + 1);
    DVM_CUDA(cudaMemcpyAsync(cnt.data(), w.lv_cnt, sizeof(int) * (nlevels + 1), cudaMemcpyDeviceToHost, P0->stream));
    DVM_CUDA(cudaStreamSynchronize(P0->stream));
    if (cnt[nlevels] != 0) {
        set_error("dvm_collide_batched_levels: a cell's level is outside [0, nlevels)");
        return DVM_E_SHAPE;
    }
    int64_t off = 0;
    for (int lv = 0; lv < nlevels; ++lv) {
        const int64_t n = cnt[lv];
        if (n == 0) continue;
        if (n == ncells) return collide_batched(plans[lv], f, Q, ncells, stride);  // one level: no gather
        // gather buffers for the whole batch once (bucket sizes change from call to call)
        if ((st = grow(&w.lv_f, &w.lv_f_elems, (size_t)ncells * g.nodes, P0->stream))) return st;
        if ((st = grow(&w.lv_q, &w.lv_q_elems, (size_t)ncells * g.nodes, P0->stream))) return st;
        const int64_t *ix = w.lv_idx + off;
        {
            LaunchScope ls(P0, KC_ZERO);
            k_copy_cells_strided<<<592, kThreads, 0, P0->stream>>>(f, stride, ix, w.lv_f, g.nodes, nullptr, n, g.nodes);
            DVM_CUDA(cudaGetLastError());
        }
        if ((st = collide_batched(plans[lv], w.lv_f, w.lv_q, n, g.nodes))) return st;
        {
            LaunchScope ls(P0, KC_ZERO);
            k_copy_cells_strided<<<592, kThreads, 0, P0->stream>>>(w.lv_q, g.nodes, nullptr, Q, stride, ix, n, g.nodes);
            DVM_CUDA(cudaGetLastError());
        }
        off += n;
    }
    return DVM_OK;
}

dvm_status_t rk2_stage(dvm_plan_s *P, int stage, double *f, double *f1, const double *q, double dt)
{
    const Geo g = geo_of(P);
    {
        LaunchScope ls(P, KC_AXPY);
        if (stage == 1)
            k_rk2_stage1<<<296, kThreads, 0, P->stream>>>(f, q, dt, f1, g.nodes);
        else
            k_rk2_stage2<<<296, kThreads, 0, P->stream>>>(f, f1, q, dt, g.nodes);
    }
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t axpy(dvm_plan_s *P, double *f, const double *q, double dt)
{
    const Geo g = geo_of(P);
    {
        LaunchScope ls(P, KC_AXPY);
        k_axpy<<<296, kThreads, 0, P->stream>>>(f, q, dt, g.nodes);
    }
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

void clear_profile(dvm_plan_s *P)
{
    for (auto &r : P->prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    P->prof.clear();
}

void free_workspace(dvm_plan_s *P)
{
    clear_profile(P);
    Workspace &w = P->ws;
    void *ptrs[] = {w.S, w.part, w.f_stage, w.q_stage, w.mom_partial, w.mom_dev, w.qtmp, w.f1tmp, w.mom_ctr, w.fft_z, w.g3_f, w.g3_t, w.g3_q, w.g3_ctr, w.p2_scr, w.p2_part, w.sp_z, w.fg_fhat, w.lv_f, w.lv_q, w.lv_idx, w.lv_cnt, w.f32_z, w.f32_part};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    w = Workspace{};
}

}  // namespace dvm
