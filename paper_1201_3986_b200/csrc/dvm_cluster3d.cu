// dvm_cluster3d.cu -- 3D evaluation on B200: one thread-block CLUSTER per pair
// of cells, persistent over all directions (one launch per collide).
//
// Frame.  For a direction e, (u, w) is the basis of e^⊥ ∩ Z^3 from the plan
// (u × w = e) and z a transverse vector with z.e = 1, so (u, w, z) is
// unimodular: every node is x = γ z + α u + β w (mod N) for exactly one
// (γ, α, β) in Z_N^3, and the lattice planes x.e ≡ γ are N×N tori in (α, β).
// The perp polygon P_e is plane 0's set of rows
// {α u + β w : lo_b <= α <= hi_b}, so T_e = Σ_{l∈P_e} f(.+l) is a 2D polygon
// filter inside every plane; the line factors are 1D windows
// along e.
//
// Layout.  Two cells are interleaved per node (double2, 16 B): every gather or
// scatter of a plane node moves 16 useful bytes of a 32-byte sector instead
// of 8 (the plane frame is a scattered permutation of the storage order).
//
// Per direction, in cluster-wide lock step:
//   phase A  CTA rank r takes planes γ = r, r + CL, ...: gathers the plane of
//            both cells into shared memory as row prefix sums, periodically
//            extended by HALO nodes each side (no wrap logic in the lookups),
//            then T(α, β) = Σ_b [P(β+b, α+hi_b) − P(β+b, α+lo_b−1)] and
//            stores T to the cluster's L2-resident T buffer.
//   cluster barrier (release/acquire: T visible to the whole cluster)
//   phase B  S = Σ_{1<=|m|<=M} f(x+me), U = Σ_{1<=|m|<=M} T(x+me),
//            Q(x) += a_e (S T(x) − f(x) U)      (eq:decD)
//            by sliding windows along segments of e-orbits (lanes on adjacent
//            orbits, coalesced when e_0 or e_1 is odd), else by a node-owned
//            stencil in storage order (always coalesced).
//   cluster barrier
// Q accumulates in direction order: bitwise deterministic, no atomics.  One
// pair of cells per cluster keeps f + T + Q of the cells in flight in L2.
// Small batches split each pair's directions into chunks (partial Q buffers,
// reduced in chunk order by k_deinterleave).
#include <cooperative_groups.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "dvm_internal.h"

namespace cg = cooperative_groups;

namespace dvm {
namespace {

constexpr int kCT = 1024;      // threads per CTA (one CTA per SM)
constexpr int kMaxRows = 256;  // perp-polygon rows held in shared memory
constexpr int kMaxM = 64;      // line half-widths held in shared memory

template <int N>
__host__ __device__ constexpr int halo()
{
    return N / 2;
}

struct C3Args {
    const double2 *f;  // [groups][N^3] two interleaved cells
    double2 *Q;        // [chunks][groups][N^3]
    double2 *Tbuf;     // [clusters][N^3]
    int64_t ngroups;
    int nchunks;
    const int *dirs;
    int ndirs;
    const int *E, *U, *W, *Z, *M;
    const double *a;
    const int *row_off, *row_b, *row_lo, *row_hi;
    uint32_t H;
    int p;
    int dbg;  // timing experiments only (DVM_C3_DEBUG): bit0 skip phase A, bit1 skip phase B
    int gsize;            // software groups: CTAs per group (SOFT kernels)
    unsigned int *gctr;   // software groups: one barrier counter per group
};

// Group barrier for SOFT (cooperative-launch) kernels: every CTA of the group
// arrives on a monotonic counter; thread 0 publishes the CTA's writes with a
// gpu-scope fence, then acquire-polls until all gsize CTAs of this epoch
// arrived (the acquire also invalidates the SM's L1, so later plain loads see
// the other CTAs' T and Q).
__device__ __forceinline__ void group_barrier(unsigned int *ctr, unsigned int target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned int v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= target) break;
            __nanosleep(32);
        }
    }
    __syncthreads();
}

template <int N>
__device__ __forceinline__ uint32_t pack3(int c0, int c1, int c2, int p)
{
    return ((uint32_t)(c0 & (N - 1)) << (2 * p)) | ((uint32_t)(c1 & (N - 1)) << p) | (uint32_t)(c2 & (N - 1));
}

__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

template <int N, bool SOFT>
__global__ void __launch_bounds__(kCT, 1) k_cluster3d(C3Args A)
{
    constexpr int HALO = halo<N>();
    constexpr int STRIDE = N + 2 * HALO;
    constexpr int NW = kCT / 32;
    constexpr int RPW = N / NW;  // scan rows per warp
    constexpr int LPL = N / 32;  // row elements per lane in the scan
    constexpr int OA = N / 32;   // outputs along α per thread (lane + 32 h)
    constexpr int OB = N / NW;   // outputs along β per thread (warp + NW g)
    constexpr int64_t NODES = (int64_t)N * N * N;
    constexpr int NN = N * N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *sP = reinterpret_cast<double2 *>(smem_raw);      // [N][STRIDE]
    int4 *sRow = reinterpret_cast<int4 *>(sP + N * STRIDE);   // {b, lo-1, hi, 0}
    uint2 *sOff = reinterpret_cast<uint2 *>(sRow + kMaxRows);  // {pack(m e), pack(-m e)}, m = 1..M
    __shared__ int s_meta[16];

    const int CL = SOFT ? A.gsize : (int)cg::this_cluster().num_blocks();
    const int rank = SOFT ? (int)(blockIdx.x % CL) : (int)cg::this_cluster().block_rank();
    const int cid = blockIdx.x / CL;
    const int nclusters = gridDim.x / CL;
    unsigned int epoch = 0;
    auto barrier = [&]() {
        if constexpr (SOFT) {
            ++epoch;
            group_barrier(A.gctr + cid, epoch * (unsigned)CL);
        } else {
            cg::this_cluster().sync();
        }
    };
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int p = A.p;
    const uint32_t H = A.H;
    double2 *Tb = A.Tbuf + (int64_t)cid * NODES;
    const int64_t items = A.ngroups * A.nchunks;

    for (int64_t item = cid; item < items; item += nclusters) {
        const int64_t grp = item / A.nchunks;
        const int chunk = (int)(item % A.nchunks);
        const int d0 = (int)((int64_t)A.ndirs * chunk / A.nchunks);
        const int d1 = (int)((int64_t)A.ndirs * (chunk + 1) / A.nchunks);
        const double2 *__restrict__ fc = A.f + grp * NODES;
        double2 *Qc = A.Q + ((int64_t)chunk * A.ngroups + grp) * NODES;

        for (int di = d0; di < d1; ++di) {
            const int dir = A.dirs[di];
            if (threadIdx.x == 0) {
                for (int j = 0; j < 3; ++j) {
                    s_meta[j] = A.E[3 * dir + j];
                    s_meta[3 + j] = A.U[3 * dir + j];
                    s_meta[6 + j] = A.W[3 * dir + j];
                    s_meta[9 + j] = A.Z[3 * dir + j];
                }
                s_meta[12] = min(A.M[dir], kMaxM);
                s_meta[13] = A.row_off[dir];
                s_meta[14] = min(A.row_off[dir + 1] - A.row_off[dir], kMaxRows);
            }
            __syncthreads();
            const int e0 = s_meta[0], e1 = s_meta[1], e2 = s_meta[2];
            const int u0 = s_meta[3], u1 = s_meta[4], u2 = s_meta[5];
            const int w0 = s_meta[6], w1 = s_meta[7], w2 = s_meta[8];
            const int z0 = s_meta[9], z1 = s_meta[10], z2 = s_meta[11];
            const int M = s_meta[12], r0 = s_meta[13], nr = s_meta[14];
            for (int k = threadIdx.x; k < nr; k += kCT)
                sRow[k] = make_int4(A.row_b[r0 + k], A.row_lo[r0 + k] - 1, A.row_hi[r0 + k], 0);
            for (int m = 1 + threadIdx.x; m <= M; m += kCT)
                sOff[m] = make_uint2(pack3<N>(m * e0, m * e1, m * e2, p), pack3<N>(-m * e0, -m * e1, -m * e2, p));
            const double aw = A.a[dir];
            __syncthreads();

            // ---------------- phase A: T on this CTA's planes (both cells)
            for (int g = rank; g < N && !(A.dbg & 1); g += CL) {
#pragma unroll
                for (int i = 0; i < RPW; ++i) {
                    const int beta = warp + NW * i;
                    const int b0 = g * z0 + beta * w0, b1 = g * z1 + beta * w1, b2 = g * z2 + beta * w2;
                    double2 v[LPL];
#pragma unroll
                    for (int j = 0; j < LPL; ++j) {
                        const int al = lane * LPL + j;
                        v[j] = __ldg(fc + pack3<N>(b0 + al * u0, b1 + al * u1, b2 + al * u2, p));
                    }
#pragma unroll
                    for (int j = 1; j < LPL; ++j) v[j] = add2(v[j], v[j - 1]);
                    double2 x = v[LPL - 1];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const double yx = __shfl_up_sync(0xffffffffu, x.x, o);
                        const double yy = __shfl_up_sync(0xffffffffu, x.y, o);
                        if (lane >= o) {
                            x.x += yx;
                            x.y += yy;
                        }
                    }
                    const double2 excl = sub2(x, v[LPL - 1]);
                    const double2 tot = make_double2(__shfl_sync(0xffffffffu, x.x, 31), __shfl_sync(0xffffffffu, x.y, 31));
                    double2 *rowp = sP + beta * STRIDE + HALO;
#pragma unroll
                    for (int j = 0; j < LPL; ++j) {
                        const int al = lane * LPL + j;
                        const double2 pv = add2(v[j], excl);
                        rowp[al] = pv;
                        if (al >= N - HALO) rowp[al - N] = sub2(pv, tot);
                        if (al < HALO) rowp[al + N] = add2(pv, tot);
                    }
                }
                __syncthreads();
                double2 acc[OB][OA];
#pragma unroll
                for (int gg = 0; gg < OB; ++gg)
#pragma unroll
                    for (int h = 0; h < OA; ++h) acc[gg][h] = make_double2(0.0, 0.0);
                for (int k = 0; k < nr; ++k) {
                    const int4 rw = sRow[k];
#pragma unroll
                    for (int gg = 0; gg < OB; ++gg) {
                        const double2 *rowp = sP + ((warp + NW * gg + rw.x) & (N - 1)) * STRIDE + HALO + lane;
                        const double2 *ph = rowp + rw.z, *pl = rowp + rw.y;
#pragma unroll
                        for (int h = 0; h < OA; ++h) acc[gg][h] = add2(acc[gg][h], sub2(ph[32 * h], pl[32 * h]));
                    }
                }
#pragma unroll
                for (int gg = 0; gg < OB; ++gg) {
                    const int beta = warp + NW * gg;
                    const int b0 = g * z0 + beta * w0, b1 = g * z1 + beta * w1, b2 = g * z2 + beta * w2;
#pragma unroll
                    for (int h = 0; h < OA; ++h) {
                        const int al = lane + 32 * h;
                        Tb[pack3<N>(b0 + al * u0, b1 + al * u1, b2 + al * u2, p)] = acc[gg][h];
                    }
                }
                __syncthreads();
            }
            barrier();

            // ---------------- phase B: S, U along e and the Q update
            if (!(A.dbg & 2)) {
                const double2 *__restrict__ Tr = Tb;
                if ((e0 & 1) || (e1 & 1)) {
                    // e-orbit segments of length N/SEGS, one per thread: lanes walk
                    // adjacent orbits (consecutive fastest-axis nodes: coalesced) and
                    // slide the windows in registers (enter/leave per step).
                    constexpr int SEGS = (16 * kCT) / NN < N / 8 ? ((16 * kCT) / NN > 0 ? (16 * kCT) / NN : 1) : N / 8;
                    constexpr int SL = N / SEGS;
                    const int ja = (e0 & 1) ? 0 : 1;
                    const uint32_t Ev = sOff[1].x;
                    const uint32_t Pin = pack3<N>((M + 1) * e0, (M + 1) * e1, (M + 1) * e2, p);
                    const uint32_t Pout = sOff[M].y;
                    for (int gt = rank * kCT + threadIdx.x; gt < NN * SEGS; gt += CL * kCT) {
                        const int r = gt % NN, seg = gt / NN;
                        const int hiF = r >> p, loF = r & (N - 1);
                        const int c0 = ja == 0 ? 0 : hiF, c1 = ja == 0 ? hiF : 0;
                        const int t0 = seg * SL;
                        uint32_t x = pack3<N>(c0 + t0 * e0, c1 + t0 * e1, loF + t0 * e2, p);
                        double2 Wf = make_double2(0.0, 0.0), WT = make_double2(0.0, 0.0);
                        uint32_t y = swar_add(x, Pout, H);
                        for (int m = -M; m <= M; ++m) {
                            Wf = add2(Wf, __ldg(fc + y));
                            WT = add2(WT, Tr[y]);
                            y = swar_add(y, Ev, H);
                        }
#pragma unroll 4
                        for (int s = 0; s < SL; ++s) {
                            const uint32_t yi = swar_add(x, Pin, H), yo = swar_add(x, Pout, H);
                            const double2 f0 = __ldg(fc + x), T0 = Tr[x];
                            const double2 fi = __ldg(fc + yi), fo = __ldg(fc + yo), ti = Tr[yi], to = Tr[yo];
                            const double2 S = sub2(Wf, f0), Uu = sub2(WT, T0);
                            double2 q = Qc[x];
                            q.x += aw * (S.x * T0.x - f0.x * Uu.x);
                            q.y += aw * (S.y * T0.y - f0.y * Uu.y);
                            Qc[x] = q;
                            Wf = add2(Wf, sub2(fi, fo));
                            WT = add2(WT, sub2(ti, to));
                            x = swar_add(x, Ev, H);
                        }
                    }
                } else {
                    // e0, e1 even: node-owned stencil in storage order (coalesced)
                    for (int64_t x = (int64_t)rank * kCT + threadIdx.x; x < NODES; x += (int64_t)CL * kCT) {
                        const uint32_t xi = (uint32_t)x;
                        const double2 f0 = __ldg(fc + xi), T0 = Tr[xi];
                        double2 S = make_double2(0.0, 0.0), Uu = make_double2(0.0, 0.0);
                        for (int m = 1; m <= M; ++m) {
                            const uint2 o = sOff[m];
                            const uint32_t xp = swar_add(xi, o.x, H), xm = swar_add(xi, o.y, H);
                            const double2 fp = __ldg(fc + xp), fm = __ldg(fc + xm), tp = Tr[xp], tm = Tr[xm];
                            S = add2(S, add2(fp, fm));
                            Uu = add2(Uu, add2(tp, tm));
                        }
                        double2 q = Qc[xi];
                        q.x += aw * (S.x * T0.x - f0.x * Uu.x);
                        q.y += aw * (S.y * T0.y - f0.y * Uu.y);
                        Qc[xi] = q;
                    }
                }
            }
            barrier();
        }
    }
}

// f [cells][stride] -> fI [groups][nodes] (double2), odd tail padded with 0
__global__ void k_interleave(const double *__restrict__ f, int64_t stride, int64_t ncells, int64_t nodes,
                             double2 *__restrict__ fI)
{
    const int64_t ngroups = (ncells + 1) / 2;
    const int64_t total = ngroups * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = i / nodes, x = i % nodes;
        const int64_t c0 = 2 * g, c1 = 2 * g + 1;
        fI[i] = make_double2(f[c0 * stride + x], c1 < ncells ? f[c1 * stride + x] : 0.0);
    }
}

// Q[cell] = Σ_chunks QI[chunk][group][.] component (chunk order: deterministic)
__global__ void k_deinterleave(const double2 *__restrict__ QI, int nchunks, int64_t ngroups, int64_t ncells,
                               int64_t nodes, double *__restrict__ Q, int64_t stride)
{
    const int64_t total = ncells * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / nodes, x = i % nodes;
        const int64_t g = c / 2;
        const bool hi = c & 1;
        double acc = 0.0;
        for (int k = 0; k < nchunks; ++k) {
            const double2 v = QI[((int64_t)k * ngroups + g) * nodes + x];
            acc += hi ? v.y : v.x;
        }
        Q[c * stride + x] = acc;
    }
}

__global__ void k_zero2(double2 *a, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = make_double2(0.0, 0.0);
}

template <int N>
size_t smem_bytes()
{
    return sizeof(double2) * (size_t)N * (N + 2 * halo<N>()) + sizeof(int4) * kMaxRows + sizeof(uint2) * (kMaxM + 1);
}

template <typename T>
dvm_status_t grow(T **ptr, size_t *cap, size_t need, cudaStream_t s)
{
    if (*cap >= need) return DVM_OK;
    DVM_CUDA(cudaStreamSynchronize(s));
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    *cap = 0;
    if (cudaMalloc(ptr, sizeof(T) * need) != cudaSuccess) {
        *ptr = nullptr;
        set_error("cluster workspace allocation failed");
        return DVM_E_NOMEM;
    }
    *cap = need;
    return DVM_OK;
}

template <int N>
dvm_status_t launch(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                    int64_t ncells, bool *handled)
{
    auto kern = k_cluster3d<N, false>;
    auto kern_soft = k_cluster3d<N, true>;
    const size_t smem = smem_bytes<N>();
    DVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    DVM_CUDA(cudaFuncSetAttribute(kern_soft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const bool verbose = getenv("DVM_VERBOSE") != nullptr;
    // Mode "soft" (default): cooperative launch, software groups of 16 CTAs
    // (one per SM) -- free of the GPC packing limits of hardware clusters.
    // Mode "cluster": hardware thread-block clusters.
    const char *mode_env = getenv("DVM_C3_MODE");
    const bool soft = !(mode_env && mode_env[0] == 'c');
    int best_cl = 0, best_nc = 0;
    const double pair_bytes = 3.0 * 16.0 * (double)N * N * N;
    if (soft) {
        int dev = 0, sms = 0, per_sm = 0, coop = 0;
        DVM_CUDA(cudaGetDevice(&dev));
        DVM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        DVM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        DVM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern_soft, kCT, smem));
        if (!coop || per_sm < 1) return DVM_OK;
        best_cl = 16;
        // groups in flight: all co-resident CTAs, capped by ~110 MB of L2 for
        // the pairs in flight (f + T + Q each)
        best_nc = std::min((sms * per_sm) / best_cl, std::max(1, (int)(110.0e6 / pair_bytes)));
        if (getenv("DVM_C3_GROUPS")) best_nc = std::min(best_nc, std::max(1, atoi(getenv("DVM_C3_GROUPS"))));
        if (verbose)
            fprintf(stderr, "[dvm] cluster3d N=%d: soft groups of %d CTAs, %d groups (co-resident CTAs %d)\n", N,
                    best_cl, best_nc, sms * per_sm);
    } else {
        const int cls[5] = {16, 8, 4, 2, 1};
        int ncl[5] = {0, 0, 0, 0, 0};
        for (int ci = 0; ci < 5; ++ci) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cls[ci];
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(cls[ci], 1, 1);
            cfg.blockDim = dim3(kCT, 1, 1);
            cfg.dynamicSmemBytes = smem;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&ncl[ci], (void *)kern, &cfg) != cudaSuccess) {
                cudaGetLastError();
                ncl[ci] = 0;
            }
        }
        // score = SMs kept busy, scaled down when the pairs in flight exceed ~100 MB of L2
        double best_score = -1.0;
        for (int ci = 0; ci < 5; ++ci) {
            if (ncl[ci] <= 0) continue;
            const double score = (double)ncl[ci] * cls[ci] * std::min(1.0, 100.0e6 / (ncl[ci] * pair_bytes));
            if (verbose) fprintf(stderr, "[dvm]   cluster %2d: %3d clusters, score %.1f\n", cls[ci], ncl[ci], score);
            if (score > best_score * 1.02) {
                best_score = score;
                best_cl = cls[ci];
                best_nc = ncl[ci];
            }
        }
        if (getenv("DVM_C3_CLUSTER")) {  // experiment override
            const int want = atoi(getenv("DVM_C3_CLUSTER"));
            for (int ci = 0; ci < 5; ++ci)
                if (cls[ci] == want && ncl[ci] > 0) {
                    best_cl = want;
                    best_nc = ncl[ci];
                }
        }
        if (best_cl == 0) return DVM_OK;  // not launchable: caller uses the orbit kernels
        if (verbose) fprintf(stderr, "[dvm] cluster3d N=%d: cluster=%d active_clusters=%d\n", N, best_cl, best_nc);
    }
    const int nloc = (int)P->local.size();
    const int64_t nodes = (int64_t)N * N * N;
    const int64_t ngroups = (ncells + 1) / 2;
    int nchunks = 1;
    if (ngroups < best_nc) nchunks = (int)std::min<int64_t>(nloc, (best_nc + ngroups - 1) / ngroups);
    const int64_t items = ngroups * nchunks;
    const int nclusters = (int)std::min<int64_t>(best_nc, items);
    Workspace &w = P->ws;
    dvm_status_t st;
    if ((st = grow(&w.c3_f, &w.c3_f_elems, (size_t)ngroups * nodes, P->stream))) return st;
    if ((st = grow(&w.c3_q, &w.c3_q_elems, (size_t)nchunks * ngroups * nodes, P->stream))) return st;
    if ((st = grow(&w.c3_t, &w.c3_t_elems, (size_t)nclusters * nodes, P->stream))) return st;
    {
        LaunchScope ls(P, KC_ZERO);
        k_interleave<<<1184, 256, 0, P->stream>>>(f, f_stride, ncells, nodes, w.c3_f);
        k_zero2<<<1184, 256, 0, P->stream>>>(w.c3_q, (int64_t)nchunks * ngroups * nodes);
        DVM_CUDA(cudaGetLastError());
    }
    C3Args a;
    a.f = w.c3_f;
    a.Q = w.c3_q;
    a.Tbuf = w.c3_t;
    a.ngroups = ngroups;
    a.nchunks = nchunks;
    a.dirs = P->t.local;
    a.ndirs = nloc;
    a.E = P->t.e;
    a.U = P->t.u;
    a.W = P->t.w;
    a.Z = P->t.z;
    a.M = P->t.M;
    a.a = P->t.a;
    a.row_off = P->t.row_off;
    a.row_b = P->t.row_b;
    a.row_lo = P->t.row_lo;
    a.row_hi = P->t.row_hi;
    a.H = P->pk.H;
    a.p = P->p;
    a.dbg = getenv("DVM_C3_DEBUG") ? atoi(getenv("DVM_C3_DEBUG")) : 0;
    a.gsize = best_cl;
    a.gctr = nullptr;
    if (soft) {
        if ((st = grow(&w.c3_ctr, &w.c3_ctr_elems, (size_t)nclusters, P->stream))) return st;
        DVM_CUDA(cudaMemsetAsync(w.c3_ctr, 0, sizeof(unsigned int) * nclusters, P->stream));
        a.gctr = w.c3_ctr;
        void *args[] = {&a};
        LaunchScope ls(P, KC_CLUSTER3D);
        DVM_CUDA(cudaLaunchCooperativeKernel((void *)kern_soft, dim3(nclusters * best_cl), dim3(kCT), args, smem,
                                             P->stream));
    } else {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = best_cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(nclusters * best_cl, 1, 1);
        cfg.blockDim = dim3(kCT, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = P->stream;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        LaunchScope ls(P, KC_CLUSTER3D);
        DVM_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    }
    {
        LaunchScope ls(P, KC_REDUCE);
        k_deinterleave<<<1184, 256, 0, P->stream>>>(w.c3_q, nchunks, ngroups, ncells, nodes, Q, q_stride);
        DVM_CUDA(cudaGetLastError());
    }
    *handled = true;
    return DVM_OK;
}

}  // namespace

dvm_status_t collide_cluster3d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                               int64_t ncells, bool *handled)
{
    *handled = false;
    if (P->d != 3 || ncells <= 0 || P->local.empty()) return DVM_OK;
    for (int i : P->local)
        if (P->h_nrows[i] > kMaxRows || P->h_M[i] > kMaxM) return DVM_OK;
    const int hl = P->N / 2;
    if (P->h_row_extent < 0 || P->h_row_extent > hl) return DVM_OK;
    switch (P->N) {
    case 32: return launch<32>(P, f, f_stride, Q, q_stride, ncells, handled);
    case 64: return launch<64>(P, f, f_stride, Q, q_stride, ncells, handled);
    default: return DVM_OK;
    }
}

}  // namespace dvm
