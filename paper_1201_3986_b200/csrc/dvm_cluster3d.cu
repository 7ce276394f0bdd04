// dvm_cluster3d.cu -- v2 3D evaluation: one thread-block CLUSTER per cell,
// persistent over all directions, one launch per collide.
//
// For a direction e, let (u, w) be the basis of e^⊥ ∩ Z^3 from the plan and z
// a transverse vector with z.e = 1, so (u, w, z) is unimodular and every node
// is x = γ z + α u + β w (mod N) for exactly one (γ, α, β) in Z_N^3: the
// lattice planes x.e ≡ γ are N×N tori in (α, β).  The perp polygon P_e
// lies in plane 0 as rows {α u + β w : lo_b <= α <= hi_b},
// so T_e = Σ_{l∈P_e} f(.+l) is a 2D polygon filter inside each plane, and the
// line factors are 1D windows along e-orbits.  Per direction:
//
//   phase A  each CTA of the cluster takes planes γ = rank, rank+CL, ...:
//            gathers the plane of f into shared memory as row prefix sums
//            P(β, α) (warp scans), then T(α, β) = Σ_b [P(β+b, α+hi_b) −
//            P(β+b, α+lo_b−1)] (+ row total on wrap) and writes T to the
//            cluster's T buffer (L2-resident, N^3 doubles).
//   cluster barrier (release/acquire: T visible, L1 invalidated)
//   phase B  threads sweep e-orbits (sliding windows, as v1): S = window of
//            f, U = window of T along e, Q(x) += a_e (S T − f U)
//            (eq:decD; U = Σ_{m≠0} T(.+me) is the loss).
//   cluster barrier
//
// Q accumulates in direction order (bitwise deterministic, no atomics).  Many
// cells in flight (one per cluster) keep the working set f + T + Q of the
// cells in flight in L2.  Small batches split each cell's directions into
// chunks with partial Q buffers reduced afterwards in chunk order.
#include <cooperative_groups.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "dvm_internal.h"

namespace cg = cooperative_groups;

namespace dvm {
namespace {

constexpr int kMaxRows = 256;  // perp-polygon rows held in shared memory

struct C3Args {
    const double *f;
    int64_t f_stride;
    double *Q;  // direct target (nchunks == 1) or partial buffer [chunk][cell][N^3]
    int64_t q_stride;
    double *Tbuf;  // [clusters][N^3]
    int64_t ncells;
    int nchunks;
    const int *dirs;
    int ndirs;
    const int *E, *U, *W, *Z, *M;
    const double *a;
    const int *row_off, *row_b, *row_lo, *row_hi;
    uint32_t H;
    int p;
    int seg_len, nseg;
    int dbg;  // timing experiments only (DVM_C3_DEBUG): bit0 skip phase A, bit1 skip phase B
};

template <int N>
__device__ __forceinline__ uint32_t pack3(int c0, int c1, int c2, int p)
{
    return ((uint32_t)(c0 & (N - 1)) << (2 * p)) | ((uint32_t)(c1 & (N - 1)) << p) | (uint32_t)(c2 & (N - 1));
}

// threads per CTA: 512 (two CTAs per SM) up to N = 64, 1024 for N = 128
template <int N>
__host__ __device__ constexpr int cta_threads()
{
    return N >= 128 ? 1024 : 512;
}

// Each shared-memory row holds the prefix sums extended periodically by HALO
// nodes on both sides (P(k) = P(k mod N) + floor(k/N) * rowtotal), so the
// window lookups of the perp-polygon rows never wrap.
template <int N>
__host__ __device__ constexpr int halo()
{
    return N >= 128 ? 32 : N / 2;
}

template <int N>
__global__ void __launch_bounds__(cta_threads<N>(), 1024 / cta_threads<N>()) k_cluster3d(C3Args A)
{
    constexpr int HALO = halo<N>();
    constexpr int STRIDE = N + 2 * HALO;
    constexpr int kCT = cta_threads<N>();
    constexpr int NW = kCT / 32;  // warps per CTA
    constexpr int LPL = N / 32;   // row elements per lane in the prefix scan
    constexpr int OA = N / 32;    // outputs per thread along α (lane + 32 h)
    constexpr int OB = N / NW;    // outputs per thread along β (warp + NW g)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *sP = reinterpret_cast<double *>(smem_raw);  // [N][STRIDE] extended row prefix sums
    int4 *sRow = reinterpret_cast<int4 *>(sP + N * STRIDE);  // {b, lo-1, hi, 0} per polygon row
    __shared__ int s_meta[16];

    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int cid = blockIdx.x / CL;
    const int nclusters = gridDim.x / CL;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int p = A.p;
    const uint32_t H = A.H;
    constexpr int NN = N * N;
    const int64_t nodes = (int64_t)N * N * N;
    double *Tb = A.Tbuf + (int64_t)cid * nodes;
    const int64_t items = A.ncells * A.nchunks;

    for (int64_t item = cid; item < items; item += nclusters) {
        const int64_t cell = item / A.nchunks;
        const int chunk = (int)(item % A.nchunks);
        const int d0 = (int)((int64_t)A.ndirs * chunk / A.nchunks);
        const int d1 = (int)((int64_t)A.ndirs * (chunk + 1) / A.nchunks);
        const double *fc = A.f + cell * A.f_stride;
        double *Qc = A.nchunks == 1 ? A.Q + cell * A.q_stride : A.Q + ((int64_t)chunk * A.ncells + cell) * nodes;

        for (int di = d0; di < d1; ++di) {
            const int dir = A.dirs[di];
            if (threadIdx.x == 0) {
                for (int j = 0; j < 3; ++j) {
                    s_meta[j] = A.E[3 * dir + j];
                    s_meta[3 + j] = A.U[3 * dir + j];
                    s_meta[6 + j] = A.W[3 * dir + j];
                    s_meta[9 + j] = A.Z[3 * dir + j];
                }
                s_meta[12] = A.M[dir];
                s_meta[13] = A.row_off[dir];
                s_meta[14] = min(A.row_off[dir + 1] - A.row_off[dir], kMaxRows);
            }
            __syncthreads();
            const int r0 = s_meta[13], nr = s_meta[14];
            for (int k = threadIdx.x; k < nr; k += kCT)
                sRow[k] = make_int4(A.row_b[r0 + k], A.row_lo[r0 + k] - 1, A.row_hi[r0 + k], 0);
            const int e0 = s_meta[0], e1 = s_meta[1], e2 = s_meta[2];
            const int u0 = s_meta[3], u1 = s_meta[4], u2 = s_meta[5];
            const int w0 = s_meta[6], w1 = s_meta[7], w2 = s_meta[8];
            const int z0 = s_meta[9], z1 = s_meta[10], z2 = s_meta[11];
            const int M = s_meta[12];
            const double aw = A.a[dir];
            __syncthreads();

            // ---------------- phase A: T on this CTA's planes
            for (int g = rank; g < N && !(A.dbg & 1); g += CL) {
                // row prefix sums of f on plane g (warp per row)
#pragma unroll
                for (int i = 0; i < N / NW; ++i) {
                    const int beta = warp + NW * i;
                    const int b0 = g * z0 + beta * w0, b1 = g * z1 + beta * w1, b2 = g * z2 + beta * w2;
                    double v[LPL];
#pragma unroll
                    for (int j = 0; j < LPL; ++j) {
                        const int al = lane * LPL + j;
                        v[j] = __ldg(fc + pack3<N>(b0 + al * u0, b1 + al * u1, b2 + al * u2, p));
                    }
#pragma unroll
                    for (int j = 1; j < LPL; ++j) v[j] += v[j - 1];
                    double x = v[LPL - 1];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        double y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    const double excl = x - v[LPL - 1];
                    const double rtot = __shfl_sync(0xffffffffu, x, 31);
                    double *rowp = sP + beta * STRIDE + HALO;
#pragma unroll
                    for (int j = 0; j < LPL; ++j) {
                        const int al = lane * LPL + j;
                        const double pv = v[j] + excl;
                        rowp[al] = pv;
                        if (al >= N - HALO) rowp[al - N] = pv - rtot;
                        if (al < HALO) rowp[al + N] = pv + rtot;
                    }
                }
                __syncthreads();
                double th[OB][OA], tl[OB][OA];
#pragma unroll
                for (int gg = 0; gg < OB; ++gg)
#pragma unroll
                    for (int h = 0; h < OA; ++h) th[gg][h] = tl[gg][h] = 0.0;
                for (int k = 0; k < nr; ++k) {
                    const int4 rw = sRow[k];
#pragma unroll
                    for (int gg = 0; gg < OB; ++gg) {
                        const double *rowp = sP + ((warp + NW * gg + rw.x) & (N - 1)) * STRIDE + HALO + lane;
                        const double *ph = rowp + rw.z, *pl = rowp + rw.y;
#pragma unroll
                        for (int h = 0; h < OA; ++h) {
                            th[gg][h] += ph[32 * h];
                            tl[gg][h] += pl[32 * h];
                        }
                    }
                }
#pragma unroll
                for (int gg = 0; gg < OB; ++gg) {
                    const int beta = warp + NW * gg;
                    const int b0 = g * z0 + beta * w0, b1 = g * z1 + beta * w1, b2 = g * z2 + beta * w2;
#pragma unroll
                    for (int h = 0; h < OA; ++h) {
                        const int al = lane + 32 * h;
                        Tb[pack3<N>(b0 + al * u0, b1 + al * u1, b2 + al * u2, p)] = th[gg][h] - tl[gg][h];
                    }
                }
                __syncthreads();
            }
            cluster.sync();

            // ---------------- phase B: e-orbit sweeps -> S, U, Q
            for (int gt = rank * kCT + threadIdx.x; gt < NN * A.nseg && !(A.dbg & 2); gt += CL * kCT) {
                {
                    const int r = gt % NN, seg = gt / NN;
                    // transversal axis: first non-fastest odd component of e
                    const int ja = (e0 & 1) ? 0 : ((e1 & 1) ? 1 : 2);
                    int c[3];
                    // insert x_ja = 0 into the 2-field orbit index r
                    const int hiF = r >> p, loF = r & (N - 1);
                    if (ja == 0) { c[0] = 0; c[1] = hiF; c[2] = loF; }
                    else if (ja == 1) { c[0] = hiF; c[1] = 0; c[2] = loF; }
                    else { c[0] = hiF; c[1] = loF; c[2] = 0; }
                    const int t0 = seg * A.seg_len;
                    uint32_t x = pack3<N>(c[0] + t0 * e0, c[1] + t0 * e1, c[2] + t0 * e2, p);
                    const uint32_t Ev = pack3<N>(e0, e1, e2, p);
                    const uint32_t Pin = pack3<N>((M + 1) * e0, (M + 1) * e1, (M + 1) * e2, p);
                    const uint32_t Pout = pack3<N>(-M * e0, -M * e1, -M * e2, p);
                    const double *__restrict__ fr = fc;
                    const double *__restrict__ Tr = Tb;
                    double *__restrict__ Qr = Qc;
                    double Wf = 0.0, WT = 0.0;
                    uint32_t y = swar_add(x, Pout, H);
                    for (int m = -M; m <= M; ++m) {
                        Wf += __ldg(fr + y);
                        WT += Tr[y];
                        y = swar_add(y, Ev, H);
                    }
#pragma unroll 4
                    for (int s = 0; s < A.seg_len; ++s) {
                        const uint32_t yi = swar_add(x, Pin, H), yo = swar_add(x, Pout, H);
                        const double fx = __ldg(fr + x), Tx = Tr[x];
                        const double fi = __ldg(fr + yi), fo = __ldg(fr + yo), ti = Tr[yi], to = Tr[yo];
                        const double S = Wf - fx, Uu = WT - Tx;
                        Qr[x] += aw * (S * Tx - fx * Uu);
                        Wf += fi - fo;
                        WT += ti - to;
                        x = swar_add(x, Ev, H);
                    }
                }
            }
            cluster.sync();
        }
    }
}

template <int N>
size_t smem_bytes()
{
    return sizeof(double) * (size_t)N * (N + 2 * halo<N>()) + sizeof(int4) * kMaxRows;
}

template <int N>
dvm_status_t launch(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                    int64_t ncells, bool *handled)
{
    auto kern = k_cluster3d<N>;
    constexpr int kCT = cta_threads<N>();
    const size_t smem = smem_bytes<N>();
    DVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    // cluster size: the one keeping the most SMs busy (ties: larger clusters,
    // fewer cells in flight, smaller L2 working set)
    int ncl[5] = {0, 0, 0, 0, 0};
    const int cls[5] = {16, 8, 4, 2, 1};
    int max_ctas = 0;
    for (int ci = 0; ci < 5; ++ci) {
        const int cl = cls[ci];
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cl, 1, 1);
        cfg.blockDim = dim3(kCT, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, (void *)kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            nc = 0;
        }
        ncl[ci] = nc;
        max_ctas = std::max(max_ctas, nc * cl);
    }
    // One cell per cluster: choose the cluster size by co-resident CTAs, scaled
    // down when the cells in flight (f + T + Q = 3 N^3 doubles each) would not
    // fit in ~96 MB of L2.
    int best_cl = 0, best_nc = 0;
    double best_score = -1.0;
    const double cell_bytes = 3.0 * 8.0 * (double)N * N * N;
    for (int ci = 0; ci < 5; ++ci) {
        if (ncl[ci] <= 0) continue;
        const double ws = ncl[ci] * cell_bytes;
        const double score = (double)ncl[ci] * cls[ci] * std::min(1.0, 96.0e6 / ws);
        if (score > best_score * 1.02) {
            best_score = score;
            best_cl = cls[ci];
            best_nc = ncl[ci];
        }
        if (getenv("DVM_VERBOSE"))
            fprintf(stderr, "[dvm]   cluster %2d: %3d clusters, score %.1f\n", cls[ci], ncl[ci], score);
    }
    if (getenv("DVM_VERBOSE"))
        fprintf(stderr, "[dvm] cluster3d N=%d: cluster=%d active_clusters=%d (max co-resident CTAs %d)\n", N,
                best_cl, best_nc, max_ctas);
    if (best_cl == 0) {
        *handled = false;
        return DVM_OK;
    }
    const int nloc = (int)P->local.size();
    const int64_t nodes = (int64_t)N * N * N;
    int nchunks = 1;
    if (ncells < best_nc) nchunks = (int)std::min<int64_t>(nloc, (best_nc + ncells - 1) / ncells);
    const int64_t items = ncells * nchunks;
    const int nclusters = (int)std::min<int64_t>(best_nc, items);
    Workspace &w = P->ws;
    const size_t need_T = (size_t)nclusters * nodes;
    const size_t need_part = nchunks > 1 ? (size_t)nchunks * ncells * nodes : 0;
    if (w.c3_T_elems < need_T || w.c3_part_elems < need_part) {
        DVM_CUDA(cudaStreamSynchronize(P->stream));
        if (w.c3_T) cudaFree(w.c3_T);
        if (w.c3_part) cudaFree(w.c3_part);
        w.c3_T = w.c3_part = nullptr;
        w.c3_T_elems = w.c3_part_elems = 0;
        if (cudaMalloc(&w.c3_T, sizeof(double) * need_T) != cudaSuccess ||
            (need_part && cudaMalloc(&w.c3_part, sizeof(double) * need_part) != cudaSuccess)) {
            set_error("cluster workspace allocation failed");
            return DVM_E_NOMEM;
        }
        w.c3_T_elems = need_T;
        w.c3_part_elems = need_part;
    }
    C3Args a;
    a.f = f;
    a.f_stride = f_stride;
    a.Q = nchunks == 1 ? Q : w.c3_part;
    a.q_stride = nchunks == 1 ? q_stride : nodes;
    a.Tbuf = w.c3_T;
    a.ncells = ncells;
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
    int nseg = 1;
    while (nseg * 2 <= best_cl * kCT / (N * N) && N / (nseg * 2) >= 8) nseg *= 2;
    a.nseg = nseg;
    a.seg_len = N / nseg;
    a.dbg = getenv("DVM_C3_DEBUG") ? atoi(getenv("DVM_C3_DEBUG")) : 0;
    // zero the accumulation target
    if (nchunks == 1) {
        dvm_status_t st = zero_cells(P, Q, q_stride, ncells, nodes);
        if (st) return st;
    } else {
        dvm_status_t st = zero_cells(P, w.c3_part, nodes, (int64_t)nchunks * ncells, nodes);
        if (st) return st;
    }
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
    {
        LaunchScope ls(P, KC_CLUSTER3D);
        DVM_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    }
    if (nchunks > 1) {
        dvm_status_t st = zero_cells(P, Q, q_stride, ncells, nodes);
        if (st) return st;
        st = reduce_slots(P, Q, q_stride, w.c3_part, (int64_t)ncells * nodes, nchunks, ncells, nodes);
        if (st) return st;
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
        if (P->h_nrows[i] > kMaxRows) return DVM_OK;
    const int hl = P->N >= 128 ? 32 : P->N / 2;
    if (P->h_row_extent < 0 || P->h_row_extent > hl) return DVM_OK;
    switch (P->N) {
    case 32: return launch<32>(P, f, f_stride, Q, q_stride, ncells, handled);
    case 64: return launch<64>(P, f, f_stride, Q, q_stride, ncells, handled);
    case 128: return launch<128>(P, f, f_stride, Q, q_stride, ncells, handled);
    default: return DVM_OK;
    }
}

}  // namespace dvm
