// dvm_gain3d.cu -- 3D evaluation of Q = D^{Ñ,N̄}(f,f) on B200 (sm_100a, fp64).
//
// The operator (eq:decD) splits into gain and loss:
//   Q = G − f Λ,   G = Σ_e a_e S_e T_e,   Λ = Σ_e a_e Σ_{m≠0} T_e(.+me) = λ ⊛ f
// with the fixed kernel λ(j) = Σ_e a_e #{(m, l) : 1<=|m|<=M_e, l ∈ P_e,
// me + l ≡ j (mod N)} (β̃ = β − β(L,L); the loss is the
// β(L,L) convolution the paper evaluates spectrally).
//
//   loss  Λ: one batched 3D FFT convolution per pair of cells (f_{2p} + i
//        f_{2p+1} packed; λ̂ is real because λ is even), hand-written radix-2
//        passes in shared memory; the last inverse pass writes Q := −f Λ.
//   gain  G: a persistent cooperative kernel; a group of CL CTAs owns one cell
//        at a time and walks the directions.  Per direction:
//          phase A (frame): each CTA takes pairs of lattice planes x.e = γ,
//            gathers them in 16-byte runs {x, x + ê_2}, builds in-row prefix
//            sums in shared memory and evaluates T_e by the sliding program of
//            dvm_frame.h; T_e is written back in storage order (L2-resident
//            ping-pong buffer of the group).
//          group barrier
//          phase B (storage order): every CTA owns a fixed slab of nodes and
//            accumulates Q += a_e T_e S_e, S_e = Σ_{1<=|m|<=M_e} f(.+me)
//            read as coalesced stencil taps.
// Q accumulates in direction order per node: bitwise deterministic.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "dvm_frame.h"
#include "dvm_g3common.h"
#include "dvm_internal.h"

namespace dvm {
namespace {
using namespace g3;

constexpr int kMaxRec = 72;     // int4 words of a direction record (6 meta + program entries)
constexpr int kMaxMS = 32;      // line half-width M_e held in shared memory

// ------------------------------------------------------------------ gain
struct GainArgs {
    const double2 *f;   // [pairs][nodes]: cells 2p, 2p+1 interleaved
    double2 *Q;         // [nchunks][pairs][nodes] interleaved accumulators (chunk 0 holds −fΛ)
    int64_t npairs;
    int nchunks;
    int nloc;
    const int4 *rec;    // [nloc][recw]: 24 ints of frame metadata, then the program entries
    int recw;
    const double *aw;   // [nloc]
    double2 *Tbuf;      // [groups][kSlots][nodes]
    unsigned int *ctr;  // [groups][2][kCL]: steps completed by each CTA's phase A / phase B
    uint32_t H;
};

constexpr int kSlots = 2;   // T ring depth per group (phase A may run kSlots-1 steps ahead)



// Shared-memory geometry (one lattice plane of a cell pair at a time).  Rows
// are padded to RS = N + 1 double2 (a thread-per-row scan is then bank-conflict
// free) and planes keep L extra rows (row N + k == row k) so a thread's L
// consecutive β-steps address rows r0 .. r0 + L - 1 without wrap logic.  The
// raw plane is double-buffered: the next plane is gathered by cp.async while
// the current one is scanned and evaluated.
template <int N, int CL = kCL>
struct G3Geom {
    static constexpr int LOGN = N == 32 ? 5 : 6;
    static constexpr int SEGS = kRoleT / N;              // β segments per column
    static constexpr int SEGLEN = N / SEGS;              // rows per segment
    static constexpr int L = SEGLEN < 8 ? SEGLEN : 8;    // rows per register chunk
    static constexpr int NCH = SEGLEN / L;
    static constexpr int ROWS = N + L;
    static constexpr int RS = N + 1;
    static constexpr int PL = ROWS * RS;
    static constexpr int NPL = N / CL;                   // planes per CTA per direction
    static constexpr size_t smem = sizeof(double2) * (3 * (size_t)PL + ROWS) + sizeof(int4) * 2 * kMaxRec +
                                   sizeof(uint32_t) * 2 * kMaxMS;
};


// Gather lattice plane g (frame z, u, w) of a cell pair into dst[ROWS][RS]
// (rows < L also into their duplicate rows) with 16-byte cp.async requests.
template <int N>
__device__ __forceinline__ void gather_plane(const double2 *fcp, double2 *dst, int g, const int *zuw, int t,
                                             uint32_t H2)
{
    using Gm = G3Geom<N>;
    constexpr int DB = kRoleT / N;  // rows advanced per pass
    const int al = t & (N - 1);
    int be = t >> Gm::LOGN;
    const int z0 = zuw[0], z1 = zuw[1], z2 = zuw[2], u0 = zuw[3], u1 = zuw[4], u2 = zuw[5];
    const int w0 = zuw[6], w1 = zuw[7], w2 = zuw[8];
    uint32_t x = pk<N>(g * z0 + al * u0 + be * w0, g * z1 + al * u1 + be * w1, g * z2 + al * u2 + be * w2);
    const uint32_t sx = pk<N>(DB * w0, DB * w1, DB * w2);
#pragma unroll 4
    for (int k = 0; k < N / DB; ++k) {
        cp_async16(dst + be * Gm::RS + al, fcp + x);
        if (be < Gm::L) cp_async16(dst + (be + N) * Gm::RS + al, fcp + x);
        be += DB;
        x = swar_add(x, sx, H2);
    }
    cp_async_commit();
}

template <int N, int CL>
__global__ void __launch_bounds__(2 * kRoleT, 1) k_gain3d(GainArgs A)
{
    using Gm = G3Geom<N, CL>;
    constexpr int LOGN = Gm::LOGN;
    constexpr int64_t NODES = (int64_t)N * N * N;
    constexpr int SEGLEN = Gm::SEGLEN;
    constexpr int L = Gm::L;
    constexpr int NCH = Gm::NCH;
    constexpr int NPR = (int)(NODES / CL);  // phase-B nodes per CTA
    static_assert(4 * (NPR / kRoleT) <= 256, "phase-B accumulators exceed the thread's 256 TMEM columns");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int RS = Gm::RS;
    constexpr int NPL = Gm::NPL;
    double2 *rawb = reinterpret_cast<double2 *>(smem_raw);  // [2][ROWS][RS] gathered planes
    double2 *pre = rawb + 2 * Gm::PL;                        // [ROWS][RS] in-row prefix sums
    double2 *tot = pre + Gm::PL;                             // [ROWS] row totals
    int4 *srec = reinterpret_cast<int4 *>(tot + Gm::ROWS);  // [2][kMaxRec] double-buffered direction records
    uint32_t *soff = reinterpret_cast<uint32_t *>(srec + 2 * kMaxRec);  // [2 * kMaxMS] (phase B)
    __shared__ int smB[4];

    const bool roleA = threadIdx.x < kRoleT;
    const int t = threadIdx.x & (kRoleT - 1);
    const int lane = t & 31, warp = t >> 5;
    const bool leader = t == 0;
    const int bar = roleA ? 1 : 2;
    const int rank = (int)(blockIdx.x % CL);
    const int grp = (int)(blockIdx.x / CL);
    const int ngroups = (int)(gridDim.x / CL);
    const uint32_t H2 = A.H;
    unsigned int *cA = A.ctr + (size_t)grp * 2 * CL, *cB = cA + CL;
    unsigned int stepi = 0;
    const int64_t items = A.npairs * A.nchunks;

    // TMEM: the B role's first warp allocates all 512 columns (one CTA per SM)
    __shared__ uint32_t s_tmem;
    if (!roleA && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"l"(
                         (uint64_t)__cvta_generic_to_shared(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (!roleA) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        role_sync(2);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // lane = 32 (warp % 4) + lane, columns: warps 8-11 -> [0, 256), 12-15 -> [256, 512)
    const uint32_t tm_base = roleA ? 0u : (s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * (warp >> 2)));

    // direction records are double-buffered: the record of step s+1 is fetched
    // into registers while step s runs and stored into the other buffer at its end
    const int recw = A.recw;
    int buf = 0;
    int4 rnext = make_int4(0, 0, 0, 0);
    int4 bnext0 = make_int4(0, 0, 0, 0), bnext3 = make_int4(0, 0, 0, 0);
    int cur = 0;  // raw plane buffer holding the next plane to evaluate
    if (grp < items) {
        const int first_di = (int)((int64_t)A.nloc * (grp % A.nchunks) / A.nchunks);
        if (roleA) {
            for (int k = t; k < recw; k += kRoleT) srec[k] = A.rec[(int64_t)first_di * recw + k];
            role_sync(bar);
            // first plane of the first step
            gather_plane<N>(A.f + (grp / A.nchunks) * NODES, rawb, rank, reinterpret_cast<const int *>(srec) + 3, t,
                            H2);
        } else if (t == 0) {
            bnext0 = A.rec[(int64_t)first_di * recw];
            bnext3 = A.rec[(int64_t)first_di * recw + 3];
        }
        role_sync(bar);
    }

    for (int64_t item = grp; item < items; item += ngroups) {
        const int64_t pair = item / A.nchunks;
        const int chunk = (int)(item % A.nchunks);
        const int d0 = (int)((int64_t)A.nloc * chunk / A.nchunks);
        const int d1 = (int)((int64_t)A.nloc * (chunk + 1) / A.nchunks);
        const double2 *__restrict__ fc = A.f + pair * NODES;
        double2 *Qc = A.Q + ((int64_t)chunk * A.npairs + pair) * NODES;

        for (int di = d0; di < d1; ++di, ++stepi) {
            double2 *Tb = A.Tbuf + ((int64_t)grp * kSlots + (stepi % kSlots)) * NODES;
            int ndi = -1;  // the direction of this group's next step
            if (di + 1 < d1) {
                ndi = di + 1;
            } else if (item + ngroups < items) {
                const int nch = (int)((item + ngroups) % A.nchunks);
                ndi = (int)((int64_t)A.nloc * nch / A.nchunks);
            }
            if (roleA) {
                // ============================================ phase A: T_e -> slot
                if (ndi >= 0 && t < recw) rnext = A.rec[(int64_t)ndi * recw + t];
                if (stepi >= kSlots) role_wait<CL>(cB, stepi - kSlots + 1, t, bar);
                const int *smA = reinterpret_cast<const int *>(srec + buf * kMaxRec);
                const int4 *sprog = srec + buf * kMaxRec + 6;
                const int z0 = smA[3], z1 = smA[4], z2 = smA[5];
                const int u0 = smA[6], u1 = smA[7], u2 = smA[8];
                const int w0 = smA[9], w1 = smA[10], w2 = smA[11];
                const int ninit = smA[16], nstep = smA[17], nraw = smA[19];
                const uint32_t SW = pk<N>(w0, w1, w2);
                const int tal = t & (N - 1);
                const int tbe = (t >> LOGN) * SEGLEN;
                // cell pair of the next step (prefetch target of the last plane)
                const double2 *fnext = (di + 1 < d1) ? fc : A.f + ((item + ngroups) / A.nchunks) * NODES;
#pragma unroll 1
                for (int kp = 0; kp < NPL; ++kp) {
                    const int g = rank + kp * CL;
                    cp_async_wait_all();
                    role_sync(bar);  // plane g is in rawb[cur] (and the next record is visible)
                    if (kp + 1 < NPL)
                        gather_plane<N>(fc, rawb + (cur ^ 1) * Gm::PL, g + CL, smA + 3, t, H2);
                    else if (ndi >= 0)
                        gather_plane<N>(fnext, rawb + (cur ^ 1) * Gm::PL, rank,
                                        reinterpret_cast<const int *>(srec + (buf ^ 1) * kMaxRec) + 3, t, H2);
                    const double2 *raw = rawb + cur * Gm::PL;
                    // A2: in-row prefix sums.  Warp w scans rows 8w .. 8w+7 (N = 64) in four
                    // 16-column quarters: lanes 8q + i take row 8w + i, quarter q, so each
                    // quarter-warp reads 8 consecutive padded rows (conflict free); the
                    // quarter totals are combined with shuffles across lanes i, i+8, ...
                    {
                        constexpr int QN = 32 / 8;          // quarters per row (lanes per row)
                        constexpr int QL = N / QN;          // columns per quarter
                        constexpr int RPWARP = 8;           // rows per warp
                        for (int rb = warp * RPWARP; rb < N; rb += (kRoleT / 32) * RPWARP) {
                            const int row = rb + (lane & 7), qd = lane >> 3;
                            const double2 *rr = raw + row * RS + qd * QL;
                            double2 v[QL];
#pragma unroll
                            for (int c = 0; c < QL; ++c) v[c] = rr[c];
#pragma unroll
                            for (int c = 1; c < QL; ++c) v[c] = add2(v[c], v[c - 1]);
                            // exclusive prefix of the quarter totals over qd = 0..3 (lanes i + 8 qd)
                            double2 x = v[QL - 1];
#pragma unroll
                            for (int o = 8; o < 32; o <<= 1) {
                                const double yx = __shfl_up_sync(0xffffffffu, x.x, o);
                                const double yy = __shfl_up_sync(0xffffffffu, x.y, o);
                                if (lane >= o) {
                                    x.x += yx;
                                    x.y += yy;
                                }
                            }
                            const double2 excl = sub2(x, v[QL - 1]);
                            double2 *pp = pre + row * RS + qd * QL;
#pragma unroll
                            for (int c = 0; c < QL; ++c) {
                                const double2 o2 = add2(v[c], excl);
                                pp[c] = o2;
                                if (row < L) pp[N * RS + c] = o2;
                            }
                            if (qd == QN - 1) {
                                tot[row] = x;
                                if (row < L) tot[row + N] = x;
                            }
                        }
                    }
                    role_sync(bar);
                    // A3: T by the sliding program (thread = column, β segment),
                    // stored straight from registers (16 bytes per node)
                    {
                        const int al = tal;
                        uint32_t x = pk<N>(g * z0 + al * u0 + tbe * w0, g * z1 + al * u1 + tbe * w1,
                                           g * z2 + al * u2 + tbe * w2);
                        double2 carry = make_double2(0.0, 0.0);
#pragma unroll 1
                        for (int c = 0; c < NCH; ++c) {
                            const int be0 = tbe + c * L;
                            double2 T[L + 1];
                            if (c == 0) {
                                double2 acc = make_double2(0.0, 0.0);
                                for (int k = 0; k < ninit; ++k) {
                                    const int4 en = sprog[k];
                                    const int r0 = (be0 + en.x) & (N - 1);
                                    const int b = al + en.z, a = al + en.y - 1;
                                    double2 v = sub2(pre[r0 * RS + (b & (N - 1))], pre[r0 * RS + (a & (N - 1))]);
                                    if ((b >> LOGN) != (a >> LOGN)) v = add2(v, tot[r0]);
                                    acc = add2(acc, v);
                                }
                                T[0] = acc;
                            } else {
                                T[0] = carry;
                            }
#pragma unroll
                            for (int q = 1; q <= L; ++q) T[q] = make_double2(0.0, 0.0);
                            // single-node entries (host-sorted first), then row ranges
#pragma unroll 2
                            for (int k = ninit; k < ninit + nraw; ++k) {
                                const int4 en = sprog[k];
                                const int r0 = (be0 + en.x) & (N - 1);
                                const double sgn = (double)en.w;
                                const double2 *q0 = raw + r0 * RS + ((al + en.y) & (N - 1));
#pragma unroll
                                for (int q = 1; q <= L; ++q) T[q] = fma2(sgn, q0[(q - 1) * RS], T[q]);
                            }
#pragma unroll 2
                            for (int k = ninit + nraw; k < ninit + nstep; ++k) {
                                const int4 en = sprog[k];
                                const int r0 = (be0 + en.x) & (N - 1);
                                const double sgn = (double)en.w;
                                const int b = al + en.z, a = al + en.y - 1;
                                const double2 *qb = pre + r0 * RS + (b & (N - 1));
                                const double2 *qa = pre + r0 * RS + (a & (N - 1));
                                const double2 *qt = tot + r0;
                                const double wr = (b >> LOGN) != (a >> LOGN) ? 1.0 : 0.0;  // periodic wrap
#pragma unroll
                                for (int q = 1; q <= L; ++q) {
                                    const double2 d = sub2(qb[(q - 1) * RS], qa[(q - 1) * RS]);
                                    const double2 tq = qt[q - 1];
                                    T[q] = fma2(sgn, make_double2(fma(wr, tq.x, d.x), fma(wr, tq.y, d.y)), T[q]);
                                }
                            }
#pragma unroll
                            for (int q = 1; q <= L; ++q) T[q] = add2(T[q], T[q - 1]);
#pragma unroll
                            for (int q = 0; q < L; ++q) {
                                st2_hint(Tb + x, T[q], l2_keep());
                                x = swar_add(x, SW, H2);
                            }
                            carry = T[L];
                        }
                    }
                    if (kp == 0 && ndi >= 0 && t < recw) srec[(buf ^ 1) * kMaxRec + t] = rnext;
                    role_sync(bar);  // rawb[cur] and pre are free again
                    cur ^= 1;
                }
                buf ^= 1;
                role_signal(cA + rank, stepi + 1, leader, bar);
            } else {
                // ============================================ phase B: Q += a_e T_e S_e
                if (t == 0) {
                    smB[0] = bnext0.x;
                    smB[1] = bnext0.y;
                    smB[2] = bnext0.z;
                    smB[3] = bnext3.w;  // M_e
                    if (ndi >= 0) {
                        bnext0 = A.rec[(int64_t)ndi * recw];
                        bnext3 = A.rec[(int64_t)ndi * recw + 3];
                    }
                }
                role_wait<CL>(cA, stepi + 1, t, bar);
                const int M = smB[3];
                if (t < 2 * M) {
                    const int m = t / 2 + 1, sg = (t & 1) ? -1 : 1;
                    soff[t] = pk<N>(sg * m * smB[0], sg * m * smB[1], sg * m * smB[2]);
                }
                role_sync(bar);
                {
                    // thread-owned nodes n0 + t + 256 j (j < NPR/256), accumulated in TMEM:
                    // 4 nodes (8 doubles, 16 columns) per batch
                    constexpr int NB = 4;
                    constexpr int NJ = NPR / kRoleT;
                    static_assert(NJ % NB == 0, "phase-B tiling");
                    const bool first = di == d0, last = di == d1 - 1;
                    const double aw = A.aw[di];
                    const int M2 = 2 * M;
                    const uint32_t n0 = (uint32_t)rank * NPR + t;
                    const uint64_t keep = l2_keep();
#pragma unroll 1
                    for (int j0 = 0; j0 < NJ; j0 += NB) {
                        uint32_t n[NB];
                        double2 T[NB], S[NB];
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            n[b] = n0 + (uint32_t)(j0 + b) * kRoleT;
                            T[b] = ld2_cg_hint(Tb + n[b], l2_drop());
                            S[b] = make_double2(0.0, 0.0);
                        }
                        for (int k = 0; k < M2; ++k) {
                            const uint32_t off = soff[k];
#pragma unroll
                            for (int b = 0; b < NB; ++b) S[b] = add2(S[b], ld2_nc_hint(fc + swar_add(n[b], off, H2), keep));
                        }
                        uint32_t r[16];
                        const uint32_t ta = tm_base + (uint32_t)(4 * j0);
                        if (first) {
#pragma unroll
                            for (int b = 0; b < NB; ++b) {
                                const double2 q = ld2_cg_hint(Qc + n[b], l2_drop());  // −fΛ (chunk 0) or 0
                                r[4 * b + 0] = __double2loint(q.x);
                                r[4 * b + 1] = __double2hiint(q.x);
                                r[4 * b + 2] = __double2loint(q.y);
                                r[4 * b + 3] = __double2hiint(q.y);
                            }
                        } else {
                            tmem_ld16(ta, r);
                        }
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            double qx = __hiloint2double(r[4 * b + 1], r[4 * b + 0]);
                            double qy = __hiloint2double(r[4 * b + 3], r[4 * b + 2]);
                            qx += aw * T[b].x * S[b].x;
                            qy += aw * T[b].y * S[b].y;
                            if (last) {
                                st2_hint(Qc + n[b], make_double2(qx, qy), l2_drop());
                            } else {
                                r[4 * b + 0] = __double2loint(qx);
                                r[4 * b + 1] = __double2hiint(qx);
                                r[4 * b + 2] = __double2loint(qy);
                                r[4 * b + 3] = __double2hiint(qy);
                            }
                        }
                        if (!last) tmem_st16(ta, r);
                    }
                    tmem_wait_st();
                }
                role_signal(cB + rank, stepi + 1, leader, bar);
            }
        }
    }
    if (!roleA) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        role_sync(2);
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
    }
}

// f [cells][stride] -> fI [pairs][nodes] (double2), odd tail padded with 0
__global__ void k_interleave(const double *__restrict__ f, int64_t stride, int64_t ncells, int64_t nodes,
                             double2 *__restrict__ fI)
{
    const int64_t npairs = (ncells + 1) / 2;
    const int64_t total = npairs * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / nodes, x = i % nodes;
        const int64_t c0 = 2 * p, c1 = c0 + 1;
        fI[i] = make_double2(f[c0 * stride + x], c1 < ncells ? f[c1 * stride + x] : 0.0);
    }
}

// Q[cell] = Σ_chunks QI[chunk][pair][.] component (chunk order: deterministic)
__global__ void k_deinterleave(const double2 *__restrict__ QI, int nchunks, int64_t npairs, int64_t ncells,
                               int64_t nodes, double *__restrict__ Q, int64_t stride)
{
    const int64_t total = ncells * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / nodes, x = i % nodes;
        const int64_t p = c / 2;
        const bool hi = c & 1;
        double acc = 0.0;
        for (int k = 0; k < nchunks; ++k) {
            const double2 v = QI[((int64_t)k * npairs + p) * nodes + x];
            acc += hi ? v.y : v.x;
        }
        Q[c * stride + x] = acc;
    }
}

size_t gain_smem_bytes(int N) { return N == 32 ? G3Geom<32>::smem : G3Geom<64>::smem; }


template <int N>
dvm_status_t launch_gain(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                         int64_t ncells, bool *fallback)
{
    *fallback = false;
    // CTAs per group: 16 (N = 64); N = 32 defaults to groups of 8 (more groups walk the
    // directions in parallel; measured on c4), dvm_set_tuning("g3_cl") overrides
    int CL = N == 32 ? 8 : 16;
    if (N == 32 && P->tune.g3_cl) CL = P->tune.g3_cl;
    auto kern = CL == 16 ? k_gain3d<N, 16> : CL == 8 ? k_gain3d<N, (N == 32 ? 8 : 16)> : k_gain3d<N, (N == 32 ? 4 : 16)>;
    const size_t smem = gain_smem_bytes(N);
    DVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    DVM_CUDA(cudaGetDevice(&dev));
    DVM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DVM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    DVM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 2 * kRoleT, smem));
    if (!coop || per_sm < 1) {  // no cooperative launch here: the v1 sweeps evaluate
        *fallback = true;
        return DVM_OK;
    }
    // every CTA allocates all 512 TMEM columns: one CTA per SM, whatever the occupancy
    // calculator would allow (a second resident CTA would block in tcgen05.alloc)
    per_sm = 1;
    int max_groups = (sms * per_sm) / CL;
    if (P->tune.max_groups) max_groups = std::max(1, std::min(max_groups, P->tune.max_groups));
    const int nloc = (int)P->local.size();
    const int64_t nodes = (int64_t)N * N * N;
    const int64_t npairs = (ncells + 1) / 2;
    int nchunks = 1;
    if (npairs < max_groups) nchunks = (int)std::min<int64_t>(std::max(1, nloc), max_groups / npairs);
    nchunks = std::max(1, nchunks);
    const int64_t items = npairs * nchunks;
    const int ngroups = (int)std::min<int64_t>(max_groups, items);
    Workspace &w = P->ws;
    dvm_status_t st;
    if ((st = grow(&w.g3_f, &w.g3_f_elems, (size_t)(npairs * nodes), P->stream))) return st;
    if ((st = grow(&w.g3_q, &w.g3_q_elems, (size_t)(nchunks * npairs * nodes), P->stream))) return st;
    if ((st = grow(&w.g3_t, &w.g3_t_elems, (size_t)ngroups * kSlots * nodes, P->stream))) return st;
    if ((st = grow(&w.g3_ctr, &w.g3_ctr_elems, (size_t)ngroups * 2 * CL, P->stream))) return st;
    {
        LaunchScope ls(P, KC_ZERO);
        k_interleave<<<1184, 256, 0, P->stream>>>(f, f_stride, ncells, nodes, w.g3_f);
        DVM_CUDA(cudaGetLastError());
    }
    if (nchunks > 1)
        DVM_CUDA(cudaMemsetAsync(w.g3_q + npairs * nodes, 0, sizeof(double2) * (size_t)((nchunks - 1) * npairs * nodes),
                                 P->stream));
    // loss first: chunk 0 := −f Λ (interleaved)
    if ((st = loss_init(P, f, f_stride, nullptr, 0, ncells, w.g3_q))) return st;
    DVM_CUDA(cudaMemsetAsync(w.g3_ctr, 0, sizeof(unsigned int) * 2 * CL * ngroups, P->stream));
    GainArgs a;
    a.f = w.g3_f;
    a.Q = w.g3_q;
    a.npairs = npairs;
    a.nchunks = nchunks;
    a.nloc = nloc;
    a.rec = P->g.rec;
    a.recw = P->g.recw;
    a.aw = P->g.aw;
    a.Tbuf = w.g3_t;
    a.ctr = w.g3_ctr;
    a.H = P->pk.H;
    if (P->tune.verbose)
        fprintf(stderr, "[dvm] gain3d N=%d: %d groups x %d CTAs, %d chunks, smem %zu\n", N, ngroups, CL, nchunks,
                smem);
    {
        void *args[] = {&a};
        LaunchScope ls(P, KC_GAIN3D);
        const cudaError_t le =
            cudaLaunchCooperativeKernel((void *)kern, dim3(ngroups * CL), dim3(2 * kRoleT), args, smem, P->stream);
        if (le == cudaErrorCooperativeLaunchTooLarge || le == cudaErrorNotSupported) {
            // the co-residency the group barriers need is not available now (e.g.
            // SMs held by another context): evaluate with the v1 sweeps instead
            cudaGetLastError();
            *fallback = true;
            return DVM_OK;
        }
        if (le != cudaSuccess) return cuda_fail(le, "cudaLaunchCooperativeKernel(k_gain3d)");
    }
    {
        LaunchScope ls(P, KC_REDUCE);
        k_deinterleave<<<1184, 256, 0, P->stream>>>(w.g3_q, nchunks, npairs, ncells, nodes, Q, q_stride);
        DVM_CUDA(cudaGetLastError());
    }
    return DVM_OK;
}

}  // namespace

// Plan-time setup of the 3D path: frames + programs of the local directions,
// twiddles, the loss kernel λ and its spectrum λ̂.
dvm_status_t build_gain3d(dvm_plan_s *P)
{
    if (P->d != 3 || (P->N != 32 && P->N != 64)) return DVM_OK;
    // line half-widths beyond the kernels' tap tables (Ñ > 16): no 3D fast path for this
    // plan; the orbit sweeps (v1) and the spectral path evaluate it
    for (int di : P->local)
        if (P->h_M[di] > kMaxMS / 2) return DVM_OK;
    const int nloc = (int)P->local.size();
    const int N = P->N;
    const int L = N == 32 ? G3Geom<32>::SEGLEN : G3Geom<64>::SEGLEN;
    std::vector<frame::DirFrame> frames(nloc);
    std::vector<double> aw(std::max(1, nloc), 0.0);
    int maxent = 0;
    for (int k = 0; k < nloc; ++k) {
        const int di = P->local[k];
        frame::DirFrame &F = frames[k];
        if (!frame::build_dir(&P->h_e[3 * di], P->Ntilde, N, L, F)) {
            set_error("gain3d: no frame for a direction");
            return DVM_E_UNSUPPORTED;
        }
        maxent = std::max(maxent, (int)(F.init.size() + F.step.size()));
        if (F.M > kMaxMS / 2) {
            set_error("gain3d: line half-width exceeds the shared-memory table");
            return DVM_E_UNSUPPORTED;
        }
        aw[k] = P->h_a[di];
    }
    // fixed-size direction records: 6 int4 of metadata + program entries
    const int recw = 6 + maxent;
    if (recw > kMaxRec) {
        set_error("gain3d: direction program exceeds the shared-memory record");
        return DVM_E_UNSUPPORTED;
    }
    std::vector<int4> rec((size_t)std::max(1, nloc) * recw, make_int4(0, 0, 0, 0));
    for (int k = 0; k < nloc; ++k) {
        const frame::DirFrame &F = frames[k];
        int m[24] = {0};
        for (int j = 0; j < 3; ++j) {
            m[j] = F.e[j];
            m[3 + j] = F.z[j];
            m[6 + j] = F.u[j];
            m[9 + j] = F.w[j];
        }
        m[12] = F.a2;
        m[13] = F.b2;
        m[14] = F.rows_mode;
        m[15] = F.M;
        m[16] = (int)F.init.size();
        m[17] = (int)F.step.size();
        int nraw = 0;
        for (const auto &x : F.step) nraw += x.t1 == x.t2;
        m[19] = nraw;
        int4 *r = &rec[(size_t)k * recw];
        for (int q = 0; q < 6; ++q) r[q] = make_int4(m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
        int q = 6;
        for (const auto &x : F.init) r[q++] = make_int4(x.rho, x.t1, x.t2, x.sign);
        // step entries: single nodes first, then row ranges (two branch-free loops)
        for (const auto &x : F.step)
            if (x.t1 == x.t2) r[q++] = make_int4(x.rho, x.t1, x.t2, x.sign);
        for (const auto &x : F.step)
            if (x.t1 != x.t2) r[q++] = make_int4(x.rho, x.t1, x.t2, x.sign);
    }
    GainTables &g = P->g;
    g.recw = recw;
    DVM_CUDA(cudaMalloc(&g.rec, sizeof(int4) * rec.size()));
    DVM_CUDA(cudaMalloc(&g.aw, sizeof(double) * aw.size()));
    g.bytes = sizeof(int4) * rec.size() + sizeof(double) * aw.size();
    DVM_CUDA(cudaMemcpyAsync(g.rec, rec.data(), sizeof(int4) * rec.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(g.aw, aw.data(), sizeof(double) * aw.size(), cudaMemcpyHostToDevice, P->stream));
    const dvm_status_t st = build_loss(P);
    if (st) return st;
    g.ready = true;
    return DVM_OK;
}

void free_gain3d(dvm_plan_s *P)
{
    GainTables &g = P->g;
    void *ptrs[] = {g.rec, g.aw, g.tw, g.lamhat, g.units, g.shat, g.that, g.fg_rec, g.fg_aw, g.fg_t2d,
                    g.f32_rec, g.f32_off, g.f32_aw, g.f32_t2d};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    g = GainTables{};
}

dvm_status_t interleave_pairs(dvm_plan_s *P, const double *f, int64_t f_stride, int64_t ncells, int64_t nodes,
                              double2 *fI)
{
    LaunchScope ls(P, KC_ZERO);
    k_interleave<<<1184, 256, 0, P->stream>>>(f, f_stride, ncells, nodes, fI);
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t deinterleave_pairs(dvm_plan_s *P, const double2 *QI, int nchunks, int64_t npairs, int64_t ncells,
                                int64_t nodes, double *Q, int64_t q_stride)
{
    LaunchScope ls(P, KC_REDUCE);
    k_deinterleave<<<1184, 256, 0, P->stream>>>(QI, nchunks, npairs, ncells, nodes, Q, q_stride);
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t collide_gain3d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                            int64_t ncells, bool *handled)
{
    *handled = false;
    if (P->d != 3 || !P->g.ready || ncells <= 0) return DVM_OK;
    *handled = true;
    switch (P->N) {
    case 32: {
        bool fb = false;
        const dvm_status_t st = launch_gain<32>(P, f, f_stride, Q, q_stride, ncells, &fb);
        *handled = !fb;
        return st;
    }
    case 64: {
        bool fb = false;
        const dvm_status_t st = launch_gain<64>(P, f, f_stride, Q, q_stride, ncells, &fb);
        *handled = !fb;
        return st;
    }
    default: *handled = false; return DVM_OK;
    }
}

}  // namespace dvm
