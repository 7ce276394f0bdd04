// dvm_fgain3d.cu -- 3D gain G = Σ_e a_e S_e T_e by per-direction FFT
// filtering (sm_100a, fp64; N = 64).
//
// The perp sums are the periodic convolution T_e = f ⊛ 1_{P_e}; their filter
// is even, so its spectrum is real and two cells share one complex transform:
//   T_{2p} + i T_{2p+1} = IFFT( f̂_p · t̂_e ),   f̂_p = FFT(f_{2p} + i f_{2p+1}),
//   t̂_e(ξ) = Σ_{l ∈ P_e} cos(2π l.ξ / N) = T2D_e(u.ξ mod N, w.ξ mod N)
// with (u, w) the basis of e^⊥ ∩ Z^3 the rows of P_e are given in
// (the paper's spectral evaluation of the α'_p
// factor; only the perp factor goes through Fourier space here, S_e stays a
// line stencil).  A persistent cooperative kernel; a group of CL CTAs owns
// one cell pair at a time and walks the directions:
//   phase A (warps 0-7): CTA `rank` takes the planes ξ_x ≡ rank (mod CL):
//     cp.async the plane of f̂ into shared memory, multiply by t̂_e, inverse
//     2D FFT over (ξ_y, ξ_z) (64 = 8 × 8 four-step, one shared-memory
//     exchange per axis), write the plane to the group's ring slot.
//   group progress counters (per CTA, monotonic)
//   phase B (warps 8-15): CTA `rank` owns the rows y ∈ [4 rank, 4 rank + 4):
//     ring columns loaded straight into registers one batch ahead, inverse FFT
//     along ξ_x of its 256 columns, then Q += a_e S_e T_e with
//     S_e = Σ_{1<=|m|<=M_e} f(.+me) read as coalesced taps; Q lives in TMEM.
//   The roles run separate loops so setmaxnreg can move registers from A (88)
//   to B (168).
// Loss and the layout conversions are shared with dvm_gain3d.cu.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "dvm_g3common.h"
#include "dvm_internal.h"

namespace dvm {
namespace {
using namespace g3;

constexpr int FN = 64;           // grid points per axis (64 = 8 × 8)
constexpr int FN2 = FN * FN;
constexpr int64_t FNODES = (int64_t)FN * FN * FN;
constexpr int FRS = FN + 1;      // padded row pitch of a plane in shared memory (double2)
constexpr int FTP = FN + 1;      // padded row pitch of the T2D table (double)
constexpr int FTR = FN / 2 + 1;  // rows of T2D kept in shared memory (the table is even: T(-p,-q) = T(p,q))
constexpr int FMS = 32;          // tap table size (2 M_e <= 32)
#ifndef FG_TAPUNROLL
#define FG_TAPUNROLL 1  // 8 loads in flight per tap pair; unrolling further measured slower
#endif
constexpr int kTapUnroll = FG_TAPUNROLL;
constexpr int kRegA = 88, kRegB = 168;
#ifndef FG_TF_REGA
#define FG_TF_REGA 96
#endif
constexpr int kRegATF = FG_TF_REGA, kRegBTF = 256 - FG_TF_REGA;  // TF: A holds 8 more TMEM words  // setmaxnreg split of the 128 x 512 register file (A + B <= 256)
#ifndef FG_TAPLD
#define FG_TAPLD ld2_nc_hint
#endif

struct FgArgs {
    const double2 *fhat;  // [pairs][N^3] f̂ of the cell pairs
    const double2 *f;     // [pairs][N^3] interleaved f
    double2 *Q;           // [nchunks][pairs][N^3] interleaved accumulators (chunk 0 holds −fΛ)
    int64_t npairs;
    int nchunks, nloc;
    const int4 *rec;      // [nloc][3]
    const double *aw;     // [nloc] a_e / N^3
    const double *t2d;    // [nloc][N][N]
    double2 *ring;        // [groups][FSLOTS][N^3]
    unsigned int *ctr;    // [groups][2][CL]
    uint32_t H;
    int slots;            // ring depth per group (phase A runs up to slots-1 steps ahead)
    int dbg;              // timing experiments (DVM_FG_DEBUG): 1 skip phase-B work, 2 skip phase-A work,
                          // 4 skip the taps
};

template <bool TF>
struct FgSmemT {
    static constexpr size_t xb = sizeof(double2) * (TF ? 1 : 2) * FN * FRS;  // plane buffer(s)
    static constexpr size_t t2 = (sizeof(double) * FTR * FTP + 127) / 128 * 128;  // T2D_e of the step, rows 0..N/2
    static constexpr size_t rb = sizeof(double2) * 2 * FN * 32;   // phase-B x-FFT exchange, 2 batches
    static constexpr size_t tw = sizeof(double2) * FN;            // W_64^k (inverse sign)
    static constexpr size_t total = xb + t2 + rb + tw;
};
using FgSmem = FgSmemT<false>;

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// inverse-sign DFTs: y_k = Σ_n a_n exp(+2πi nk / n_pts), natural order in and out
__device__ __forceinline__ void idft4(double2 &a0, double2 &a1, double2 &a2, double2 &a3)
{
    const double2 t0 = add2(a0, a2), t1 = sub2(a0, a2), t2 = add2(a1, a3), d = sub2(a1, a3);
    const double2 t3 = make_double2(-d.y, d.x);  // i (a1 − a3)
    a0 = add2(t0, t2);
    a2 = sub2(t0, t2);
    a1 = add2(t1, t3);
    a3 = sub2(t1, t3);
}

__device__ __forceinline__ void idft8(double2 (&v)[8])
{
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    idft4(e0, e1, e2, e3);
    idft4(o0, o1, o2, o3);
    constexpr double c = 0.70710678118654752440;
    o1 = make_double2(c * (o1.x - o1.y), c * (o1.x + o1.y));     // × e^{iπ/4}
    o2 = make_double2(-o2.y, o2.x);                               // × i
    o3 = make_double2(-c * (o3.x + o3.y), c * (o3.x - o3.y));    // × e^{3iπ/4}
    v[0] = add2(e0, o0);
    v[4] = sub2(e0, o0);
    v[1] = add2(e1, o1);
    v[5] = sub2(e1, o1);
    v[2] = add2(e2, o2);
    v[6] = sub2(e2, o2);
    v[3] = add2(e3, o3);
    v[7] = sub2(e3, o3);
}

// position of element z of a row after the in-row four-step (z = k2 + 8 k1 is
// kept where its thread read it: 8 k2 + ((k1 + k2) & 7)); bank-conflict free
// for lanes along rows and along columns
__device__ __forceinline__ int zpos(int z) { return 8 * (z & 7) + (((z >> 3) + (z & 7)) & 7); }

__device__ __forceinline__ void cp_async16_pol(void *smem_dst, const void *gsrc, uint64_t pol)
{
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// 32 columns of this thread's TMEM lane (8 double2)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// progress counters of a group of CL CTAs (role_wait of dvm_g3common.h for CL <= 32)
template <int CL>
__device__ __forceinline__ void group_wait(const unsigned int *ctrs, unsigned int target, int t, int id)
{
    static_assert(CL <= 32, "one polling lane per CTA");
    if (t < 32) {
        bool ok = t >= CL;
        for (;;) {
            if (!ok) {
                unsigned int v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctrs + t) : "memory");
                ok = v >= target;
            }
            if (__all_sync(0xffffffffu, ok)) break;
#ifndef FG_SLEEP
#define FG_SLEEP 32
#endif
            if (FG_SLEEP) __nanosleep(FG_SLEEP);
        }
    }
    role_sync(id);
}

// TF: f̂ of the group's cell pair resident in TMEM (groups of 32 CTAs: each CTA's 2
// planes are 128 KB = TMEM columns 256-511; Q takes columns 0-255), no plane loads
template <int CL, bool TF>
__global__ void __launch_bounds__(2 * kRoleT, 1) k_fgain3d(FgArgs A)
{
    static_assert(!TF || CL == 32, "TMEM-resident f̂ needs 2 planes per CTA");
    using Sm = FgSmemT<TF>;
    constexpr int FPL = FN / CL;  // ξ_x planes per CTA per direction
    constexpr int FRY = FN / CL;  // phase-B rows y per CTA
    constexpr int NBAT = 2 * FRY; // phase-B batches (one row y, 32 columns z)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *xb = reinterpret_cast<double2 *>(smem_raw);                            // [2][FN][FRS]
    double *t2 = reinterpret_cast<double *>(smem_raw + Sm::xb);                      // [FTR][FTP]
    double2 *rb = reinterpret_cast<double2 *>(smem_raw + Sm::xb + Sm::t2);           // [2][FN][32]
    double2 *tw = rb + 2 * FN * 32;                                                  // [FN]
    __shared__ uint32_t soff[FMS];
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

    if (threadIdx.x < FN) {
        double s, c;
        sincospi(2.0 * threadIdx.x / FN, &s, &c);
        tw[threadIdx.x] = make_double2(c, s);
    }
    __shared__ uint32_t s_tmem;
    if (!roleA && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"l"(
                         (uint64_t)__cvta_generic_to_shared(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // B: Q accumulators (64 or 32 node pairs per thread); A (TF): the f̂ planes
    constexpr uint32_t QCOLS = TF ? 128 : 256;
    const uint32_t tm_lane = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    const uint32_t tm_base = roleA ? (TF ? tm_lane + 256u + 128u * (warp >> 2) : 0u) : tm_lane + QCOLS * (warp >> 2);

    // phase A loads: T2D_e (8-byte pieces into padded rows) and planes of f̂
    auto load_t2d = [&](int di) {
        const double *src = A.t2d + (int64_t)di * FN2;
        for (int i = t; i < FTR * FN; i += kRoleT) cp_async8(t2 + (i >> 6) * FTP + (i & 63), src + i);
        cp_async_commit();
    };
    auto load_plane = [&](const double2 *fh, int g, double2 *dst) {
        const double2 *src = fh + (int64_t)g * FN2;
        // f̂ streams (evict first): L2 is kept for f (taps) and the ring
        const uint64_t pol = (A.dbg & 32) ? l2_keep() : l2_drop();
        for (int i = t; i < FN2; i += kRoleT) cp_async16_pol(dst + (i >> 6) * FRS + (i & 63), src + i, pol);
        cp_async_commit();
    };
    // TF: the planes ξ_x = rank + CL kp of a pair into this thread's TMEM columns,
    // [kp][h][n2] x double2: exactly the row-pass inputs of thread (n1 = warp, r = lane + 32 h)
    auto load_fhat_tmem = [&](const double2 *fh) {
#pragma unroll 1
        for (int kp = 0; kp < 2; ++kp)
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                uint32_t r[32];
                const double2 *src = fh + (int64_t)(rank + CL * kp) * FN2 + (lane + 32 * h) * FN + warp;
#pragma unroll
                for (int n2 = 0; n2 < 8; ++n2) {
                    const double2 x = src[8 * n2];
                    r[4 * n2 + 0] = __double2loint(x.x);
                    r[4 * n2 + 1] = __double2hiint(x.x);
                    r[4 * n2 + 2] = __double2loint(x.y);
                    r[4 * n2 + 3] = __double2hiint(x.y);
                }
                __syncwarp();
                tmem_st32(tm_base + 64u * kp + 32u * h, r);
            }
        tmem_wait_st();
    };
    if (roleA && grp < items && !(A.dbg & 2)) {
        if constexpr (!TF) load_plane(A.fhat + (grp / A.nchunks) * FNODES, rank, xb);
        load_t2d((int)((int64_t)A.nloc * (grp % A.nchunks) / A.nchunks));
    }

    if (roleA) {
        // phase A fits in 88 registers; phase B takes the rest (register prefetch of the ring)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(TF ? kRegATF : kRegA));
    for (int64_t item = grp; item < items; item += ngroups) {
        const int64_t pair = item / A.nchunks;
        const int chunk = (int)(item % A.nchunks);
        const int d0 = (int)((int64_t)A.nloc * chunk / A.nchunks);
        const int d1 = (int)((int64_t)A.nloc * (chunk + 1) / A.nchunks);
        const double2 *__restrict__ fh = A.fhat + pair * FNODES;
        if constexpr (TF) {
            if (!(A.dbg & 2)) load_fhat_tmem(fh);
        }

        for (int di = d0; di < d1; ++di, ++stepi) {
            double2 *Tb = A.ring + ((int64_t)grp * A.slots + (stepi % A.slots)) * FNODES;
            // the group's next step (direction, cell pair), -1 at the end
            int ndi = -1;
            const double2 *fh_next = fh;
            if (di + 1 < d1) {
                ndi = di + 1;
            } else if (item + ngroups < items) {
                ndi = (int)((int64_t)A.nloc * ((item + ngroups) % A.nchunks) / A.nchunks);
                fh_next = A.fhat + ((item + ngroups) / A.nchunks) * FNODES;
            }
            {
                // ============================================ phase A: planes of IFFT_yz(f̂ t̂_e)
                // (T2D_e and the first plane are in flight since the previous step)
                if (stepi >= (unsigned)A.slots) group_wait<CL>(cB, stepi - A.slots + 1, t, bar);
                const int4 ru = A.rec[(int64_t)di * 3 + 1], rw = A.rec[(int64_t)di * 3 + 2];
                const uint64_t keep = l2_keep();
                int cur = 0;
#pragma unroll 1
                for (int kp = 0; kp < ((A.dbg & 2) ? 0 : FPL); ++kp) {
                    const int g = rank + kp * CL;
                    const bool lastp = kp + 1 == FPL;
                    if constexpr (TF) {
                        if (kp == 0) {
                            cp_async_wait_all();  // T2D_e of this step
                            role_sync(bar);
                        }
                    } else {
                        if (!lastp) {
                            load_plane(fh, g + CL, xb + (cur ^ 1) * FN * FRS);
                            cp_async_wait1();
                        } else {
                            cp_async_wait_all();
                        }
                        role_sync(bar);
                        // the last plane: the next step's first plane goes into the other buffer
                        if (lastp && ndi >= 0) load_plane(fh_next, rank, xb + (cur ^ 1) * FN * FRS);
                    }
                    double2 *X = xb + (TF ? 0 : cur) * FN * FRS;
                    double2 v[8];
                    // --- rows: t̂ multiply, inverse FFT along ξ_z (four-step 8 × 8)
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        const int r = lane + 32 * h;  // ξ_y
                        {
                            const int n1 = warp;
                            int pu = (ru.x * g + ru.y * r + ru.z * n1) & (FN - 1);
                            int pw = (rw.x * g + rw.y * r + rw.z * n1) & (FN - 1);
                            const int du = (8 * ru.z) & (FN - 1), dw = (8 * rw.z) & (FN - 1);
                            uint32_t fr[TF ? 32 : 1];
                            if constexpr (TF) {
                                __syncwarp();
                                tmem_ld32(tm_base + 64u * kp + 32u * h, fr);
                            }
#pragma unroll
                            for (int n2 = 0; n2 < 8; ++n2) {
                                // rows p > N/2 from the even symmetry T(p, q) = T(N - p, N - q)
                                const bool up = pu > FN / 2;
                                const int tp = up ? FN - pu : pu, tq = up ? (FN - pw) & (FN - 1) : pw;
                                const double tv = t2[tp * FTP + tq];
                                double2 x;
                                if constexpr (TF)
                                    x = make_double2(__hiloint2double(fr[4 * n2 + 1], fr[4 * n2]),
                                                     __hiloint2double(fr[4 * n2 + 3], fr[4 * n2 + 2]));
                                else
                                    x = X[r * FRS + n1 + 8 * n2];
                                v[n2] = make_double2(x.x * tv, x.y * tv);
                                pu = (pu + du) & (FN - 1);
                                pw = (pw + dw) & (FN - 1);
                            }
                            idft8(v);
#pragma unroll
                            for (int k2 = 1; k2 < 8; ++k2) v[k2] = cmul(v[k2], tw[(n1 * k2) & (FN - 1)]);
                            if constexpr (!TF) role_sync(bar);  // other warps still read the staged plane
#pragma unroll
                            for (int k2 = 0; k2 < 8; ++k2) X[r * FRS + 8 * k2 + ((n1 + k2) & 7)] = v[k2];
                        }
                        role_sync(bar);
                        {
                            const int k2 = warp;
#pragma unroll
                            for (int n1 = 0; n1 < 8; ++n1) v[n1] = X[r * FRS + 8 * k2 + ((n1 + k2) & 7)];
                            idft8(v);
#pragma unroll
                            for (int k1 = 0; k1 < 8; ++k1) X[r * FRS + 8 * k2 + ((k1 + k2) & 7)] = v[k1];
                        }
                    }
                    role_sync(bar);
                    if (lastp && ndi >= 0) load_t2d(ndi);  // t2 is free: the next direction's table
                    // --- columns: inverse FFT along ξ_y, plane -> ring slot [ξ_x][y][z]
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        const int z = lane + 32 * h;
                        const int pz = zpos(z);
                        {
                            const int n1 = warp;
#pragma unroll
                            for (int n2 = 0; n2 < 8; ++n2) v[n2] = X[(n1 + 8 * n2) * FRS + pz];
                            idft8(v);
#pragma unroll
                            for (int k2 = 1; k2 < 8; ++k2) v[k2] = cmul(v[k2], tw[(n1 * k2) & (FN - 1)]);
                            role_sync(bar);
#pragma unroll
                            for (int k2 = 0; k2 < 8; ++k2) X[(8 * k2 + ((n1 + k2) & 7)) * FRS + pz] = v[k2];
                        }
                        role_sync(bar);
                        {
                            const int k2 = warp;
#pragma unroll
                            for (int n1 = 0; n1 < 8; ++n1) v[n1] = X[(8 * k2 + ((n1 + k2) & 7)) * FRS + pz];
                            idft8(v);
                            double2 *dst = Tb + (int64_t)g * FN2 + z;
#pragma unroll
                            for (int k1 = 0; k1 < 8; ++k1) st2_hint(dst + (k2 + 8 * k1) * FN, v[k1], keep);
                        }
                    }
                    role_sync(bar);  // X is free for the next prefetch
                    cur ^= 1;
                }
                role_signal(cA + rank, stepi + 1, leader, bar);
            }
        }
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(TF ? kRegBTF : kRegB));
    for (int64_t item = grp; item < items; item += ngroups) {
        const int64_t pair = item / A.nchunks;
        const int chunk = (int)(item % A.nchunks);
        const int d0 = (int)((int64_t)A.nloc * chunk / A.nchunks);
        const int d1 = (int)((int64_t)A.nloc * (chunk + 1) / A.nchunks);
        const double2 *__restrict__ fh = A.fhat + pair * FNODES;
        const double2 *__restrict__ fc = A.f + pair * FNODES;
        double2 *Qc = A.Q + ((int64_t)chunk * A.npairs + pair) * FNODES;

        for (int di = d0; di < d1; ++di, ++stepi) {
            double2 *Tb = A.ring + ((int64_t)grp * A.slots + (stepi % A.slots)) * FNODES;
            // the group's next step (direction, cell pair), -1 at the end
            int ndi = -1;
            const double2 *fh_next = fh;
            if (di + 1 < d1) {
                ndi = di + 1;
            } else if (item + ngroups < items) {
                ndi = (int)((int64_t)A.nloc * ((item + ngroups) % A.nchunks) / A.nchunks);
                fh_next = A.fhat + ((item + ngroups) / A.nchunks) * FNODES;
            }
            {
                // ============================================ phase B: IFFT_x, Q += a_e S_e T_e
                if (t == 0) {
                    const int4 re = A.rec[(int64_t)di * 3];
                    smB[0] = re.x;
                    smB[1] = re.y;
                    smB[2] = re.z;
                    smB[3] = re.w;
                }
                group_wait<CL>(cA, stepi + 1, t, bar);
                const int M = smB[3];
                if (t < 2 * M) {
                    const int m = t / 2 + 1, sg = (t & 1) ? -1 : 1;
                    soff[t] = pk<FN>(sg * m * smB[0], sg * m * smB[1], sg * m * smB[2]);
                }
                const bool first = di == d0, last = di == d1 - 1;
                const double aw = A.aw[di];
                const int M2 = 2 * M;
                const uint64_t keep = l2_keep(), drop = l2_drop();
                // ring columns straight into registers, one batch ahead (coalesced 512 B per warp row)
                double2 pre[8];
                auto fetch = [&](int b) {
                    const int y = FRY * rank + (b >> 1), z = 32 * (b & 1) + lane;
#pragma unroll
                    for (int n2 = 0; n2 < 8; ++n2) pre[n2] = ld2_cg_hint(Tb + ((int64_t)(warp + 8 * n2) * FN + y) * FN + z, drop);
                };
                if (!(A.dbg & 1)) fetch(0);
#pragma unroll 1
                for (int b = 0; b < ((A.dbg & 1) ? 0 : NBAT); ++b) {
                    const int y = FRY * rank + (b >> 1), z = 32 * (b & 1) + lane;
                    double2 v[8];
                    // buffer of pass-1 outputs: batch b - 2 used it, every thread is past b - 1's barrier
                    double2 *R = rb + (b & 1) * FN * 32;
                    {
                        const int n1 = warp;
#pragma unroll
                        for (int n2 = 0; n2 < 8; ++n2) v[n2] = pre[n2];
                        if (b + 1 < NBAT) fetch(b + 1);
                        idft8(v);
#pragma unroll
                        for (int k2 = 1; k2 < 8; ++k2) v[k2] = cmul(v[k2], tw[(n1 * k2) & (FN - 1)]);
#pragma unroll
                        for (int k2 = 0; k2 < 8; ++k2) R[(n1 + 8 * k2) * 32 + lane] = v[k2];
                    }
                    if (!(A.dbg & 64)) {
                        // the ring lines this warp read for batch b are dead (32 lines of 128 B, one per lane)
                        __syncwarp();
                        const double2 *line = Tb + ((int64_t)(warp + 8 * (lane >> 2)) * FN + y) * FN + 32 * (b & 1) + 8 * (lane & 3);
                        asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
                    }
                    role_sync(bar);
                    const int k2 = warp;
#pragma unroll
                    for (int n1 = 0; n1 < 8; ++n1) v[n1] = R[(n1 + 8 * k2) * 32 + lane];
                    idft8(v);  // v[k1] = N^3 T_e(x = k2 + 8 k1, y, z)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        uint32_t n[4];
                        double2 S[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            n[q] = (uint32_t)((((k2 + 8 * (4 * hh + q)) * FN) + y) * FN + z);
                            S[q] = make_double2(0.0, 0.0);
                        }
                        // taps ±m e in pairs (M2 is even): 8 independent loads per iteration
#pragma unroll kTapUnroll
                        for (int k = 0; k < ((A.dbg & 4) ? 0 : M2); k += 2) {
                            const uint32_t o0 = soff[k], o1 = soff[k + 1];
                            double2 a[4], c[4];
                            // the 4 nodes differ only in x (the top field, 8 q apart): one carry-less
                            // add per tap, then plain adds modulo N^3 for the other nodes
                            const uint32_t b0 = swar_add(n[0], o0, H2), b1 = swar_add(n[0], o1, H2);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                a[q] = FG_TAPLD(fc + ((b0 + (uint32_t)q * 8u * FN2) & (uint32_t)(FNODES - 1)), keep);
                                c[q] = FG_TAPLD(fc + ((b1 + (uint32_t)q * 8u * FN2) & (uint32_t)(FNODES - 1)), keep);
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) S[q] = add2(S[q], add2(a[q], c[q]));
                        }
                        uint32_t r[16];
                        const uint32_t ta = tm_base + (uint32_t)(32 * b + 16 * hh);
                        // the TMEM load and store are unconditional (.sync.aligned: every lane must
                        // execute the same instruction; no data-dependent branch around them)
                        __syncwarp();
                        tmem_ld16(ta, r);
                        if (first) {
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const double2 qv = ld2_cg_hint(Qc + n[q], drop);
                                r[4 * q + 0] = __double2loint(qv.x);
                                r[4 * q + 1] = __double2hiint(qv.x);
                                r[4 * q + 2] = __double2loint(qv.y);
                                r[4 * q + 3] = __double2hiint(qv.y);
                            }
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const double2 T = v[4 * hh + q];
                            double qx = __hiloint2double(r[4 * q + 1], r[4 * q + 0]);
                            double qy = __hiloint2double(r[4 * q + 3], r[4 * q + 2]);
                            qx += aw * T.x * S[q].x;
                            qy += aw * T.y * S[q].y;
                            if (last) st2_hint(Qc + n[q], make_double2(qx, qy), drop);
                            r[4 * q + 0] = __double2loint(qx);
                            r[4 * q + 1] = __double2hiint(qx);
                            r[4 * q + 2] = __double2loint(qy);
                            r[4 * q + 3] = __double2hiint(qy);
                        }
                        __syncwarp();
                        tmem_st16(ta, r);
                    }
                }
                __syncwarp();
                tmem_wait_st();
                role_signal(cB + rank, stepi + 1, leader, bar);
            }
        }
    }
    }
    if (!roleA) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        role_sync(2);
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
    }
}

// T2D_e(p, q) = Σ_{(α, β) ∈ P_e} cos(2π(α p + β q) / N): one thread per (direction, p, q)
__global__ void k_fg_t2d(int N, int nloc, const int *local, const int *row_off, const int *row_b, const int *row_lo,
                         const int *row_hi, double *out)
{
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)nloc * N * N) return;
    const int k = (int)(gid / (N * N));
    const int p = (int)((gid / N) % N), q = (int)(gid % N);
    const int di = local[k];
    double acc = 0.0;
    for (int r = row_off[di]; r < row_off[di + 1]; ++r) {
        const int b = row_b[r];
        for (int a = row_lo[r]; a <= row_hi[r]; ++a) {
            const int ph = ((a * p + b * q) % N + N) % N;
            acc += cospi(2.0 * ph / N);
        }
    }
    out[gid] = acc;
}

dvm_status_t build_fg_tables(dvm_plan_s *P)
{
    GainTables &g = P->g;
    if (g.fg_rec) return DVM_OK;
    const int nloc = (int)P->local.size();
    const int A = P->A;
    std::vector<int> hu((size_t)A * 3), hw((size_t)A * 3);
    DVM_CUDA(cudaMemcpy(hu.data(), P->t.u, sizeof(int) * hu.size(), cudaMemcpyDeviceToHost));
    DVM_CUDA(cudaMemcpy(hw.data(), P->t.w, sizeof(int) * hw.size(), cudaMemcpyDeviceToHost));
    std::vector<int4> rec((size_t)std::max(1, nloc) * 3);
    std::vector<double> aw(std::max(1, nloc));
    for (int k = 0; k < nloc; ++k) {
        const int di = P->local[k];
        if (P->h_M[di] > FMS / 2) {
            set_error("fgain3d: line half-width exceeds the tap table");
            return DVM_E_UNSUPPORTED;
        }
        rec[3 * k] = make_int4(P->h_e[3 * di], P->h_e[3 * di + 1], P->h_e[3 * di + 2], P->h_M[di]);
        rec[3 * k + 1] = make_int4(hu[3 * di], hu[3 * di + 1], hu[3 * di + 2], 0);
        rec[3 * k + 2] = make_int4(hw[3 * di], hw[3 * di + 1], hw[3 * di + 2], 0);
        aw[k] = P->h_a[di] / (double)FNODES;  // the inverse transforms are unnormalised
    }
    DVM_CUDA(cudaMalloc(&g.fg_rec, sizeof(int4) * rec.size()));
    DVM_CUDA(cudaMalloc(&g.fg_aw, sizeof(double) * aw.size()));
    DVM_CUDA(cudaMalloc(&g.fg_t2d, sizeof(double) * (size_t)std::max(1, nloc) * FN2));
    DVM_CUDA(cudaMemcpyAsync(g.fg_rec, rec.data(), sizeof(int4) * rec.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(g.fg_aw, aw.data(), sizeof(double) * aw.size(), cudaMemcpyHostToDevice, P->stream));
    if (nloc > 0) {
        LaunchScope ls(P, KC_PLAN);
        const int64_t tot = (int64_t)nloc * FN2;
        k_fg_t2d<<<(unsigned)((tot + 255) / 256), 256, 0, P->stream>>>(FN, nloc, P->t.local, P->t.row_off, P->t.row_b,
                                                                      P->t.row_lo, P->t.row_hi, g.fg_t2d);
    }
    DVM_CUDA(cudaGetLastError());
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    g.bytes += sizeof(int4) * rec.size() + sizeof(double) * aw.size() + sizeof(double) * (size_t)nloc * FN2;
    return DVM_OK;
}

}  // namespace

dvm_status_t collide_fgain3d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                             int64_t ncells, bool *handled)
{
    *handled = false;
    if (P->d != 3 || P->N != FN || !P->g.ready || ncells <= 0) return DVM_OK;
    // the tap table holds 2 M_e <= 32 offsets (M_e <= Ñ): such plans have no 3D fast
    // path (build_gain3d leaves g.ready unset) and are evaluated by the v1 sweeps
    for (int di : P->local)
        if (P->h_M[di] > FMS / 2) return DVM_OK;
    dvm_status_t st;
    if ((st = build_fg_tables(P))) return st;
    // DVM_FG_TMEM=1: groups of 32 CTAs with f̂ resident in TMEM (k_fgain3d<32, true>)
    const bool tf = getenv("DVM_FG_TMEM") && atoi(getenv("DVM_FG_TMEM")) != 0;
    const int CL = tf ? 32 : (getenv("DVM_FG_CL") ? atoi(getenv("DVM_FG_CL")) : 16);
    if (CL != 16 && CL != 32) {
        set_error("DVM_FG_CL must be 16 or 32");
        return DVM_E_UNSUPPORTED;
    }
    auto kern = tf ? k_fgain3d<32, true> : (CL == 16 ? k_fgain3d<16, false> : k_fgain3d<32, false>);
    const size_t smem = tf ? FgSmemT<true>::total : FgSmemT<false>::total;
    DVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    DVM_CUDA(cudaGetDevice(&dev));
    DVM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DVM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    DVM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 2 * kRoleT, smem));
    if (!coop || per_sm < 1) return DVM_OK;  // the caller evaluates another path
    int max_groups = (sms * per_sm) / CL;
    if (getenv("DVM_G3_GROUPS")) max_groups = std::max(1, std::min(max_groups, atoi(getenv("DVM_G3_GROUPS"))));
    const int nloc = (int)P->local.size();
    const int64_t npairs = (ncells + 1) / 2;
    // direction chunks per pair: the persistent groups take (pair, chunk) items round-robin;
    // pick the fewest chunks whose busiest group does within 0.5 % of the balanced share
    // (256 pairs on 9 groups: 2 chunks, 28.5 instead of 29 pair-times)
    int nchunks = 1;
    {
        auto rounds = [&](int c) { return (double)((npairs * c + max_groups - 1) / max_groups) / c; };
        double best = 1e30;
        const int cmax = (int)std::max<int64_t>(1, std::min<int64_t>(nloc, std::max<int64_t>(16, max_groups / npairs)));
        for (int c = 1; c <= cmax; ++c) best = std::min(best, rounds(c));
        while (nchunks < cmax && rounds(nchunks) > best * 1.005) ++nchunks;
    }
    const int64_t items = npairs * nchunks;
    const int ngroups = (int)std::min<int64_t>(max_groups, items);
    Workspace &w = P->ws;
    if ((st = grow(&w.g3_f, &w.g3_f_elems, (size_t)(npairs * FNODES), P->stream))) return st;
    if ((st = grow(&w.fg_fhat, &w.fg_fhat_elems, (size_t)(npairs * FNODES), P->stream))) return st;
    if ((st = grow(&w.g3_q, &w.g3_q_elems, (size_t)(nchunks * npairs * FNODES), P->stream))) return st;
    const int slots = getenv("DVM_FG_SLOTS") ? std::max(2, std::min(4, atoi(getenv("DVM_FG_SLOTS")))) : 2;
    if ((st = grow(&w.g3_t, &w.g3_t_elems, (size_t)ngroups * slots * FNODES, P->stream))) return st;
    if ((st = grow(&w.g3_ctr, &w.g3_ctr_elems, (size_t)ngroups * 2 * CL, P->stream))) return st;
    if ((st = interleave_pairs(P, f, f_stride, ncells, FNODES, w.g3_f))) return st;
    if ((st = fft_forward_pairs(P, f, f_stride, ncells, w.fg_fhat))) return st;
    if (nchunks > 1)
        DVM_CUDA(cudaMemsetAsync(w.g3_q + npairs * FNODES, 0,
                                 sizeof(double2) * (size_t)((nchunks - 1) * npairs * FNODES), P->stream));
    if ((st = loss_init(P, f, f_stride, nullptr, 0, ncells, w.g3_q))) return st;
    DVM_CUDA(cudaMemsetAsync(w.g3_ctr, 0, sizeof(unsigned int) * 2 * CL * ngroups, P->stream));
    FgArgs a;
    a.fhat = w.fg_fhat;
    a.f = w.g3_f;
    a.Q = w.g3_q;
    a.npairs = npairs;
    a.nchunks = nchunks;
    a.nloc = nloc;
    a.rec = P->g.fg_rec;
    a.aw = P->g.fg_aw;
    a.t2d = P->g.fg_t2d;
    a.ring = w.g3_t;
    a.ctr = w.g3_ctr;
    a.H = P->pk.H;
    a.slots = slots;
    a.dbg = getenv("DVM_FG_DEBUG") ? atoi(getenv("DVM_FG_DEBUG")) : 0;
    if (getenv("DVM_VERBOSE"))
        fprintf(stderr, "[dvm] fgain3d: %d groups x %d CTAs, %d chunks, smem %zu\n", ngroups, CL, nchunks, smem);
    {
        void *args[] = {&a};
        LaunchScope ls(P, KC_FGAIN3D);
        const cudaError_t le =
            cudaLaunchCooperativeKernel((void *)kern, dim3(ngroups * CL), dim3(2 * kRoleT), args, smem, P->stream);
        if (le == cudaErrorCooperativeLaunchTooLarge || le == cudaErrorNotSupported) {
            cudaGetLastError();
            return DVM_OK;  // not handled: the caller evaluates another path
        }
        if (le != cudaSuccess) return cuda_fail(le, "cudaLaunchCooperativeKernel(k_fgain3d)");
    }
    if ((st = deinterleave_pairs(P, w.g3_q, nchunks, npairs, ncells, FNODES, Q, q_stride))) return st;
    *handled = true;
    return DVM_OK;
}

}  // namespace dvm
