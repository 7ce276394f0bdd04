// dvm_fgain3d.cu -- 3D gain G = Σ_e a_e S_e T_e by per-direction FFT
// filtering (sm_100a, fp64; N = 64): k_fg2.
//
// The perp sums are the periodic convolution T_e = f ⊛ 1_{P_e}; their filter
// is even, so its spectrum is real and two cells share one complex transform:
//   T_{2p} + i T_{2p+1} = IFFT( f̂_p · t̂_e ),   f̂_p = FFT(f_{2p} + i f_{2p+1}),
//   t̂_e(ξ) = Σ_{l ∈ P_e} cos(2π l.ξ / N) = T2D_e(u.ξ mod N, w.ξ mod N)
// with (u, w) the basis of e^⊥ ∩ Z^3 the rows of P_e are given in
// (the paper's spectral evaluation of the α'_p
// factor; only the perp factor goes through Fourier space here, S_e stays a
// line stencil).  A persistent cooperative kernel; a group of 16 CTAs owns
// one cell pair at a time and walks the directions, warp-specialised:
//   phase A (warps 0-7): CTA `rank` takes the planes ξ_x ≡ rank (mod 16):
//     bulk-copy the plane of f̂ into shared memory, multiply by t̂_e, inverse
//     2D FFT over (ξ_y, ξ_z) with 16 points per thread (details below), write
//     the plane to the group's ring slot [ξ_x][y][z] in L2.
//   group progress counters (per CTA, monotonic, acquire/release)
//   phase B (warps 8-15): CTA `rank` owns the rows y ∈ [4 rank, 4 rank + 4):
//     ring columns loaded straight into registers one batch ahead, inverse FFT
//     along ξ_x (64 = 8 × 8, one shared-memory exchange), then Q += a_e S_e T_e
//     with S_e = Σ_{1<=|m|<=M_e} f(.+me) read as coalesced taps; Q lives in TMEM.
//   The roles run separate loops so setmaxnreg can move registers between them.
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
constexpr int FMS = 32;          // tap table size (2 M_e <= 32)
#ifndef FG2_REGA
#define FG2_REGA 104  // k_fg2 setmaxnreg split: phase A, phase B gets 256 - FG2_REGA
#endif
// T2D_e lookups of phase A: a half-warp (ξ_z = zl + const) reads one table row
// at q = c + g_z zl in the basis of perp_basis_zfree (dvm_internal.h): distinct
// banks for odd g_z, the t2d_col swizzle for even g_z (1.06 wavefronts per phase
// on average over the c5 directions instead of 2.27 in the plan's basis).

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
    int dbg;              // timing experiments (dvm_set_tuning "timing_dbg"; Q wrong): 1 skip phase-B work, 2 skip phase-A work,
                          // 4 skip the taps
};

// tap loads of phase B, not allocated in L1 (no reuse there: hit rate 1.8 %)
__device__ __forceinline__ double2 ld2_tap(const double2 *a, uint64_t pol)
{
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(a), "l"(pol));
    return v;
}

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
            __nanosleep(32);
        }
    }
    role_sync(id);
}

// ============================================================================
// Phase A of k_fg2: 16 points per thread, 64 = 4 × 16 in both in-plane passes
// (radix-4 over the high index in registers, one warp-private 16 × 16
// transpose, a 16-point DFT; one CTA-wide exchange between the two axes), so
// a plane costs 2 role barriers plus one mbarrier only the storing warp waits on.  Plane ξ_x = g, thread t = (yl, zl), zl = t & 15,
// yl = t >> 4, holds f̂(g, ξ_y = yl + 16 b, ξ_z = zl + 16 a), a, b < 4:
//   z: radix-4 over a, × ω^{zl kp1}; y: radix-4 over b, × ω^{yl kq1}    (ω = e^{2πi/64})
//   warp-private transpose: thread (yl, c = kp1 + 4 kq1) gets the 16 zl
//   16-point DFT over zl → z = kp1 + 4 kp2
//   CTA exchange: thread (z, kq1) gets the 16 yl;  16-point DFT → y = kq1 + 4 kq2
//   ring slot [ξ_x][y][z] (coalesced along z)
// Phase B: thread (k2 = warp, z = lane + 32 (b & 1)) of batch b (row
// y = 4 rank + b / 2) holds H(ξ_x = k2 + 8 n2, y, z), n2 < 8: DFT-8,
// twiddle, one shared-memory exchange across the 8 warps, DFT-8 → x = k2 + 8 k1.
// Lanes run along z, so every ring load and every tap load of a warp covers
// 512 contiguous bytes.
// ============================================================================
constexpr int kRegA2 = FG2_REGA, kRegB2 = 256 - FG2_REGA;
constexpr int kStoreWarp = 0;  // phase-A warp issuing the ring bulk stores (warp 7 measured 1.5 % slower)
constexpr int F2Q = FN2 / 4 + 4;  // CTA-exchange pitch of one kq1 quarter [16 yl][64 z] (+4: conflict-free writes)

struct Fg2Smem {
    static constexpr size_t st = sizeof(double2) * FN2;                        // f̂ plane staging / ex1 scratch
    static constexpr size_t ex = sizeof(double2) * (3 * F2Q + FN2 / 4);        // CTA exchange [kq1][yl][z]
    static constexpr size_t t2 = sizeof(double) * FN2;                         // T2D_e, full 64 × 64
    static constexpr size_t tw = sizeof(double2) * FN;                         // ω^k
    static constexpr size_t rb = sizeof(double2) * 2 * FN * 32;                // phase-B exchange, 2 batches
    static constexpr size_t total = st + ex + t2 + tw + rb;
};

// inverse 16-point DFT, natural order in and out: n = n1 + 4 n2, k = k1 + 4 k2
__device__ __forceinline__ void idft16(double2 (&v)[16])
{
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, c2 = 0.70710678118654752440;
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) idft4(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);  // v[n1 + 4 k1]
    // × ω16^{n1 k1}
    auto rot = [](double2 x, double c, double s) { return make_double2(x.x * c - x.y * s, x.x * s + x.y * c); };
    v[5] = rot(v[5], c1, s1);                                            // n1 = 1, k1 = 1: ω^1
    v[9] = make_double2(c2 * (v[9].x - v[9].y), c2 * (v[9].x + v[9].y));  // n1 = 1, k1 = 2: ω^2
    v[13] = rot(v[13], s1, c1);                                          // n1 = 1, k1 = 3: ω^3
    v[6] = make_double2(c2 * (v[6].x - v[6].y), c2 * (v[6].x + v[6].y));  // n1 = 2, k1 = 1: ω^2
    v[10] = make_double2(-v[10].y, v[10].x);                             // n1 = 2, k1 = 2: ω^4 = i
    v[14] = make_double2(-c2 * (v[14].x + v[14].y), c2 * (v[14].x - v[14].y));  // n1 = 2, k1 = 3: ω^6
    v[7] = rot(v[7], s1, c1);                                            // n1 = 3, k1 = 1: ω^3
    v[11] = make_double2(-c2 * (v[11].x + v[11].y), c2 * (v[11].x - v[11].y));  // n1 = 3, k1 = 2: ω^6
    v[15] = rot(v[15], -c1, -s1);                                        // n1 = 3, k1 = 3: ω^9
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) idft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);  // v[4 k1 + k2]
    double2 o[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) o[k1 + 4 * k2] = v[4 * k1 + k2];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = o[k];
}

__device__ __forceinline__ void mbar_init(uint64_t *m, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *m)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t phase)
{
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(m);
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(a), "r"(phase)
                     : "memory");
}
// one thread: expect `bytes` on the barrier, then bulk copies (TMA engine) complete them
__device__ __forceinline__ void mbar_expect(uint64_t *m, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *m, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(m)), "l"(pol)
        : "memory");
}

template <int CL>
__global__ void __launch_bounds__(2 * kRoleT, 1) k_fg2(FgArgs A)
{
    constexpr int FPL = FN / CL;  // ξ_x planes per CTA per direction
    constexpr int FRY = FN / CL;  // phase-B rows y per CTA (one batch each)
    static_assert(FRY == 4, "TMEM holds 4 rows of node pairs per CTA");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *stg = reinterpret_cast<double2 *>(smem_raw);                                 // [FN][FN]
    double2 *ex = reinterpret_cast<double2 *>(smem_raw + Fg2Smem::st);                    // [4][F2Q]
    double *t2 = reinterpret_cast<double *>(smem_raw + Fg2Smem::st + Fg2Smem::ex);        // [FN][FN]
    double2 *tw = reinterpret_cast<double2 *>(smem_raw + Fg2Smem::st + Fg2Smem::ex + Fg2Smem::t2);  // [FN]
    double2 *rb = tw + FN;  // phase-B x-FFT exchange [2][FN][32]
    __shared__ uint32_t soff[2][FMS];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_mbar;  // FG_BULK: completion of the phase-A bulk loads
    __shared__ __align__(8) uint64_t s_xbar[2], s_rbar[2];  // phase-B exchange buffer written / read
    __shared__ __align__(8) uint64_t s_obar;  // phase A: the plane's output rows are in the exchange buffer

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
    if (!roleA && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"l"(
                         (uint64_t)__cvta_generic_to_shared(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        mbar_init(&s_mbar, 1);
        mbar_init(&s_obar, kRoleT);
        for (int k = 0; k < 2; ++k) {
            mbar_init(&s_xbar[k], kRoleT);
            mbar_init(&s_rbar[k], kRoleT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // one bulk copy per table: the plane of f̂ (64 KB) and T2D_e (32 KB), issued by
    // thread 0 of phase A, completing the phase of s_mbar
    auto issue = [&](const double2 *fh, int g, int di) {
        if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect(&s_mbar, (uint32_t)(sizeof(double2) * FN2 + (di >= 0 ? sizeof(double) * FN2 : 0)));
            bulk_g2s(stg, fh + (int64_t)g * FN2, (uint32_t)(sizeof(double2) * FN2), &s_mbar, l2_drop());
            if (di >= 0) bulk_g2s(t2, A.t2d + (int64_t)di * FN2, (uint32_t)(sizeof(double) * FN2), &s_mbar, l2_keep());
        }
    };
    uint32_t mph = 0;
    uint32_t oph = 0;

    if (roleA) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegA2));
        const int zl = t & 15, yl = t >> 4;
        // ex1 scratch of this half-warp: the 4 staging rows it read, yl + 16 b
        double2 *x1w = stg + yl * FN;
        const int c_me = zl;  // after the transpose: c = kp1 + 4 kq1
        const int sw = c_me & 7;
        const int zr = t & 63, kq1r = t >> 6;  // CTA exchange reader: (z, kq1)
        if (grp < items && !(A.dbg & 2)) {
            issue(A.fhat + (grp / A.nchunks) * FNODES, rank, (int)((int64_t)A.nloc * (grp % A.nchunks) / A.nchunks));
        }
        for (int64_t item = grp; item < items; item += ngroups) {
            const int64_t pair = item / A.nchunks;
            const int chunk = (int)(item % A.nchunks);
            const int d0 = (int)((int64_t)A.nloc * chunk / A.nchunks);
            const int d1 = (int)((int64_t)A.nloc * (chunk + 1) / A.nchunks);
            const double2 *__restrict__ fh = A.fhat + pair * FNODES;
            for (int di = d0; di < d1; ++di, ++stepi) {
                double2 *Tb = A.ring + ((int64_t)grp * A.slots + (stepi % A.slots)) * FNODES;
                int ndi = -1;
                const double2 *fh_next = fh;
                if (di + 1 < d1) {
                    ndi = di + 1;
                } else if (item + ngroups < items) {
                    ndi = (int)((int64_t)A.nloc * ((item + ngroups) % A.nchunks) / A.nchunks);
                    fh_next = A.fhat + ((item + ngroups) / A.nchunks) * FNODES;
                }
                if (stepi >= (unsigned)A.slots) group_wait<CL>(cB, stepi - A.slots + 1, t, bar);
                const int4 ru = A.rec[(int64_t)di * 3 + 1], rw = A.rec[(int64_t)di * 3 + 2];
                const uint64_t keep = l2_keep();
#pragma unroll 1
                for (int kp = 0; kp < ((A.dbg & 2) ? 0 : FPL); ++kp) {
                    const int g = rank + kp * CL;
                    const bool lastp = kp + 1 == FPL;
                    mbar_wait(&s_mbar, mph);  // [1] the plane (and at kp = 0 T2D_e) is in shared memory
                    mph ^= 1;
                    double2 v[16];
                    {
                        // stage 1: f̂ t̂_e, radix-4 over ξ_z high and ξ_y high
                        const int pu0 = ru.x * g + ru.y * yl + ru.z * zl, pw0 = rw.x * g + rw.y * yl + rw.z * zl;
                        const int dua = 16 * ru.z, dub = 16 * ru.y, dwa = 16 * rw.z, dwb = 16 * rw.y;
#pragma unroll
                        for (int b = 0; b < 4; ++b)
#pragma unroll
                            for (int a = 0; a < 4; ++a) {
                                const int pu = (pu0 + a * dua + b * dub) & (FN - 1);
                                const int pw = (pw0 + a * dwa + b * dwb) & (FN - 1);
                                const double tv = t2[pu * FN + t2d_col(pw, rw.w)];
                                const double2 x = stg[(yl + 16 * b) * FN + zl + 16 * a];
                                v[a + 4 * b] = make_double2(x.x * tv, x.y * tv);
                            }
#pragma unroll
                        for (int b = 0; b < 4; ++b) idft4(v[4 * b], v[4 * b + 1], v[4 * b + 2], v[4 * b + 3]);
#pragma unroll
                        for (int b = 0; b < 4; ++b)
#pragma unroll
                            for (int k = 1; k < 4; ++k) v[k + 4 * b] = cmul(v[k + 4 * b], tw[(zl * k) & (FN - 1)]);  // ω^{zl kp1}
#pragma unroll
                        for (int k = 0; k < 4; ++k) idft4(v[k], v[k + 4], v[k + 8], v[k + 12]);
#pragma unroll
                        for (int q = 1; q < 4; ++q)
#pragma unroll
                            for (int k = 0; k < 4; ++k) v[k + 4 * q] = cmul(v[k + 4 * q], tw[(yl * q) & (FN - 1)]);  // ω^{yl kq1}
                    }
                    // warp-private 16 × 16 transpose in the rows this half-warp read:
                    // entry (c, zl) at c·16 + (zl ^ (c & 7)) of the 256-entry block
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        x1w[(c >> 2) * 16 * FN + 16 * (c & 3) + (zl ^ (c & 7))] = v[c];
                    __syncwarp();
#pragma unroll
                    for (int n = 0; n < 16; ++n)
                        v[n] = x1w[(c_me >> 2) * 16 * FN + 16 * (c_me & 3) + (n ^ sw)];
                    idft16(v);  // z = kp1 + 4 kp2: v[kp2], kp1 = c_me & 3
                    if (warp == kStoreWarp) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // ex is read
                    role_sync(bar);  // [2] staging and the exchange buffer are free
                    if (!lastp)
                        issue(fh, g + CL, -1);
                    else if (ndi >= 0)
                        issue(fh_next, rank, ndi);
                    {
                        const int kp1 = c_me & 3, kq1 = c_me >> 2;
                        double2 *dst = ex + kq1 * F2Q + yl * FN + kp1;
#pragma unroll
                        for (int k = 0; k < 16; ++k) dst[4 * k] = v[k];
                    }
                    role_sync(bar);  // [3]
                    {
                        const double2 *src = ex + kq1r * F2Q + zr;
#pragma unroll
                        for (int n = 0; n < 16; ++n) v[n] = src[n * FN];
                    }
                    idft16(v);  // y = kq1r + 4 kq2: v[kq2]
                    // back into the entries this thread read (row kq2 of quarter kq1r = ring row
                    // y = kq1r + 4 kq2), then warp 0 bulk-stores the 64 rows (1 KB each)
                    {
                        double2 *own = ex + kq1r * F2Q + zr;
#pragma unroll
                        for (int k = 0; k < 16; ++k) own[k * FN] = v[k];
                    }
                    // [4] as an mbarrier only the storing warp waits on
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive(&s_obar);
                    if (warp == kStoreWarp) {
                        mbar_wait(&s_obar, oph);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int idx = lane + 32 * h, q = idx >> 4, r = idx & 15;
                            asm volatile(
                                "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                                    Tb + (int64_t)g * FN2 + (q + 4 * r) * FN),
                                "r"((uint32_t)__cvta_generic_to_shared(ex + q * F2Q + r * FN)),
                                "r"((uint32_t)(sizeof(double2) * FN)), "l"(keep)
                                : "memory");
                        }
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    oph ^= 1;
                }
                if (warp == kStoreWarp) {
                    // the step's planes are in global memory before the release below
                    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                role_signal(cA + rank, stepi + 1, leader, bar);
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegB2));
        const uint32_t tm_base = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (uint32_t)(warp >> 2);
        // batch b -> (row, z half)
        auto b_row = [](int b) { return b >> 1; };
        auto b_zh = [](int b) { return b & 1; };
        for (int64_t item = grp; item < items; item += ngroups) {
            const int64_t pair = item / A.nchunks;
            const int chunk = (int)(item % A.nchunks);
            const int d0 = (int)((int64_t)A.nloc * chunk / A.nchunks);
            const int d1 = (int)((int64_t)A.nloc * (chunk + 1) / A.nchunks);
            const double2 *__restrict__ fc = A.f + pair * FNODES;
            double2 *Qc = A.Q + ((int64_t)chunk * A.npairs + pair) * FNODES;
            for (int di = d0; di < d1; ++di, ++stepi) {
                const double2 *Tb = A.ring + ((int64_t)grp * A.slots + (stepi % A.slots)) * FNODES;
                const int4 re = A.rec[(int64_t)di * 3];
                const int M2 = 2 * re.w;
                uint32_t *so = soff[stepi & 1];
                if (t < M2) {
                    const int m = t / 2 + 1, sg = (t & 1) ? -1 : 1;
                    so[t] = pk<FN>(sg * m * re.x, sg * m * re.y, sg * m * re.z);
                }
                const double aw = A.aw[di];
                const bool first = di == d0, last = di == d1 - 1;
                group_wait<CL>(cA, stepi + 1, t, bar);  // the ring slot is complete (and soff visible)
                const uint64_t keep = l2_keep(), drop = l2_drop();
                // ring columns straight into registers, one batch ahead (coalesced 512 B per warp row)
                double2 pre[8];
                auto fetch = [&](int b) {
                    const int y = FRY * rank + b_row(b), z = 32 * b_zh(b) + lane;
#pragma unroll
                    for (int n2 = 0; n2 < 8; ++n2) pre[n2] = ld2_cg_hint(Tb + ((int64_t)(warp + 8 * n2) * FN + y) * FN + z, drop);
                };
                // stage 1 of a batch (DFT-8 over n2, twiddle) from the prefetched ring values
                // into exchange buffer b & 1, then every B thread arrives on s_xbar[b & 1];
                // stage 2 waits on that barrier only, and arrives on s_rbar[b & 1] once read.
                // Each buffer completes 4 phases per step: parity (b >> 1) & 1.
                auto stage1 = [&](int b) {
                    const int y = FRY * rank + b_row(b);
                    double2 u[8];
#pragma unroll
                    for (int n2 = 0; n2 < 8; ++n2) u[n2] = pre[n2];
                    idft8(u);
#pragma unroll
                    for (int k2 = 1; k2 < 8; ++k2) u[k2] = cmul(u[k2], tw[(warp * k2) & (FN - 1)]);
                    double2 *Rw = rb + (b & 1) * FN * 32;
#pragma unroll
                    for (int k2 = 0; k2 < 8; ++k2) Rw[(warp + 8 * k2) * 32 + lane] = u[k2];
                    __syncwarp();
                    const double2 *line = Tb + ((int64_t)(warp + 8 * (lane >> 2)) * FN + y) * FN + 32 * b_zh(b) + 8 * (lane & 3);
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
                    mbar_arrive(&s_xbar[b & 1]);
                };
                if (!(A.dbg & 1)) {
                    fetch(0);
                    stage1(0);
                    fetch(1);
                }
#pragma unroll 1
                for (int b = 0; b < ((A.dbg & 1) ? 0 : (2 * FRY)); ++b) {
                    const int y = FRY * rank + b_row(b), z = 32 * b_zh(b) + lane;
                    double2 v[8];
                    const double2 *R = rb + (b & 1) * FN * 32;
                    mbar_wait(&s_xbar[b & 1], (uint32_t)((b >> 1) & 1));
                    // every B warp has staged the step's last batch (its ring loads and
                    // discards precede its arrival): the slot is free for phase A now, not
                    // after this batch's taps (144 c5 cells 476.1 -> 466.9 ms)
                    if (b == 2 * FRY - 1 && leader)
                        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(cB + rank), "r"(stepi + 1) : "memory");
                    const int k2 = warp;
#pragma unroll
                    for (int n1 = 0; n1 < 8; ++n1) v[n1] = R[(n1 + 8 * k2) * 32 + lane];
                    mbar_arrive(&s_rbar[b & 1]);
                    idft8(v);  // v[k1] = N^3 T_e(x = k2 + 8 k1, y, z)
                    if (b + 1 < (2 * FRY)) {
                        // buffer (b + 1) & 1 was batch b - 1's: wait until every thread has read it
                        if (b >= 1) mbar_wait(&s_rbar[(b + 1) & 1], (uint32_t)(((b - 1) >> 1) & 1));
                        stage1(b + 1);
                        if (b + 2 < (2 * FRY)) fetch(b + 2);
                    }
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        uint32_t n[4];
                        double2 S[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            n[q] = (uint32_t)((((k2 + 8 * (4 * hh + q)) * FN) + y) * FN + z);
                            S[q] = make_double2(0.0, 0.0);
                        }
                        // the accumulators' TMEM load is issued before the taps; its wait follows them
                        uint32_t r[16];
                        const uint32_t ta = tm_base + (uint32_t)(32 * b + 16 * hh);
                        __syncwarp();
                        tmem_ld16_nowait(ta, r);
                        // taps ±m e in pairs (M2 is even): 8 independent loads per iteration
                        int k0 = 0;
                        // two tap pairs per iteration while 4 taps remain: 16 loads in flight
#pragma unroll 1
                        for (; k0 + 4 <= ((A.dbg & 4) ? 0 : M2); k0 += 4) {
                            double2 a[4], c[4], a2[4], c2[4];
                            const uint32_t b0 = swar_add(n[0], so[k0], H2), b1 = swar_add(n[0], so[k0 + 1], H2);
                            const uint32_t b2 = swar_add(n[0], so[k0 + 2], H2), b3 = swar_add(n[0], so[k0 + 3], H2);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                a[q] = ld2_tap(fc + ((b0 + (uint32_t)q * 8u * FN2) & (uint32_t)(FNODES - 1)), keep);
                                c[q] = ld2_tap(fc + ((b1 + (uint32_t)q * 8u * FN2) & (uint32_t)(FNODES - 1)), keep);
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                a2[q] = ld2_tap(fc + ((b2 + (uint32_t)q * 8u * FN2) & (uint32_t)(FNODES - 1)), keep);
                                c2[q] = ld2_tap(fc + ((b3 + (uint32_t)q * 8u * FN2) & (uint32_t)(FNODES - 1)), keep);
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) S[q] = add2(S[q], add2(a[q], c[q]));
#pragma unroll
                            for (int q = 0; q < 4; ++q) S[q] = add2(S[q], add2(a2[q], c2[q]));
                        }
#pragma unroll 1
                        for (int k = k0; k < ((A.dbg & 4) ? 0 : M2); k += 2) {
                            const uint32_t o0 = so[k], o1 = so[k + 1];
                            double2 a[4], c[4];
                            // the 4 nodes differ only in x (the top field, 8 q apart): one carry-less
                            // add per tap, then plain adds modulo N^3 for the other nodes
                            const uint32_t b0 = swar_add(n[0], o0, H2), b1 = swar_add(n[0], o1, H2);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                a[q] = ld2_tap(fc + ((b0 + (uint32_t)q * 8u * FN2) & (uint32_t)(FNODES - 1)), keep);
                                c[q] = ld2_tap(fc + ((b1 + (uint32_t)q * 8u * FN2) & (uint32_t)(FNODES - 1)), keep);
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) S[q] = add2(S[q], add2(a[q], c[q]));
                        }
                        __syncwarp();
                        tmem_wait_ld();
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
                role_sync(bar);  // exchange buffer 0 is rewritten by the next step's first batch
                if ((A.dbg & 1) && leader)  // timing mode without phase-B work: no batch released the slot
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(cB + rank), "r"(stepi + 1) : "memory");
            }
        }
    }
    if (!roleA) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        role_sync(2);
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
    }
}

// T2D_e(p, q) = Σ_{(α, β) ∈ P_e} cos(2π(α p + β q) / N) in the plan's basis (u, w)
// of the rows, stored in the kernel's basis u' = c0 u + c1 w, w' = c2 u + c3 w
// (det 1): entry (p', q') holds T2D_e(c3 p' − c1 q', −c2 p' + c0 q') at column
// t2d_col(q', m).  One thread per (direction, p', q').
__global__ void k_fg_t2d(int N, int nloc, const int *local, const int *row_off, const int *row_b, const int *row_lo,
                         const int *row_hi, const int4 *basis, const int *mask, double *out)
{
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)nloc * N * N) return;
    const int k = (int)(gid / (N * N));
    const int pp = (int)((gid / N) % N), qq = (int)(gid % N);
    const int4 c = basis[k];
    const int p = ((c.w * pp - c.y * qq) % N + N) % N, q = ((-c.z * pp + c.x * qq) % N + N) % N;
    const int di = local[k];
    double acc = 0.0;
    for (int r = row_off[di]; r < row_off[di + 1]; ++r) {
        const int b = row_b[r];
        for (int a = row_lo[r]; a <= row_hi[r]; ++a) {
            const int ph = ((a * p + b * q) % N + N) % N;
            acc += cospi(2.0 * ph / N);
        }
    }
    out[(int64_t)k * N * N + pp * N + t2d_col(qq, mask[k])] = acc;
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
    std::vector<int4> rec((size_t)std::max(1, nloc) * 3), basis((size_t)std::max(1, nloc));
    std::vector<int> mask((size_t)std::max(1, nloc));
    std::vector<double> aw(std::max(1, nloc));
    for (int k = 0; k < nloc; ++k) {
        const int di = P->local[k];
        if (P->h_M[di] > FMS / 2) {
            set_error("fgain3d: line half-width exceeds the tap table");
            return DVM_E_UNSUPPORTED;
        }
        rec[3 * k] = make_int4(P->h_e[3 * di], P->h_e[3 * di + 1], P->h_e[3 * di + 2], P->h_M[di]);
        int c[4], up[3], wp[3], gz = 0;
        if (!perp_basis_zfree(&hu[3 * di], &hw[3 * di], c, up, wp, &gz)) {
            set_error("fgain3d: perp basis normalisation failed");
            return DVM_E_UNSUPPORTED;
        }
        const int c0 = c[0], c1 = c[1], c2 = c[2], c3 = c[3];
        basis[k] = make_int4(c0, c1, c2, c3);
        mask[k] = (gz & 1) ? 0 : 15;
        rec[3 * k + 1] = make_int4(up[0], up[1], up[2], 0);
        rec[3 * k + 2] = make_int4(wp[0], wp[1], wp[2], mask[k]);
        aw[k] = P->h_a[di] / (double)FNODES;  // the inverse transforms are unnormalised
    }
    DVM_CUDA(cudaMalloc(&g.fg_rec, sizeof(int4) * rec.size()));
    DVM_CUDA(cudaMalloc(&g.fg_aw, sizeof(double) * aw.size()));
    DVM_CUDA(cudaMalloc(&g.fg_t2d, sizeof(double) * (size_t)std::max(1, nloc) * FN2));
    DVM_CUDA(cudaMemcpyAsync(g.fg_rec, rec.data(), sizeof(int4) * rec.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(g.fg_aw, aw.data(), sizeof(double) * aw.size(), cudaMemcpyHostToDevice, P->stream));
    int4 *d_basis = nullptr;
    int *d_mask = nullptr;
    DVM_CUDA(cudaMalloc(&d_basis, sizeof(int4) * basis.size()));
    DVM_CUDA(cudaMalloc(&d_mask, sizeof(int) * mask.size()));
    DVM_CUDA(cudaMemcpyAsync(d_basis, basis.data(), sizeof(int4) * basis.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(d_mask, mask.data(), sizeof(int) * mask.size(), cudaMemcpyHostToDevice, P->stream));
    if (nloc > 0) {
        LaunchScope ls(P, KC_PLAN);
        const int64_t tot = (int64_t)nloc * FN2;
        k_fg_t2d<<<(unsigned)((tot + 255) / 256), 256, 0, P->stream>>>(FN, nloc, P->t.local, P->t.row_off, P->t.row_b,
                                                                      P->t.row_lo, P->t.row_hi, d_basis, d_mask,
                                                                      g.fg_t2d);
    }
    DVM_CUDA(cudaGetLastError());
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    cudaFree(d_basis);
    cudaFree(d_mask);
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
    constexpr int CL = 16;
    auto kern = k_fg2<CL>;
    const size_t smem = Fg2Smem::total;
    DVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    DVM_CUDA(cudaGetDevice(&dev));
    DVM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DVM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    DVM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 2 * kRoleT, smem));
    if (!coop || per_sm < 1) return DVM_OK;  // the caller evaluates another path
    // every CTA allocates all 512 TMEM columns: one CTA per SM (a second resident
    // CTA would block in tcgen05.alloc while its group waits for it)
    per_sm = 1;
    int max_groups = (sms * per_sm) / CL;
    if (P->tune.max_groups) max_groups = std::max(1, std::min(max_groups, P->tune.max_groups));
    const int nloc = (int)P->local.size();
    const int64_t npairs = (ncells + 1) / 2;
    // direction chunks per pair: the persistent groups take (pair, chunk) items round-robin;
    // pick the fewest chunks whose busiest group does within 0.5 % of the balanced share
    // (small batches; larger ones below)
    int nchunks = 1;
    {
        auto rounds = [&](int c) { return (double)((npairs * c + max_groups - 1) / max_groups) / c; };
        double best = 1e30;
        const int cmax = (int)std::max<int64_t>(1, std::min<int64_t>(nloc, std::max<int64_t>(16, max_groups / npairs)));
        for (int c = 1; c <= cmax; ++c) best = std::min(best, rounds(c));
        while (nchunks < cmax && rounds(nchunks) > best * 1.005) ++nchunks;
        // batches of >= 16 pairs: 8 or 16 chunks (the one with fewer rounds, ties to
        // 8) measured fastest at every bench size (ms, auto rule -> this rule:
        // 512 cells 1605 -> 1585, 256: 792.5 -> 792.0, 128: 398.1 -> 397.8, 64:
        // 199.8 -> 199.5, 32: 103.7 -> 100.5; tools/sweep_chunks.sh)
        if (npairs >= 16 && nloc >= 16) {
            const int c = rounds(16) < rounds(8) ? 16 : 8;
            // the chunk partials take c x the batch's Q: keep them under 24 GB (huge
            // batches keep the balance rule's fewer chunks)
            if ((double)c * (double)npairs * (double)FNODES * sizeof(double2) <= 24e9) nchunks = std::max(nchunks, c);
        }
    }
    if (P->tune.fg_chunks) nchunks = std::min(P->tune.fg_chunks, nloc);
    const int64_t items = npairs * nchunks;
    const int ngroups = (int)std::min<int64_t>(max_groups, items);
    Workspace &w = P->ws;
    if ((st = grow(&w.g3_f, &w.g3_f_elems, (size_t)(npairs * FNODES), P->stream))) return st;
    if ((st = grow(&w.fg_fhat, &w.fg_fhat_elems, (size_t)(npairs * FNODES), P->stream))) return st;
    if ((st = grow(&w.g3_q, &w.g3_q_elems, (size_t)(nchunks * npairs * FNODES), P->stream))) return st;
    const int slots = P->tune.ring_slots ? P->tune.ring_slots : 2;  // ring depth: A runs up to slots-1 steps ahead
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
    a.dbg = P->tune.fg_dbg;
    if (P->tune.verbose)
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
