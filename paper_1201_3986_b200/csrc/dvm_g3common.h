// dvm_g3common.h -- device helpers shared by the persistent 3D gain kernels
// (dvm_gain3d.cu: frame-plane sliding program; dvm_fgain3d.cu: per-direction
// FFT filter): role barriers and per-CTA progress counters of the warp-
// specialised groups, TMEM accumulator access, L2 cache-policy loads/stores,
// cp.async, and small double2 arithmetic.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dvm {
namespace g3 {

constexpr int kCL = 16;      // CTAs per cell group
constexpr int kRoleT = 256;  // threads per role (warps 0-7: phase A, warps 8-15: phase B)

template <int N>
__device__ __forceinline__ uint32_t pk(int c0, int c1, int c2)
{
    constexpr int P = N == 32 ? 5 : 6;
    return ((uint32_t)(c0 & (N - 1)) << (2 * P)) | ((uint32_t)(c1 & (N - 1)) << P) | (uint32_t)(c2 & (N - 1));
}

__device__ __forceinline__ void role_sync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kRoleT) : "memory"); }

// Wait until every CTA of the group has published progress >= target on its
// own monotonic counter (ctrs[0..kCL)): lanes of the role's first warp poll one
// counter each (acquire), then the role syncs.  Per-CTA counters, not a sum:
// a CTA running ahead must not stand in for a slower one.
template <int CL = kCL>
__device__ __forceinline__ void role_wait(const unsigned int *ctrs, unsigned int target, int t, int id)
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

// publish this CTA's role progress: the role barrier orders every role thread's
// writes before the leader's release store (release is cumulative; the CTA
// barrier + one st/red.release pattern of grid barriers, no separate fence)
__device__ __forceinline__ void role_signal(unsigned int *own, unsigned int value, bool leader, int id)
{
    role_sync(id);
    if (leader) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(own), "r"(value) : "memory");
}

// ---- tensor memory (TMEM) as the phase-B accumulator store: each B-role thread
// owns one TMEM lane and 256 32-bit columns (its 64 nodes × 2 cells in fp64).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// the same load without its wait (tcgen05.wait::ld before the registers are read)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 fma2(double s, double2 a, double2 c)
{
    return make_double2(fma(s, a.x, c.x), fma(s, a.y, c.y));
}

// L2 residency policies: the T ring and f stay (evict_last); T once consumed
// and the per-pair Q init/final go first (evict_first).
__device__ __forceinline__ uint64_t l2_keep()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_drop()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st2_hint(double2 *a, double2 v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ double2 ld2_cg_hint(const double2 *a, uint64_t pol)
{
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ld2_nc_hint(const double2 *a, uint64_t pol)
{
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
    return v;
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc)
{
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc), "l"(l2_keep())
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

}  // namespace g3
}  // namespace dvm
