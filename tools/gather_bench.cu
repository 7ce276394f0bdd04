// gather_bench.cu -- calibration (not product code): scattered 16-byte gathers
// into shared memory on B200 via cp.async (LSU) vs cp.async.bulk (TMA, mbarrier),
// alone and while other warps stream LDS.128 (interference with the smem pipe).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/gather_bench.cu -o tools/gather_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kN = 4096;  // 16-byte pieces per round per CTA (one plane of a cell pair)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>  // 0 cp.async, 1 cp.async.bulk (TMA), 2 none
__global__ void __launch_bounds__(512, 1) k_gather(const double2 *__restrict__ src, size_t mask, int rounds, int lds_warps,
                                                   double *out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    double2 *dst = reinterpret_cast<double2 *>(sm);          // kN pieces
    double2 *work = dst + kN;                                 // LDS streaming area (16 KB)
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5;
    const bool gather_thread = warp >= lds_warps;
    const int gt = tid - lds_warps * 32, ng = blockDim.x - lds_warps * 32;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = tid; i < 1024; i += blockDim.x) work[i] = make_double2(i, i);
    __syncthreads();
    double acc = 0;
    uint32_t phase = 0;
    for (int r = 0; r < rounds; ++r) {
        if (gather_thread && MODE != 2) {
            if (MODE == 1 && gt == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)),
                             "r"(kN * 16));
            if (MODE == 1) asm volatile("bar.sync 1, %0;" ::"r"(ng));
            for (int i = gt; i < kN; i += ng) {
                const size_t idx = ((size_t)(blockIdx.x * 7919 + r * 104729 + i) * 2654435761ull) & mask;
                if (MODE == 0) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + i)), "l"(src + idx));
                } else {
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                            smem_u32(dst + i)),
                        "l"(src + idx), "r"(smem_u32(&mbar))
                        : "memory");
                }
            }
            if (MODE == 0) {
                asm volatile("cp.async.commit_group;");
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            } else {
                uint32_t done = 0;
                while (!done) {
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done)
                                 : "r"(smem_u32(&mbar)), "r"(phase));
                }
                phase ^= 1;
            }
            if (MODE == 1) asm volatile("bar.sync 1, %0;" ::"r"(ng));
            acc += dst[gt].x;
        } else if (!gather_thread) {
            // LDS.128 streaming (the sliding program's load pattern)
            for (int k = 0; k < 64; ++k) {
                const double2 v = work[(tid + 37 * k) & 1023];
                acc += v.x + v.y;
            }
        }
    }
    out[blockIdx.x * blockDim.x + tid] = acc;
}

template <int MODE>
void run(const double2 *src, size_t n, double *out, int sms, int lds_warps, const char *name)
{
    auto k = k_gather<MODE>;
    const size_t smem = kN * 16 + 1024 * 16;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int rounds = 200;
    k<<<sms, 512, smem>>>(src, n - 1, 4, lds_warps, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<sms, 512, smem>>>(src, n - 1, rounds, lds_warps, out);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double pieces = (double)sms * rounds * kN;
    printf("{\"mode\": \"%s\", \"lds_warps\": %d, \"ms\": %.3f, \"ns_per_round\": %.1f, \"cycles_per_piece_per_SM\": %.3f, \"err\": \"%s\"}\n",
           name, lds_warps, ms, ms * 1e6 / rounds, ms * 1e-3 * 1.965e9 / (rounds * (double)kN), cudaGetErrorString(e));
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t n = (64ull << 20) / 16;  // 64 MB source (L2 resident)
    double2 *src;
    double *out;
    cudaMalloc(&src, n * 16);
    cudaMemset(src, 0, n * 16);
    cudaMalloc(&out, sizeof(double) * sms * 512);
    for (int lw : {0, 8}) {
        run<0>(src, n, out, sms, lw, "cp.async");
        run<1>(src, n, out, sms, lw, "cp.async.bulk");
    }
    run<2>(src, n, out, sms, 8, "lds-only");
    return 0;
}
