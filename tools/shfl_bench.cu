// shfl_bench.cu -- exchange cost on B200 (not product code): warp shuffles of
// 32-bit words vs a shared-memory STS.128 + LDS.128 round trip, per SM and clock.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/shfl_bench.cu -o tools/shfl_bench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_shfl(unsigned *out, int iters)
{
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 + 9, a5 = a0 + 11, a6 = a0 + 13, a7 = a0 + 17;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 1; k < 8; ++k) {
            a0 = __shfl_xor_sync(0xffffffffu, a0, k);
            a1 = __shfl_xor_sync(0xffffffffu, a1, k);
            a2 = __shfl_xor_sync(0xffffffffu, a2, k);
            a3 = __shfl_xor_sync(0xffffffffu, a3, k);
            a4 = __shfl_xor_sync(0xffffffffu, a4, k);
            a5 = __shfl_xor_sync(0xffffffffu, a5, k);
            a6 = __shfl_xor_sync(0xffffffffu, a6, k);
            a7 = __shfl_xor_sync(0xffffffffu, a7, k);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// warp-private 8x8 transpose of double2 through shared memory: 8 STS.128 + 8 LDS.128 per thread
__global__ void k_smx(double *out, int iters)
{
    extern __shared__ double2 sm[];
    double2 *w = sm + (threadIdx.x >> 5) * 32 * 9;
    const int lane = threadIdx.x & 31;
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = make_double2(lane + k, k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) w[lane * 9 + k] = v[k];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = w[((lane & ~7) + k) * 9 + (lane & 7)];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k].x += 1.0;
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half the warps shuffle, half exchange through shared memory: do the two share a pipe?
__global__ void k_mix(unsigned *out, double *outd, int iters)
{
    extern __shared__ double2 sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w & 1) {
        unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 + 9, a5 = a0 + 11, a6 = a0 + 13, a7 = a0 + 17;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 1; k < 8; ++k) {
                a0 = __shfl_xor_sync(0xffffffffu, a0, k); a1 = __shfl_xor_sync(0xffffffffu, a1, k);
                a2 = __shfl_xor_sync(0xffffffffu, a2, k); a3 = __shfl_xor_sync(0xffffffffu, a3, k);
                a4 = __shfl_xor_sync(0xffffffffu, a4, k); a5 = __shfl_xor_sync(0xffffffffu, a5, k);
                a6 = __shfl_xor_sync(0xffffffffu, a6, k); a7 = __shfl_xor_sync(0xffffffffu, a7, k);
            }
        }
        out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    } else {
        double2 *wp = sm + (w >> 1) * 32 * 9;
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = make_double2(lane + k, k);
        // the smem half does 2x the iterations' worth per shuffle-iteration ratio measured alone
        for (int i = 0; i < iters * 7 / 4; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) wp[lane * 9 + k] = v[k];
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = wp[((lane & ~7) + k) * 9 + (lane & 7)];
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k].x += 1.0;
        }
        double s = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y;
        outd[blockIdx.x * blockDim.x + threadIdx.x] = s;
    }
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned *o;
    double *od;
    cudaMalloc(&o, sizeof(unsigned) * sms * 1024);
    cudaMalloc(&od, sizeof(double) * sms * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4000;
    for (int thr : {256, 512, 1024}) {
        k_shfl<<<sms, thr>>>(o, 10);
        cudaEventRecord(e0);
        k_shfl<<<sms, thr>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double shfl = (double)sms * thr / 32 * iters * 56;  // warp-level SHFL instructions
        printf("shfl threads=%d: %.3f warp-shfl/clk/SM (at %d MHz)\n", thr, shfl / sms / (ms * 1e-3) / (clk * 1e3), clk / 1000);
        const size_t smem = (size_t)(thr / 32) * 32 * 9 * sizeof(double2);
        cudaFuncSetAttribute(k_smx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_smx<<<sms, thr, smem>>>(od, 10);
        cudaEventRecord(e0);
        k_smx<<<sms, thr, smem>>>(od, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double ex = (double)sms * thr * iters * 8;  // double2 elements exchanged (thread level)
        printf("smem x threads=%d: %.2f double2/clk/SM exchanged (%.2f wavefront-equiv B/clk)\n", thr,
               ex / sms / (ms * 1e-3) / (clk * 1e3), 32.0 * ex / sms / (ms * 1e-3) / (clk * 1e3));
    }
    {
        const int thr = 1024;
        const size_t smem = (size_t)(thr / 64) * 32 * 9 * sizeof(double2);
        cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_mix<<<sms, thr, smem>>>(o, od, 10);
        cudaEventRecord(e0);
        k_mix<<<sms, thr, smem>>>(o, od, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        // alone: shfl half = (thr/2/32)*iters*56 shfl at 1/clk; smem half = (thr/2)*iters*7/4*8 double2 at 4/clk
        double t_sh = (double)(thr / 64) * iters * 56;
        double t_sm = (double)(thr / 2) * iters * 7 / 4 * 8 / 4.0;
        printf("mix: %.3f ms; alone-sum estimate %.3f ms, alone-max %.3f ms\n", ms,
               (t_sh + t_sm) / (clk * 1e3) * 1e3 / 1, (t_sh > t_sm ? t_sh : t_sm) / (clk * 1e3) * 1e3);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
