// dsmem_bench.cu -- calibration (not product code): distributed shared memory
// gather/scatter bandwidth inside a thread-block cluster on B200.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/dsmem_bench.cu -o tools/dsmem_bench
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <typename T, int MODE>  // MODE 0: local smem gather, 1: remote (random rank) gather, 2: remote scatter
__global__ void k_ds(double *out, int iters, int words)
{
    extern __shared__ __align__(16) unsigned char sm[];
    T *s = reinterpret_cast<T *>(sm);
    cg::cluster_group cl = cg::this_cluster();
    const int n = words;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { T v; *reinterpret_cast<double *>(&v) = i; s[i] = v; }
    cl.sync();
    const unsigned nb = cl.num_blocks();
    double acc = 0;
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x * 97u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int k = 0; k < 8; ++k) {
            x = x * 1664525u + 1013904223u;
            unsigned idx = (x >> 8) % n;
            unsigned rk = (x >> 3) % nb;
            if (MODE == 0) {
                T v = s[(idx + threadIdx.x) % n];
                acc += *reinterpret_cast<double *>(&v);
            } else if (MODE == 1) {
                T *r = cl.map_shared_rank(s, rk);
                T v = r[idx];
                acc += *reinterpret_cast<double *>(&v);
            } else {
                T *r = cl.map_shared_rank(s, rk);
                T v; *reinterpret_cast<double *>(&v) = acc + k;
                r[idx] = v;
            }
        }
    }
    cl.sync();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename T, int MODE>
void run(int csize, double *out, int sms)
{
    auto k = k_ds<T, MODE>;
    size_t smem = 128 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    int ncl = 0;
    cfg.gridDim = dim3(csize); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem; cfg.attrs = attr; cfg.numAttrs = 1;
    cudaOccupancyMaxActiveClusters(&ncl, (void *)k, &cfg);
    cfg.gridDim = dim3(ncl * csize);
    int words = smem / sizeof(T);
    int iters = 256;
    cudaLaunchKernelEx(&cfg, k, out, 4, words);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k, out, iters, words);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)ncl * csize * 1024 * iters * 8 * sizeof(T);
    int ctas = ncl * csize;
    printf("{\"mode\": %d, \"elem\": %zu, \"cluster\": %d, \"ctas\": %d, \"GBps_total\": %.1f, \"B_per_clk_per_SM\": %.2f, \"err\": \"%s\"}\n", MODE, sizeof(T), csize, ctas,
           bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / ctas / 1.965e9, cudaGetErrorString(e));
}
int main()
{
    double *out; cudaMalloc(&out, 1 << 26);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cs : {2, 8, 16}) {
        run<double, 0>(cs, out, sms);
        run<double, 1>(cs, out, sms);
        run<double2, 1>(cs, out, sms);
        run<double4, 1>(cs, out, sms);
        run<double, 2>(cs, out, sms);
        run<double2, 2>(cs, out, sms);
    }
    return 0;
}
