// microbench.cu -- calibration of the B200 resources the DVM path is bound by
// (not product code): fp64 add / fma issue rate, shared-memory LDS.64
// bandwidth, L2-resident and HBM read bandwidth.  Prints one JSON line.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench.cu -o tools/microbench
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_dadd(double *out, int iters, double s)
{
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 += s; a1 += s; a2 += s; a3 += s; a4 += s; a5 += s; a6 += s; a7 += s;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dfma(double *out, int iters, double s, double t)
{
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fma(a0, s, t); a1 = fma(a1, s, t); a2 = fma(a2, s, t); a3 = fma(a3, s, t);
            a4 = fma(a4, s, t); a5 = fma(a5, s, t); a6 = fma(a6, s, t); a7 = fma(a7, s, t);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_lds(double *out, int iters)
{
    __shared__ double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    double acc = 0;
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += sm[(idx + k * 37) & 4095];
        idx = (idx + 32) & 4095;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_read(const double2 *in, size_t n, int reps, double *out)
{
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            double2 v = in[i];
            acc += v.x + v.y;
        }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename T>
__global__ void k_gather(const T *in, size_t mask, size_t stride, int reps, double *out)
{
    double acc = 0;
    const size_t n = mask + 1;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            T v = in[(i * stride + r) & mask];
            acc += *reinterpret_cast<double *>(&v);
        }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <typename T>
__global__ void k_scatter(T *buf, size_t mask, size_t stride, int reps)
{
    const size_t n = mask + 1;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            T v;
            *reinterpret_cast<double *>(&v) = (double)i;
            buf[(i * stride + r) & mask] = v;
        }
}
template <typename T>
double time_gather(const void *buf, size_t bytes, size_t stride, int sms, double *out)
{
    size_t n = bytes / sizeof(T);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_gather<T><<<sms * 8, 256>>>((const T *)buf, n - 1, stride, 2, out);
    cudaEventRecord(a);
    k_gather<T><<<sms * 8, 256>>>((const T *)buf, n - 1, stride, 20, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return 20.0 * n * sizeof(T) / (ms * 1e-3);
}
template <typename T>
double time_scatter(void *buf, size_t bytes, size_t stride, int sms)
{
    size_t n = bytes / sizeof(T);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_scatter<T><<<sms * 8, 256>>>((T *)buf, n - 1, stride, 2);
    cudaEventRecord(a);
    k_scatter<T><<<sms * 8, 256>>>((T *)buf, n - 1, stride, 20);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return 20.0 * n * sizeof(T) / (ms * 1e-3);
}

int main()
{
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double *out;
    CK(cudaMalloc(&out, sizeof(double) * 1 << 24));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    int blocks = sms * 8, threads = 256, iters = 4096;
    k_dadd<<<blocks, threads>>>(out, 16, 1.0);
    cudaEventRecord(a);
    k_dadd<<<blocks, threads>>>(out, iters, 1e-9);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double dadd = (double)blocks * threads * iters * 16 * 8 / (ms * 1e-3);
    k_dfma<<<blocks, threads>>>(out, 16, 1.0, 1.0);
    cudaEventRecord(a);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double dfma = (double)blocks * threads * iters * 16 * 8 / (ms * 1e-3);
    k_lds<<<blocks, threads>>>(out, 16);
    cudaEventRecord(a);
    k_lds<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double lds = (double)blocks * threads * iters * 16 * 8 / (ms * 1e-3);
    // L2-resident read: 32 MB buffer read 20 times; HBM read: 4 GB once
    size_t n2 = (32u << 20) / 16;
    double2 *buf;
    size_t nh = (4ull << 30) / 16;
    CK(cudaMalloc(&buf, nh * 16));
    cudaMemset(buf, 0, nh * 16);
    k_read<<<sms * 8, 256>>>(buf, n2, 2, out);
    cudaEventRecord(a);
    k_read<<<sms * 8, 256>>>(buf, n2, 20, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double l2 = 20.0 * n2 * 16 / (ms * 1e-3);
    k_read<<<sms * 8, 256>>>(buf, nh, 1, out);
    cudaEventRecord(a);
    k_read<<<sms * 8, 256>>>(buf, nh, 1, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double hbm = (double)nh * 16 / (ms * 1e-3);
    // L2-resident gathers/scatters over 32 MB: stride 1 (coalesced) vs odd stride (one element per sector)
    for (size_t st : {(size_t)1, (size_t)4099}) {
        printf("{\"l2_32MB_stride\": %zu, \"gather8\": %.4e, \"gather16\": %.4e, \"gather32\": %.4e, \"scatter8\": %.4e, \"scatter16\": %.4e, \"scatter32\": %.4e}\n", st,
               time_gather<double>(buf, 32u << 20, st, sms, out), time_gather<double2>(buf, 32u << 20, st, sms, out),
               time_gather<double4>(buf, 32u << 20, st, sms, out), time_scatter<double>(buf, 32u << 20, st, sms),
               time_scatter<double2>(buf, 32u << 20, st, sms), time_scatter<double4>(buf, 32u << 20, st, sms));
    }
    for (size_t mb : {(size_t)8, (size_t)64, (size_t)96}) {
        printf("{\"l2_MB\": %zu, \"read16\": %.4e, \"gather16_odd\": %.4e}\n", mb,
               time_gather<double2>(buf, mb << 20, 1, sms, out), time_gather<double2>(buf, mb << 20, 4099, sms, out));
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"dadd_per_s\": %.4e, \"dfma_flops\": %.4e, \"lds64_bytes_per_s\": %.4e, "
           "\"l2_read_bytes_per_s\": %.4e, \"hbm_read_bytes_per_s\": %.4e}\n",
           sms, clk, dadd, 2 * dfma, lds, l2, hbm);
    return 0;
}
