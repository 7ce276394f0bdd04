// dvm_fg32.cu -- 3D gain at N = 32 by batched spectral filtering of direction
// pairs (sm_100a, fp64): the single-cell counterpart of k_fg2 (c4).
//
// For one real cell f, two directions share one complex transform (both perp
// filters are real and even, f is real):
//   T_a + i T_b = IFFT( f̂ (t̂_a + i t̂_b) ),   t̂_e(ξ) = T2D_e(u.ξ mod N, w.ξ mod N)
// (the paper's spectral evaluation of the α'_p factor, PAPER.md:561-570,
// 816-819; reading R23).  All A/2 pair arrays are formed at once (k_f32_mult),
// transformed by the batched inverse passes of dvm_loss.cu (3 launches for the
// whole batch, L2-resident: A/2 × 512 KB, 74 MB for c4), then one kernel adds
// a_e S_e T_e for every node and direction chunk with S_e = Σ_{1<=|m|<=M_e}
// f(.+me) read as taps, and the chunk partials are summed in
// chunk order on top of −fΛ (the loss, one FFT convolution, reading R21).
// Deterministic: fixed summation order everywhere.
#include <math.h>

#include <algorithm>
#include <vector>

#include "dvm_internal.h"

namespace dvm {
namespace {

constexpr int K32 = 32;
constexpr int K32N = K32 * K32 * K32;
constexpr int K32CHUNKS = 16;  // direction-pair chunks of the gain kernel (partials summed in order)

// T2D_e(p, q) = Σ_{(α, β) ∈ P_e} cos(2π(α p + β q) / N), one thread per (direction, p, q)
__global__ void k_f32_t2d(int nloc, const int *local, const int *row_off, const int *row_b, const int *row_lo,
                          const int *row_hi, double *out)
{
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)nloc * K32 * K32) return;
    const int k = (int)(gid / (K32 * K32)), p = (int)((gid / K32) % K32), q = (int)(gid % K32);
    const int di = local[k];
    double acc = 0.0;
    for (int r = row_off[di]; r < row_off[di + 1]; ++r)
        for (int a = row_lo[r]; a <= row_hi[r]; ++a) {
            const int ph = ((a * p + row_b[r] * q) % K32 + K32) % K32;
            acc += cospi(2.0 * ph / K32);
        }
    out[gid] = acc;
}

// Z[p][ξ] = f̂(ξ) (t̂_{2p}(ξ) + i t̂_{2p+1}(ξ))   (t̂ of a missing partner: 0)
__global__ void k_f32_mult(const double2 *__restrict__ fhat, const double *__restrict__ t2d,
                           const int4 *__restrict__ ru, const int4 *__restrict__ rw, int nloc, int npairs,
                           double2 *__restrict__ Z)
{
    const int64_t total = (int64_t)npairs * K32N;
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)(gid / K32N), x = (int)(gid % K32N);
        const int x0 = x >> 10, x1 = (x >> 5) & 31, x2 = x & 31;
        auto filt = [&](int k) {
            const int4 u = ru[k], w = rw[k];
            const int pu = (u.x * x0 + u.y * x1 + u.z * x2) & (K32 - 1);
            const int pw = (w.x * x0 + w.y * x1 + w.z * x2) & (K32 - 1);
            return t2d[(int64_t)k * K32 * K32 + pu * K32 + pw];
        };
        const double ta = filt(2 * p), tb = 2 * p + 1 < nloc ? filt(2 * p + 1) : 0.0;
        const double2 fh = fhat[x];
        Z[gid] = make_double2(fh.x * ta - fh.y * tb, fh.x * tb + fh.y * ta);
    }
}

// part[chunk][x] = Σ_{pairs of the chunk, in order} a_a S_a(x) T_a(x) + a_b S_b(x) T_b(x)
__global__ void __launch_bounds__(256) k_f32_gain(const double *__restrict__ f, const double2 *__restrict__ Z,
                                                  const uint32_t *__restrict__ off, int mmax2,
                                                  const int4 *__restrict__ ru, const double *__restrict__ aw,
                                                  int nloc, int npairs, int ppc, uint32_t H,
                                                  double *__restrict__ part)
{
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int chunk = blockIdx.y;
    if (x >= K32N) return;
    const int p0 = chunk * ppc, p1 = min(npairs, p0 + ppc);
    double acc = 0.0;
    for (int p = p0; p < p1; ++p) {
        const double2 z = Z[(int64_t)p * K32N + x];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int k = 2 * p + s;
            if (k >= nloc) break;
            const int m2 = 2 * ru[k].w;
            const uint32_t *o = off + (int64_t)k * mmax2;
            double S = 0.0;
            for (int t = 0; t < m2; t += 2)
                S += __ldg(f + swar_add((uint32_t)x, o[t], H)) + __ldg(f + swar_add((uint32_t)x, o[t + 1], H));
            acc += aw[k] * (s ? z.y : z.x) * S;
        }
    }
    part[(int64_t)chunk * K32N + x] = acc;
}

// Q[x] += Σ_chunk part[chunk][x], chunks in order (Q holds −fΛ)
__global__ void k_f32_sum(const double *__restrict__ part, int nchunks, double *__restrict__ Q)
{
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= K32N) return;
    double g = 0.0;
    for (int c = 0; c < nchunks; ++c) g += part[(int64_t)c * K32N + x];
    Q[x] += g;
}

dvm_status_t build_f32_tables(dvm_plan_s *P)
{
    GainTables &g = P->g;
    if (g.f32_rec) return DVM_OK;
    const int nloc = (int)P->local.size();
    const int A = P->A;
    std::vector<int> hu((size_t)A * 3), hw((size_t)A * 3);
    DVM_CUDA(cudaMemcpy(hu.data(), P->t.u, sizeof(int) * hu.size(), cudaMemcpyDeviceToHost));
    DVM_CUDA(cudaMemcpy(hw.data(), P->t.w, sizeof(int) * hw.size(), cudaMemcpyDeviceToHost));
    int mmax = 1;
    for (int di : P->local) mmax = std::max(mmax, P->h_M[di]);
    std::vector<int4> rec((size_t)std::max(1, 2 * nloc));
    std::vector<uint32_t> off((size_t)std::max(1, nloc) * 2 * mmax, 0u);
    std::vector<double> aw(std::max(1, nloc));
    for (int k = 0; k < nloc; ++k) {
        const int di = P->local[k];
        rec[k] = make_int4(hu[3 * di], hu[3 * di + 1], hu[3 * di + 2], P->h_M[di]);
        rec[nloc + k] = make_int4(hw[3 * di], hw[3 * di + 1], hw[3 * di + 2], 0);
        for (int m = 1; m <= P->h_M[di]; ++m)
            for (int sg = 0; sg < 2; ++sg) {
                int c[3];
                for (int j = 0; j < 3; ++j) c[j] = (sg ? -m : m) * P->h_e[3 * di + j];
                off[(size_t)k * 2 * mmax + 2 * (m - 1) + sg] = pack_vec(c, 3, P->p, P->N);
            }
        aw[k] = P->h_a[di] / (double)K32N;  // the inverse transforms are unnormalised
    }
    DVM_CUDA(cudaMalloc(&g.f32_rec, sizeof(int4) * rec.size()));
    DVM_CUDA(cudaMalloc(&g.f32_off, sizeof(uint32_t) * off.size()));
    DVM_CUDA(cudaMalloc(&g.f32_aw, sizeof(double) * aw.size()));
    DVM_CUDA(cudaMalloc(&g.f32_t2d, sizeof(double) * (size_t)std::max(1, nloc) * K32 * K32));
    DVM_CUDA(cudaMemcpyAsync(g.f32_rec, rec.data(), sizeof(int4) * rec.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(g.f32_off, off.data(), sizeof(uint32_t) * off.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(g.f32_aw, aw.data(), sizeof(double) * aw.size(), cudaMemcpyHostToDevice, P->stream));
    if (nloc > 0) {
        LaunchScope ls(P, KC_PLAN);
        const int64_t tot = (int64_t)nloc * K32 * K32;
        k_f32_t2d<<<(unsigned)((tot + 255) / 256), 256, 0, P->stream>>>(nloc, P->t.local, P->t.row_off, P->t.row_b,
                                                                       P->t.row_lo, P->t.row_hi, g.f32_t2d);
    }
    DVM_CUDA(cudaGetLastError());
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    g.f32_mmax = mmax;
    g.bytes += sizeof(int4) * rec.size() + sizeof(uint32_t) * off.size() + sizeof(double) * aw.size() +
               sizeof(double) * (size_t)nloc * K32 * K32;
    return DVM_OK;
}

}  // namespace

dvm_status_t collide_fg32(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                          int64_t ncells, bool *handled)
{
    *handled = false;
    if (P->d != 3 || P->N != K32 || !P->g.lamhat || ncells <= 0) return DVM_OK;
    dvm_status_t st;
    if ((st = build_f32_tables(P))) return st;
    const int nloc = (int)P->local.size();
    const int npairs = (nloc + 1) / 2;
    const int nchunks = std::max(1, std::min(K32CHUNKS, npairs));
    const int ppc = npairs > 0 ? (npairs + nchunks - 1) / nchunks : 0;
    Workspace &w = P->ws;
    if ((st = grow(&w.f32_z, &w.f32_z_elems, (size_t)(std::max(1, npairs) + 1) * K32N, P->stream))) return st;
    if ((st = grow(&w.f32_part, &w.f32_part_elems, (size_t)nchunks * K32N, P->stream))) return st;
    // Q := −f Λ for every cell (the loss, one FFT convolution per cell pair)
    if ((st = loss_init(P, f, f_stride, Q, q_stride, ncells, nullptr))) return st;
    if (nloc == 0) {
        *handled = true;
        return DVM_OK;
    }
    double2 *fhat = w.f32_z + (size_t)npairs * K32N;
    const GainTables &g = P->g;
    for (int64_t c = 0; c < ncells; ++c) {
        if ((st = fft_forward_pairs(P, f + c * f_stride, f_stride, 1, fhat))) return st;
        {
            LaunchScope ls(P, KC_FG32);
            k_f32_mult<<<1184, 256, 0, P->stream>>>(fhat, g.f32_t2d, g.f32_rec, g.f32_rec + nloc, nloc, npairs,
                                                    w.f32_z);
            DVM_CUDA(cudaGetLastError());
        }
        if ((st = ifft_batch(P, w.f32_z, npairs))) return st;
        {
            LaunchScope ls(P, KC_FG32);
            k_f32_gain<<<dim3(K32N / 256, nchunks), 256, 0, P->stream>>>(f + c * f_stride, w.f32_z, g.f32_off,
                                                                         2 * g.f32_mmax, g.f32_rec, g.f32_aw, nloc,
                                                                         npairs, ppc, P->pk.H, w.f32_part);
            DVM_CUDA(cudaGetLastError());
        }
        {
            LaunchScope ls(P, KC_REDUCE);
            k_f32_sum<<<K32N / 256, 256, 0, P->stream>>>(w.f32_part, nchunks, Q + c * q_stride);
            DVM_CUDA(cudaGetLastError());
        }
    }
    *handled = true;
    return DVM_OK;
}

}  // namespace dvm
