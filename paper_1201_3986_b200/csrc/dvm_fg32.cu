// dvm_fg32.cu -- 3D gain at N = 32 by batched spectral filtering of direction
// pairs (sm_100a, fp64): the single-cell counterpart of k_fg2 (c4).
//
// For one real cell f, two directions share one complex transform (both perp
// filters are real and even, f is real):
//   T_a + i T_b = IFFT( f̂ (t̂_a + i t̂_b) ),   t̂_e(ξ) = T2D_e(u.ξ mod N, w.ξ mod N)
// (the paper's spectral evaluation of the α'_p factor, PAPER.md:561-570,
// 816-819; reading R23).  k_f32_plane forms each plane ξ_0 of every pair
// product (T2D lookups in the basis of perp_basis_zfree: a warp reads one
// table row) and runs the inverse 2D DFT over (ξ_1, ξ_2) into
// Z[pair][ξ_0][y][z] (A/2 × 512 KB, 74 MB for c4, L2-resident); k_f32_xgain
// runs the inverse DFT along ξ_0 for one row y and a chunk of pairs, then adds
// a_e S_e T_e for its nodes with S_e = Σ_{1<=|m|<=M_e} f(.+me) read as taps
// (PAPER.md:817); the chunk partials are summed in chunk order on top of −fΛ
// (the loss, one FFT convolution through the same plane kernel, reading R21).
// Deterministic: fixed summation order everywhere.
#include <math.h>

#include <algorithm>
#include <vector>

#include "dvm_g3common.h"
#include "dvm_internal.h"

namespace dvm {
namespace {

constexpr int K32 = 32;
constexpr int K32N = K32 * K32 * K32;
constexpr int K32CHUNKS = 32;  // direction-pair chunks of the gain kernel (partials summed in order)

// T2D_e(p, q) = Σ_{(α, β) ∈ P_e} cos(2π(α p + β q) / N) in the plan's basis (u, w),
// stored in the basis of perp_basis_zfree (u' = c0 u + c1 w, w' = c2 u + c3 w):
// entry (p', q') holds T2D_e(c3 p' − c1 q', −c2 p' + c0 q') at column
// t2d_col(q', m) of row p'.  One thread per (direction, p', q').
__global__ void k_f32_t2d(int nloc, const int *local, const int *row_off, const int *row_b, const int *row_lo,
                          const int *row_hi, const int4 *basis, const int *mask, double *out)
{
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)nloc * K32 * K32) return;
    const int k = (int)(gid / (K32 * K32)), pp = (int)((gid / K32) % K32), qq = (int)(gid % K32);
    const int4 cb = basis[k];
    const int p = ((cb.w * pp - cb.y * qq) % K32 + K32) % K32, q = ((-cb.z * pp + cb.x * qq) % K32 + K32) % K32;
    const int di = local[k];
    double acc = 0.0;
    for (int r = row_off[di]; r < row_off[di + 1]; ++r)
        for (int a = row_lo[r]; a <= row_hi[r]; ++a) {
            const int ph = ((a * p + row_b[r] * q) % K32 + K32) % K32;
            acc += cospi(2.0 * ph / K32);
        }
    out[(int64_t)k * K32 * K32 + pp * K32 + t2d_col(qq, mask[k])] = acc;
}

constexpr int P32 = K32 + 1;  // padded pitch of a 32 x 32 tile in shared memory (double2)

__device__ __forceinline__ double2 cmul32(double2 a, double2 b)
{
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 add2_(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2_(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// inverse-sign DFTs (y_k = Σ_n a_n e^{+2πi nk/n}), natural order in and out
__device__ __forceinline__ void idft4_(double2 &a0, double2 &a1, double2 &a2, double2 &a3)
{
    const double2 t0 = add2_(a0, a2), t1 = sub2_(a0, a2), t2 = add2_(a1, a3), d = sub2_(a1, a3);
    const double2 t3 = make_double2(-d.y, d.x);
    a0 = add2_(t0, t2);
    a2 = sub2_(t0, t2);
    a1 = add2_(t1, t3);
    a3 = sub2_(t1, t3);
}
__device__ __forceinline__ void idft8_(double2 (&v)[8])
{
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    idft4_(e0, e1, e2, e3);
    idft4_(o0, o1, o2, o3);
    constexpr double c = 0.70710678118654752440;
    o1 = make_double2(c * (o1.x - o1.y), c * (o1.x + o1.y));
    o2 = make_double2(-o2.y, o2.x);
    o3 = make_double2(-c * (o3.x + o3.y), c * (o3.x - o3.y));
    v[0] = add2_(e0, o0);
    v[4] = sub2_(e0, o0);
    v[1] = add2_(e1, o1);
    v[5] = sub2_(e1, o1);
    v[2] = add2_(e2, o2);
    v[6] = sub2_(e2, o2);
    v[3] = add2_(e3, o3);
    v[7] = sub2_(e3, o3);
}

// Inverse 32-point DFTs of the 32 lines of a 32 x 32 tile in shared memory, in
// place: element n of line l at buf[l * ls + n * es].  128 threads: thread
// (l = t & 31, j = t >> 5) takes n = j + 4 q (q < 8): DFT-8 over q -> k1,
// × ω32^{j k1}, then DFT-4 over j for k1 = 2 j', 2 j' + 1 -> k = k1 + 8 k2.
__device__ __forceinline__ void ifft32_lines(double2 *buf, int ls, int es, const double2 *tw32)
{
    const int t = threadIdx.x, l = t & 31, j = t >> 5;  // 8 lanes of a phase: 8 lines, distinct banks
    double2 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = buf[l * ls + (j + 4 * q) * es];
    idft8_(v);
#pragma unroll
    for (int k1 = 1; k1 < 8; ++k1) v[k1] = cmul32(v[k1], tw32[(j * k1) & (K32 - 1)]);
    __syncthreads();
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) buf[l * ls + (j + 4 * k1) * es] = v[k1];
    __syncthreads();
    double2 a[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k1 = 2 * j + h;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) a[h][jj] = buf[l * ls + (jj + 4 * k1) * es];
        idft4_(a[h][0], a[h][1], a[h][2], a[h][3]);
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) buf[l * ls + (2 * j + h + 8 * k2) * es] = a[h][k2];
    __syncthreads();
}

// One CTA per (direction pair p, plane ξ_0): the plane of f̂ (t̂_{2p} + i t̂_{2p+1}),
// inverse 2D DFT over (ξ_1, ξ_2), written to Z[p][ξ_0][y][z].
__global__ void __launch_bounds__(128) k_f32_plane(const double2 *__restrict__ fhat, const double *__restrict__ t2d,
                                                   const int4 *__restrict__ ru, const int4 *__restrict__ rw,
                                                   int nloc, int npairs, const double *__restrict__ lamhat,
                                                   double2 *__restrict__ Z)
{
    __shared__ double2 buf[K32 * P32];
    __shared__ double2 tw32[K32];
    const int p = blockIdx.x / K32, x0 = blockIdx.x % K32;
    const int t = threadIdx.x;
    if (t < K32) {
        double s, c;
        sincospi(2.0 * t / K32, &s, &c);
        tw32[t] = make_double2(c, s);
    }
    if (p == npairs) {
        // the loss array: f̂ λ̂ (λ̂ real, the spectrum of the loss kernel λ, reading R21)
        for (int i = t; i < K32 * K32; i += 128) {
            const double2 fh = fhat[x0 * K32 * K32 + i];
            const double l = lamhat[x0 * K32 * K32 + i];
            buf[(i >> 5) * P32 + (i & 31)] = make_double2(fh.x * l, fh.y * l);
        }
        __syncthreads();
        ifft32_lines(buf, P32, 1, tw32);
        ifft32_lines(buf, 1, P32, tw32);
        double2 *dst = Z + ((int64_t)p * K32 + x0) * K32 * K32;
        for (int i = t; i < K32 * K32; i += 128) dst[i] = buf[(i >> 5) * P32 + (i & 31)];
        return;
    }
    const int ka = 2 * p, kb = 2 * p + 1;
    const int4 ua = ru[ka], wa = rw[ka];
    const bool hb = kb < nloc;
    const int4 ub = hb ? ru[kb] : make_int4(0, 0, 0, 0), wb = hb ? rw[kb] : make_int4(0, 0, 0, 0);
    const double *Ta = t2d + (int64_t)ka * K32 * K32, *Tb = t2d + (int64_t)(hb ? kb : ka) * K32 * K32;
    for (int i = t; i < K32 * K32; i += 128) {
        const int x1 = i >> 5, x2 = i & 31;
        // a warp steps ξ_2 = x2: one row of each table (u'.z = 0), 2 lines per lookup
        const double ta = Ta[((ua.x * x0 + ua.y * x1 + ua.z * x2) & 31) * K32 +
                                  t2d_col((wa.x * x0 + wa.y * x1 + wa.z * x2) & 31, wa.w)];
        const double tb = hb ? Tb[((ub.x * x0 + ub.y * x1 + ub.z * x2) & 31) * K32 +
                                       t2d_col((wb.x * x0 + wb.y * x1 + wb.z * x2) & 31, wb.w)]
                             : 0.0;
        const double2 fh = fhat[x0 * K32 * K32 + i];
        buf[x1 * P32 + x2] = make_double2(fh.x * ta - fh.y * tb, fh.x * tb + fh.y * ta);
    }
    __syncthreads();
    ifft32_lines(buf, P32, 1, tw32);  // along ξ_2 -> z
    ifft32_lines(buf, 1, P32, tw32);  // along ξ_1 -> y
    double2 *dst = Z + ((int64_t)p * K32 + x0) * K32 * K32;
    // Z is read once, by k_f32_xgain: stored evict_last, read evict_first, so the
    // 74 MB stay in L2 between the two kernels (c4 0.111 -> 0.106 ms)
    const uint64_t keep = g3::l2_keep();
    for (int i = t; i < K32 * K32; i += 128) g3::st2_hint(dst + i, buf[(i >> 5) * P32 + (i & 31)], keep);
}

// Q := −f Λ for row y from the loss array's plane transform (the loss of eq:decD
// as one convolution, reading R21): the inverse DFT along ξ_0 gives N^3 Λ.
__device__ __forceinline__ void f32_xloss_row(const double *__restrict__ f, const double2 *__restrict__ Zl,
                                              double *__restrict__ Q, int y, double2 *buf, const double2 *tw32)
{
    const int t = threadIdx.x;
    const double2 *src = Zl + y * K32;
    for (int i = t; i < K32 * K32; i += 128) buf[(i >> 5) * P32 + (i & 31)] = src[(i >> 5) * K32 * K32 + (i & 31)];
    __syncthreads();
    ifft32_lines(buf, 1, P32, tw32);
    constexpr double inv = 1.0 / (double)K32N;
    for (int i = t; i < K32 * K32; i += 128) {
        const int x = i >> 5, z = i & 31;
        const int n = (x * K32 + y) * K32 + z;
        Q[n] = -f[n] * (buf[x * P32 + z].x * inv);
    }
}

// One CTA per (row y, pair chunk): for every pair of the chunk, the inverse DFT
// along ξ_0 of Z[p][:][y][:] gives T_a + i T_b on the 32 x 32 nodes (x, y, z);
// then G += a_a S_a T_a + a_b S_b T_b (S as taps of f), G in registers, written
// as this chunk's partial.  Thread t owns z = t & 31, x = (t >> 5) + 4 i.
__global__ void __launch_bounds__(128) k_f32_xgain(const double *__restrict__ f, const double2 *__restrict__ Z,
                                                   const uint32_t *__restrict__ off, int mmax2,
                                                   const int4 *__restrict__ ru, const double *__restrict__ aw,
                                                   int nloc, int npairs, int ppc, uint32_t H,
                                                   double *__restrict__ part, const double2 *__restrict__ Zl,
                                                   double *__restrict__ Q)
{
    __shared__ double2 buf[K32 * P32];
    __shared__ double2 tw32[K32];
    const int y = blockIdx.x, chunk = blockIdx.y;
    const int t = threadIdx.x, z = t & 31, xb = t >> 5;
    if (t < K32) {
        double s, c;
        sincospi(2.0 * t / K32, &s, &c);
        tw32[t] = make_double2(c, s);
    }
    if (chunk == (int)gridDim.y - 1) {  // the last row of blocks: Q := −f Λ (concurrent with the gain chunks)
        __syncthreads();
        f32_xloss_row(f, Zl, Q, y, buf, tw32);
        return;
    }
    double G[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) G[i] = 0.0;
    const int p0 = chunk * ppc, p1 = min(npairs, p0 + ppc);
    for (int p = p0; p < p1; ++p) {
        __syncthreads();
        const double2 *src = Z + (int64_t)p * K32N + y * K32;
        const uint64_t drop = g3::l2_drop();
        for (int i = t; i < K32 * K32; i += 128)
            buf[(i >> 5) * P32 + (i & 31)] = g3::ld2_cg_hint(src + (i >> 5) * K32 * K32 + (i & 31), drop);
        __syncthreads();
        ifft32_lines(buf, 1, P32, tw32);  // along ξ_0 -> x: buf[x][z]
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int k = 2 * p + s;
            if (k >= nloc) break;
            const int m2 = 2 * ru[k].w;
            const uint32_t *o = off + (int64_t)k * mmax2;
            const double a = aw[k];
            double S[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) S[i] = 0.0;
            const uint32_t n0 = (uint32_t)((xb * K32 + y) * K32 + z);
            // taps ±m e: 16 independent loads per pair of taps (8 nodes 4 x-planes apart)
            for (int q = 0; q < m2; q += 2) {
                const uint32_t b0 = swar_add(n0, o[q], H), b1 = swar_add(n0, o[q + 1], H);
                double va[8], vb[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    va[i] = __ldg(f + ((b0 + (uint32_t)(4 * i * K32 * K32)) & (uint32_t)(K32N - 1)));
                    vb[i] = __ldg(f + ((b1 + (uint32_t)(4 * i * K32 * K32)) & (uint32_t)(K32N - 1)));
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) S[i] += va[i] + vb[i];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double2 T = buf[(xb + 4 * i) * P32 + z];
                G[i] += a * (s ? T.y : T.x) * S[i];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) part[(int64_t)chunk * K32N + ((xb + 4 * i) * K32 + y) * K32 + z] = G[i];
}

// One CTA per row y: the loss array's transform along ξ_0 gives N^3 Λ(x, y, z);
// Q := −f Λ (the loss of eq:decD as one convolution, reading R21).
__global__ void __launch_bounds__(128) k_f32_xloss(const double *__restrict__ f, const double2 *__restrict__ Zl,
                                                   double *__restrict__ Q)
{
    __shared__ double2 buf[K32 * P32];
    __shared__ double2 tw32[K32];
    const int t = threadIdx.x;
    if (t < K32) {
        double s, c;
        sincospi(2.0 * t / K32, &s, &c);
        tw32[t] = make_double2(c, s);
    }
    __syncthreads();
    f32_xloss_row(f, Zl, Q, blockIdx.x, buf, tw32);
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
    std::vector<int4> rec((size_t)std::max(1, 2 * nloc)), basis((size_t)std::max(1, nloc));
    std::vector<int> mask((size_t)std::max(1, nloc));
    std::vector<uint32_t> off((size_t)std::max(1, nloc) * 2 * mmax, 0u);
    std::vector<double> aw(std::max(1, nloc));
    for (int k = 0; k < nloc; ++k) {
        const int di = P->local[k];
        int c[4], up[3], wp[3], gz = 0;
        if (!perp_basis_zfree(&hu[3 * di], &hw[3 * di], c, up, wp, &gz)) {
            set_error("fg32: perp basis normalisation failed");
            return DVM_E_UNSUPPORTED;
        }
        basis[k] = make_int4(c[0], c[1], c[2], c[3]);
        mask[k] = (gz & 1) ? 0 : 15;
        rec[k] = make_int4(up[0], up[1], up[2], P->h_M[di]);
        rec[nloc + k] = make_int4(wp[0], wp[1], wp[2], mask[k]);
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
    int4 *d_basis = nullptr;
    int *d_mask = nullptr;
    DVM_CUDA(cudaMalloc(&d_basis, sizeof(int4) * basis.size()));
    DVM_CUDA(cudaMalloc(&d_mask, sizeof(int) * mask.size()));
    DVM_CUDA(cudaMemcpyAsync(d_basis, basis.data(), sizeof(int4) * basis.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(d_mask, mask.data(), sizeof(int) * mask.size(), cudaMemcpyHostToDevice, P->stream));
    if (nloc > 0) {
        LaunchScope ls(P, KC_PLAN);
        const int64_t tot = (int64_t)nloc * K32 * K32;
        k_f32_t2d<<<(unsigned)((tot + 255) / 256), 256, 0, P->stream>>>(nloc, P->t.local, P->t.row_off, P->t.row_b,
                                                                       P->t.row_lo, P->t.row_hi, d_basis, d_mask,
                                                                       g.f32_t2d);
    }
    DVM_CUDA(cudaGetLastError());
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    cudaFree(d_basis);
    cudaFree(d_mask);
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
    // arrays: npairs direction pairs, the loss array, f̂
    if ((st = grow(&w.f32_z, &w.f32_z_elems, (size_t)(npairs + 2) * K32N, P->stream))) return st;
    if ((st = grow(&w.f32_part, &w.f32_part_elems, (size_t)nchunks * K32N, P->stream))) return st;
    double2 *fhat = w.f32_z + (size_t)(npairs + 1) * K32N;
    const GainTables &g = P->g;
    for (int64_t c = 0; c < ncells; ++c) {
        if ((st = fft_forward_pairs(P, f + c * f_stride, f_stride, 1, fhat))) return st;
        {
            LaunchScope ls(P, KC_FG32);
            k_f32_plane<<<(npairs + 1) * K32, 128, 0, P->stream>>>(fhat, g.f32_t2d, g.f32_rec, g.f32_rec + nloc,
                                                                   nloc, npairs, g.lamhat, w.f32_z);
            DVM_CUDA(cudaGetLastError());
        }
        if (nloc == 0) {
            LaunchScope ls(P, KC_FG32);
            k_f32_xloss<<<K32, 128, 0, P->stream>>>(f + c * f_stride, w.f32_z + (size_t)npairs * K32N, Q + c * q_stride);
            DVM_CUDA(cudaGetLastError());
            continue;
        }
        {
            // the gain chunks and, in one more row of blocks, the loss Q := −fΛ
            LaunchScope ls(P, KC_FG32);
            k_f32_xgain<<<dim3(K32, nchunks + 1), 128, 0, P->stream>>>(
                f + c * f_stride, w.f32_z, g.f32_off, 2 * g.f32_mmax, g.f32_rec, g.f32_aw, nloc, npairs, ppc, P->pk.H,
                w.f32_part, w.f32_z + (size_t)npairs * K32N, Q + c * q_stride);
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
