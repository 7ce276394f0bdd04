// dvm_loss.cu -- the loss term of Q = D^{Ñ,N̄}(f,f) as one periodic convolution
// (reading R21): Σ_e a_e f U_e = f Λ, Λ = λ ⊛ f with the fixed kernel
//   λ(j) = Σ_e a_e #{(m, l) : 1 <= |m| <= M_e, l ∈ P_e, me + l ≡ j (mod N)}
// (β̃ = β − β(L,L); the paper evaluates this convolution
// spectrally).  λ is even, so λ̂ is real and two real cells
// share one complex transform (f_{2p} + i f_{2p+1}).
//
//   plan time   k_lambda (one thread per node, directions in order) and
//               λ̂ = FFT(λ) with the passes below (k_take_real)
//   per collide loss_init: 2d − 1 passes: d − 1 forward, one along axis 0 that
//               runs forward, × λ̂ and inverse in shared memory, d − 1
//               inverse (the last writes −f Λ)
// k_fft_pass is a radix-2 fp64 pass along one axis over tiles of lines in
// shared memory (two stages per barrier), twiddles exp(−2πik/N) from sincospi.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "dvm_internal.h"

namespace dvm {
namespace {

constexpr int kFT = 256;  // FFT threads per CTA

struct FftArgs {
    int d, ax, inverse;
    int64_t npairs;
    // real input (first forward pass): cells 2p, 2p+1 of r0 (cell stride r_stride, r_cells cells)
    const double *r0;
    int64_t r_stride, r_cells, r_first;  // r_first: index of the batch's first cell
    const double2 *zin;
    double2 *zout;
    const double *mult;  // optional real multiplier per node (λ̂)
    int roundtrip;       // forward stages, × mult, inverse stages in one pass (the middle axis pair)
    // epilogue (last inverse pass): Q[c] = -f[c] * Λ[c]
    double *q;
    int64_t q_stride;
    double2 *qI;  // epilogue, interleaved mode: qI[pair][node] = (-f_{2p} Λ_{2p}, -f_{2p+1} Λ_{2p+1})
    const double *f;
    int64_t f_stride;
    double scale;
    const double2 *tw;  // exp(-2πik/N), k < N/2
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Radix-2 DIT stages over LINES lines of N points in shared memory (input in
// bit-reversed order, output natural), two stages per barrier: a thread takes
// the 4 elements i0 + {0, 1, 2, 3} half of one 4-half block and applies stage
// `half` and stage `2 half` in registers (the same butterflies and twiddles as
// one stage at a time).  Every thread of the block calls it; it ends with a
// barrier.
template <int N, int LINES>
__device__ __forceinline__ void fft_stages(double2 *buf, const double2 *stw, bool inverse)
{
    auto bfly = [](double2 u, double2 x, double2 w, double2 &lo, double2 &hi) {
        const double2 v = cmul(x, w);
        lo = make_double2(u.x + v.x, u.y + v.y);
        hi = make_double2(u.x - v.x, u.y - v.y);
    };
    int half = 1;
    for (; 4 * half <= N; half <<= 2) {
        for (int b = threadIdx.x; b < LINES * N / 4; b += blockDim.x) {
            const int i = b / (N / 4), k = b % (N / 4);
            const int pos = k % half, grp = k / half;
            const int i0 = grp * 4 * half + pos;
            double2 w1 = stw[pos * (N / (2 * half))];
            double2 wa = stw[pos * (N / (4 * half))], wb = stw[(pos + half) * (N / (4 * half))];
            if (inverse) w1.y = -w1.y, wa.y = -wa.y, wb.y = -wb.y;
            double2 *r = buf + i * N + i0;
            double2 y0, y1, y2, y3, z0, z1, z2, z3;
            bfly(r[0], r[half], w1, y0, y1);
            bfly(r[2 * half], r[3 * half], w1, y2, y3);
            bfly(y0, y2, wa, z0, z2);
            bfly(y1, y3, wb, z1, z3);
            r[0] = z0, r[half] = z1, r[2 * half] = z2, r[3 * half] = z3;
        }
        __syncthreads();
    }
    if (half < N) {  // log2 N odd: the last stage alone
        for (int b = threadIdx.x; b < LINES * N / 2; b += blockDim.x) {
            const int i = b / (N / 2), k = b % (N / 2);
            const int pos = k & (half - 1), grp = k / half;
            const int i0 = grp * 2 * half + pos, i1 = i0 + half;
            double2 w = stw[pos * (N / (2 * half))];
            if (inverse) w.y = -w.y;
            double2 lo, hi;
            bfly(buf[i * N + i0], buf[i * N + i1], w, lo, hi);
            buf[i * N + i0] = lo, buf[i * N + i1] = hi;
        }
        __syncthreads();
    }
}

// One radix-2 FFT pass of length N along axis `ax` for every line of every
// pair in the batch.  Tile = B lines (contiguous rows for the last axis,
// lines adjacent in the last axis otherwise).
#ifndef FFT_B256
#define FFT_B256 1
#endif
// lines per CTA (the kernel's tile and the launcher's grid): 16 KB tiles, but fewer
// lines for N = 256 (a 2D cell has only 256 lines: more CTAs per pass), and 4
// lines when the default tiling gives fewer CTAs than SMs (fft_pass)
__host__ __device__ constexpr int fft_lines_per_cta(int N)
{
    return N == 256 ? FFT_B256 : ((1024 / N) < N ? (1024 / N) : N);
}

template <int N, int B>
__global__ void __launch_bounds__(kFT) k_fft_pass(FftArgs A)
{
    constexpr int LOGN = N == 16 ? 4 : N == 32 ? 5 : N == 64 ? 6 : N == 128 ? 7 : 8;
    __shared__ double2 buf[B * N];
    __shared__ double2 stw[N / 2];
    for (int k = threadIdx.x; k < N / 2; k += kFT) stw[k] = A.tw[k];
    const int d = A.d, ax = A.ax;
    int64_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= N;
    const int64_t lines = nodes / N;
    const int64_t tiles_per_pair = lines / B;
    const int64_t tile_all = blockIdx.x;
    const int64_t pair = tile_all / tiles_per_pair;
    const int64_t tile = tile_all % tiles_per_pair;
    if (pair >= A.npairs) return;
    const bool last_axis = ax == d - 1;
    int64_t sax = 1;
    for (int j = ax + 1; j < d; ++j) sax *= N;
    // address of element t of line i of this tile (within the pair's cell)
    auto addr = [&](int i, int t) -> int64_t {
        if (last_axis) return (tile * B + i) * N + t;
        const int64_t x_last0 = (tile % (N / B)) * B;
        const int64_t outer = tile / (N / B);  // the remaining coordinate (d = 3) or 0
        int64_t o = 0;
        if (d == 3) o = ax == 0 ? outer * N : outer * (int64_t)N * N;
        return o + (int64_t)t * sax + x_last0 + i;
    };
    // load (bit-reversed)
    for (int idx = threadIdx.x; idx < B * N; idx += kFT) {
        int i, t;
        if (last_axis) { i = idx / N; t = idx % N; }
        else { i = idx % B; t = idx / B; }
        const int64_t a = addr(i, t);
        double2 v;
        if (A.r0) {
            const int64_t c0 = A.r_first + 2 * pair, c1 = c0 + 1;
            v.x = A.r0[c0 * A.r_stride + a];
            v.y = c1 < A.r_cells ? A.r0[c1 * A.r_stride + a] : 0.0;
        } else {
            v = A.zin[pair * nodes + a];
        }
        const int tr = (int)(__brev((unsigned)t) >> (32 - LOGN));
        buf[i * N + tr] = v;
    }
    __syncthreads();
    auto stages = [&](bool inverse) { fft_stages<N, B>(buf, stw, inverse); };
    stages(A.inverse != 0);
    if (A.roundtrip) {
        // the same arithmetic as a forward pass storing × λ̂ and an inverse pass
        // loading bit-reversed: multiply, permute in shared memory, inverse stages
        for (int idx = threadIdx.x; idx < B * N; idx += kFT) {
            int i, t;
            if (last_axis) { i = idx / N; t = idx % N; }
            else { i = idx % B; t = idx / B; }
            const double m = A.mult[addr(i, t)];
            buf[i * N + t].x *= m;
            buf[i * N + t].y *= m;
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < B * N; idx += kFT) {
            const int i = idx / N, t = idx % N;
            const int tr = (int)(__brev((unsigned)t) >> (32 - LOGN));
            if (t < tr) {
                const double2 x = buf[i * N + t];
                buf[i * N + t] = buf[i * N + tr];
                buf[i * N + tr] = x;
            }
        }
        __syncthreads();
        stages(true);
    }
    for (int idx = threadIdx.x; idx < B * N; idx += kFT) {
        int i, t;
        if (last_axis) { i = idx / N; t = idx % N; }
        else { i = idx % B; t = idx / B; }
        const int64_t a = addr(i, t);
        double2 v = buf[i * N + t];
        if (A.mult && !A.roundtrip) {
            const double m = A.mult[a];
            v.x *= m;
            v.y *= m;
        }
        if (A.qI) {
            const int64_t c0 = A.r_first + 2 * pair, c1 = c0 + 1;
            double2 o;
            o.x = -A.f[c0 * A.f_stride + a] * (v.x * A.scale);
            o.y = c1 < A.r_cells ? -A.f[c1 * A.f_stride + a] * (v.y * A.scale) : 0.0;
            A.qI[(A.r_first / 2 + pair) * nodes + a] = o;
        } else if (A.q) {
            const int64_t c0 = A.r_first + 2 * pair, c1 = c0 + 1;
            A.q[c0 * A.q_stride + a] = -A.f[c0 * A.f_stride + a] * (v.x * A.scale);
            if (c1 < A.r_cells) A.q[c1 * A.q_stride + a] = -A.f[c1 * A.f_stride + a] * (v.y * A.scale);
        } else {
            A.zout[pair * nodes + a] = v;
        }
    }
}

__global__ void k_twiddles(int N, double2 *tw)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N / 2) return;
    double s, c;
    sincospi(2.0 * k / N, &s, &c);
    tw[k] = make_double2(c, -s);
}

// λ(j) = Σ_e a_e #{(m, l): 1 <= |m| <= M_e, l ∈ e^⊥ ∩ [-Ñ,Ñ]^d, me + l ≡ j},
// one thread per node j, directions in local-list order (deterministic).
// (2D: e^⊥ ∩ box = {n e^⊥ : |n| <= M_e}, the perp line of PAPER.md:803, 818.)
__global__ void k_lambda(int d, int N, int p, int Nt, const int *local, int nloc, const int *E, const int *M,
                         const double *aw, double *lam)
{
    int64_t nodes = 1;
    for (int q = 0; q < d; ++q) nodes *= N;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nodes) return;
    int jc[3] = {0, 0, 0};
    for (int q = d - 1, sh = 0; q >= 0; --q, sh += p) jc[q] = (int)((j >> sh) & (N - 1));
    double acc = 0.0;
    for (int k = 0; k < nloc; ++k) {
        const int di = local[k];
        const int ee[3] = {E[3 * di], E[3 * di + 1], E[3 * di + 2]};
        const int m_e = M[di];
        int cnt = 0;
        for (int m = 1; m <= m_e; ++m)
            for (int s = -1; s <= 1; s += 2) {
                bool ok = true;
                int dot = 0;
                for (int q = 0; q < d; ++q) {
                    int v = (jc[q] - s * m * ee[q]) % N;
                    if (v < 0) v += N;
                    if (v > N / 2) v -= N;  // centred representative (|l| <= Ñ < N/2)
                    if (v > Nt || v < -Nt) ok = false;
                    dot += v * ee[q];
                }
                if (ok && dot == 0) ++cnt;
            }
        if (cnt) acc += aw[di] * cnt;
    }
    lam[j] = acc;
}

// Weighted loss kernel (eq:decoup, general a(k) b(l)):
//   λ_w(j) = Σ_e Σ_{1<=|m|<=M_e, l ∈ e^⊥ ∩ [-Ñ,Ñ]^d, me + l ≡ j} a(me) b(l)
// (2Ñ+1 <= N: at most one l per residue class).  Box tables indexed k + Ñ.
__device__ __forceinline__ int box_index(int d, int Nt, const int *v)
{
    int idx = 0;
    for (int q = 0; q < d; ++q) idx = idx * (2 * Nt + 1) + (v[q] + Nt);
    return idx;
}

__global__ void k_lambda_w(int d, int N, int p, int Nt, const int *local, int nloc, const int *E, const int *M,
                           const double *wa, const double *wb, double *lam)
{
    int64_t nodes = 1;
    for (int q = 0; q < d; ++q) nodes *= N;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nodes) return;
    int jc[3] = {0, 0, 0};
    for (int q = d - 1, sh = 0; q >= 0; --q, sh += p) jc[q] = (int)((j >> sh) & (N - 1));
    double acc = 0.0;
    for (int k = 0; k < nloc; ++k) {
        const int di = local[k];
        const int ee[3] = {E[3 * di], E[3 * di + 1], E[3 * di + 2]};
        const int m_e = M[di];
        for (int m = 1; m <= m_e; ++m)
            for (int s = -1; s <= 1; s += 2) {
                bool ok = true;
                int dot = 0, kv[3] = {0, 0, 0}, lv[3] = {0, 0, 0};
                for (int q = 0; q < d; ++q) {
                    kv[q] = s * m * ee[q];
                    int v = (jc[q] - kv[q]) % N;
                    if (v < 0) v += N;
                    if (v > N / 2) v -= N;
                    if (v > Nt || v < -Nt) ok = false;
                    lv[q] = v;
                    dot += v * ee[q];
                }
                if (ok && dot == 0) acc += wa[box_index(d, Nt, kv)] * wb[box_index(d, Nt, lv)];
            }
    }
    lam[j] = acc;
}

__global__ void k_take_real(const double2 *z, int64_t n, double *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = z[i].x;
}

template <int N>
dvm_status_t fft_pass(dvm_plan_s *P, const FftArgs &a)
{
    constexpr int B = fft_lines_per_cta(N);
    constexpr int BS = B < 4 ? B : 4;  // small batches (a single cell at N <= 64): 4 lines per CTA, more CTAs
    int64_t nodes = 1;
    for (int j = 0; j < a.d; ++j) nodes *= N;
    const int64_t tiles = a.npairs * (nodes / N / B);
    LaunchScope ls(P, KC_FFT);
    if (tiles < 148)
        k_fft_pass<N, BS><<<(unsigned)(a.npairs * (nodes / N / BS)), kFT, 0, P->stream>>>(a);
    else
        k_fft_pass<N, B><<<(unsigned)tiles, kFT, 0, P->stream>>>(a);
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t fft_dispatch(dvm_plan_s *P, const FftArgs &a)
{
    switch (P->N) {
    case 16: return fft_pass<16>(P, a);
    case 32: return fft_pass<32>(P, a);
    case 64: return fft_pass<64>(P, a);
    case 128: return fft_pass<128>(P, a);
    case 256: return fft_pass<256>(P, a);
    default: set_error("FFT length unsupported"); return DVM_E_UNSUPPORTED;
    }
}

// ---------------------------------------------------------------- spectral reference path
// (dvm_set_path(3); the paper's per-direction spectral evaluation, PAPER.md:
// 561-570, 816-819): S_e = IFFT(f̂ ŝ_e), T_e = IFFT(f̂ t̂_e) from one complex
// transform, S_e + i T_e = IFFT(f̂ (ŝ_e + i t̂_e)); Q += a_e S_e T_e on top of −fΛ.
// ŝ_e(ξ) = Σ_{1<=|m|<=M_e} cos(2π m e.ξ / N), t̂_e(ξ) = Σ_{l ∈ P_e} cos(2π l.ξ / N):
// the line and perp-set filters are even, their spectra real.  Phases are
// integers mod N: cos values come from one table (identical for every term).
__global__ void k_spec_tables(int d, int N, int p, int nloc, const int *local, const int *E, const int *M,
                              const int *U, const int *W, const int *row_off, const int *row_b, const int *row_lo,
                              const int *row_hi, const double *ctab, double *shat, double *that)
{
    int64_t nodes = 1;
    for (int q = 0; q < d; ++q) nodes *= N;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= nodes * nloc) return;
    const int k = (int)(gid / nodes);
    const int64_t j = gid % nodes;
    int xi[3] = {0, 0, 0};
    for (int q = d - 1, sh = 0; q >= 0; --q, sh += p) xi[q] = (int)((j >> sh) & (N - 1));
    const int di = local[k];
    auto dot = [&](const int *v) {
        int s = 0;
        for (int q = 0; q < d; ++q) s += v[q] * xi[q];
        s %= N;
        return s < 0 ? s + N : s;
    };
    const int ev = dot(E + 3 * di), m_e = M[di];
    double sh_ = 0.0;
    for (int m = 1; m <= m_e; ++m) sh_ += 2.0 * ctab[(m * ev) & (N - 1)];
    double th = 0.0;
    if (d == 2) {
        const int ep[2] = {-E[3 * di + 1], E[3 * di]};
        int pv = (ep[0] * xi[0] + ep[1] * xi[1]) % N;
        if (pv < 0) pv += N;
        for (int n = -m_e; n <= m_e; ++n) th += ctab[((n * pv) % N + N) & (N - 1)];
    } else {
        const int uv = dot(U + 3 * di), wv = dot(W + 3 * di);
        for (int r = row_off[di]; r < row_off[di + 1]; ++r) {
            const int b = row_b[r];
            for (int a = row_lo[r]; a <= row_hi[r]; ++a) th += ctab[(((a * uv + b * wv) % N) + N) & (N - 1)];
        }
    }
    shat[(int64_t)k * nodes + j] = sh_;
    that[(int64_t)k * nodes + j] = th;
}

// Weighted filters (even a, b): ŝ_e(ξ) = Σ_{m=1}^{M_e} 2 a(me) cos(2π m e.ξ/N),
// t̂_e(ξ) = Σ_{l ∈ P_e} b(l) cos(2π l.ξ/N); a(me) sits in ŝ_e (Q += S_e T_e).
__global__ void k_spec_tables_w(int d, int N, int p, int Nt, int nloc, const int *local, const int *E, const int *M,
                                const int *U, const int *W, const int *row_off, const int *row_b,
                                const int *row_lo, const int *row_hi, const double *ctab, const double *wa,
                                const double *wb, double *shat, double *that)
{
    int64_t nodes = 1;
    for (int q = 0; q < d; ++q) nodes *= N;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= nodes * nloc) return;
    const int k = (int)(gid / nodes);
    const int64_t j = gid % nodes;
    int xi[3] = {0, 0, 0};
    for (int q = d - 1, sh = 0; q >= 0; --q, sh += p) xi[q] = (int)((j >> sh) & (N - 1));
    const int di = local[k];
    const int *e = E + 3 * di;
    int ev = 0;
    for (int q = 0; q < d; ++q) ev += e[q] * xi[q];
    ev %= N;
    if (ev < 0) ev += N;
    const int m_e = M[di];
    double sh_ = 0.0;
    for (int m = 1; m <= m_e; ++m) {
        const int kv[3] = {m * e[0], m * e[1], m * e[2]};
        sh_ += 2.0 * wa[box_index(d, Nt, kv)] * ctab[(m * ev) & (N - 1)];
    }
    double th = 0.0;
    if (d == 2) {
        const int ep[2] = {-e[1], e[0]};
        int pv = (ep[0] * xi[0] + ep[1] * xi[1]) % N;
        if (pv < 0) pv += N;
        for (int n = -m_e; n <= m_e; ++n) {
            const int lv[3] = {n * ep[0], n * ep[1], 0};
            th += wb[box_index(2, Nt, lv)] * ctab[((n * pv) % N + N) & (N - 1)];
        }
    } else {
        const int *u = U + 3 * di, *w = W + 3 * di;
        int uv = 0, wv = 0;
        for (int q = 0; q < 3; ++q) {
            uv += u[q] * xi[q];
            wv += w[q] * xi[q];
        }
        uv = ((uv % N) + N) % N;
        wv = ((wv % N) + N) % N;
        for (int r = row_off[di]; r < row_off[di + 1]; ++r) {
            const int b = row_b[r];
            for (int a = row_lo[r]; a <= row_hi[r]; ++a) {
                const int lv[3] = {a * u[0] + b * w[0], a * u[1] + b * w[1], a * u[2] + b * w[2]};
                th += wb[box_index(3, Nt, lv)] * ctab[(((a * uv + b * wv) % N) + N) & (N - 1)];
            }
        }
    }
    shat[(int64_t)k * nodes + j] = sh_;
    that[(int64_t)k * nodes + j] = th;
}

__global__ void k_cos_table(int N, double *ctab)
{
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N) ctab[n] = cospi(2.0 * n / N);
}

// z1 = z0 (ŝ + i t̂)
__global__ void k_spec_mul(const double2 *__restrict__ z0, const double *__restrict__ sh, const double *__restrict__ th,
                           double2 *__restrict__ z1, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 a = z0[i];
        const double s = sh[i], t = th[i];
        z1[i] = make_double2(a.x * s - a.y * t, a.x * t + a.y * s);
    }
}

// Q += a (Re z / n)(Im z / n)   (z = unnormalised inverse transform)
__global__ void k_spec_acc(const double2 *__restrict__ z, double aw, double scale, double *__restrict__ Q, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = z[i];
        Q[i] += aw * (v.x * scale) * (v.y * scale);
    }
}

}  // namespace


// λ (computed by `fill` into a scratch array) -> its real spectrum `lamhat`
// (λ even: FFT(λ) is real), with twiddles `tw`.
template <typename Fill>
dvm_status_t lambda_spectrum(dvm_plan_s *P, const double2 *tw, double *lamhat, Fill fill)
{
    const int d = P->d, N = P->N;
    int64_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= N;
    double *lam = nullptr;
    double2 *z = nullptr;
    DVM_CUDA(cudaMalloc(&lam, sizeof(double) * nodes));
    if (cudaMalloc(&z, sizeof(double2) * nodes) != cudaSuccess) {
        cudaFree(lam);
        return cuda_fail(cudaGetLastError(), "cudaMalloc");
    }
    {
        LaunchScope ls(P, KC_PLAN);
        fill(lam, nodes);
    }
    const cudaError_t le = cudaGetLastError();
    dvm_status_t st = le == cudaSuccess ? DVM_OK : cuda_fail(le, "k_lambda");
    for (int k = 0; k < d && !st; ++k) {
        FftArgs a = {};
        a.d = d;
        a.npairs = 1;
        a.tw = tw;
        a.r_cells = 1;
        a.r_first = 0;
        a.ax = d - 1 - k;
        a.zin = z;
        a.zout = z;
        if (k == 0) {
            a.r0 = lam;
            a.r_stride = nodes;
        }
        st = fft_dispatch(P, a);
    }
    if (!st) {
        LaunchScope ls(P, KC_PLAN);
        k_take_real<<<256, 256, 0, P->stream>>>(z, nodes, lamhat);
    }
    cudaStreamSynchronize(P->stream);
    cudaFree(lam);
    cudaFree(z);
    if (st) return st;
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

// Plan-time tables of the loss: twiddles, λ of the plan's (local) directions
// and its real spectrum λ̂.
dvm_status_t build_loss(dvm_plan_s *P)
{
    const int d = P->d, N = P->N;
    int64_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= N;
    GainTables &g = P->g;
    DVM_CUDA(cudaMalloc(&g.tw, sizeof(double2) * N / 2));
    DVM_CUDA(cudaMalloc(&g.lamhat, sizeof(double) * nodes));
    g.bytes += sizeof(double2) * N / 2 + sizeof(double) * nodes;
    {
        LaunchScope ls(P, KC_PLAN);
        k_twiddles<<<1, 128, 0, P->stream>>>(N, g.tw);
    }
    return lambda_spectrum(P, g.tw, g.lamhat, [&](double *lam, int64_t n) {
        k_lambda<<<(unsigned)((n + 127) / 128), 128, 0, P->stream>>>(d, N, P->p, P->Ntilde, P->t.local,
                                                                     (int)P->local.size(), P->t.e, P->t.M, P->t.a,
                                                                     lam);
    });
}

void free_weights(dvm_plan_s *P)
{
    WeightTables &w = P->wt;
    if (w.a_box || w.tw) cudaStreamSynchronize(P->stream);
    void *ptrs[] = {w.a_box, w.b_box, w.tw, w.lamhat, w.shat, w.that};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    w = WeightTables{};
}

// dvm_set_weights: validate the box tables (finite, even), upload them and
// build the weighted loss spectrum; the filter spectra follow lazily.
dvm_status_t set_weights(dvm_plan_s *P, const double *a_box, const double *b_box)
{
    free_weights(P);
    if (!a_box && !b_box) return DVM_OK;  // back to the built-in weights
    const int d = P->d, N = P->N, Nt = P->Ntilde;
    if (N < 16 || N > 256) {
        set_error("custom weights need the spectral path: N in [16, 256]");
        return DVM_E_UNSUPPORTED;
    }
    const int side = 2 * Nt + 1;
    int64_t box = 1;
    for (int j = 0; j < d; ++j) box *= side;
    std::vector<double> a(box), b(box);
    for (int64_t i = 0; i < box; ++i) {
        int v[3] = {0, 0, 0};
        int64_t r = i;
        for (int j = d - 1; j >= 0; --j) {
            v[j] = (int)(r % side) - Nt;
            r /= side;
        }
        if (a_box) {
            a[i] = a_box[i];
        } else {  // built-in a(k) = h^{d+1} |k| / gcd(k)
            int g = 0;
            double n2 = 0.0;
            for (int j = 0; j < d; ++j) {
                int x = v[j] < 0 ? -v[j] : v[j], y = g;
                while (y) {
                    const int t = x % y;
                    x = y;
                    y = t;
                }
                g = x;
                n2 += (double)v[j] * v[j];
            }
            a[i] = g ? pow(P->h, d + 1) * sqrt(n2) / g : 0.0;
        }
        b[i] = b_box ? b_box[i] : 1.0;
    }
    for (int64_t i = 0; i < box; ++i) {
        // reversing the row-major index negates every coordinate
        if (!std::isfinite(a[i]) || !std::isfinite(b[i]) || a[i] != a[box - 1 - i] || b[i] != b[box - 1 - i]) {
            set_error("weights must be finite and even: a(-k) = a(k), b(-l) = b(l)");
            return DVM_E_UNSUPPORTED;
        }
    }
    WeightTables &w = P->wt;
    int64_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= N;
    if (cudaMalloc(&w.a_box, sizeof(double) * box) != cudaSuccess ||
        cudaMalloc(&w.b_box, sizeof(double) * box) != cudaSuccess ||
        cudaMalloc(&w.tw, sizeof(double2) * N / 2) != cudaSuccess ||
        cudaMalloc(&w.lamhat, sizeof(double) * nodes) != cudaSuccess) {
        cudaGetLastError();
        free_weights(P);
        set_error("weight table allocation failed");
        return DVM_E_NOMEM;
    }
    DVM_CUDA(cudaMemcpyAsync(w.a_box, a.data(), sizeof(double) * box, cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(w.b_box, b.data(), sizeof(double) * box, cudaMemcpyHostToDevice, P->stream));
    {
        LaunchScope ls(P, KC_PLAN);
        k_twiddles<<<1, 128, 0, P->stream>>>(N, w.tw);
    }
    const double *wa = w.a_box, *wb = w.b_box;
    dvm_status_t st = lambda_spectrum(P, w.tw, w.lamhat, [&](double *lam, int64_t n) {
        k_lambda_w<<<(unsigned)((n + 127) / 128), 128, 0, P->stream>>>(d, N, P->p, Nt, P->t.local,
                                                                       (int)P->local.size(), P->t.e, P->t.M, wa,
                                                                       wb, lam);
    });
    if (st) {
        free_weights(P);
        return st;
    }
    w.on = true;
    return DVM_OK;
}

// f̂ of cell pairs: out[p] = FFT_d(f_{2p} + i f_{2p+1}) (forward, unnormalised;
// an odd tail cell is paired with zero).
// d unnormalised inverse passes, in place, over `narrays` complex N^d arrays
dvm_status_t ifft_batch(dvm_plan_s *P, double2 *z, int64_t narrays)
{
    const int d = P->d;
    for (int k = 0; k < d; ++k) {
        FftArgs a = {};
        a.d = d;
        a.npairs = narrays;
        a.tw = P->g.tw;
        a.inverse = 1;
        a.ax = k;
        a.zin = z;
        a.zout = z;
        dvm_status_t st = fft_dispatch(P, a);
        if (st) return st;
    }
    return DVM_OK;
}

dvm_status_t fft_forward_pairs(dvm_plan_s *P, const double *f, int64_t f_stride, int64_t ncells, double2 *out)
{
    const int d = P->d;
    int64_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= P->N;
    const int64_t npairs = (ncells + 1) / 2;
    const double2 *tw = P->wt.on ? P->wt.tw : P->g.tw;
    constexpr int64_t kBatch = 64;  // pairs per launch (grid size)
    for (int64_t p0 = 0; p0 < npairs; p0 += kBatch) {
        const int64_t np = std::min(kBatch, npairs - p0);
        for (int k = 0; k < d; ++k) {
            FftArgs a = {};
            a.d = d;
            a.npairs = np;
            a.tw = tw;
            a.r_cells = ncells;
            a.r_first = 2 * p0;
            a.ax = d - 1 - k;
            a.zin = out + p0 * nodes;
            a.zout = out + p0 * nodes;
            if (k == 0) {
                a.r0 = f;
                a.r_stride = f_stride;
            }
            dvm_status_t st = fft_dispatch(P, a);
            if (st) return st;
        }
    }
    return DVM_OK;
}

// Loss initialisation Q[c] := −f[c] Λ[c] for cells [0, ncells) (Λ = λ ⊛ f).
dvm_status_t loss_init(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride, int64_t ncells,
                       double2 *QI)
{
    const int d = P->d;
    int64_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= P->N;
    const int64_t npairs_all = (ncells + 1) / 2;
    const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(npairs_all, (int64_t)((256ull << 20) / (16 * nodes))));
    Workspace &w = P->ws;
    dvm_status_t st;
    if ((st = grow(&w.fft_z, &w.fft_z_elems, (size_t)(batch * nodes), P->stream))) return st;
    double scale = 1.0 / (double)nodes;
    const double2 *tw = P->wt.on ? P->wt.tw : P->g.tw;
    const double *lamhat = P->wt.on ? P->wt.lamhat : P->g.lamhat;
    for (int64_t p0 = 0; p0 < npairs_all; p0 += batch) {
        const int64_t np = std::min(batch, npairs_all - p0);
        for (int k = 0; k < 2 * d; ++k) {
            if (k == d) continue;  // the first inverse pass ran inside pass d - 1 (roundtrip)
            FftArgs a = {};
            a.d = d;
            a.npairs = np;
            a.tw = tw;
            a.r_cells = ncells;
            a.r_first = 2 * p0;
            const bool fwd = k < d;
            a.inverse = fwd ? 0 : 1;
            a.ax = fwd ? d - 1 - k : k - d;
            a.zin = w.fft_z;
            a.zout = w.fft_z;
            if (k == 0) {
                a.r0 = f;
                a.r_stride = f_stride;
            }
            if (k == d - 1) {
                a.mult = lamhat;
                a.roundtrip = 1;
            }
            if (k == 2 * d - 1) {
                a.qI = QI;
                a.q = Q;
                a.q_stride = q_stride;
                a.f = f;
                a.f_stride = f_stride;
                a.scale = scale;
            }
            if ((st = fft_dispatch(P, a))) return st;
        }
    }
    return DVM_OK;
}


dvm_status_t collide_spectral(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                              int64_t ncells)
{
    const int d = P->d, N = P->N;
    int64_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= N;
    const int nloc = (int)P->local.size();
    GainTables &g = P->g;
    WeightTables &wt = P->wt;
    const bool wtd = wt.on;  // caller weights a(k) b(l) (dvm_set_weights)
    if (!wtd && !g.lamhat) {
        set_error("spectral path needs the FFT loss tables (3D N in {32, 64}, 2D 16 <= N <= 256)");
        return DVM_E_UNSUPPORTED;
    }
    if ((double)nodes * nloc * 16.0 > 4.0e9) {
        set_error("spectral path tables would exceed 4 GB");
        return DVM_E_UNSUPPORTED;
    }
    dvm_status_t st;
    Workspace &w = P->ws;
    double *&shat = wtd ? wt.shat : g.shat;
    double *&that = wtd ? wt.that : g.that;
    const double2 *tw = wtd ? wt.tw : g.tw;
    if (!shat && nloc > 0) {  // lazily, on first use
        DVM_CUDA(cudaMalloc(&shat, sizeof(double) * nodes * nloc));
        DVM_CUDA(cudaMalloc(&that, sizeof(double) * nodes * nloc));
        double *ctab = nullptr;
        DVM_CUDA(cudaMalloc(&ctab, sizeof(double) * N));
        {
            LaunchScope ls(P, KC_PLAN);
            k_cos_table<<<(N + 127) / 128, 128, 0, P->stream>>>(N, ctab);
            const int64_t tot = nodes * nloc;
            if (wtd)
                k_spec_tables_w<<<(unsigned)((tot + 127) / 128), 128, 0, P->stream>>>(
                    d, N, P->p, P->Ntilde, nloc, P->t.local, P->t.e, P->t.M, P->t.u, P->t.w, P->t.row_off,
                    P->t.row_b, P->t.row_lo, P->t.row_hi, ctab, wt.a_box, wt.b_box, shat, that);
            else
                k_spec_tables<<<(unsigned)((tot + 127) / 128), 128, 0, P->stream>>>(
                    d, N, P->p, nloc, P->t.local, P->t.e, P->t.M, P->t.u, P->t.w, P->t.row_off, P->t.row_b,
                    P->t.row_lo, P->t.row_hi, ctab, shat, that);
        }
        DVM_CUDA(cudaGetLastError());
        DVM_CUDA(cudaStreamSynchronize(P->stream));
        cudaFree(ctab);
    }
    // Q := −f Λ (the loss, one convolution), then the gain direction by direction
    if ((st = loss_init(P, f, f_stride, Q, q_stride, ncells, nullptr))) return st;
    if ((st = grow(&w.sp_z, &w.sp_z_elems, (size_t)(2 * nodes), P->stream))) return st;
    double2 *z0 = w.sp_z, *z1 = w.sp_z + nodes;
    const double scale = 1.0 / (double)nodes;
    for (int64_t c = 0; c < ncells; ++c) {
        for (int k = 0; k < d; ++k) {  // f̂ of this cell
            FftArgs a = {};
            a.d = d;
            a.npairs = 1;
            a.tw = tw;
            a.r_cells = 1;
            a.ax = d - 1 - k;
            a.zin = z0;
            a.zout = z0;
            if (k == 0) {
                a.r0 = f + c * f_stride;
                a.r_stride = nodes;
            }
            if ((st = fft_dispatch(P, a))) return st;
        }
        for (int kd = 0; kd < nloc; ++kd) {
            {
                LaunchScope ls(P, KC_FFT);
                k_spec_mul<<<256, 256, 0, P->stream>>>(z0, shat + (int64_t)kd * nodes, that + (int64_t)kd * nodes,
                                                     z1, nodes);
            }
            for (int k = 0; k < d; ++k) {
                FftArgs a = {};
                a.d = d;
                a.npairs = 1;
                a.tw = tw;
                a.inverse = 1;
                a.ax = k;
                a.zin = z1;
                a.zout = z1;
                if ((st = fft_dispatch(P, a))) return st;
            }
            {
                // weighted: a(me) is inside ŝ_e; built-in: the line constant a_e
                const double aw = wtd ? 1.0 : P->h_a[P->local[kd]];
                LaunchScope ls(P, KC_FFT);
                k_spec_acc<<<256, 256, 0, P->stream>>>(z1, aw, scale, Q + c * q_stride, nodes);
            }
        }
        DVM_CUDA(cudaGetLastError());
    }
    return DVM_OK;
}

}  // namespace dvm
