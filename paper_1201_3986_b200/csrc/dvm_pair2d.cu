// dvm_pair2d.cu -- 2D evaluation of Q = D^{Ñ,N̄}(f,f) (Maxwell molecules).
//
// In 2D the perp set of direction e is the line P_e = {n e⊥ : |n| <= M_e}
// and e⊥ is again a direction of the table with the same
// M_e and a_e (|e⊥| = |e|, |e⊥|_inf = |e|_inf).  With the inclusive line windows
//     W_e(x) = Σ_{|m| <= M_e} f(x + m e)
// the factors of eq:decD are S_e = W_e − f and T_e = W_{e⊥}, so a pair of
// directions {e, e⊥} contributes
//     G_e + G_{e⊥} = a_e [ (W_e − f) W_{e⊥} + (W_{e⊥} − f) W_e ]
// (each term only if that direction belongs to the plan's shard).  The loss is
// the FFT convolution −f (λ ⊛ f) of dvm_loss.cu (reading R21).
//
//   k_wline2d  W along the first direction of every pair unit (sliding window
//              along its lattice lines) -> scratch
//   k_pair2d   W along the second direction (always one with an odd first
//              component: its lines start on the transversal x0 = 0 and warp
//              lanes walk adjacent lines, so every access is coalesced), combined
//              with the scratch and f into one partial gain per pair unit
//   k_sum_units Q += Σ_units partial in unit order (bitwise deterministic)
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "dvm_internal.h"

#ifndef TILE2D_COLS
#define TILE2D_COLS 32
#endif

namespace dvm {
namespace {

constexpr int kPT = 128;  // threads per CTA

struct Unit2D {
    int a0, a1;   // first direction A (pass 1)
    int b0, b1;   // second direction B (pass 2, odd first component)
    int M;        // common M_e
    int flags;    // bit0: A is local, bit1: B is local
    double aw;    // common a_e
};

__device__ __forceinline__ uint32_t pk2(int c0, int c1, int p, int N)
{
    return ((uint32_t)(c0 & (N - 1)) << p) | (uint32_t)(c1 & (N - 1));
}

// Walks along the lines of a primitive v in Z_N^2 (N = 2^p), coalesced.  With
// v0 = 2^s · odd (s < p), a line returns to the same row residue every
// Lv = N / 2^s steps; the segments starting at every node (c, j) of the rows
// c < 2^s partition all lines, and warp lanes on consecutive columns j stay in
// one row at every step (consecutive addresses).  Segments are cut further into
// `seglen` pieces.  v0 = 0 (v = (0, ±1): the lines are the rows) walks from the
// column x1 = 0 instead (strided, one direction only).
struct LineWalk {
    uint32_t x;     // packed current node
    uint32_t step;  // packed v
    uint32_t fwd;   // packed (M+1) v
    uint32_t back;  // packed -M v
};

struct WalkShape {
    int R;       // rows of starts (2^s), N for v0 == 0 (see below)
    int seglen;  // steps per work item
    int nsub;    // work items per (row, column) start
};

__host__ __device__ inline WalkShape walk_shape(int v0, int N)
{
    WalkShape w;
    int R = 1;
    if (v0 == 0) {
        R = 0;  // rows as lines: starts (j, 0), one item per line
        w.R = 0;
        w.seglen = N;
        w.nsub = 1;
        return w;
    }
    int a = v0 < 0 ? -v0 : v0;
    while (!(a & 1) && R < N) {
        a >>= 1;
        R <<= 1;
    }
    const int Lv = N / R;
    w.R = R;
    w.seglen = Lv < 64 ? Lv : 64;
    w.nsub = Lv / w.seglen;
    return w;
}

__host__ __device__ inline int walk_items(const WalkShape &w, int N) { return w.R == 0 ? N : w.nsub * w.R * N; }

__device__ __forceinline__ LineWalk line_start(int v0, int v1, int M, int item, const WalkShape &ws, int p, int N)
{
    LineWalk w;
    if (ws.R == 0) {
        w.x = pk2(item, 0, p, N);
    } else {
        const int j = item % N, c = (item / N) % ws.R, k = item / (N * ws.R);
        const int t0 = k * ws.seglen;
        w.x = pk2(c + t0 * v0, j + t0 * v1, p, N);
    }
    w.step = pk2(v0, v1, p, N);
    w.fwd = pk2((M + 1) * v0, (M + 1) * v1, p, N);
    w.back = pk2(-M * v0, -M * v1, p, N);
    return w;
}

__device__ __forceinline__ double window_at(const double *__restrict__ fc, uint32_t x, int v0, int v1, int M, int p,
                                            int N, uint32_t H)
{
    double W = 0.0;
    for (int m = -M; m <= M; ++m) W += __ldg(fc + swar_add(x, pk2(m * v0, m * v1, p, N), H));
    return W;
}

// pass 1: scratch[u][c][x] = W_A(x)
__global__ void __launch_bounds__(kPT) k_wline2d(const double *__restrict__ f, int64_t f_stride, int ncells,
                                                 const Unit2D *__restrict__ units, int p, int N, uint32_t H,
                                                 double *__restrict__ scratch)
{
    const int u = blockIdx.y, c = blockIdx.z;
    const Unit2D U = units[u];
    const int64_t nodes = (int64_t)N * N;
    const double *fc = f + (int64_t)c * f_stride;
    double *out = scratch + ((int64_t)u * ncells + c) * nodes;
    const WalkShape ws = walk_shape(U.a0, N);
    const int item = blockIdx.x * kPT + threadIdx.x;
    if (item >= walk_items(ws, N)) return;
    LineWalk w = line_start(U.a0, U.a1, U.M, item, ws, p, N);
    double W = window_at(fc, w.x, U.a0, U.a1, U.M, p, N, H);
#pragma unroll 4
    for (int i = 0; i < ws.seglen; ++i) {
        out[w.x] = W;
        W += __ldg(fc + swar_add(w.x, w.fwd, H)) - __ldg(fc + swar_add(w.x, w.back, H));
        w.x = swar_add(w.x, w.step, H);
    }
}

// pass 2: part[u][c][x] = a [A local](W_A − f) W_B + a [B local](W_B − f) W_A
__global__ void __launch_bounds__(kPT) k_pair2d(const double *__restrict__ f, int64_t f_stride, int ncells,
                                                const Unit2D *__restrict__ units, int p, int N, uint32_t H,
                                                const double *__restrict__ scratch,
                                                double *__restrict__ part)
{
    const int u = blockIdx.y, c = blockIdx.z;
    const Unit2D U = units[u];
    const int64_t nodes = (int64_t)N * N;
    const double *fc = f + (int64_t)c * f_stride;
    const double *WA = scratch + ((int64_t)u * ncells + c) * nodes;
    double *out = part + ((int64_t)u * ncells + c) * nodes;
    const WalkShape ws = walk_shape(U.b0, N);
    const int item = blockIdx.x * kPT + threadIdx.x;
    if (item >= walk_items(ws, N)) return;
    LineWalk w = line_start(U.b0, U.b1, U.M, item, ws, p, N);
    double W = window_at(fc, w.x, U.b0, U.b1, U.M, p, N, H);
    const double ca = (U.flags & 1) ? U.aw : 0.0, cb = (U.flags & 2) ? U.aw : 0.0;
#pragma unroll 4
    for (int i = 0; i < ws.seglen; ++i) {
        const double wa = WA[w.x], f0 = __ldg(fc + w.x);
        out[w.x] = ca * (wa - f0) * W + cb * (W - f0) * wa;
        W += __ldg(fc + swar_add(w.x, w.fwd, H)) - __ldg(fc + swar_add(w.x, w.back, H));
        w.x = swar_add(w.x, w.step, H);
    }
}

// Q[c][x] += Σ_u part[u][c][x], u ascending
__global__ void k_sum_units(const double *__restrict__ part, int nunits, int ncells, int64_t nodes,
                            double *__restrict__ Q, int64_t q_stride)
{
    const int64_t total = (int64_t)ncells * nodes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / nodes, x = i % nodes;
        double acc = Q[c * q_stride + x];
        for (int u = 0; u < nunits; ++u) acc += part[(int64_t)u * total + i];
        Q[c * q_stride + x] = acc;
    }
}

// ---- small grids (N <= 64): one CTA per (pair unit, cell) holds f and W_B in shared
// memory; the loss is evaluated per pair as well (no FFT):
//   U_A = Σ_{1<=|m|<=M} T_A(x + m A) = Box − W_B,  U_B = Box − W_A,
//   Box(x) = Σ_{|m|,|n| <= M} f(x + m A + n B)  (the window of W_B along A),
//   part_u = ca (W_A − f) W_B + cb (W_B − f) W_A − f [ca (Box − W_B) + cb (Box − W_A)]
// with ca = a [A local], cb = a [B local] (eq:decD with β̃ = β − β(L,L), PAPER.md:545,
// 822-831; in 2D the perp set of A is the line of B).  Direct
// window sums from shared memory (2M+1 loads each); partials summed in unit order.
#ifndef S2_THREADS
#define S2_THREADS 1024  // c2: 256 threads 40 us, 512 31 us, 1024 29 us
#endif
constexpr int kST = S2_THREADS;

__global__ void __launch_bounds__(kST) k_small2d(const double *__restrict__ f, int64_t f_stride,
                                                const Unit2D *__restrict__ units, int nunits, int nslice, int p,
                                                double *__restrict__ part)
{
    extern __shared__ double sm2[];
    const int N = 1 << p, mask = N - 1;
    const int nodes = N * N;
    double *F = sm2, *WB = sm2 + nodes;
    // CTA (unit u, slice s): W_B over the whole grid, the partial on slice s of the nodes
    const int u = blockIdx.x / nslice, sl = blockIdx.x % nslice, c = blockIdx.y;
    const Unit2D U = units[u];
    const double *fc = f + (int64_t)c * f_stride;
    for (int i = threadIdx.x; i < nodes; i += kST) F[i] = fc[i];
    __syncthreads();
    const int M = U.M;
    // W_B(x) = Σ_{|m| <= M} f(x + m B)
    for (int i = threadIdx.x; i < nodes; i += kST) {
        const int x0 = i >> p, x1 = i & mask;
        double w = 0.0;
        for (int m = -M; m <= M; ++m) w += F[(((x0 + m * U.b0) & mask) << p) | ((x1 + m * U.b1) & mask)];
        WB[i] = w;
    }
    __syncthreads();
    const double ca = (U.flags & 1) ? U.aw : 0.0, cb = (U.flags & 2) ? U.aw : 0.0;
    double *out = part + ((int64_t)c * nunits + u) * nodes;
    const int i0 = (int)((int64_t)nodes * sl / nslice), i1 = (int)((int64_t)nodes * (sl + 1) / nslice);
    for (int i = i0 + threadIdx.x; i < i1; i += kST) {
        const int x0 = i >> p, x1 = i & mask;
        double wa = 0.0, box = 0.0;
        for (int m = -M; m <= M; ++m) {
            const int j = (((x0 + m * U.a0) & mask) << p) | ((x1 + m * U.a1) & mask);
            wa += F[j];
            box += WB[j];
        }
        const double f0 = F[i], wb = WB[i];
        out[i] = ca * (wa - f0) * wb + cb * (wb - f0) * wa - f0 * (ca * (box - wb) + cb * (box - wa));
    }
}

// The same unit partials as k_small2d in two fine-grained launches, so the
// large-M units no longer set the critical path of one CTA each: k_s2_wb
// writes W_B of every (unit, row block) to scratch, k_s2_part the partial of
// every (unit, row block) from f and that scratch (both read through L1/L2).
// Same sums in the same order: bitwise the k_small2d partials.
__global__ void __launch_bounds__(256) k_s2_wb(const double *__restrict__ f, int64_t f_stride,
                                              const Unit2D *__restrict__ units, int nunits, int nrb, int p,
                                              double *__restrict__ wb)
{
    const int N = 1 << p, mask = N - 1, nodes = N * N;
    const int u = blockIdx.x / nrb, rb = blockIdx.x % nrb, c = blockIdx.y;
    const Unit2D U = units[u];
    const double *fc = f + (int64_t)c * f_stride;
    double *wc = wb + ((int64_t)c * nunits + u) * nodes;
    const int i0 = nodes / nrb * rb, i1 = i0 + nodes / nrb;
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const int x0 = i >> p, x1 = i & mask;
        double w = 0.0;
        for (int m = -U.M; m <= U.M; ++m) w += __ldg(fc + ((((x0 + m * U.b0) & mask) << p) | ((x1 + m * U.b1) & mask)));
        wc[i] = w;
    }
}

__global__ void __launch_bounds__(256) k_s2_part(const double *__restrict__ f, int64_t f_stride,
                                                const Unit2D *__restrict__ units, int nunits, int nrb, int p,
                                                const double *__restrict__ wb, double *__restrict__ part)
{
    const int N = 1 << p, mask = N - 1, nodes = N * N;
    const int u = blockIdx.x / nrb, rb = blockIdx.x % nrb, c = blockIdx.y;
    const Unit2D U = units[u];
    const double *fc = f + (int64_t)c * f_stride;
    const double *wc = wb + ((int64_t)c * nunits + u) * nodes;
    double *out = part + ((int64_t)c * nunits + u) * nodes;
    const double ca = (U.flags & 1) ? U.aw : 0.0, cb = (U.flags & 2) ? U.aw : 0.0;
    const int i0 = nodes / nrb * rb, i1 = i0 + nodes / nrb;
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const int x0 = i >> p, x1 = i & mask;
        double wa = 0.0, box = 0.0;
        for (int m = -U.M; m <= U.M; ++m) {
            const int j = (((x0 + m * U.a0) & mask) << p) | ((x1 + m * U.a1) & mask);
            wa += __ldg(fc + j);
            box += wc[j];
        }
        const double f0 = __ldg(fc + i), w0 = wc[i];
        out[i] = ca * (wa - f0) * w0 + cb * (w0 - f0) * wa - f0 * (ca * (box - w0) + cb * (box - wa));
    }
}

// Q[c][x] = Σ_u part[c][u][x], u ascending
// Q[c][x] = Σ_units part[c][u][x]: a block takes 32 consecutive nodes; its 8
// warps sum the units in 8 contiguous groups (loads of a group in flight
// together), then warp 0 adds the 8 group sums in group order.  Fixed order:
// deterministic.  (One thread per node summing all units serialised ~44 L2
// round trips per node and took 17 us on c2.)
__global__ void __launch_bounds__(256) k_small2d_sum(const double *__restrict__ part, int nunits, int ncells,
                                                     int nodes, double *__restrict__ Q, int64_t q_stride)
{
    __shared__ double gs[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t total = (int64_t)ncells * nodes;
    const int per = (nunits + 7) / 8, u0 = min(nunits, w * per), u1 = min(nunits, u0 + per);
    for (int64_t base = (int64_t)blockIdx.x * 32; base < total; base += (int64_t)gridDim.x * 32) {
        const int64_t i = base + lane;
        double acc = 0.0;
        if (i < total) {
            const int64_t c = i / nodes, x = i % nodes;
            const double *pc = part + c * nunits * (int64_t)nodes + x;
#pragma unroll 4
            for (int uu = u0; uu < u1; ++uu) acc += pc[(int64_t)uu * nodes];
        }
        gs[w][lane] = acc;
        __syncthreads();
        if (w == 0 && i < total) {
            double q = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) q += gs[k][lane];
            Q[(i / nodes) * q_stride + i % nodes] = q;
        }
        __syncthreads();
    }
}

// The same sum for one cell fused with an explicit Euler step and the moments
// partials of the new f (time stepping of small grids, config c2): Q is written,
// f <- f + dt Q exactly as k_axpy does, and every block (32 nodes) writes its
// mass / momentum / energy partial sums (reading R16; a fixed xor-shuffle tree)
// for the final fixed-order tree of dvm_collide.cu.  One launch instead of three.
__global__ void __launch_bounds__(256) k_small2d_sum_euler(const double *__restrict__ part, int nunits, int nodes,
                                                           double *__restrict__ Q, double *__restrict__ f,
                                                           double dt, int p, int N, double h,
                                                           double *__restrict__ mpart)
{
    __shared__ double gs[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per = (nunits + 7) / 8, u0 = min(nunits, w * per), u1 = min(nunits, u0 + per);
    const int i = blockIdx.x * 32 + lane;
    double acc = 0.0;
    if (i < nodes) {
        const double *pc = part + i;
#pragma unroll 4
        for (int uu = u0; uu < u1; ++uu) acc += pc[(int64_t)uu * nodes];
    }
    gs[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
        double m[4] = {0.0, 0.0, 0.0, 0.0};
        if (i < nodes) {
            double q = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) q += gs[k][lane];
            Q[i] = q;
            const double fn = f[i] + dt * q;
            f[i] = fn;
            const double v0 = ((i >> p) - N / 2) * h, v1 = ((i & (N - 1)) - N / 2) * h;
            m[0] = fn;
            m[1] = v0 * fn;
            m[2] = v1 * fn;
            m[3] = (v0 * v0 + v1 * v1) * fn;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
        if (lane == 0) {
            double *mp = mpart + (int64_t)blockIdx.x * 5;
#pragma unroll
            for (int k = 0; k < 4; ++k) mp[k] = m[k];
            mp[4] = 0.0;
        }
    }
}

// ---------------------------------------------------------------- 2D tile kernel (N >= 128)
// One CTA per 16 x 32 node tile and cell (a warp per tile row): the tile plus a halo of Ñ (every
// window offset m e has |m e|_inf <= M_e |e|_inf <= Ñ) is loaded into shared
// memory once (periodic wrap), then every thread walks the pair units in order
// for its node: W_A = Σ_{|m|<=M} f(x + mA), W_B likewise (direct windows from
// shared memory, 4 partial sums), G += a [(W_A − f) W_B + (W_B − f) W_A]
// (each term if that direction is in the plan's shard).
// G stays in a register; Q := −fΛ + G.  No scratch, no per-unit partials.
// c3: 0.123 ms (the line-walk kernels + partial sum: 0.194 ms); bound by the
// shared-memory loads (Σ_e (2M_e + 1) = 4568 per node for c3) with 16 warps per SM.
constexpr int kTile = 16;             // tile rows (at most; a launch may use fewer, see collide_tiles)
constexpr int kTileC = TILE2D_COLS;    // tile columns (one warp per row)

// the tile kernel's body; getU(u) returns unit u (shared memory, or the kernel
// parameter space for up to kParamUnits units: warp-uniform constant-cache loads
// instead of shared-memory wavefronts)
template <class GetU>
__device__ __forceinline__ void tile2d_body(const double *__restrict__ f, int64_t f_stride, int nunits, int N, int H,
                                            double *__restrict__ Q, int64_t q_stride, double *s2, int R, GetU getU)
{
    const int PR = R + 2 * H, P = kTileC + 2 * H;  // rows, pitch of the tile + halo (R tile rows)
    const int t = threadIdx.x;
    const int64_t cell = blockIdx.z;
    const int r0 = blockIdx.y * R, c0 = blockIdx.x * kTileC;
    const double *fc = f + cell * f_stride;
    for (int i = t; i < PR * P; i += blockDim.x) {
        const int rr = i / P, cc = i - rr * P;
        const int gr = (r0 - H + rr) & (N - 1), gc = (c0 - H + cc) & (N - 1);
        s2[i] = fc[(int64_t)gr * N + gc];
    }
    __syncthreads();
    const int ty = t / kTileC, tx = t % kTileC;
    if (r0 + ty >= N) return;  // rows past the grid in the last, ragged row of tiles
    const double *c = s2 + (H + ty) * P + (H + tx);
    const double fx = c[0];
    double g = 0.0;
    for (int u = 0; u < nunits; ++u) {
        const Unit2D U = getU(u);
        const int M = U.M, oa = U.a0 * P + U.a1, ob = U.b0 * P + U.b1;
        double wa0 = fx, wa1 = 0.0, wb0 = fx, wb1 = 0.0, wa2 = 0.0, wa3 = 0.0, wb2 = 0.0, wb3 = 0.0;
        int m = 1;
        for (; m + 1 <= M; m += 2) {
            wa0 += c[m * oa];
            wa1 += c[-m * oa];
            wa2 += c[(m + 1) * oa];
            wa3 += c[-(m + 1) * oa];
            wb0 += c[m * ob];
            wb1 += c[-m * ob];
            wb2 += c[(m + 1) * ob];
            wb3 += c[-(m + 1) * ob];
        }
        if (m <= M) {
            wa0 += c[m * oa];
            wa1 += c[-m * oa];
            wb0 += c[m * ob];
            wb1 += c[-m * ob];
        }
        const double WA = (wa0 + wa1) + (wa2 + wa3), WB = (wb0 + wb1) + (wb2 + wb3);
        double term = 0.0;
        if (U.flags & 1) term += (WA - fx) * WB;
        if (U.flags & 2) term += (WB - fx) * WA;
        g += U.aw * term;
    }
    double *q = Q + cell * q_stride + (int64_t)(r0 + ty) * N + (c0 + tx);
    *q += g;
}

__global__ void __launch_bounds__(kTile * kTileC) k_tile2d(const double *__restrict__ f, int64_t f_stride,
                                                const Unit2D *__restrict__ units, int nunits, int N, int H,
                                                double *__restrict__ Q, int64_t q_stride, int R)
{
    extern __shared__ __align__(16) double s2[];
    const int PR = R + 2 * H, P = kTileC + 2 * H;
    Unit2D *su = reinterpret_cast<Unit2D *>(s2 + ((PR * P + 1) & ~1));
    for (int i = threadIdx.x; i < nunits; i += blockDim.x) su[i] = units[i];
    tile2d_body(f, f_stride, nunits, N, H, Q, q_stride, s2, R, [&](int u) { return su[u]; });
}

constexpr int kParamUnits = 256;
struct TileUnits {
    Unit2D u[kParamUnits];
};

__global__ void __launch_bounds__(kTile * kTileC) k_tile2d_pu(const double *__restrict__ f, int64_t f_stride,
                                                   int nunits, int N, int H, double *__restrict__ Q,
                                                   int64_t q_stride, int R, const __grid_constant__ TileUnits pu)
{
    extern __shared__ __align__(16) double s2[];
    tile2d_body(f, f_stride, nunits, N, H, Q, q_stride, s2, R, [&](int u) { return pu.u[u]; });
}

}  // namespace

size_t tile2d_smem(int Ntilde, int nunits, int R = kTile)
{
    const int PR = R + 2 * Ntilde, P = kTileC + 2 * Ntilde;
    return sizeof(double) * (size_t)((PR * P + 1) & ~1) + sizeof(Unit2D) * (size_t)nunits;
}

// the per-unit partials of one cell (k_small2d only), into P->ws.p2_part
dvm_status_t collide_small2d_parts(dvm_plan_s *P, const double *f, bool *handled);

dvm_status_t euler_small2d(dvm_plan_s *P, double *f, double *Q, double dt, double *mpart, int *nblocks,
                           bool *handled)
{
    *handled = false;
    if (P->d != 2 || P->N > 64 || !P->g.ready || P->g.nunits == 0 || !mpart) return DVM_OK;
    const int N = P->N, nodes = N * N, nunits = P->g.nunits;
    if ((nodes + 31) / 32 > 128) return DVM_OK;  // the moments tree holds 128 partials
    bool h1 = false;
    // the partials of one cell (k_small2d), then the fused sum + Euler + moments partials
    dvm_status_t st = collide_small2d_parts(P, f, &h1);
    if (st || !h1) return st;
    {
        LaunchScope ls(P, KC_REDUCE);
        k_small2d_sum_euler<<<(nodes + 31) / 32, 256, 0, P->stream>>>(P->ws.p2_part, nunits, nodes, Q, f, dt, P->p,
                                                                     N, P->h, mpart);
        DVM_CUDA(cudaGetLastError());
    }
    *nblocks = (nodes + 31) / 32;
    *handled = true;
    return DVM_OK;
}

// small 2D grids (N <= 64): gain and loss per pair unit in shared memory, two launches
dvm_status_t collide_small2d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                             int64_t ncells, bool *handled)
{
    *handled = false;
    if (P->d != 2 || P->N > 64 || !P->g.ready || ncells <= 0) return DVM_OK;
    *handled = true;
    const int N = P->N, p = P->p;
    const int nodes = N * N;
    const int nunits = P->g.nunits;
    Workspace &w = P->ws;
    dvm_status_t st;
    if (nunits == 0) {
        LaunchScope ls(P, KC_ZERO);
        for (int64_t c = 0; c < ncells; ++c) DVM_CUDA(cudaMemsetAsync(Q + c * q_stride, 0, sizeof(double) * nodes, P->stream));
        return DVM_OK;
    }
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>({ncells, 65535, (int64_t)((256ull << 20) / (sizeof(double) * (uint64_t)nunits * nodes))}));
    if ((st = grow(&w.p2_part, &w.p2_part_elems, (size_t)(chunk * nunits * nodes), P->stream))) return st;
    const size_t smem = sizeof(double) * 2 * nodes;
    const Unit2D *units = reinterpret_cast<const Unit2D *>(P->g.units);
    int sms = 148;
    {
        int dev = 0;
        DVM_CUDA(cudaGetDevice(&dev));
        DVM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        // the 64 KB shared-memory opt-in is a per-device (per-context) attribute:
        // set once per device, under a lock (plans on several devices / threads)
        static std::mutex mu;
        static std::vector<char> done;
        std::lock_guard<std::mutex> lk(mu);
        if ((int)done.size() <= dev) done.resize(dev + 1, 0);
        if (!done[dev]) {
            DVM_CUDA(cudaFuncSetAttribute(k_small2d, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(sizeof(double) * 2 * 64 * 64)));
            done[dev] = 1;
        }
    }
    if (N >= 32) {
        // two fine-grained launches over (unit, 256-node row block) items (c2: 1 + 100
        // Euler steps 2.04 -> 1.86 ms); a 16 x 16 grid keeps the one-launch kernel
        const int nrb = nodes / 256;
        if ((st = grow(&w.p2_scr, &w.p2_scr_elems, (size_t)(chunk * nunits * nodes), P->stream))) return st;
        const int64_t nq = Q ? ncells : 1;
        for (int64_t c0 = 0; c0 < nq; c0 += chunk) {
            const int nc = (int)std::min<int64_t>(chunk, nq - c0);
            {
                LaunchScope ls(P, KC_SMALL2D);
                k_s2_wb<<<dim3(nunits * nrb, nc), 256, 0, P->stream>>>(f + c0 * f_stride, f_stride, units, nunits, nrb,
                                                                        p, w.p2_scr);
                k_s2_part<<<dim3(nunits * nrb, nc), 256, 0, P->stream>>>(f + c0 * f_stride, f_stride, units, nunits,
                                                                          nrb, p, w.p2_scr, w.p2_part);
            }
            if (Q) {
                LaunchScope ls(P, KC_REDUCE);
                const int64_t tot = (int64_t)nc * nodes;
                k_small2d_sum<<<(unsigned)std::min<int64_t>(2368, (tot + 31) / 32), 256, 0, P->stream>>>(
                    w.p2_part, nunits, nc, nodes, Q + c0 * q_stride, q_stride);
            }
            DVM_CUDA(cudaGetLastError());
        }
        return DVM_OK;
    }
    if (!Q) {  // collide_small2d_parts: the partials of one cell only
        const int nslice = (int)std::max<int64_t>(1, std::min<int64_t>(8, sms / (int64_t)nunits));
        LaunchScope ls(P, KC_SMALL2D);
        k_small2d<<<dim3(nunits * nslice, 1), kST, smem, P->stream>>>(f, f_stride, units, nunits, nslice, p, w.p2_part);
        DVM_CUDA(cudaGetLastError());
        return DVM_OK;
    }
    for (int64_t c0 = 0; c0 < ncells; c0 += chunk) {
        const int nc = (int)std::min<int64_t>(chunk, ncells - c0);
        // node slices per unit so that one wave covers the SMs (the widest windows dominate)
        const int nslice = (int)std::max<int64_t>(1, std::min<int64_t>(8, sms / ((int64_t)nunits * nc)));
        {
            LaunchScope ls(P, KC_SMALL2D);
            k_small2d<<<dim3(nunits * nslice, nc), kST, smem, P->stream>>>(f + c0 * f_stride, f_stride, units,
                                                                           nunits, nslice, p, w.p2_part);
        }
        {
            LaunchScope ls(P, KC_REDUCE);
            const int64_t tot = (int64_t)nc * nodes;
            k_small2d_sum<<<(unsigned)std::min<int64_t>(2368, (tot + 31) / 32), 256, 0, P->stream>>>(
                w.p2_part, nunits, nc, nodes, Q + c0 * q_stride, q_stride);
        }
        DVM_CUDA(cudaGetLastError());
    }
    return DVM_OK;
}

// Plan-time: pair units of the (local) directions, loss tables.
dvm_status_t build_pair2d(dvm_plan_s *P)
{
    if (P->d != 2 || P->N < 16 || P->N > 256) return DVM_OK;  // FFT lengths of dvm_loss.cu; else v1
    const int A = P->A;
    auto canon = [](int a, int b) {
        if (a < 0 || (a == 0 && b < 0)) {
            a = -a;
            b = -b;
        }
        return std::make_pair(a, b);
    };
    auto find = [&](int a, int b) {
        for (int i = 0; i < A; ++i)
            if (P->h_e[3 * i] == a && P->h_e[3 * i + 1] == b) return i;
        return -1;
    };
    std::vector<Unit2D> units;
    std::vector<uint8_t> used(A, 0);
    for (int i = 0; i < A; ++i) {
        if (used[i]) continue;
        const int e0 = P->h_e[3 * i], e1 = P->h_e[3 * i + 1];
        const auto pp = canon(-e1, e0);
        const int k = find(pp.first, pp.second);
        if (k < 0 || P->h_M[k] != P->h_M[i]) {
            set_error("2D direction table is not closed under e -> e^perp");
            return DVM_E_UNSUPPORTED;
        }
        used[i] = used[k] = 1;
        const bool li = P->is_local[i], lk = P->is_local[k];
        if (!li && !lk) continue;
        Unit2D U;
        // pass 2 (coalesced) takes the direction with an odd first component
        const bool i_second = (e0 & 1) != 0;
        const int sA = i_second ? k : i, sB = i_second ? i : k;
        U.a0 = P->h_e[3 * sA];
        U.a1 = P->h_e[3 * sA + 1];
        U.b0 = P->h_e[3 * sB];
        U.b1 = P->h_e[3 * sB + 1];
        U.M = P->h_M[i];
        U.flags = (P->is_local[sA] ? 1 : 0) | (P->is_local[sB] ? 2 : 0);
        U.aw = P->h_a[i];
        units.push_back(U);
    }
    P->g.nunits = (int)units.size();
    int maxitems = 1;
    for (const Unit2D &U : units)
        maxitems = std::max({maxitems, walk_items(walk_shape(U.a0, P->N), P->N), walk_items(walk_shape(U.b0, P->N), P->N)});
    P->g.maxitems2d = maxitems;
    P->g.h_units2d.assign(reinterpret_cast<const char *>(units.data()),
                          reinterpret_cast<const char *>(units.data() + units.size()));
    if (!units.empty()) {
        DVM_CUDA(cudaMalloc(&P->g.units, sizeof(Unit2D) * units.size()));
        DVM_CUDA(cudaMemcpyAsync(P->g.units, units.data(), sizeof(Unit2D) * units.size(), cudaMemcpyHostToDevice,
                                 P->stream));
        P->g.bytes += sizeof(Unit2D) * units.size();
    }
    dvm_status_t st = build_loss(P);
    if (st) return st;
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    P->g.ready = true;
    return DVM_OK;
}

size_t pair2d_unit_bytes() { return sizeof(Unit2D); }

dvm_status_t collide_small2d_parts(dvm_plan_s *P, const double *f, bool *handled)
{
    return collide_small2d(P, f, P->N * P->N, nullptr, 0, 1, handled);
}

dvm_status_t collide_pair2d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                            int64_t ncells, bool *handled)
{
    *handled = false;
    if (P->d != 2 || !P->g.ready || ncells <= 0) return DVM_OK;
    *handled = true;
    const int N = P->N, p = P->p;
    const int64_t nodes = (int64_t)N * N;
    // loss: Q := −f Λ for all cells
    dvm_status_t st = loss_init(P, f, f_stride, Q, q_stride, ncells, nullptr);
    if (st) return st;
    const int nunits = P->g.nunits;
    if (nunits == 0) return DVM_OK;
    // the tile kernel when its tile + halo fits shared memory and the batch has enough
    // tiles for most SMs (c3: 128 tiles; dvm_set_path 7 forces it, 2 the line walks)
    const int64_t ntiles = (int64_t)(N / kTileC) * (N / kTile) * ncells;
    // tile rows R <= 16 minimising (waves of CTAs) x R: c3 (one 256^2 grid) takes
    // R = 15, 18 x 8 = 144 CTAs in one wave instead of 128 of 16 rows (the last
    // row of tiles ragged); ties keep 16
    int R = kTile;
    {
        int sms = 148, dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        auto cost = [&](int r) {
            const int64_t tl = (int64_t)(N / kTileC) * ((N + r - 1) / r) * ncells;
            return ((tl + sms - 1) / sms) * r;
        };
        for (int r = kTile - 1; r >= 8; --r)
            if (cost(r) < cost(R)) R = r;
    }
    const size_t tsm = tile2d_smem(P->Ntilde, nunits, R);
    const unsigned tile_rows = (unsigned)((N + R - 1) / R);
    const bool tile = P->path_mode != 2 && N >= kTileC && tsm <= 227u * 1024u &&
                      (P->path_mode == 7 || ntiles >= 96);
    if (tile) {
        static std::mutex mu;
        static std::vector<size_t> set_to;
        int dev = 0;
        DVM_CUDA(cudaGetDevice(&dev));
        {
            std::lock_guard<std::mutex> lk(mu);
            if ((int)set_to.size() <= dev) set_to.resize(dev + 1, 0);
            if (set_to[dev] < tsm) {
                DVM_CUDA(cudaFuncSetAttribute(k_tile2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
                DVM_CUDA(cudaFuncSetAttribute(k_tile2d_pu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
                set_to[dev] = tsm;
            }
        }
        for (int64_t c0 = 0; c0 < ncells; c0 += 65535) {
            const int nc = (int)std::min<int64_t>(65535, ncells - c0);
            LaunchScope ls(P, KC_PAIR2D);
            if (nunits <= kParamUnits && (int)P->g.h_units2d.size() == nunits * (int)sizeof(Unit2D)) {
                TileUnits pu;
                std::memcpy(pu.u, P->g.h_units2d.data(), sizeof(Unit2D) * (size_t)nunits);
                k_tile2d_pu<<<dim3(N / kTileC, tile_rows, nc), R * kTileC, tsm, P->stream>>>(
                    f + c0 * f_stride, f_stride, nunits, N, P->Ntilde, Q + c0 * q_stride, q_stride, R, pu);
            } else {
                k_tile2d<<<dim3(N / kTileC, tile_rows, nc), R * kTileC, tsm, P->stream>>>(
                    f + c0 * f_stride, f_stride, reinterpret_cast<const Unit2D *>(P->g.units), nunits, N, P->Ntilde,
                    Q + c0 * q_stride, q_stride, R);
            }
            DVM_CUDA(cudaGetLastError());
        }
        return DVM_OK;
    }
    // the line-walk kernels: cell chunks bounded by the scratch + partial budget
    const size_t per_cell = sizeof(double) * 2 * (size_t)nunits * nodes;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(ncells, (int64_t)((512ull << 20) / per_cell)));
    Workspace &w = P->ws;
    if ((st = grow(&w.p2_scr, &w.p2_scr_elems, (size_t)(chunk * nunits * nodes), P->stream))) return st;
    if ((st = grow(&w.p2_part, &w.p2_part_elems, (size_t)(chunk * nunits * nodes), P->stream))) return st;
    const int items = P->g.maxitems2d;  // largest walk of any unit (shorter walks exit early)
    for (int64_t c0 = 0; c0 < ncells; c0 += chunk) {
        const int nc = (int)std::min<int64_t>(chunk, ncells - c0);
        dim3 grid((items + kPT - 1) / kPT, nunits, nc);
        {
            LaunchScope ls(P, KC_WLINE2D);
            k_wline2d<<<grid, kPT, 0, P->stream>>>(f + c0 * f_stride, f_stride, nc,
                                                   reinterpret_cast<const Unit2D *>(P->g.units), p, N, P->pk.H,
                                                   w.p2_scr);
        }
        {
            LaunchScope ls(P, KC_PAIR2D);
            k_pair2d<<<grid, kPT, 0, P->stream>>>(f + c0 * f_stride, f_stride, nc,
                                                  reinterpret_cast<const Unit2D *>(P->g.units), p, N, P->pk.H,
                                                  w.p2_scr, w.p2_part);
        }
        {
            LaunchScope ls(P, KC_REDUCE);
            k_sum_units<<<592, 256, 0, P->stream>>>(w.p2_part, nunits, nc, nodes, Q + c0 * q_stride, q_stride);
        }
        DVM_CUDA(cudaGetLastError());
    }
    return DVM_OK;
}

}  // namespace dvm
