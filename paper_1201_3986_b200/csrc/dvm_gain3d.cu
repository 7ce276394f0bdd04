// dvm_gain3d.cu -- 3D evaluation of Q = D^{Ñ,N̄}(f,f) on B200 (sm_100a, fp64).
//
// The operator (eq:decD) splits into gain and loss:
//   Q = G − f Λ,   G = Σ_e a_e S_e T_e,   Λ = Σ_e a_e Σ_{m≠0} T_e(.+me) = λ ⊛ f
// with the fixed kernel λ(j) = Σ_e a_e #{(m, l) : 1<=|m|<=M_e, l ∈ P_e,
// me + l ≡ j (mod N)} (β̃ = β − β(L,L); the loss is the
// β(L,L) convolution the paper evaluates spectrally).
//
//   loss  Λ: one batched 3D FFT convolution per pair of cells (f_{2p} + i
//        f_{2p+1} packed; λ̂ is real because λ is even), hand-written radix-2
//        passes in shared memory; the last inverse pass writes Q := −f Λ.
//   gain  G: a persistent cooperative kernel; a group of CL CTAs owns one cell
//        at a time and walks the directions.  Per direction:
//          phase A (frame): each CTA takes pairs of lattice planes x.e = γ,
//            gathers them in 16-byte runs {x, x + ê_2}, builds in-row prefix
//            sums in shared memory and evaluates T_e by the sliding program of
//            dvm_frame.h; T_e is written back in storage order (L2-resident
//            ping-pong buffer of the group).
//          group barrier
//          phase B (storage order): every CTA owns a fixed slab of nodes and
//            accumulates Q += a_e T_e S_e, S_e = Σ_{1<=|m|<=M_e} f(.+me)
//            read as coalesced stencil taps.
// Q accumulates in direction order per node: bitwise deterministic.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "dvm_frame.h"
#include "dvm_internal.h"

namespace dvm {
namespace {

constexpr int kGT = 512;        // threads per gain CTA (1 CTA per SM)
constexpr int kCL = 16;         // CTAs per cell group
constexpr int kMaxProg = 448;   // program entries (init + step) held in shared memory
constexpr int kMeta = 24;       // ints of per-direction metadata
constexpr int kMaxMS = 32;      // line half-width M_e held in shared memory
constexpr int kFT = 256;        // FFT threads per CTA

// ------------------------------------------------------------------ FFT
struct FftArgs {
    int d, ax, inverse;
    int64_t npairs;
    // real input (first forward pass): cells 2p, 2p+1 of r0 (cell stride r_stride, r_cells cells)
    const double *r0;
    int64_t r_stride, r_cells, r_first;  // r_first: index of the batch's first cell
    const double2 *zin;
    double2 *zout;
    const double *mult;  // optional real multiplier per node (λ̂)
    // epilogue (last inverse pass): Q[c] = -f[c] * Λ[c]
    double *q;
    int64_t q_stride;
    const double *f;
    int64_t f_stride;
    double scale;
    const double2 *tw;  // exp(-2πik/N), k < N/2
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// One radix-2 FFT pass of length N along axis `ax` for every line of every
// pair in the batch.  Tile = B lines (contiguous rows for the last axis,
// lines adjacent in the last axis otherwise).
template <int N>
__global__ void __launch_bounds__(kFT) k_fft_pass(FftArgs A)
{
    constexpr int B = (1024 / N) < N ? (1024 / N) : N;
    constexpr int LOGN = N == 16 ? 4 : N == 32 ? 5 : N == 64 ? 6 : N == 128 ? 7 : 8;
    __shared__ double2 buf[B * N];
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
    for (int half = 1; half < N; half <<= 1) {
        for (int b = threadIdx.x; b < B * N / 2; b += kFT) {
            const int i = b / (N / 2), k = b % (N / 2);
            const int pos = k & (half - 1), grp = k / half;
            const int i0 = grp * 2 * half + pos, i1 = i0 + half;
            double2 w = A.tw[pos * (N / (2 * half))];
            if (A.inverse) w.y = -w.y;
            const double2 u = buf[i * N + i0], v = cmul(buf[i * N + i1], w);
            buf[i * N + i0] = make_double2(u.x + v.x, u.y + v.y);
            buf[i * N + i1] = make_double2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < B * N; idx += kFT) {
        int i, t;
        if (last_axis) { i = idx / N; t = idx % N; }
        else { i = idx % B; t = idx / B; }
        const int64_t a = addr(i, t);
        double2 v = buf[i * N + t];
        if (A.mult) {
            const double m = A.mult[a];
            v.x *= m;
            v.y *= m;
        }
        if (A.q) {
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

// λ(j) = Σ_e a_e #{(m, l): 1 <= |m| <= M_e, l ∈ e^⊥ ∩ [-Ñ,Ñ]^3, me + l ≡ j},
// one thread per node j, directions in local-list order (deterministic).
__global__ void k_lambda(int N, int p, int Nt, const int *local, int nloc, const int *E, const int *M,
                         const double *aw, double *lam)
{
    const int64_t nodes = (int64_t)N * N * N;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nodes) return;
    const int jc[3] = {(int)(j >> (2 * p)), (int)((j >> p) & (N - 1)), (int)(j & (N - 1))};
    double acc = 0.0;
    for (int k = 0; k < nloc; ++k) {
        const int di = local[k];
        const int e0 = E[3 * di], e1 = E[3 * di + 1], e2 = E[3 * di + 2];
        const int m_e = M[di];
        int cnt = 0;
        for (int m = 1; m <= m_e; ++m)
            for (int s = -1; s <= 1; s += 2) {
                int l[3];
                const int ee[3] = {e0, e1, e2};
                bool ok = true;
                for (int q = 0; q < 3; ++q) {
                    int v = (jc[q] - s * m * ee[q]) % N;
                    if (v < 0) v += N;
                    if (v > N / 2) v -= N;  // centred representative (|l| <= Ñ < N/2)
                    l[q] = v;
                    if (v > Nt || v < -Nt) ok = false;
                }
                if (ok && l[0] * e0 + l[1] * e1 + l[2] * e2 == 0) ++cnt;
            }
        if (cnt) acc += aw[di] * cnt;
    }
    lam[j] = acc;
}

__global__ void k_take_real(const double2 *z, int64_t n, double *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = z[i].x;
}

// ------------------------------------------------------------------ gain
struct GainArgs {
    const double *f;
    int64_t f_stride;
    double *Q;  // accumulation target: [nchunks][ncells] blocks (see qc())
    int64_t q_stride, q_chunk_stride;
    int64_t ncells;
    int nchunks;
    int nloc;
    const int *meta;    // [nloc][kMeta]
    const int4 *prog;   // program entries
    const double *aw;   // [nloc]
    double *Tbuf;       // [groups][2][nodes]
    unsigned int *ctr;  // [groups] barrier counters
    uint32_t H;
    int p;
    int dbg;
};

__device__ __forceinline__ void group_barrier(unsigned int *ctr, unsigned int target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned int v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= target) break;
            __nanosleep(20);
        }
    }
    __syncthreads();
}

template <int N>
__device__ __forceinline__ uint32_t pk(int c0, int c1, int c2)
{
    constexpr int P = N == 32 ? 5 : 6;
    return ((uint32_t)(c0 & (N - 1)) << (2 * P)) | ((uint32_t)(c1 & (N - 1)) << P) | (uint32_t)(c2 & (N - 1));
}

// Shared-memory geometry of the gain kernel: planes are stored with L-1
// duplicated rows (row N + k == row k) so that the L consecutive β-steps of a
// thread address rows r0 .. r0 + L - 1 without wrap logic.
template <int N>
struct G3Geom {
    static constexpr int LOGN = N == 32 ? 5 : 6;
    static constexpr int NN = N * N;
    static constexpr int SEGS = kGT / (2 * N);  // β segments per column
    static constexpr int L = N / SEGS;           // outputs per segment
    static constexpr int ROWS = N + L - 1;       // stored rows per plane
    static constexpr int PL = ROWS * N;          // doubles per stored plane
    static constexpr size_t smem = sizeof(double) * (4 * (size_t)PL + 2 * ROWS) + sizeof(int4) * kMaxProg +
                                   sizeof(uint32_t) * 2 * kMaxMS;
};

template <int N>
__global__ void __launch_bounds__(kGT, 1) k_gain3d(GainArgs A)
{
    using Gm = G3Geom<N>;
    constexpr int LOGN = Gm::LOGN;
    constexpr int NN = Gm::NN;
    constexpr int64_t NODES = (int64_t)N * N * N;
    constexpr int SEGS = Gm::SEGS;
    constexpr int L = Gm::L;
    constexpr int ROWS = Gm::ROWS;
    constexpr int PL = Gm::PL;
    constexpr int NPR = (int)(NODES / kCL);   // phase-B nodes per CTA
    constexpr int GIT = 2 * NN / kGT;          // gathered nodes per thread per slab
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *raw = reinterpret_cast<double *>(smem_raw);   // [2][ROWS][N] (T overlays it after phase A3)
    double *pre = raw + 2 * PL;                            // [2][ROWS][N] in-row prefix sums
    double *tot = pre + 2 * PL;                            // [2][ROWS] row totals
    int4 *sprog = reinterpret_cast<int4 *>(tot + 2 * ROWS);  // [kMaxProg]
    uint32_t *soff = reinterpret_cast<uint32_t *>(sprog + kMaxProg);  // [2 * kMaxMS]
    __shared__ int sm[kMeta];

    const int tid = threadIdx.x;
    const int rank = (int)(blockIdx.x % kCL);
    const int grp = (int)(blockIdx.x / kCL);
    const int ngroups = (int)(gridDim.x / kCL);
    const uint32_t H = A.H;
    unsigned int epoch = 0;
    unsigned int step = 0;
    const int64_t items = A.ncells * A.nchunks;

    for (int64_t item = grp; item < items; item += ngroups) {
        const int64_t cell = item / A.nchunks;
        const int chunk = (int)(item % A.nchunks);
        const int d0 = (int)((int64_t)A.nloc * chunk / A.nchunks);
        const int d1 = (int)((int64_t)A.nloc * (chunk + 1) / A.nchunks);
        const double *__restrict__ fc = A.f + cell * A.f_stride;
        double *Qc = A.Q + chunk * A.q_chunk_stride + cell * A.q_stride;

        for (int di = d0; di < d1; ++di, ++step) {
            __syncthreads();  // previous direction's phase B done with sm/soff
            if (tid < kMeta) sm[tid] = A.meta[di * kMeta + tid];
            __syncthreads();
            const int nprog = sm[16] + sm[17];
            for (int k = tid; k < nprog && k < kMaxProg; k += kGT) sprog[k] = A.prog[sm[18] + k];
            {
                const int M = sm[15];
                if (tid < 2 * M) {
                    const int m = tid / 2 + 1, s = (tid & 1) ? -1 : 1;
                    soff[tid] = pk<N>(s * m * sm[0], s * m * sm[1], s * m * sm[2]);
                }
            }
            __syncthreads();
            double *Tb = A.Tbuf + ((int64_t)grp * 2 + (step & 1)) * NODES;

            // ---------------------------------------------------------- phase A
            if (!(A.dbg & 1)) {
                const int z0 = sm[3], z1 = sm[4], z2 = sm[5];
                const int u0 = sm[6], u1 = sm[7], u2 = sm[8];
                const int w0 = sm[9], w1 = sm[10], w2 = sm[11];
                const int a2 = sm[12], b2 = sm[13];
                const int rows_mode = sm[14];
                const int e2m = sm[2] & (N - 1);
                const int ninit = sm[16], nstep = sm[17];
                const int gg = rows_mode ? 1 : (e2m & -e2m);  // gcd(e2, N)
                // per-thread gather/scatter pattern: GIT nodes, fixed column and plane,
                // rows advancing by a constant (packed storage step sx)
                int gj, gal, gbe0, gdbe;
                if (rows_mode) {
                    gj = 0;  // plane switches half-way (k >= GIT/2)
                    gal = tid & (N - 1);
                    gbe0 = tid >> LOGN;
                    gdbe = kGT >> LOGN;
                } else {
                    gj = tid & 1;
                    gal = (tid >> 1) & (N - 1);
                    gbe0 = (tid >> 1) >> LOGN;
                    gdbe = (kGT / 2) >> LOGN;
                }
                const uint32_t sx = pk<N>(gdbe * w0, gdbe * w1, gdbe * w2);
                for (int s = rank; s < N / 2; s += kCL) {
                    int g0, g1;
                    if (rows_mode) {
                        g0 = 2 * s;
                        g1 = 2 * s + 1;
                    } else {
                        const int c = s % gg, i = s / gg;
                        g0 = (c + 2 * i * e2m) & (N - 1);
                        g1 = (g0 + e2m) & (N - 1);
                    }
                    // A1: gather (16-byte runs {x, x + ê_2}, or contiguous rows)
                    {
                        const int sal = rows_mode ? gal : ((gal + gj * a2) & (N - 1));
                        const int g = g0;
                        uint32_t x = pk<N>(g * z0 + gal * u0 + gbe0 * w0, g * z1 + gal * u1 + gbe0 * w1,
                                           g * z2 + gal * u2 + gbe0 * w2 + (rows_mode ? 0 : gj));
                        double v[GIT];
#pragma unroll
                        for (int k = 0; k < GIT; ++k) {
                            if (rows_mode && k == GIT / 2)
                                x = pk<N>(g1 * z0 + gal * u0 + gbe0 * w0, g1 * z1 + gal * u1 + gbe0 * w1,
                                          g1 * z2 + gal * u2 + gbe0 * w2);
                            v[k] = __ldg(fc + x);
                            x = swar_add(x, sx, H);
                        }
#pragma unroll
                        for (int k = 0; k < GIT; ++k) {
                            int j, row;
                            if (rows_mode) {
                                j = k >= GIT / 2;
                                row = (gbe0 + (k % (GIT / 2)) * gdbe) & (N - 1);
                            } else {
                                j = gj;
                                row = (gbe0 + k * gdbe + gj * b2) & (N - 1);
                            }
                            double *dst = raw + j * PL + row * N + sal;
                            dst[0] = v[k];
                            if (row < L - 1) dst[NN] = v[k];
                        }
                    }
                    __syncthreads();
                    // A2: in-row prefix sums of all stored rows (periodic rows; totals apart)
                    {
                        const int lane = tid & 31, warp = tid >> 5;
                        constexpr int PLN = N / 32;
                        for (int row = warp; row < 2 * ROWS; row += kGT / 32) {
                            const double *src = raw + row * N;
                            double v[PLN];
#pragma unroll
                            for (int q = 0; q < PLN; ++q) v[q] = src[lane * PLN + q];
#pragma unroll
                            for (int q = 1; q < PLN; ++q) v[q] += v[q - 1];
                            double x = v[PLN - 1];
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const double y = __shfl_up_sync(0xffffffffu, x, o);
                                if (lane >= o) x += y;
                            }
                            const double excl = x - v[PLN - 1];
                            double *dst = pre + row * N;
#pragma unroll
                            for (int q = 0; q < PLN; ++q) dst[lane * PLN + q] = v[q] + excl;
                            if (lane == 31) tot[row] = x;
                        }
                    }
                    __syncthreads();
                    // A3: T by the sliding program; thread = (plane j, column al, β segment)
                    {
                        const int j = tid / (N * SEGS);
                        const int rem = tid % (N * SEGS);
                        const int al = rem & (N - 1), sg = rem >> LOGN;
                        const double *R = raw + j * PL;
                        const double *Pp = pre + j * PL;
                        const double *Tt = tot + j * ROWS;
                        const int be0 = sg * L;
                        double T[L];
                        {
                            double acc = 0.0;
                            for (int k = 0; k < ninit; ++k) {
                                const int4 en = sprog[k];
                                const int r0 = (be0 + en.x) & (N - 1);
                                const int b = al + en.z, a = al + en.y - 1;
                                double v = Pp[r0 * N + (b & (N - 1))] - Pp[r0 * N + (a & (N - 1))];
                                if ((b >> LOGN) != (a >> LOGN)) v += Tt[r0];
                                acc += v;
                            }
                            T[0] = acc;
                        }
#pragma unroll
                        for (int q = 1; q < L; ++q) T[q] = 0.0;
                        // T[q] (q >= 1) collects the step difference D(β0 + q − 1)
                        for (int k = ninit; k < ninit + nstep; ++k) {
                            const int4 en = sprog[k];
                            const int r0 = (be0 + en.x) & (N - 1);
                            const double sgn = (double)en.w;
                            if (en.y == en.z) {
                                const double *q0 = R + r0 * N + ((al + en.y) & (N - 1));
#pragma unroll
                                for (int q = 1; q < L; ++q) T[q] = fma(sgn, q0[(q - 1) * N], T[q]);
                            } else {
                                const int b = al + en.z, a = al + en.y - 1;
                                const double *qb = Pp + r0 * N + (b & (N - 1));
                                const double *qa = Pp + r0 * N + (a & (N - 1));
                                if ((b >> LOGN) != (a >> LOGN)) {
                                    const double *qt = Tt + r0;
#pragma unroll
                                    for (int q = 1; q < L; ++q)
                                        T[q] = fma(sgn, (qb[(q - 1) * N] - qa[(q - 1) * N]) + qt[q - 1], T[q]);
                                } else {
#pragma unroll
                                    for (int q = 1; q < L; ++q)
                                        T[q] = fma(sgn, qb[(q - 1) * N] - qa[(q - 1) * N], T[q]);
                                }
                            }
                        }
#pragma unroll
                        for (int q = 1; q < L; ++q) T[q] += T[q - 1];
                        __syncthreads();  // every thread is done reading raw: overlay T on it
                        double *To = raw + j * PL + al;
#pragma unroll
                        for (int q = 0; q < L; ++q) To[(be0 + q) * N] = T[q];
                    }
                    __syncthreads();
                    // A4: write T back in storage order (same runs as the gather)
                    {
                        const int sal = rows_mode ? gal : ((gal + gj * a2) & (N - 1));
                        uint32_t x = pk<N>(g0 * z0 + gal * u0 + gbe0 * w0, g0 * z1 + gal * u1 + gbe0 * w1,
                                           g0 * z2 + gal * u2 + gbe0 * w2 + (rows_mode ? 0 : gj));
#pragma unroll
                        for (int k = 0; k < GIT; ++k) {
                            int j, row;
                            if (rows_mode) {
                                if (k == GIT / 2)
                                    x = pk<N>(g1 * z0 + gal * u0 + gbe0 * w0, g1 * z1 + gal * u1 + gbe0 * w1,
                                              g1 * z2 + gal * u2 + gbe0 * w2);
                                j = k >= GIT / 2;
                                row = (gbe0 + (k % (GIT / 2)) * gdbe) & (N - 1);
                            } else {
                                j = gj;
                                row = (gbe0 + k * gdbe + gj * b2) & (N - 1);
                            }
                            __stcg(Tb + x, raw[j * PL + row * N + sal]);
                            x = swar_add(x, sx, H);
                        }
                    }
                    // (the next slab's A1 rewrites raw only after every thread passed A4:
                    //  A1 of the next slab is separated by the barrier below)
                    __syncthreads();
                }
            }
            ++epoch;
            group_barrier(A.ctr + grp, epoch * (unsigned)kCL);

            // ---------------------------------------------------------- phase B
            if (!(A.dbg & 2)) {
                constexpr int NB = (NPR / kGT) < 8 ? (NPR / kGT) : 8;
                static_assert(NPR % (kGT * NB) == 0, "phase-B tiling");
                const double aw = A.aw[di];
                const int M2 = 2 * sm[15];
                const uint32_t n0 = (uint32_t)rank * NPR;
                for (int i0 = tid; i0 < NPR; i0 += kGT * NB) {
                    uint32_t n[NB];
                    double T[NB], S[NB];
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        n[b] = n0 + i0 + b * kGT;
                        T[b] = __ldcg(Tb + n[b]);
                        S[b] = 0.0;
                    }
                    for (int k = 0; k < M2; ++k) {
                        const uint32_t off = soff[k];
#pragma unroll
                        for (int b = 0; b < NB; ++b) S[b] += __ldg(fc + swar_add(n[b], off, H));
                    }
#pragma unroll
                    for (int b = 0; b < NB; ++b) Qc[n[b]] += aw * T[b] * S[b];
                }
            }
        }
    }
}

size_t gain_smem_bytes(int N) { return N == 32 ? G3Geom<32>::smem : G3Geom<64>::smem; }

template <typename T>
dvm_status_t grow(T **ptr, size_t *cap, size_t need, cudaStream_t s)
{
    if (*cap >= need) return DVM_OK;
    DVM_CUDA(cudaStreamSynchronize(s));
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    *cap = 0;
    if (cudaMalloc(ptr, sizeof(T) * need) != cudaSuccess) {
        *ptr = nullptr;
        cudaGetLastError();
        set_error("gain3d workspace allocation failed");
        return DVM_E_NOMEM;
    }
    *cap = need;
    return DVM_OK;
}

template <int N>
dvm_status_t fft_pass(dvm_plan_s *P, const FftArgs &a)
{
    constexpr int B = (1024 / N) < N ? (1024 / N) : N;
    int64_t nodes = 1;
    for (int j = 0; j < a.d; ++j) nodes *= N;
    const int64_t tiles = a.npairs * (nodes / N / B);
    LaunchScope ls(P, KC_FFT);
    k_fft_pass<N><<<(unsigned)tiles, kFT, 0, P->stream>>>(a);
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

// Loss initialisation Q[c] := −f[c] Λ[c] for cells [0, ncells) (Λ = λ ⊛ f).
dvm_status_t loss_init(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride, int64_t ncells)
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
    for (int64_t p0 = 0; p0 < npairs_all; p0 += batch) {
        const int64_t np = std::min(batch, npairs_all - p0);
        for (int k = 0; k < 2 * d; ++k) {
            FftArgs a = {};
            a.d = d;
            a.npairs = np;
            a.tw = P->g.tw;
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
            if (k == d - 1) a.mult = P->g.lamhat;
            if (k == 2 * d - 1) {
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

template <int N>
dvm_status_t launch_gain(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                         int64_t ncells)
{
    auto kern = k_gain3d<N>;
    const size_t smem = gain_smem_bytes(N);
    DVM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    DVM_CUDA(cudaGetDevice(&dev));
    DVM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DVM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    DVM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGT, smem));
    if (!coop || per_sm < 1) {
        set_error("gain3d kernel cannot be launched cooperatively on this device");
        return DVM_E_CUDA;
    }
    int max_groups = (sms * per_sm) / kCL;
    if (getenv("DVM_G3_GROUPS")) max_groups = std::max(1, std::min(max_groups, atoi(getenv("DVM_G3_GROUPS"))));
    const int nloc = (int)P->local.size();
    const int64_t nodes = (int64_t)N * N * N;
    int nchunks = 1;
    if (ncells < max_groups) nchunks = (int)std::min<int64_t>(nloc, max_groups / ncells);
    nchunks = std::max(1, nchunks);
    const int64_t items = ncells * nchunks;
    const int ngroups = (int)std::min<int64_t>(max_groups, items);
    Workspace &w = P->ws;
    dvm_status_t st;
    if ((st = grow(&w.g3_t, &w.g3_t_elems, (size_t)ngroups * 2 * nodes, P->stream))) return st;
    if ((st = grow(&w.g3_ctr, &w.g3_ctr_elems, (size_t)ngroups, P->stream))) return st;
    double *Qacc = Q;
    int64_t qs = q_stride, qcs = 0;
    if (nchunks > 1) {
        if ((st = grow(&w.g3_q, &w.g3_q_elems, (size_t)nchunks * ncells * nodes, P->stream))) return st;
        Qacc = w.g3_q;
        qs = nodes;
        qcs = ncells * nodes;
        DVM_CUDA(cudaMemsetAsync(w.g3_q + qcs, 0, sizeof(double) * (size_t)(nchunks - 1) * qcs, P->stream));
    }
    // loss first: Q_acc(chunk 0) := −f Λ
    if ((st = loss_init(P, f, f_stride, Qacc, qs, ncells))) return st;
    DVM_CUDA(cudaMemsetAsync(w.g3_ctr, 0, sizeof(unsigned int) * ngroups, P->stream));
    GainArgs a;
    a.f = f;
    a.f_stride = f_stride;
    a.Q = Qacc;
    a.q_stride = qs;
    a.q_chunk_stride = qcs;
    a.ncells = ncells;
    a.nchunks = nchunks;
    a.nloc = nloc;
    a.meta = P->g.meta;
    a.prog = P->g.prog;
    a.aw = P->g.aw;
    a.Tbuf = w.g3_t;
    a.ctr = w.g3_ctr;
    a.H = P->pk.H;
    a.p = P->p;
    a.dbg = getenv("DVM_G3_DEBUG") ? atoi(getenv("DVM_G3_DEBUG")) : 0;
    if (getenv("DVM_VERBOSE"))
        fprintf(stderr, "[dvm] gain3d N=%d: %d groups x %d CTAs, %d chunks, smem %zu\n", N, ngroups, kCL, nchunks,
                smem);
    {
        void *args[] = {&a};
        LaunchScope ls(P, KC_GAIN3D);
        DVM_CUDA(cudaLaunchCooperativeKernel((void *)kern, dim3(ngroups * kCL), dim3(kGT), args, smem, P->stream));
    }
    if (nchunks > 1) {
        if ((st = zero_cells(P, Q, q_stride, ncells, nodes))) return st;
        if ((st = reduce_slots(P, Q, q_stride, w.g3_q, ncells * nodes, nchunks, ncells, nodes))) return st;
    }
    return DVM_OK;
}

}  // namespace

// Plan-time setup of the 3D path: frames + programs of the local directions,
// twiddles, the loss kernel λ and its spectrum λ̂.
dvm_status_t build_gain3d(dvm_plan_s *P)
{
    if (P->d != 3 || (P->N != 32 && P->N != 64)) return DVM_OK;
    const int nloc = (int)P->local.size();
    const int N = P->N;
    const int SEGS = kGT / (2 * N), L = N / SEGS;
    std::vector<int> meta((size_t)std::max(1, nloc) * kMeta, 0);
    std::vector<int4> prog;
    std::vector<double> aw(std::max(1, nloc), 0.0);
    for (int k = 0; k < nloc; ++k) {
        const int di = P->local[k];
        frame::DirFrame F;
        if (!frame::build_dir(&P->h_e[3 * di], P->Ntilde, N, L, F)) {
            set_error("gain3d: no frame for a direction");
            return DVM_E_UNSUPPORTED;
        }
        if ((int)(F.init.size() + F.step.size()) > kMaxProg || F.M > kMaxMS / 2) {
            set_error("gain3d: direction program exceeds the shared-memory table");
            return DVM_E_UNSUPPORTED;
        }
        int *m = &meta[(size_t)k * kMeta];
        for (int j = 0; j < 3; ++j) {
            m[j] = F.e[j];
            m[3 + j] = F.z[j];
            m[6 + j] = F.u[j];
            m[9 + j] = F.w[j];
        }
        m[12] = F.a2;
        m[13] = F.b2;
        m[14] = F.rows_mode;
        m[15] = F.M;
        m[16] = (int)F.init.size();
        m[17] = (int)F.step.size();
        m[18] = (int)prog.size();
        for (const auto &x : F.init) prog.push_back(make_int4(x.rho, x.t1, x.t2, x.sign));
        for (const auto &x : F.step) prog.push_back(make_int4(x.rho, x.t1, x.t2, x.sign));
        aw[k] = P->h_a[di];
    }
    if (prog.empty()) prog.push_back(make_int4(0, 0, 0, 0));
    GainTables &g = P->g;
    DVM_CUDA(cudaMalloc(&g.meta, sizeof(int) * meta.size()));
    DVM_CUDA(cudaMalloc(&g.prog, sizeof(int4) * prog.size()));
    DVM_CUDA(cudaMalloc(&g.aw, sizeof(double) * aw.size()));
    DVM_CUDA(cudaMalloc(&g.tw, sizeof(double2) * N / 2));
    const int64_t nodes = (int64_t)N * N * N;
    DVM_CUDA(cudaMalloc(&g.lamhat, sizeof(double) * nodes));
    g.bytes = sizeof(int) * meta.size() + sizeof(int4) * prog.size() + sizeof(double) * aw.size() +
              sizeof(double2) * N / 2 + sizeof(double) * nodes;
    DVM_CUDA(cudaMemcpyAsync(g.meta, meta.data(), sizeof(int) * meta.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(g.prog, prog.data(), sizeof(int4) * prog.size(), cudaMemcpyHostToDevice, P->stream));
    DVM_CUDA(cudaMemcpyAsync(g.aw, aw.data(), sizeof(double) * aw.size(), cudaMemcpyHostToDevice, P->stream));
    {
        LaunchScope ls(P, KC_PLAN);
        k_twiddles<<<1, 128, 0, P->stream>>>(N, g.tw);
    }
    // λ on the grid, then λ̂ = FFT(λ) (real: λ is even)
    double *lam = nullptr;
    double2 *z = nullptr;
    DVM_CUDA(cudaMalloc(&lam, sizeof(double) * nodes));
    DVM_CUDA(cudaMalloc(&z, sizeof(double2) * nodes));
    {
        LaunchScope ls(P, KC_PLAN);
        k_lambda<<<(unsigned)((nodes + 127) / 128), 128, 0, P->stream>>>(N, P->p, P->Ntilde, P->t.local, nloc,
                                                                         P->t.e, P->t.M, P->t.a, lam);
    }
    DVM_CUDA(cudaGetLastError());
    dvm_status_t st = DVM_OK;
    for (int k = 0; k < 3 && !st; ++k) {
        FftArgs a = {};
        a.d = 3;
        a.npairs = 1;
        a.tw = g.tw;
        a.r_cells = 1;
        a.r_first = 0;
        a.ax = 2 - k;
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
        k_take_real<<<256, 256, 0, P->stream>>>(z, nodes, g.lamhat);
    }
    cudaStreamSynchronize(P->stream);
    cudaFree(lam);
    cudaFree(z);
    if (st) return st;
    DVM_CUDA(cudaGetLastError());
    g.ready = true;
    return DVM_OK;
}

void free_gain3d(dvm_plan_s *P)
{
    GainTables &g = P->g;
    void *ptrs[] = {g.meta, g.prog, g.aw, g.tw, g.lamhat};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    g = GainTables{};
}

dvm_status_t collide_gain3d(dvm_plan_s *P, const double *f, int64_t f_stride, double *Q, int64_t q_stride,
                            int64_t ncells, bool *handled)
{
    *handled = false;
    if (P->d != 3 || !P->g.ready || ncells <= 0) return DVM_OK;
    *handled = true;
    switch (P->N) {
    case 32: return launch_gain<32>(P, f, f_stride, Q, q_stride, ncells);
    case 64: return launch_gain<64>(P, f, f_stride, Q, q_stride, ncells);
    default: *handled = false; return DVM_OK;
    }
}

}  // namespace dvm
