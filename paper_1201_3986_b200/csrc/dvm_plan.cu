// dvm_plan.cu -- plan construction: direction table (K1) and per-direction
// geometry (K2) built on the device, once per plan.
//
// K1 (k_dirgen): the canonical primitive directions of order <= N̄ ("primal
//     representants of directions of lines"; Farey series
//     F^1 / F^2 of PAPER.md:597-681).  One thread per candidate of
//     [-N̄,N̄]^d; order-preserving block-scan compaction, so the table is in
//     lexicographic order (reading R7: brute-force enumeration replaces the
//     simplex subdivision of PAPER.md:915-920 and the over-counting closed form
//     of PAPER.md:674-677).
// K2 (k_dirmeta / k_dirrows): per direction e, M_e = floor(Ñ/|e|_inf), the
//     weight a_e = h^{d+1}|e|, and the perp set
//     P_e = e^⊥ ∩ [-Ñ,Ñ]^d as rows along a lattice vector u:
//     2D: P_e = {n e^⊥ : |n| <= M_e} (one row); 3D: an integer basis (u, w) of
//     the lattice e^⊥ ∩ Z^3 (Bezout basis, Lagrange-Gauss reduced) and the rows
//     {α u + β w : lo_β <= α <= hi_β} of the polygon.
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>
#include <numeric>

#include "dvm_internal.h"

namespace dvm {
namespace {

constexpr int kScanThreads = 1024;

__device__ __host__ inline int igcd(int a, int b)
{
    a = a < 0 ? -a : a;
    b = b < 0 ? -b : b;
    while (b) {
        int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

__device__ inline long long floor_div(long long a, long long b)
{
    long long q = a / b, r = a % b;
    if (r != 0 && ((r < 0) != (b < 0))) --q;
    return q;
}
__device__ inline long long ceil_div(long long a, long long b) { return -floor_div(-a, b); }

// Block-wide exclusive scan of one int per thread (blockDim.x == kScanThreads).
__device__ int block_exclusive_scan(int v, int *total)
{
    __shared__ int warp_sums[32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = warp_sums[lane];
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    int excl = x - v + (wid > 0 ? warp_sums[wid - 1] : 0);
    *total = warp_sums[31];
    __syncthreads();
    return excl;
}

// K1: single CTA sweeps the candidate cube in chunks; keeps lexicographic order.
__global__ void k_dirgen(int d, int Nbar, int *out_e, int cap, int *out_count)
{
    const int side = 2 * Nbar + 1;
    long long total = 1;
    for (int j = 0; j < d; ++j) total *= side;
    int base = 0;
    for (long long c0 = 0; c0 < total; c0 += blockDim.x) {
        long long c = c0 + threadIdx.x;
        int e[3] = {0, 0, 0};
        int flag = 0;
        if (c < total) {
            long long r = c;
            for (int j = d - 1; j >= 0; --j) {
                e[j] = (int)(r % side) - Nbar;
                r /= side;
            }
            int first = 0, g = 0;
            for (int j = 0; j < d; ++j) {
                if (!first && e[j] != 0) first = e[j];
                g = igcd(g, e[j]);
            }
            flag = (first > 0 && g == 1) ? 1 : 0;
        }
        int tot;
        int pos = base + block_exclusive_scan(flag, &tot);
        if (flag && pos < cap)
            for (int j = 0; j < 3; ++j) out_e[pos * 3 + j] = e[j];
        base += tot;
    }
    if (threadIdx.x == 0) *out_count = base;
}

__device__ inline void cross3(const long long *a, const long long *b, long long *c)
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

// Rows of P_e = {α u + β w : |α u_j + β w_j| <= Ñ  for j = 0..2}.  Calls
// emit(β, lo, hi) for every non-empty row in increasing β; returns the count.
template <typename F>
__device__ int enumerate_rows(const int *u, const int *w, const int *e, int Nt, F emit)
{
    double nu = sqrt((double)(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]));
    double ne = sqrt((double)(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]));
    // |β| = |(u × x)·e| / |e|^2 <= |u| sqrt(3) Ñ / |e| for x in the box
    int Bmax = (int)ceil(nu * 1.7320508075688772 * Nt / ne) + 2;
    int count = 0;
    for (int b = -Bmax; b <= Bmax; ++b) {
        long long lo = -(1LL << 40), hi = (1LL << 40);
        bool empty = false;
        for (int j = 0; j < 3; ++j) {
            long long c = u[j], s = (long long)b * w[j];
            if (c == 0) {
                if (s > Nt || s < -Nt) empty = true;
            } else if (c > 0) {
                lo = max(lo, ceil_div(-Nt - s, c));
                hi = min(hi, floor_div(Nt - s, c));
            } else {
                lo = max(lo, ceil_div(Nt - s, c));
                hi = min(hi, floor_div(-Nt - s, c));
            }
        }
        if (empty || lo > hi) continue;
        emit(b, (int)lo, (int)hi);
        ++count;
    }
    return count;
}

// Orbits of a primitive vector can be walked with warp lanes on consecutive
// fastest-axis nodes iff one of its non-fastest components is odd.
__device__ inline bool coalescable(const int *v, int d)
{
    for (int j = 0; j < d - 1; ++j)
        if (v[j] & 1) return true;
    return false;
}

// Integer basis (u, w) of e^⊥ ∩ Z^3 with u × w = e: Bezout basis
// v1 = (b/g, -a/g, 0), v2 = (c s, c t, -g) with a s + b t = g, then
// Lagrange-Gauss reduction; finally the row vector u is chosen among
// {v1, v2, v1+v2, v1-v2} to minimise the row count (coalescable preferred).
__device__ void perp_basis(const int *e, int Nt, int *u_out, int *w_out)
{
    long long a = e[0], b = e[1], c = e[2];
    long long v1[3], v2[3];
    int g = igcd((int)a, (int)b);
    if (g == 0) {  // e = (0,0,1)
        v1[0] = 1; v1[1] = 0; v1[2] = 0;
        v2[0] = 0; v2[1] = 1; v2[2] = 0;
    } else {
        // extended Euclid on |a|, |b|
        long long r0 = a < 0 ? -a : a, r1 = b < 0 ? -b : b, s0 = 1, s1 = 0, t0 = 0, t1 = 1;
        while (r1) {
            long long q = r0 / r1, tmp;
            tmp = r0 - q * r1; r0 = r1; r1 = tmp;
            tmp = s0 - q * s1; s0 = s1; s1 = tmp;
            tmp = t0 - q * t1; t0 = t1; t1 = tmp;
        }
        long long s = a < 0 ? -s0 : s0, t = b < 0 ? -t0 : t0;  // a s + b t = g
        v1[0] = b / g; v1[1] = -a / g; v1[2] = 0;
        v2[0] = c * s; v2[1] = c * t; v2[2] = -g;
    }
    for (int it = 0; it < 64; ++it) {  // Lagrange-Gauss reduction
        long long n1 = v1[0] * v1[0] + v1[1] * v1[1] + v1[2] * v1[2];
        long long n2 = v2[0] * v2[0] + v2[1] * v2[1] + v2[2] * v2[2];
        if (n2 < n1) {
            for (int j = 0; j < 3; ++j) {
                long long tmp = v1[j]; v1[j] = v2[j]; v2[j] = tmp;
            }
            long long tmp = n1; n1 = n2; n2 = tmp;
        }
        long long dot = v1[0] * v2[0] + v1[1] * v2[1] + v1[2] * v2[2];
        long long mu = floor_div(2 * dot + n1, 2 * n1);
        if (mu == 0) break;
        for (int j = 0; j < 3; ++j) v2[j] -= mu * v1[j];
    }
    long long cr[3];
    cross3(v1, v2, cr);
    if (cr[0] != a || cr[1] != b || cr[2] != c)
        for (int j = 0; j < 3; ++j) v2[j] = -v2[j];
    int cand_u[4][3], cand_w[4][3];
    for (int j = 0; j < 3; ++j) {
        cand_u[0][j] = (int)v1[j];          cand_w[0][j] = (int)v2[j];
        cand_u[1][j] = (int)v2[j];          cand_w[1][j] = (int)-v1[j];
        cand_u[2][j] = (int)(v1[j] + v2[j]); cand_w[2][j] = (int)v2[j];
        cand_u[3][j] = (int)(v1[j] - v2[j]); cand_w[3][j] = (int)v2[j];
    }
    int best = 0;
    long long best_score = -1;
    for (int k = 0; k < 4; ++k) {
        int n = enumerate_rows(cand_u[k], cand_w[k], e, Nt, [](int, int, int) {});
        long long score = (long long)n * (coalescable(cand_u[k], 3) ? 1 : 4);
        if (best_score < 0 || score < best_score) {
            best_score = score;
            best = k;
        }
    }
    for (int j = 0; j < 3; ++j) {
        u_out[j] = cand_u[best][j];
        w_out[j] = cand_w[best][j];
    }
}

// z with z.e = 1 (e primitive): Bezout on (a, b) -> g, then on (g, c) -> 1.
__device__ void transverse(const int *e, int *z)
{
    auto egcd = [](long long a, long long b, long long &x, long long &y) {
        long long r0 = a < 0 ? -a : a, r1 = b < 0 ? -b : b, s0 = 1, s1 = 0, t0 = 0, t1 = 1;
        while (r1) {
            long long q = r0 / r1, tmp;
            tmp = r0 - q * r1; r0 = r1; r1 = tmp;
            tmp = s0 - q * s1; s0 = s1; s1 = tmp;
            tmp = t0 - q * t1; t0 = t1; t1 = tmp;
        }
        x = a < 0 ? -s0 : s0;
        y = b < 0 ? -t0 : t0;
        return r0;
    };
    long long s, t, s2, t2;
    long long g = egcd(e[0], e[1], s, t);   // s e0 + t e1 = g
    egcd(g, e[2], s2, t2);                   // s2 g + t2 e2 = 1
    z[0] = (int)(s2 * s);
    z[1] = (int)(s2 * t);
    z[2] = (int)t2;
}

// K2a: one thread per direction.
__global__ void k_dirmeta(int d, int A, int Nt, double hd1, const int *E, int *M, double *aw, int *U,
                          int *W, int *Z, int *nrows, int *cost)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= A) return;
    int e[3] = {E[3 * t], E[3 * t + 1], E[3 * t + 2]};
    int inf = 0;
    long long n2 = 0;
    for (int j = 0; j < 3; ++j) {
        int c = e[j] < 0 ? -e[j] : e[j];
        inf = c > inf ? c : inf;
        n2 += (long long)e[j] * e[j];
    }
    int m = Nt / inf;
    M[t] = m;
    aw[t] = hd1 * sqrt((double)n2);  // a(me) = h^{d+1}|me|/|m|
    int u[3] = {0, 0, 0}, w[3] = {0, 0, 0}, z[3] = {0, 0, 0};
    int nr;
    if (d == 3) transverse(e, z);
    if (d == 2) {
        u[0] = -e[1];
        u[1] = e[0];
        nr = 1;
    } else {
        perp_basis(e, Nt, u, w);
        nr = enumerate_rows(u, w, e, Nt, [](int, int, int) {});
    }
    for (int j = 0; j < 3; ++j) {
        U[3 * t + j] = u[j];
        W[3 * t + j] = w[j];
        Z[3 * t + j] = z[j];
    }
    nrows[t] = nr;
    cost[t] = 4 * nr + 8;
}

__global__ void k_scan_rows(int A, const int *nrows, int *row_off)
{
    int base = 0;
    for (int c0 = 0; c0 < A; c0 += blockDim.x) {
        int c = c0 + threadIdx.x;
        int v = c < A ? nrows[c] : 0;
        int tot;
        int ex = block_exclusive_scan(v, &tot);
        if (c < A) row_off[c] = base + ex;
        base += tot;
    }
    if (threadIdx.x == 0) row_off[A] = base;
}

// K2b: fill the rows and their packed stencil offsets.
__global__ void k_dirrows(int d, int A, int Nt, int p, int N, const int *E, const int *M, const int *U,
                          const int *W, const int *row_off, int *rb, int *rlo, int *rhi, uint32_t *oin,
                          uint32_t *oout)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= A) return;
    const int *e = E + 3 * t, *u = U + 3 * t, *w = W + 3 * t;
    int base = row_off[t];
    auto emit = [&](int b, int lo, int hi) {
        int k = base++;
        rb[k] = b;
        rlo[k] = lo;
        rhi[k] = hi;
        int vin[3], vout[3];
        for (int j = 0; j < 3; ++j) {
            vin[j] = (hi + 1) * u[j] + b * w[j];
            vout[j] = lo * u[j] + b * w[j];
        }
        oin[k] = pack_vec(vin, d, p, N);
        oout[k] = pack_vec(vout, d, p, N);
    };
    if (d == 2) {
        emit(0, -M[t], M[t]);
    } else {
        enumerate_rows(u, w, e, Nt, emit);
    }
}

template <typename T>
dvm_status_t dalloc(T **p, size_t n, size_t *acc)
{
    cudaError_t err = cudaMalloc((void **)p, sizeof(T) * (n ? n : 1));
    if (err != cudaSuccess) {
        set_error("cudaMalloc of plan table failed");
        return err == cudaErrorMemoryAllocation ? DVM_E_NOMEM : cuda_fail(err, "cudaMalloc");
    }
    *acc += sizeof(T) * (n ? n : 1);
    return DVM_OK;
}

}  // namespace

dvm_status_t build_table(dvm_plan_s *P)
{
    const int d = P->d, Nb = P->Nbar;
    long long cand = 1;
    for (int j = 0; j < d; ++j) cand *= (2 * Nb + 1);
    int cap = (int)(cand / 2 + 1);
    size_t acc = 0;
    dvm_status_t st;
    int *d_e = nullptr, *d_count = nullptr;
    if ((st = dalloc(&d_e, (size_t)cap * 3, &acc))) return st;
    if ((st = dalloc(&d_count, 1, &acc))) return st;
    {
        LaunchScope ls(P, KC_PLAN);
        k_dirgen<<<1, kScanThreads, 0, P->stream>>>(d, Nb, d_e, cap, d_count);
    }
    DVM_CUDA(cudaGetLastError());
    int A = 0;
    DVM_CUDA(cudaMemcpyAsync(&A, d_count, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    cudaFree(d_count);
    if (A <= 0 || A > cap) {
        set_error("direction generation produced an invalid count");
        return DVM_E_CUDA;
    }
    // Plan-time self-check of the table size against closed forms that share
    // nothing with k_dirgen: 2D A = 4 Σ_{q<=N̄} φ(q); any d,
    // by Möbius inversion over the gcd, #{e primitive, |e|_inf <= N̄} =
    // Σ_k μ(k) ((2⌊N̄/k⌋+1)^d − 1), and A is half of it (one of ±e).
    {
        auto mu = [](int k) {
            int r = 1;
            for (int q = 2; q * q <= k; ++q)
                if (k % q == 0) {
                    k /= q;
                    if (k % q == 0) return 0;
                    r = -r;
                }
            return k > 1 ? -r : r;
        };
        long long prim = 0;
        for (int k = 1; k <= Nb; ++k) {
            long long side = 2 * (Nb / k) + 1, pw = 1;
            for (int j = 0; j < d; ++j) pw *= side;
            prim += mu(k) * (pw - 1);
        }
        long long want = prim / 2;
        if (d == 2) {
            long long phis = 0;
            for (int q = 1; q <= Nb; ++q) {
                int ph = 0;
                for (int a = 1; a <= q; ++a) {
                    int x = a, y = q;
                    while (y) {
                        const int r = x % y;
                        x = y;
                        y = r;
                    }
                    ph += x == 1;
                }
                phis += ph;
            }
            if (4 * phis != want) want = -1;  // the two closed forms disagree: flag below
            else want = 4 * phis;
        }
        if (A != want) {
            set_error("direction table self-check failed: A = " + std::to_string(A) + ", closed form " +
                      std::to_string(want));
            return DVM_E_STATE;
        }
    }
    P->A = A;
    P->t.e = d_e;
    DirTable &t = P->t;
    if ((st = dalloc(&t.M, A, &acc))) return st;
    if ((st = dalloc(&t.a, A, &acc))) return st;
    if ((st = dalloc(&t.u, (size_t)A * 3, &acc))) return st;
    if ((st = dalloc(&t.w, (size_t)A * 3, &acc))) return st;
    if ((st = dalloc(&t.z, (size_t)A * 3, &acc))) return st;
    if ((st = dalloc(&t.nrows, A, &acc))) return st;
    if ((st = dalloc(&t.row_off, A + 1, &acc))) return st;
    if ((st = dalloc(&t.cost, A, &acc))) return st;
    double hd1 = pow(P->h, d + 1);
    int blocks = (A + 127) / 128;
    {
        LaunchScope ls(P, KC_PLAN);
        k_dirmeta<<<blocks, 128, 0, P->stream>>>(d, A, P->Ntilde, hd1, t.e, t.M, t.a, t.u, t.w, t.z, t.nrows, t.cost);
    }
    {
        LaunchScope ls(P, KC_PLAN);
        k_scan_rows<<<1, kScanThreads, 0, P->stream>>>(A, t.nrows, t.row_off);
    }
    DVM_CUDA(cudaGetLastError());
    int R = 0;
    DVM_CUDA(cudaMemcpyAsync(&R, t.row_off + A, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    P->R = R;
    if ((st = dalloc(&t.row_b, R, &acc))) return st;
    if ((st = dalloc(&t.row_lo, R, &acc))) return st;
    if ((st = dalloc(&t.row_hi, R, &acc))) return st;
    if ((st = dalloc(&t.off_in, R, &acc))) return st;
    if ((st = dalloc(&t.off_out, R, &acc))) return st;
    {
        LaunchScope ls(P, KC_PLAN);
        k_dirrows<<<blocks, 128, 0, P->stream>>>(d, A, P->Ntilde, P->p, P->N, t.e, t.M, t.u, t.w, t.row_off,
                                                  t.row_b, t.row_lo, t.row_hi, t.off_in, t.off_out);
    }
    DVM_CUDA(cudaGetLastError());
    // small host mirrors (plan-time only)
    P->h_e.resize((size_t)A * 3);
    P->h_M.resize(A);
    P->h_a.resize(A);
    P->h_nrows.resize(A);
    P->h_row_off.resize(A + 1);
    P->h_cost.resize(A);
    DVM_CUDA(cudaMemcpyAsync(P->h_e.data(), t.e, sizeof(int) * A * 3, cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaMemcpyAsync(P->h_M.data(), t.M, sizeof(int) * A, cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaMemcpyAsync(P->h_a.data(), t.a, sizeof(double) * A, cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaMemcpyAsync(P->h_nrows.data(), t.nrows, sizeof(int) * A, cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaMemcpyAsync(P->h_row_off.data(), t.row_off, sizeof(int) * (A + 1), cudaMemcpyDeviceToHost,
                             P->stream));
    DVM_CUDA(cudaMemcpyAsync(P->h_cost.data(), t.cost, sizeof(int) * A, cudaMemcpyDeviceToHost, P->stream));
    P->table_bytes = acc;

    // Direction sharding (the decomposition eq:decD is a sum
    // over directions, hence completely parallelisable): longest-processing-time
    // assignment by the cost estimate, ties to the lowest rank; deterministic.
    P->is_local.assign(A, 0);
    P->local.clear();
    if (P->shard_world <= 1) {
        for (int i = 0; i < A; ++i) P->is_local[i] = 1;
    } else if (d == 2) {
        // 2D: shard whole pair units {e, e⊥} (both members share M_e and a_e; the
        // pair kernels evaluate a unit together, so splitting one would evaluate
        // it twice).  Unit i < mate[i], in order of its first member; cost per
        // unit: the pair kernels' per-node work is O(1) per unit (sliding
        // windows) plus an O(M_e) prologue per line segment -> 64 + 2 M_e + 1.
        // LPT over the units, ties to the lowest rank, stable.  Mirrored by
        // paper_1201_3986_b200.parallel.pair_units_2d / lpt_assign.
        std::vector<int> mate(A, -1);
        for (int i = 0; i < A; ++i) {
            int a = -P->h_e[3 * i + 1], b = P->h_e[3 * i];
            if (a < 0 || (a == 0 && b < 0)) {
                a = -a;
                b = -b;
            }
            for (int k = 0; k < A; ++k)
                if (P->h_e[3 * k] == a && P->h_e[3 * k + 1] == b) mate[i] = k;
            if (mate[i] < 0) {
                set_error("2D direction table is not closed under e -> e^perp");
                return DVM_E_STATE;
            }
        }
        std::vector<int> unit_first;
        for (int i = 0; i < A; ++i)
            if (i < mate[i]) unit_first.push_back(i);
        const int U = (int)unit_first.size();
        std::vector<long long> ucost(U);
        for (int u = 0; u < U; ++u) ucost[u] = 64 + 2LL * P->h_M[unit_first[u]] + 1;
        std::vector<int> order(U);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return ucost[x] > ucost[y]; });
        std::vector<long long> load(P->shard_world, 0);
        for (int u : order) {
            int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
            load[r] += ucost[u];
            if (r == P->shard_rank) P->is_local[unit_first[u]] = P->is_local[mate[unit_first[u]]] = 1;
        }
    } else {
        std::vector<int> order(A);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(),
                         [&](int x, int y) { return P->h_cost[x] > P->h_cost[y]; });
        std::vector<long long> load(P->shard_world, 0);
        for (int i : order) {
            int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
            load[r] += P->h_cost[i];
            if (r == P->shard_rank) P->is_local[i] = 1;
        }
    }
    for (int i = 0; i < A; ++i)
        if (P->is_local[i]) P->local.push_back(i);
    int maxrows = 0;
    for (int i = 0; i < A; ++i) maxrows = std::max(maxrows, P->h_nrows[i]);
    if (maxrows > 512) {
        set_error("perp polygon has more than 512 rows");
        return DVM_E_UNSUPPORTED;
    }
    if ((st = dalloc(&t.local, P->local.size(), &acc))) return st;
    if (!P->local.empty())
        DVM_CUDA(cudaMemcpyAsync(t.local, P->local.data(), sizeof(int) * P->local.size(), cudaMemcpyHostToDevice,
                                 P->stream));
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    if ((st = build_gain3d(P))) return st;
    if ((st = build_pair2d(P))) return st;
    P->table_bytes = acc;  // plan tables; dvm_plan_info adds the path tables (g.bytes, grown lazily)
    return DVM_OK;
}

void free_table(dvm_plan_s *P)
{
    DirTable &t = P->t;
    void *ptrs[] = {t.e, t.M, t.a, t.u, t.w, t.z, t.nrows, t.row_off, t.cost, t.row_b, t.row_lo, t.row_hi,
                    t.off_in, t.off_out, t.local};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    t = DirTable{};
    free_gain3d(P);
    free_weights(P);
}

}  // namespace dvm
