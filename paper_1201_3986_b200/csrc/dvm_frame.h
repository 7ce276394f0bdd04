// dvm_frame.h -- plan-time (host) geometry of the 3D gain kernel: for every
// direction e, a unimodular lattice frame (z, u, w) and the "sliding program"
// that evaluates the perp-polygon sum T_e inside the
// lattice planes x.e = γ.  Product code of libdvm (never shared with oracle/).
//
// Frame.  (u, w) is a basis of the plane lattice e^⊥ ∩ Z^3 and z.e = 1, so
// x = γ z + α u + β w (mod N) is a bijection of Z_N^3 and plane γ is the N×N
// torus of (α, β).  The polygon P_e = e^⊥ ∩ [-Ñ,Ñ]^3 is a set of rows
// {(t, r) : lo_r <= t <= hi_r} (t along u, r along w), so
//     T(α, β) = Σ_r Σ_{t=lo_r}^{hi_r} f(α + t, β + r)        (in-plane indices).
// Sliding the polygon one step along w:
//     T(α, β+1) = T(α, β) + Σ_ρ Σ_t [1(t∈seg_{ρ-1}) − 1(t∈seg_ρ)] f(α + t, β + ρ),
// a short list of single nodes ("raw" entries) and row ranges ("range"
// entries, evaluated as differences of in-row prefix sums).  The basis is
// chosen per direction to minimise the smem loads of that program.
//
// Storage runs.  For e_2 = 0 the frame uses u = ê_2 (the fastest storage
// axis), so every plane row is one contiguous storage row and the kernel's
// gathers and stores are coalesced.  (a2, b2) with ê_2 = e_2 z + a2 u + b2 w
// locate the storage neighbour x + ê_2 in the frame (checked by
// tools/frame_check.cpp).
#pragma once

#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace dvm {
namespace frame {

struct Entry {  // one term of the init sum or of a sliding step
    int rho;    // row offset (along w)
    int t1, t2; // column range t1..t2 (along u); t1 == t2: single node
    int sign;   // +1 / -1
};

struct DirFrame {
    int e[3];
    int z[3], u[3], w[3];
    int a2, b2;        // ê_2 = e2 z + a2 u + b2 w
    int rows_mode;     // 1: e2 == 0, u = ê_2 (plane rows are storage rows)
    int M;             // M_e = floor(Ñ / |e|_inf)
    std::vector<Entry> init;  // T(α, β) = Σ init ranges at rows β + rho
    std::vector<Entry> step;  // T(α, β+1) − T(α, β)
    double cost;       // modelled smem loads per output
    int tmax;          // max |t| over entries (incl. t1 − 1)
};

inline long long fdiv(long long a, long long b)
{
    long long q = a / b, r = a % b;
    if (r != 0 && ((r < 0) != (b < 0))) --q;
    return q;
}
inline long long cdiv(long long a, long long b) { return -fdiv(-a, b); }

inline void cross(const long long *a, const long long *b, long long *c)
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

inline long long egcd(long long a, long long b, long long &x, long long &y)
{
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
}

// Reduced basis (v1, v2) of e^⊥ ∩ Z^3 with v1 × v2 = e (Bezout, Lagrange-Gauss).
inline void plane_basis(const int *e, long long *v1, long long *v2)
{
    long long a = e[0], b = e[1], c = e[2];
    long long s, t;
    long long g = egcd(a, b, s, t);
    if (g == 0) {
        v1[0] = 1; v1[1] = 0; v1[2] = 0;
        v2[0] = 0; v2[1] = 1; v2[2] = 0;
    } else {
        v1[0] = b / g; v1[1] = -a / g; v1[2] = 0;
        v2[0] = c * s; v2[1] = c * t; v2[2] = -g;
    }
    for (int it = 0; it < 128; ++it) {
        long long n1 = v1[0] * v1[0] + v1[1] * v1[1] + v1[2] * v1[2];
        long long n2 = v2[0] * v2[0] + v2[1] * v2[1] + v2[2] * v2[2];
        if (n2 < n1) {
            for (int j = 0; j < 3; ++j) std::swap(v1[j], v2[j]);
            std::swap(n1, n2);
        }
        long long dot = v1[0] * v2[0] + v1[1] * v2[1] + v1[2] * v2[2];
        long long mu = fdiv(2 * dot + n1, 2 * n1);
        if (mu == 0) break;
        for (int j = 0; j < 3; ++j) v2[j] -= mu * v1[j];
    }
    long long cr[3];
    cross(v1, v2, cr);
    if (cr[0] != a || cr[1] != b || cr[2] != c)
        for (int j = 0; j < 3; ++j) v2[j] = -v2[j];
}

// z with z.e = 1.
inline void transverse(const int *e, int *z)
{
    long long s, t, s2, t2;
    long long g = egcd(e[0], e[1], s, t);
    egcd(g, e[2], s2, t2);
    z[0] = (int)(s2 * s);
    z[1] = (int)(s2 * t);
    z[2] = (int)t2;
}

// Rows of P_e in the basis (u, w): for r in [rmin, rmax], lo[r-rmin]..hi[r-rmin]
// (lo > hi: empty row).  Returns false if the polygon is empty.
inline bool polygon_rows(const int *u, const int *w, int Nt, int &rmin, std::vector<int> &lo, std::vector<int> &hi)
{
    // |r| is bounded: r = (u × x).e / |e|^2 ... use a generous scan.
    const int R = 4 * Nt + 4;
    int first = 1 << 30, last = -(1 << 30);
    std::vector<int> L(2 * R + 1), H(2 * R + 1);
    for (int r = -R; r <= R; ++r) {
        long long l = -(1LL << 40), h = (1LL << 40);
        bool empty = false;
        for (int j = 0; j < 3; ++j) {
            long long c = u[j], s = (long long)r * w[j];
            if (c == 0) {
                if (s > Nt || s < -Nt) empty = true;
            } else if (c > 0) {
                l = std::max(l, cdiv(-Nt - s, c));
                h = std::min(h, fdiv(Nt - s, c));
            } else {
                l = std::max(l, cdiv(Nt - s, c));
                h = std::min(h, fdiv(-Nt - s, c));
            }
        }
        if (empty || l > h) {
            L[r + R] = 1;
            H[r + R] = 0;
            continue;
        }
        L[r + R] = (int)l;
        H[r + R] = (int)h;
        first = std::min(first, r);
        last = std::max(last, r);
    }
    if (first > last) return false;
    rmin = first;
    lo.assign(L.begin() + (first + R), L.begin() + (last + R + 1));
    hi.assign(H.begin() + (first + R), H.begin() + (last + R + 1));
    return true;
}

// 1_A − 1_B for intervals A = [a1, a2], B = [b1, b2] (empty if lo > hi) as
// signed runs.
inline void interval_diff(int a1, int a2, int b1, int b2, std::vector<Entry> &out, int rho)
{
    const bool ea = a1 > a2, eb = b1 > b2;
    auto emit = [&](int x1, int x2, int sg) {
        if (x1 <= x2) out.push_back({rho, x1, x2, sg});
    };
    if (ea && eb) return;
    if (ea) { emit(b1, b2, -1); return; }
    if (eb) { emit(a1, a2, +1); return; }
    if (a2 < b1 || b2 < a1) {  // disjoint
        emit(a1, a2, +1);
        emit(b1, b2, -1);
        return;
    }
    if (a1 < b1) emit(a1, b1 - 1, +1);
    if (b1 < a1) emit(b1, a1 - 1, -1);
    if (a2 > b2) emit(b2 + 1, a2, +1);
    if (b2 > a2) emit(a2 + 1, b2, -1);
}

constexpr double kRangeCost = 2.25;  // two prefix loads + a broadcast total

// Build the program for basis (u, w); seg_len = outputs per init.
inline bool make_program(const int *u, const int *w, int Nt, int seg_len, DirFrame &F)
{
    int rmin;
    std::vector<int> lo, hi;
    if (!polygon_rows(u, w, Nt, rmin, lo, hi)) return false;
    const int nr = (int)lo.size();
    F.init.clear();
    F.step.clear();
    for (int k = 0; k < nr; ++k)
        if (lo[k] <= hi[k]) F.init.push_back({rmin + k, lo[k], hi[k], +1});
    std::vector<Entry> raw;
    for (int k = 0; k <= nr; ++k) {  // rho = rmin + k: seg_{rho-1} - seg_rho
        const int rho = rmin + k;
        int a1 = 1, a2 = 0, b1 = 1, b2 = 0;
        if (k - 1 >= 0) { a1 = lo[k - 1]; a2 = hi[k - 1]; }
        if (k < nr) { b1 = lo[k]; b2 = hi[k]; }
        raw.clear();
        interval_diff(a1, a2, b1, b2, raw, rho);
        for (const Entry &x : raw) {
            if (x.t2 - x.t1 + 1 <= 2) {
                for (int t = x.t1; t <= x.t2; ++t) F.step.push_back({rho, t, t, x.sign});
            } else {
                F.step.push_back(x);
            }
        }
    }
    double c = 0, ci = 0;
    int tm = 0;
    for (const Entry &x : F.step) {
        c += x.t1 == x.t2 ? 1.0 : kRangeCost;
        tm = std::max({tm, std::abs(x.t1 - 1), std::abs(x.t2), std::abs(x.t1)});
    }
    for (const Entry &x : F.init) {
        ci += kRangeCost;
        tm = std::max({tm, std::abs(x.t1 - 1), std::abs(x.t2)});
    }
    F.cost = c + ci / seg_len;
    F.tmax = tm;
    for (int j = 0; j < 3; ++j) {
        F.u[j] = u[j];
        F.w[j] = w[j];
    }
    return true;
}

// Solve ê_2 − e2 z = a2 u + b2 w.
inline bool run_offsets(DirFrame &F)
{
    long long v[3] = {-(long long)F.e[2] * F.z[0], -(long long)F.e[2] * F.z[1], 1 - (long long)F.e[2] * F.z[2]};
    long long U[3] = {F.u[0], F.u[1], F.u[2]}, W[3] = {F.w[0], F.w[1], F.w[2]}, E[3] = {F.e[0], F.e[1], F.e[2]};
    long long uw[3], vw[3], uv[3];
    cross(U, W, uw);
    cross(v, W, vw);
    cross(U, v, uv);
    long long den = uw[0] * E[0] + uw[1] * E[1] + uw[2] * E[2];
    long long na = vw[0] * E[0] + vw[1] * E[1] + vw[2] * E[2];
    long long nb = uv[0] * E[0] + uv[1] * E[1] + uv[2] * E[2];
    if (den == 0 || na % den || nb % den) return false;
    F.a2 = (int)(na / den);
    F.b2 = (int)(nb / den);
    for (int j = 0; j < 3; ++j)
        if (F.a2 * (long long)F.u[j] + F.b2 * (long long)F.w[j] != v[j]) return false;
    return true;
}

// Frame + program of direction e (primitive), Ñ = Nt, plane side N.
inline bool build_dir(const int *e, int Nt, int N, int seg_len, DirFrame &out)
{
    DirFrame F;
    for (int j = 0; j < 3; ++j) F.e[j] = e[j];
    int inf = std::max({std::abs(e[0]), std::abs(e[1]), std::abs(e[2])});
    F.M = Nt / inf;
    transverse(e, F.z);
    F.rows_mode = e[2] == 0;
    long long v1[3], v2[3];
    plane_basis(e, v1, v2);
    bool have = false;
    DirFrame best;
    auto consider = [&](const long long *uu, const long long *ww) {
        int u[3] = {(int)uu[0], (int)uu[1], (int)uu[2]}, w[3] = {(int)ww[0], (int)ww[1], (int)ww[2]};
        DirFrame C = F;
        if (!make_program(u, w, Nt, seg_len, C)) return;
        if (C.tmax >= N / 2) return;  // ranges must stay within one periodic row
        if (!run_offsets(C)) return;
        if (!have || C.cost < best.cost - 1e-9) {
            best = C;
            have = true;
        }
    };
    if (F.rows_mode) {
        // u = ê_2 (in e^⊥ since e2 = 0); w completes the basis: (-e1, e0, 0)
        long long u[3] = {0, 0, 1}, w0[3] = {-(long long)e[1], (long long)e[0], 0};
        for (int k = -4; k <= 4; ++k) {
            long long w[3] = {w0[0], w0[1], w0[2] + k};
            long long wn[3] = {-w[0], -w[1], -w[2]};
            consider(u, w);
            consider(u, wn);
        }
    } else {
        static const int T[][4] = {{1, 0, 0, 1},  {0, 1, -1, 0}, {1, 1, 0, 1},  {1, -1, 0, 1}, {1, 0, 1, 1},
                                   {1, 0, -1, 1}, {1, 2, 0, 1},  {1, -2, 0, 1}, {1, 0, 2, 1},  {1, 0, -2, 1},
                                   {2, 1, 1, 1},  {1, 1, 1, 2},  {2, -1, -1, 1}, {1, -1, -1, 2}, {0, 1, -1, 1},
                                   {0, 1, -1, -1}, {1, 1, -1, 0}, {1, -1, 1, 0}, {0, 1, -1, 2}, {0, 1, -1, -2}};
        for (const auto &m : T) {
            long long u[3], w[3];
            for (int j = 0; j < 3; ++j) {
                u[j] = m[0] * v1[j] + m[1] * v2[j];
                w[j] = m[2] * v1[j] + m[3] * v2[j];
            }
            long long un[3] = {-u[0], -u[1], -u[2]};
            consider(u, w);    // slide along +w
            consider(w, u);    // rows along w, slide along u
            consider(un, w);
            consider(w, un);
        }
    }
    if (!have) return false;
    out = best;
    return true;
}

}  // namespace frame
}  // namespace dvm
