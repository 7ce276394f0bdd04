// frame_check.cpp -- CPU check of the 3D gain-kernel geometry (not product
// code): frames are bijections, the run offsets (a2, b2) hold, and the sliding
// program reproduces the direct perp-polygon sum T_e on random data.
// g++ -O2 -std=c++17 -I paper_1201_3986_b200/csrc tools/frame_check.cpp -o /tmp/frame_check
#include <array>
#include <cmath>
#include <cstdio>
#include <random>
#include "dvm_frame.h"
using namespace dvm::frame;

int main(int argc, char **argv)
{
    int N = argc > 1 ? atoi(argv[1]) : 32, Nb = argc > 2 ? atoi(argv[2]) : 4, Nt = argc > 3 ? atoi(argv[3]) : 7;
    int seg = argc > 4 ? atoi(argv[4]) : 16;
    int sample = argc > 5 ? atoi(argv[5]) : 1;
    std::vector<std::array<int, 3>> dirs;
    for (int a = -Nb; a <= Nb; ++a)
        for (int b = -Nb; b <= Nb; ++b)
            for (int c = -Nb; c <= Nb; ++c) {
                int first = a ? a : (b ? b : c);
                if (first <= 0) continue;
                long long x, y;
                long long g = egcd(egcd(a, b, x, y), c, x, y);
                if (g != 1) continue;
                dirs.push_back({a, b, c});
            }
    printf("A=%zu\n", dirs.size());
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    const int NN = N * N, NODES = N * N * N;
    std::vector<double> f(NODES), T(NODES), Td(NODES);
    for (auto &v : f) v = U(rng);
    auto idx = [&](long long a, long long b, long long c) {
        a = ((a % N) + N) % N; b = ((b % N) + N) % N; c = ((c % N) + N) % N;
        return (int)((a * N + b) * N + c);
    };
    double tot_cost = 0, tot_init = 0, tot_step = 0;
    int bad = 0, checked = 0, rows_mode = 0;
    for (size_t di = 0; di < dirs.size(); ++di) {
        DirFrame F;
        if (!build_dir(dirs[di].data(), Nt, N, seg, F)) { printf("build failed %zu\n", di); return 1; }
        tot_cost += F.cost;
        tot_init += F.init.size();
        tot_step += F.step.size();
        rows_mode += F.rows_mode;
        if (di % sample) continue;
        ++checked;
        const int *e = F.e;
        // frame bijection + planes
        std::vector<int> seen(NODES, 0);
        for (int g = 0; g < N; ++g)
            for (int be = 0; be < N; ++be)
                for (int al = 0; al < N; ++al) {
                    int x = idx((long long)g * F.z[0] + (long long)al * F.u[0] + (long long)be * F.w[0],
                                (long long)g * F.z[1] + (long long)al * F.u[1] + (long long)be * F.w[1],
                                (long long)g * F.z[2] + (long long)al * F.u[2] + (long long)be * F.w[2]);
                    seen[x]++;
                }
        for (int x = 0; x < NODES; ++x) if (seen[x] != 1) { printf("not a bijection dir %zu\n", di); return 1; }
        // run offsets: x + e2hat = frame(g + e2, al + a2, be + b2)
        for (int j = 0; j < 3; ++j) {
            long long v = (long long)e[2] * F.z[j] + (long long)F.a2 * F.u[j] + (long long)F.b2 * F.w[j];
            if (v != (j == 2)) { printf("run offset wrong dir %zu\n", di); return 1; }
        }
        if (F.rows_mode && !(F.u[0] == 0 && F.u[1] == 0 && F.u[2] == 1)) { printf("rows mode u\n"); return 1; }
        // direct T
        std::vector<std::array<int, 3>> P;
        for (int a = -Nt; a <= Nt; ++a) for (int b = -Nt; b <= Nt; ++b) for (int c = -Nt; c <= Nt; ++c)
            if (a * e[0] + b * e[1] + c * e[2] == 0) P.push_back({a, b, c});
        for (int x0 = 0; x0 < N; ++x0) for (int x1 = 0; x1 < N; ++x1) for (int x2 = 0; x2 < N; ++x2) {
            double s = 0;
            for (auto &l : P) s += f[idx(x0 + l[0], x1 + l[1], x2 + l[2])];
            Td[(x0 * N + x1) * N + x2] = s;
        }
        // program T, plane by plane, emulating the kernel (periodic prefix + total)
        std::vector<double> raw(NN), pre(NN), tot(N);
        for (int g = 0; g < N; ++g) {
            for (int be = 0; be < N; ++be)
                for (int al = 0; al < N; ++al)
                    raw[be * N + al] = f[idx((long long)g * F.z[0] + (long long)al * F.u[0] + (long long)be * F.w[0],
                                             (long long)g * F.z[1] + (long long)al * F.u[1] + (long long)be * F.w[1],
                                             (long long)g * F.z[2] + (long long)al * F.u[2] + (long long)be * F.w[2])];
            for (int be = 0; be < N; ++be) {
                double s = 0;
                for (int al = 0; al < N; ++al) { s += raw[be * N + al]; pre[be * N + al] = s; }
                tot[be] = s;
            }
            auto range = [&](int row, int a, int b) {
                int r = row & (N - 1);
                int am = a - 1;
                double v = pre[r * N + (b & (N - 1))] - pre[r * N + (am & (N - 1))];
                int k = (int)(dvm::frame::fdiv((long long)b, (long long)N) - dvm::frame::fdiv((long long)am, (long long)N));
                return v + k * tot[r];
            };
            for (int al = 0; al < N; ++al)
                for (int s0 = 0; s0 < N; s0 += seg) {
                    double acc = 0;
                    for (auto &x : F.init) acc += range(s0 + x.rho, al + x.t1, al + x.t2);
                    for (int s = 0; s < seg; ++s) {
                        int be = s0 + s;
                        int xs = idx((long long)g * F.z[0] + (long long)al * F.u[0] + (long long)be * F.w[0],
                                     (long long)g * F.z[1] + (long long)al * F.u[1] + (long long)be * F.w[1],
                                     (long long)g * F.z[2] + (long long)al * F.u[2] + (long long)be * F.w[2]);
                        T[xs] = acc;
                        double pos = 0, neg = 0;
                        for (auto &x : F.step) {
                            double v = x.t1 == x.t2 ? raw[((be + x.rho) & (N - 1)) * N + ((al + x.t1) & (N - 1))]
                                                    : range(be + x.rho, al + x.t1, al + x.t2);
                            if (x.sign > 0) pos += v; else neg += v;
                        }
                        acc += pos - neg;
                    }
                }
        }
        double md = 0;
        for (int x = 0; x < NODES; ++x) md = std::max(md, std::fabs(T[x] - Td[x]) / std::max(1.0, std::fabs(Td[x])));
        if (md > 1e-12) { printf("dir %zu (%d,%d,%d): T mismatch %.3e\n", di, e[0], e[1], e[2], md); ++bad; }
    }
    printf("checked %d dirs, bad %d, rows_mode %d; per-output cost %.1f (init entries %.0f, step entries %.0f)\n",
           checked, bad, rows_mode, tot_cost, tot_init, tot_step);
    return bad != 0;
}
