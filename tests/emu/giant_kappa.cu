// giant_kappa.cu -- ANALYSIS HARNESS (not product code, not a test): the giant-step
// distance excess kappa = dist(mu'_k) - dist(mu'_{k-1}) - dist(stride) (nats) over
// K giant steps of each seeded d (stdin), min and max over all d.  The two-sided
// window's margin M (walk_bsgs.cuh two_sided_margin2, R35, R38) must
// exceed what this measures.
//   nvcc -x cu -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a \
//        -o giant_kappa tests/emu/giant_kappa.cu;  giant_kappa ALPHA_X16 K < d-list
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2507_06579_b200/csrc/walk_bsgs.cuh"
int main(int argc, char **argv) {
    const float alpha = atoi(argv[1]) / 16.0f;
    const int K = atoi(argv[2]);
    BsgsArgs B; B.plain_th = 50; B.giant_cap_mul = 20.f; B.two_sided = 1;
    std::vector<u32> lst(1 << 12);
    unsigned long long d;
    double gmin = 1e9, gmax = -1e9;
    long n = 0;
    while (scanf("%llu", &d) == 1) {
        const BsgsSizes z = bsgs_sizes(d, alpha, 1);
        B.nw = z.nw; B.j1 = z.j1; B.nb = z.nb; B.lcap = z.lcap;
        WinLane w; u32 e0, e1, err = 0;
        if (!win_begin(w, d, e0, e1)) continue;
        for (int j = 2; j < B.nw && w.live; j++) {
            win_step(w);
            if ((j & 3) == 3) win_flush(w);
            if (j == B.j1 && w.live) win_mark_mu1(w);
        }
        if (!w.live) continue;
        const BabyRec br = win_pack(w, 0, (u32)B.nw);
        GiantLane g;
        giant_init(g, B, d, br, &err);
        giant_start(g, B, &err);
        float prev = g.distc;
        double mn = 1e9, mx = -1e9;
        for (int k = 0; k < K; k++) {
            giant_advance(g, B, &err, 0xffffffffu, false);
            const double kap = (double)(g.distc - prev - g.dist1) * 0.6931471805599453;
            mn = std::min(mn, kap); mx = std::max(mx, kap);
            prev = g.distc;
        }
        gmin = std::min(gmin, mn); gmax = std::max(gmax, mx); n++;
        if (err) fprintf(stderr, "err %llu\n", d);
    }
    printf("%ld d: kappa min %.3f max %.3f nats\n", n, gmin, gmax);
}
