// giant_profile.cu -- ANALYSIS HARNESS (not product code, not a test): runs the
// giant kernel's per-lane state machine on the CPU for seeded d (stdin) and
// prints, per giant step, the host-only event counters of EIS_PROF
// (common.cuh): 0 xgcd iterations, 1 F not | s branch, 2 partial-Euclid
// iterations, 3 rho steps of the reduction, 4 NUCOMP calls, 5 F != 1, 6 z == 0,
// 7 bx == 0, 8 rare path (plain product / generic), 9 key-match checks,
// 10 second-bucket loads.  scripts/giant_divergence.py turns the rows into
// expected warp-level trip counts (max over 32 lanes) -- the SIMT divergence
// of each loop and branch (K3 BSGS giant).
//   nvcc -x cu -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a \
//        -o giant_profile tests/emu/giant_profile.cu;  giant_profile ALPHA_X16 < d-list
#define EIS_HOST_PROFILE 1
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2507_06579_b200/csrc/walk_bsgs.cuh"
unsigned eis_prof[16];
int main(int argc, char **argv) {
    const float alpha = atoi(argv[1]) / 16.0f;
    BsgsArgs B; B.plain_th = 50; B.giant_cap_mul = 20.f; B.two_sided = 1;
    std::vector<u32> tab(1 << 16), lst(1 << 12);
    unsigned long long d;
    while (scanf("%llu", &d) == 1) {
        const BsgsSizes z = bsgs_sizes(d, alpha, 1);
        B.nw = z.nw; B.j1 = z.j1; B.nb = z.nb; B.lcap = z.lcap;
        std::fill(tab.begin(), tab.begin() + (size_t)B.nb * BKT, 0u);
        WinLane w; u32 e0, e1, err = 0;
        if (!win_begin(w, d, e0, e1)) continue;
        lst[0] = e0; lst[1] = e1;
        for (int j = 2; j < B.nw && w.live; j++) {
            lst[j] = win_step(w);
            if ((j & 3) == 3) win_flush(w);
            if (j == B.j1 && w.live) win_mark_mu1(w);
        }
        if (!w.live) continue;
        store_build_seq(tab.data(), (u32)B.nb, lst.data(), (u32)B.nw);
        const BabyRec br = win_pack(w, 0, (u32)B.nw);
        GiantLane g;
        giant_init(g, B, d, br, &err);
        giant_start(g, B, &err);
        // giant kernel steps: one line per step with counter deltas
        int k = 0;
        for (;;) {
            unsigned before[16]; std::copy(eis_prof, eis_prof + 16, before);
            bool done = giant_lookup(g, tab.data(), lst.data(), B);
            if (done) { unsigned dd[16]; for (int i=0;i<16;i++) dd[i]=eis_prof[i]-before[i];
                printf("%llu L %d", d, k); for (int i=0;i<11;i++) printf(" %u", dd[i]); printf("\n"); break; }
            giant_advance(g, B, &err, 0xffffffffu, false);
            unsigned dd[16]; for (int i=0;i<16;i++) dd[i]=eis_prof[i]-before[i];
            printf("%llu S %d", d, k); for (int i=0;i<11;i++) printf(" %u", dd[i]); printf("\n");
            k++;
        }
        if (err) fprintf(stderr, "err %llu\n", d);
    }
}
