// kernel_emu.cu -- TEST HARNESS: runs the walk kernels' per-lane state machines
// (the __host__ __device__ functions of walk_half.cuh / walk_bsgs.cuh) on the
// CPU, one d at a time, so their arithmetic can be checked against the oracle
// without a GPU.  Not part of the product library.
//
// usage: kernel_emu MODE ALPHA_X16 NB [PLAIN_TH [TWO_SIDED]] < d-list  (MODE: half | bsgs;
//        NB: table buckets per d, 0 = sized from d; half mode: 99 = integer step)
// prints per d: "d t baby giant reduce fallback err kinds(plain,comp,dupl)"
// MODE dupl (ALPHA_X16 = ideals per d): squares the first ideals of the principal
// cycle with NUDUPL twice, the generic int64 nudupl() and the fp64 nudupl_d(),
// and prints per d: "d checked mismatches err" (outputs u3 v3 x y G compared;
// both stop the partial Euclid at the fast path's bound, R38).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

#include "../../paper_2507_06579_b200/csrc/walk_bsgs.cuh"

int main(int argc, char **argv) {
    if (argc < 4) {
        fprintf(stderr, "usage: %s half|bsgs alpha_x16 ns_log2(0=auto)\n", argv[0]);
        return 2;
    }
    const bool bsgs = strcmp(argv[1], "bsgs") == 0;
    if (strcmp(argv[1], "dupl") == 0) {
        const int per_d = atoi(argv[2]);
        const i64 plain_th = argc > 4 ? atoi(argv[4]) : 50;
        unsigned long long dd;
        while (scanf("%llu", &dd) == 1) {
            u32 err = 0, r1;
            int checked = 0, bad = 0;
            BabyState st;
            const i64 L = (i64)isqrt_u64_dev((u64)isqrt_u64_dev(dd));
            // the fast path stops its partial Euclid at kEuclidBound L (DESIGN.md
            // R38); the generic nudupl() is given that bound as an integer
            const i64 Lg = (i64)((float)L * kEuclidBound);
            if (!baby_init(st, dd, &r1)) {
                for (int k = 0; k < per_d; k++) {
                    if ((i64)st.Q > plain_th) {
                        const Mu1Form m = mu1_form((i64)st.Q, (i64)st.P, (i64)dd, &err);
                        i64 u3, v3, w3, G, x, y;
                        nudupl((i64)(m.Q >> 1), -(i64)m.P, m.w, Lg, u3, v3, w3, G, x, y, &err);
                        CompD o;
                        nudupl_d((double)(m.Q >> 1), -(double)m.P, (double)m.w, (float)L, o, &err,
                                 0xffffffffu);
                        checked++;
                        if ((i64)o.u3 != u3 || (i64)o.v3 != v3 || (i64)o.w3 != w3 ||
                            (i64)o.x != x || (i64)o.y != y || (i64)o.G != G ||
                            !disc_ok(o.u3, o.v3, o.w3, (double)dd))
                            bad++;
                    }
                    if (baby_step(st)) break;
                }
            }
            printf("%llu %d %d %u\n", dd, checked, bad, err);
        }
        return 0;
    }
    BsgsArgs B;
    const float alpha = atoi(argv[2]) / 16.0f;
    const int nb_fixed = atoi(argv[3]);
    B.plain_th = argc > 4 ? atoi(argv[4]) : 50;
    B.giant_cap_mul = 20.0f;
    B.two_sided = argc > 5 ? atoi(argv[5]) : 1;
    std::vector<u32> bm(1 << 10);
    std::vector<u32> tab(1 << 16), lst(1 << 12);
    unsigned long long d;
    while (scanf("%llu", &d) == 1) {
        u32 res = 0, err = 0;
        u64 baby = 0, giant = 0, red = 0, fb = 0, kinds[3] = {0, 0, 0};
        if (!bsgs) {
            BabyState st;
            u32 r1;
            baby = 1;
            if (baby_init(st, d, &r1)) res = r1;
            else if (nb_fixed == 99) {                      // integer form of the step
                for (;;) { baby++; if (baby_step(st)) break; }
                res = baby_result(st);
            } else {                                        // FP32 form (the kernel's)
                BabyStateF sf = baby_to_f(st);
                for (;;) { baby++; if (baby_step_f(sf)) break; }
                res = baby_result_f(sf);
            }
        } else {
            const BsgsSizes z = bsgs_sizes(d, alpha, B.two_sided);
            B.nw = z.nw;
            B.j1 = z.j1;
            B.nb = nb_fixed ? nb_fixed : z.nb;
            B.lcap = z.lcap;
            std::fill(tab.begin(), tab.begin() + (size_t)B.nb * BKT, 0u);
            WinLane w;
            u32 e0, e1;
            baby = 1;
            if (!win_begin(w, d, e0, e1)) {
                res = w.res;
            } else {                                        // window kernel, one lane
                lst[0] = e0;
                lst[1] = e1;
                for (int j = 2; j < B.nw && w.live; j++) {
                    lst[j] = win_step(w);
                    if ((j & 3) == 3) win_flush(w);
                    baby++;
                    if (j == B.j1 && w.live) win_mark_mu1(w);
                }
                if (!w.live) {
                    res = w.res;
                } else {
                    store_build_seq(tab.data(), (u32)B.nb, lst.data(), (u32)B.nw);
                    // table invariant: every entry j is reached from its bucket h(key)
                    // by following only buckets flagged SLOT_PASSED (counted as errors)
                    for (int j = 0; j < B.nw; j++) {
                        const u32 key = entry_key(lst[j]);
                        u32 b = store_bucket(key, (u32)B.nb), hops = 0;
                        for (;;) {
                            bool found = false;
                            for (int i = 0; i < BKT; i++) {
                                const u32 sl = tab[b * BKT + i];
                                if (sl && (sl & 0x3FFFFu) == key && slot_j1(sl) == (u32)j + 1) found = true;
                            }
                            if (found) break;
                            if (!(tab[b * BKT + BKT - 1] & SLOT_PASSED) || ++hops > (u32)B.nb) {
                                err++;
                                break;
                            }
                            b = next_bucket(b, (u32)B.nb);
                        }
                    }
                    const BabyRec br = win_pack(w, 0, (u32)B.nw);
                    GiantLane g;
                    giant_init(g, B, d, br, &err);
                    GiantInfo gi = giant_start(g, B, &err);   // prep kernel
                    giant++;
                    red += gi.nred;
                    kinds[gi.kind]++;
                    while (!giant_lookup(g, tab.data(), lst.data(), B)) {   // giant kernel
                        gi = giant_advance(g, B, &err, 0xffffffffu, true);   // (squarings: fp64 NUDUPL)
                        giant++;
                        red += gi.nred;
                        kinds[gi.kind]++;
                    }
                    if (g.phase == PH_HALF) {
                        fb++;
                        const HalfOne h = half_walk_one(d);
                        g.res = h.res;
                        baby += h.steps;
                        err += h.err;
                    }
                    res = g.res;
                }
            }
        }
        printf("%llu %u %llu %llu %llu %llu %u %llu %llu %llu\n", d, res % 3,
               (unsigned long long)baby, (unsigned long long)giant, (unsigned long long)red,
               (unsigned long long)fb, err, (unsigned long long)kinds[0],
               (unsigned long long)kinds[1], (unsigned long long)kinds[2]);
    }
    return 0;
}
