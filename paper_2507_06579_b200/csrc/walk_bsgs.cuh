// walk_bsgs.cuh -- K3 in BSGS mode: the paper's Algorithm 1
// with residues in Z/3 (l.585-603): baby steps rho into a per-d store, then
// giant steps mu_k = mu_1 * mu'_{k-1} by NUCOMPchoose (forms.cuh), rho-reduction,
// and a store lookup.
//
// Three kernels per segment (K3 BSGS):
//   bsgs_baby_kernel   persistent lanes, per-lane refill: bsgs_begin + baby steps in
//                      the half walk's exact FP32 form, each entry APPENDED to a dense
//                      per-d list (sequential writes: full sectors, no L2 capacity
//                      limit).  Symmetry exits (l.553-556) finish the d; completed
//                      windows are queued for the build kernel.
//   bsgs_build_kernel  one warp per 32 queued d: each store is built as a hash table
//                      in shared memory from the list and written out with coalesced
//                      full-line stores; then the 32 lanes take the k = 2 giant step
//                      (always NUDUPL, Alg. 4 l.745) together and queue the d for
//   bsgs_giant_kernel  persistent lanes with per-lane refill (giant counts are
//                      heavy-tailed) and a software-pipelined lookup.
//
// The store ("dictionary of ideals", l.549, l.607).  list[j] = Q_j | t_j << 20 for
// the j-th baby entry (theta_{j+1} <-> (Q_j, P_j); t unreduced, < 2^12); the
// table maps Q to j: slot = (Q >> 2) | (j + 1) << 18 | (t_j mod 3) << 29, 0 =
// empty.  P is not stored: on the principal cycle P_j^2 = d - Q_{j-1} Q_j with
// P_j > 0 (rho), so a reduced (Q*, P*) matches entry j >= 1 iff Q* = Q_j and
// P*^2 = d - Q_{j-1} Q* (exact, u64); entry 0 is (2, P_1), the only reduced
// ideal of norm 1 (R34).  The paper's Bloom filter plays the table's
// role (no false negatives; positives verified exactly).
//
// The guard (R14): a hit counts if log mu'_k - log theta >= 1.  With
// log theta <= the distance of the last stored entry, a hit with log mu'_k -
// dist_last >= 1 always passes; any other hit (only possible for tiny d, where
// mu'_2 can land inside the window) sends the d to the exact half walk.
//
// Per-lane state machines are __host__ __device__ and are run by the CPU
// emulation harness tests/emu/kernel_emu.cu.
#pragma once
#include "common.cuh"
#include "forms.cuh"
#include "walk_half.cuh"

constexpr float LN2F = 0.69314718f;
constexpr float GUARD_LOG2 = 1.0f / LN2F;    // "log mu'_k - log theta >= 1" in log2 units

enum LanePhase : u32 { PH_IDLE = 0, PH_BABY = 1, PH_GIANT = 2, PH_HALF = 3, PH_DONE = 4 };

struct BsgsArgs {
    int ns_log2;        // table slots per d = 1 << ns_log2
    int cap;            // max list entries per d (<= 2040)
    int lcap;           // list stride per d (>= cap, multiple of 32)
    float alpha;        // baby window factor: W = alpha d^(1/4)
    int plain_th;       // Alg. 4 plain-product threshold on Q (paper: 50)
    float giant_cap_mul;// giant-step cap = giant_cap_mul * (d^(1/4) + 10)
    int two_sided;      // R35: conjugate hits + doubled stride (0 = the paper's one-sided Alg. 1)
};

EIS_HD u32 mod3(u32 v) { return v % 3u; }

// Two-sided window (R35).  Conjugation reverses the principal cycle
// (R13: a_{j+1} = conj(a_j) when Q_j = Q_{j-1}), so the conjugates of the stored
// ideals theta_1..theta_n are the n cycle ideals just before a_p = O: the store
// covers the arc of distances [R - dist_last + O(log sqrt d), R + dist_last]
// around every multiple of R.  A giant ideal mu = (alpha) whose conjugate is the
// stored theta_j = (beta) gives conj(alpha) = +-eps^-1 beta, so t(eps) = t(mu) +
// t(theta_j) (t(conj x) = -t(x), R13); a direct match gives t(mu) - t(theta_j).
// Both are read from one probe (same Q, P or -P mod Q).  The arc is ~2 dist_last
// long, so the giant stride may be mu_1^2 with mu_1 a margin M below the window
// end: stride 2 dist_1 + kappa <= 2 dist_last - 2M + kappa stays shorter than the
// arc while 2M >= kappa_2 + kappa_k + log sqrt d + (largest rho-step distance),
// kappa being the composition excess (< 2 log sqrt d; <= 16.4 nats seen at 1e11,
// SURVEY.md 8(c) #14).  M = 2 ln d + 4 nats (= 4 log sqrt d + 4) is used.
EIS_HD float two_sided_margin2(u64 d) {            // M in log2 units
    return 2.f * log2_approx((float)d) + 4.f / LN2F;
}

// ---------------------------------------------------------------- the store --
EIS_HD u32 list_entry(u32 Q, u32 traw) { return Q | (traw << 20); }
EIS_HD u32 slot_entry(u32 Q, u32 j, u32 t3) { return (Q >> 2) | ((j + 1) << 18) | (t3 << 29); }
EIS_HD u32 store_hash(u32 Q, int ns_log2) { return (Q * 0x9E3779B1u) >> (32 - ns_log2); }

// host/emulation build: sequential linear probing into a zeroed table
EIS_HD void store_build_seq(u32 *tab, int ns_log2, const u32 *list, u32 n) {
    const u32 mask = (1u << ns_log2) - 1;
    for (u32 j = 0; j < n; j++) {
        const u32 e = list[j], Q = e & 0xFFFFFu;
        u32 h = store_hash(Q, ns_log2);
        while (tab[h] != 0) h = (h + 1) & mask;
        tab[h] = slot_entry(Q, j, mod3(e >> 20));
    }
}

// Lookup of a reduced (Q, P) (P canonical): tables are zero-filled, so linear
// probing stops at the first empty slot; slots are read four at a time (one
// 16-byte load per aligned group).  Split so the giant kernel can issue the
// first group load, compute the next giant step, then resolve.
struct Probe {
    u32 h;
    uint4 grp;
};

EIS_HD uint4 load_group(const u32 *tab, u32 h) {
    return *reinterpret_cast<const uint4 *>(tab + (h & ~3u));
}

EIS_HD Probe store_probe(const u32 *tab, int ns_log2, u32 Q) {
    Probe p;
    p.h = store_hash(Q, ns_log2);
    p.grp = load_group(tab, p.h);
    return p;
}

// Hit kinds of a lookup of the reduced (Q, P): the stored ideal is (Q, P) itself
// or its conjugate (Q, -P mod Q) (R35).
enum HitKind : int { HIT_NONE = 0, HIT_DIRECT = 1, HIT_CONJ = 2 };

// P-bar: the canonical representative in (s - Q, s] of -P mod Q
EIS_HD u32 conj_P(u32 Q, u32 P, u32 s) {
    const u32 r = (s + P) % Q;
    return s - r;
}

// Entry jj >= 1 holds (Q_j, P_j) with P_j^2 = d - Q_{j-1} Q_j, P_j > 0 on reduced
// ideals, so Q_{j-1} identifies P_j; entry 0 is (2, P_1) = O, the only reduced
// ideal with Q = 2 (self-conjugate).
EIS_HD int match_kind(u64 d, u32 Q, u32 P, u32 s, u32 jj, u32 Qprev) {
    if (jj == 0) return HIT_DIRECT;
    const u64 nrm = d - (u64)Qprev * Q;
    if ((u64)P * P == nrm) return HIT_DIRECT;
    const u32 Pb = conj_P(Q, P, s);
    if ((u64)Pb * Pb == nrm) return HIT_CONJ;
    return HIT_NONE;
}

// Resolve a probe of (Q, P): the hit kind, t3 = t(theta) mod 3, j = the entry.
EIS_HD int store_resolve(const u32 *tab, const u32 *list, int ns_log2, Probe p, u64 d, u32 s,
                         u32 Q, u32 P, u32 &t3, u32 &j) {
    const u32 mask = (1u << ns_log2) - 1;
    const u32 qk = Q >> 2;
    u32 h = p.h;
    uint4 g = p.grp;
    for (;;) {
        const u32 i0 = h & 3u;
#pragma unroll
        for (u32 i = 0; i < 4; i++) {
            const u32 e = i == 0 ? g.x : (i == 1 ? g.y : (i == 2 ? g.z : g.w));
            if (i < i0) continue;
            if (e == 0) return HIT_NONE;
            if ((e & 0x3FFFFu) == qk) {
                const u32 jj = ((e >> 18) & 0x7FFu) - 1;
                const u32 Qprev = jj ? (list[jj - 1] & 0xFFFFFu) : 0u;
                const int k = match_kind(d, Q, P, s, jj, Qprev);
                if (k != HIT_NONE) {
                    t3 = e >> 29;
                    j = jj;
                    return k;
                }
            }
        }
        h = ((h | 3u) + 1) & mask;
        g = load_group(tab, h);
    }
}

// ------------------------------------------------------------ baby phase --
// Baby steps in the half walk's exact FP32 form (walk_half.cuh) plus the log2
// distance of each generator multiplier (P_j + sqrt d)/Q_{j-1}.
struct BabyLane {
    BabyStateF st;
    float dist;         // log2 theta_{j+1} of the current ideal
    float sqd_m;        // sqrt(d) - 2^23 (P + sqrt d = Pm + sqd_m)
    float W2;           // window in log2 units
    u32 n;              // list entries (those of the last partial group are pending)
    u32 pe0, pe1, pe2;  // pending entries of the group [n & ~3, n), not yet in memory
    int extras;         // -1 before the window is complete, then 2, 1
    float M2;           // two-sided margin (log2 units), 0 = one-sided
    u32 Q1, P1, t1;     // mu_1 (Q1 = 0: not chosen yet)
    float dist1;
    u32 phase, res;
};

struct __align__(32) BabyRec {       // baby kernel -> build kernel
    u32 off;            // survivor-list entry (offset | PRIME_BIT)
    u32 n;              // list entries
    u32 Q1, P1, t1;     // mu_1
    float dist1, dist_last;
    u32 pad;
};

EIS_HD bool baby_step_fd(BabyStateF &st, float sqd_m, float &dist) {
    const float num = st.Pm + st.sm;
    const float rq = rcp_approx(st.Q);
    const float rqb = rq * 1.000000476837158203125f;
    const float q = fma_rz(num, rqb, 8388608.0f) - 8388608.0f;
    const float r = fmaf(-q, st.Q, num);
    const float Pnm = st.sp - r;
    const float Qn = fmaf(q, st.Pm - Pnm, st.Qp);
    st.t2 += (f2u_bits(Pnm) & 2u) + 2u;
    dist += log2_approx((Pnm + sqd_m) * rq);
    const bool eP = (Pnm == st.Pm);
    st.Qp = st.Q;
    st.Q = Qn;
    st.Pm = Pnm;
    return (Qn == st.Qp) | eP;
}

EIS_HD u32 f_to_u(float v) { return f2u_bits(v + 8388608.0f) - 0x4B000000u; }   // v < 2^23

// Start d: entries theta_1 = (2, P_1) and theta_2 = (Q_1, P_1).  True if finished.
EIS_HD bool bsgs_begin(BabyLane &ln, u32 *list, const BsgsArgs &B, u64 d) {
    BabyState b;
    u32 r1;
    const bool fin = baby_init(b, d, &r1);
    if (fin) {
        ln.res = r1;
        ln.phase = PH_DONE;
        return true;
    }
    ln.st = baby_to_f(b);
    const float sqd = (float)sqrt((double)d);
    ln.sqd_m = sqd - 8388608.0f;
    ln.W2 = B.alpha * sqrtf(sqd) / LN2F;
    (void)list;
    ln.pe0 = list_entry(2u, 0u);                      // entries 0 and 1, written with
    ln.pe1 = list_entry(b.Q, b.t2 >> 1);              // the first full group
    ln.pe2 = 0;
    ln.dist = log2_approx(((float)b.P + sqd) * 0.5f);
    ln.n = 2;
    ln.extras = -1;
    ln.phase = PH_BABY;
    ln.M2 = two_sided_margin2(d);
    if (!B.two_sided || ln.W2 < 3.f * ln.M2) ln.M2 = 0.f;   // one-sided (paper's Alg. 1)
    ln.Q1 = 0;
    if (ln.dist >= ln.W2 - ln.M2) {         // mu_1 = theta_2
        ln.Q1 = b.Q;
        ln.P1 = b.P;
        ln.t1 = mod3(b.t2 >> 1);
        ln.dist1 = ln.dist;
    }
    if (ln.dist >= ln.W2) ln.extras = 2;    // window already complete at theta_2
    return false;
}

// Up to `kmax` baby steps (Alg. 1 l.549-561).  Sets PH_DONE (symmetry exit) or
// PH_GIANT (window + two more ideals stored).  Returns the steps taken.
// List entries are gathered four at a time in registers and written with one
// 16-byte store (per-lane lists are 16-byte aligned); a 4-byte store per step
// makes the kernel store-transaction bound (32 lines per warp instruction).
EIS_HD void list_flush(u32 *list, u32 n, u32 e0, u32 e1, u32 e2, u32 e3) {
    // entries n-? .. n-1 are pending: n % 4 of them (e0 oldest); at n % 4 == 0 all four
    const u32 k = n & 3u, b = n - (k ? k : 4u);
    if (k == 0) {
        *reinterpret_cast<uint4 *>(list + b) = make_uint4(e0, e1, e2, e3);
    } else {
        list[b] = e0;
        if (k > 1) list[b + 1] = e1;
        if (k > 2) list[b + 2] = e2;
    }
}

EIS_HD int bsgs_baby(BabyLane &ln, u32 *list, const BsgsArgs &B, int kmax) {
    int k = 0;
    // pending group: entries [n & ~3, n) live in e0..e2 (list is written up to n & ~3)
    u32 e0 = ln.pe0, e1 = ln.pe1, e2 = ln.pe2, e3 = 0;
    while (k < kmax) {
        const bool ex = baby_step_fd(ln.st, ln.sqd_m, ln.dist);
        k++;
        const u32 e = list_entry(f_to_u(ln.st.Q), ln.st.t2 >> 1);
        const u32 p = ln.n & 3u;
        if (p == 0) e0 = e; else if (p == 1) e1 = e; else if (p == 2) e2 = e; else e3 = e;
        ln.n++;
        if (p == 3) list_flush(list, ln.n, e0, e1, e2, e3);
        if (ex) {
            if ((ln.n & 3u) != 0) list_flush(list, ln.n, e0, e1, e2, e3);
            ln.res = baby_result_f(ln.st);
            ln.phase = PH_DONE;
            return k;
        }
        if (ln.extras < 0) {
            const bool end = ln.dist >= ln.W2 || (int)ln.n >= B.cap - 2;
            if (ln.Q1 == 0 && (end || ln.dist >= ln.W2 - ln.M2)) {
                ln.Q1 = f_to_u(ln.st.Q);                 // mu_1 = theta_j (just stored)
                ln.P1 = f2u_bits(ln.st.Pm) - 0x4B000000u;
                ln.t1 = mod3(ln.st.t2 >> 1);
                ln.dist1 = ln.dist;
            }
            if (end) ln.extras = 2;                      // "Compute two more ideals" (l.560)
        } else if (--ln.extras == 0) {
            if ((ln.n & 3u) != 0) list_flush(list, ln.n, e0, e1, e2, e3);
            ln.phase = PH_GIANT;
            return k;
        }
    }
    ln.pe0 = e0;                                    // chunk end: keep the group pending
    ln.pe1 = e1;
    ln.pe2 = e2;
    return k;
}

EIS_HD BabyRec baby_pack(const BabyLane &ln, u32 off) {
    BabyRec r;
    r.off = off;
    r.n = ln.n;
    r.Q1 = ln.Q1;
    r.P1 = ln.P1;
    r.t1 = ln.t1;
    r.dist1 = ln.dist1;
    r.dist_last = ln.dist;
    r.pad = 0;
    return r;
}

// ----------------------------------------------------------- giant phase --
struct GiantLane {
    u64 d;
    i64 s, L;           // isqrt(d), floor(d^(1/4))
    double sqrtd;
    Mu1Form m1;
    u32 t1;
    float dist1, dist_last;
    u32 Qc, Pc, tc;     // mu'_{k-1}
    float distc;
    int k, kcap;
    u32 phase, res;
};

EIS_HD void giant_init(GiantLane &g, const BsgsArgs &B, u64 d, const BabyRec &br, u32 *err) {
    g.d = d;
    g.s = (i64)isqrt_u64_dev(d);
    g.L = (i64)isqrt_u64_dev((u64)g.s);            // floor(d^(1/4))
    g.sqrtd = sqrt((double)d);
    g.m1 = mu1_form((i64)br.Q1, (i64)br.P1, (i64)d, err);
    g.t1 = br.t1;
    g.dist1 = br.dist1;
    g.dist_last = br.dist_last;
    g.Qc = br.Q1;
    g.Pc = br.P1;
    g.tc = br.t1;
    g.distc = br.dist1;
    g.k = 1;
    g.kcap = (int)(B.giant_cap_mul * (sqrtf((float)g.s) + 10.f));
    g.phase = PH_GIANT;
}

struct GiantInfo {
    u32 kind;       // composition kind
    u32 nred;       // rho steps in the reduction
};

// Advance: mu'_k = rho-reduce(NUCOMPchoose(mu_1, mu'_{k-1})) with its residue and
// distance; no lookup.  *err counts invariant violations.
EIS_HD GiantInfo giant_advance(GiantLane &g, const BsgsArgs &B, u32 *err, u32 wmask = 0xffffffffu) {
    GiantInfo gi;
    const i64 d = (i64)g.d;
    const i64 s = g.s;
    const GiantComp c = giant_compose(g.m1, (i64)g.Qc, (i64)g.Pc, d, s, g.L, (float)g.sqrtd,
                                      B.plain_th, err, wmask);
    warp_reconverge(wmask);
    gi.kind = c.kind;
    u32 t = mod3(g.t1 + g.tc + 3u - c.tg);       // theta(mu_k) = theta(mu_1) theta(mu'_{k-1}) / gamma
    float dist = g.dist1 + g.distc - c.lg;
    i64 Q = c.Q, P = c.P;                        // P canonical in (s - Q, s]
    u32 nred = 0;
    if (Q - P > s) {                             // not reduced (R18): apply rho
        // exact fp64 integers (|P|, Q < 2^32); Q' = (d - P'^2)/Q with d - P'^2 in int64
        const double sd = (double)s;
        double Qd = (double)Q, Pd = (double)P, rQ = rcp64(Qd);
        do {
            const double num = Pd + sd;
            double q = floor(num * rQ);              // floor((P + sqrt d)/Q)
            const double rr = fma(-q, Qd, num);
            q = rr < 0.0 ? q - 1.0 : (rr >= Qd ? q + 1.0 : q);
            const double Pn = fma(q, Qd, -Pd);
            const i64 Pni = (i64)Pn;
            const i64 nQ = d - Pni * Pni;
            const double Qn = rint((double)nQ * rQ);
            if ((i64)Qn * (i64)Qd != nQ) *err += 1;
            t = mod3(t + 1u + (u32)((Pni >> 1) & 1));
            dist += log2_approx((float)fabs(Pn + g.sqrtd)) - log2_approx((float)Qd);
            Qd = fabs(Qn);
            rQ = rcp64(Qd);
            Pd = sd - dfloor_mod(sd - Pn, Qd, rQ);   // canonical P in (s - Q, s]
            if (++nred > 4096) { *err += 1; break; }
        } while (Qd - Pd > sd);
        Q = (i64)Qd;
        P = (i64)Pd;
    }
    warp_reconverge(wmask);
    gi.nred = nred;
    g.k++;
    g.Qc = (u32)Q;
    g.Pc = (u32)P;
    g.tc = t;
    g.distc = dist;
    return gi;
}

// Verdict for a store hit on mu'_k = (t, dist) (R14):
// 1 = accepted, result in res (eps = mu'_k / theta); 0 = inconclusive guard
// (caller switches the d to the exact half walk).
// A conjugate hit of mu = (Q, P) is the relation eps^-m = conj(alpha)/beta with
// m R = dist + log theta_j - log N(mu) >= dist - log(Q/2) (R35): it is
// nontrivial once dist - log2(Q/2) >= the guard.
EIS_HD int giant_hit(const GiantLane &g, int kind, u32 te, u32 t, float dist, u32 Q, u32 &res) {
    if (kind == HIT_CONJ) {
        if (dist - log2_approx(0.5f * (float)Q) >= GUARD_LOG2) {
            res = mod3(t + te);
            return 1;
        }
    } else if (dist - g.dist_last >= GUARD_LOG2) {
        res = mod3(t + 3u - te);
        return 1;
    }
    return 0;
}

// k = 2: mu'_2 = rho-reduce(mu_1 * mu_1) (NUDUPL).  With the two-sided window
// (R35) and enough margin, mu'_2 becomes the giant stride: mu''_1 = mu'_2 and
// mu''_k = mu'_2 * mu''_{k-1}.  Same lane mask rules as giant_advance.
EIS_HD GiantInfo giant_start(GiantLane &g, const BsgsArgs &B, u32 *err, u32 wmask = 0xffffffffu) {
    const GiantInfo gi = giant_advance(g, B, err, wmask);
    const float M2 = two_sided_margin2(g.d);
    if (B.two_sided && g.dist1 >= 2.f * M2 && g.dist_last - g.dist1 >= M2) {
        g.m1 = mu1_form((i64)g.Qc, (i64)g.Pc, (i64)g.d, err);
        g.t1 = g.tc;
        g.dist1 = g.distc;
    }
    return gi;
}

// Unpipelined lookup of the current giant ideal (CPU emulation).  Sets PH_DONE
// on an accepted hit, PH_HALF on an inconclusive guard or past the cap; returns
// true when the d is decided.
EIS_HD bool giant_lookup(GiantLane &g, const u32 *tab, const u32 *list, const BsgsArgs &B) {
    u32 te, j;
    const int kind = store_resolve(tab, list, B.ns_log2, store_probe(tab, B.ns_log2, g.Qc), g.d,
                                   (u32)g.s, g.Qc, g.Pc, te, j);
    if (kind != HIT_NONE) {
        g.phase = giant_hit(g, kind, te, g.tc, g.distc, g.Qc, g.res) ? PH_DONE : PH_HALF;
        return true;
    }
    if (g.k > g.kcap) {
        g.phase = PH_HALF;
        return true;
    }
    return false;
}

// Everything the giant kernel needs to resume a d (written by the build kernel
// after k = 2), so a refill is two 32-byte loads.
struct __align__(64) GiantRec {
    double sqrtd;
    i64 w1;                        // mu_1's form coefficient (P1^2 - d)/(2 Q1)
    u32 off, Q1, P1, Qc;           // P1 normalised mod Q1
    u32 Pc, tk, s, Lk;             // tk = t1 | tc << 2 | k << 4; Lk = L | kcap << 16
    float dist1, distc, dist_last;
    u32 pad;
};

EIS_HD GiantRec giant_pack(const GiantLane &g, u32 off) {
    GiantRec r;
    r.sqrtd = g.sqrtd;
    r.w1 = g.m1.w;
    r.off = off;
    r.Q1 = (u32)g.m1.Q;
    r.P1 = (u32)g.m1.P;
    r.Qc = g.Qc;
    r.Pc = g.Pc;
    r.tk = g.t1 | (g.tc << 2) | ((u32)g.k << 4);
    r.s = (u32)g.s;
    r.Lk = (u32)g.L | ((u32)g.kcap << 16);
    r.dist1 = g.dist1;
    r.distc = g.distc;
    r.dist_last = g.dist_last;
    r.pad = 0;
    return r;
}

EIS_HD void giant_unpack(GiantLane &g, const GiantRec &r, u64 d) {
    g.d = d;
    g.s = (i64)r.s;
    g.L = (i64)(r.Lk & 0xFFFFu);
    g.kcap = (int)(r.Lk >> 16);
    g.sqrtd = r.sqrtd;
    g.m1.Q = (i64)r.Q1;
    g.m1.P = (i64)r.P1;
    g.m1.w = r.w1;
    g.t1 = r.tk & 3u;
    g.tc = (r.tk >> 2) & 3u;
    g.k = (int)(r.tk >> 4);
    g.dist1 = r.dist1;
    g.dist_last = r.dist_last;
    g.Qc = r.Qc;
    g.Pc = r.Pc;
    g.distc = r.distc;
    g.phase = PH_GIANT;
}

// exact half walk for one d (guard inconclusive / cap exceeded)
EIS_HD u32 half_walk_one(u64 d, u64 &steps, u32 &err) {
    BabyState st;
    u32 r1;
    if (baby_init(st, d, &r1)) return r1;
    const u32 cap = half_step_cap(st.s);
    u32 j = 0;
    bool ok;
    do { steps++; ok = baby_step(st); } while (!ok && ++j <= cap);
    if (ok) return baby_result(st);
    err++;
    return 0xFFu;
}

// ------------------------------------------------------------------ kernels --
struct BsgsOut {
    u32 *lists;         // [survivors][lcap] baby entries
    u32 *tables;        // [survivors][ns] store slots
    BabyRec *brecs;     // [survivors]
    GiantRec *grecs;    // [survivors]
    u32 *bqueue;        // survivor indices with a complete window
    u32 *gqueue;        // survivor indices needing giant steps
    u32 *ctr;           // device: [0] bqueue len, [1] build work, [2] gqueue len, [3] giant work
};

#ifdef __CUDACC__
__device__ __forceinline__ void record_result(const WalkArgs &a, u32 *hist, u32 le, u64 d,
                                              u32 res) {
    const u32 t = res % 3;
    if (a.flags) a.flags[le & ~PRIME_BIT] = (u8)t;
    if (a.ckpt) hist_record(a, hist, d, t, (le & PRIME_BIT) != 0);
}

__device__ __forceinline__ void flush_stats(const WalkArgs &a, u64 baby, u64 giant, u64 red,
                                            u64 done, u64 sym, u64 fb, u32 err) {
    const int lane = threadIdx.x & 31;
    const u64 s_baby = warp_sum_u64(baby), s_giant = warp_sum_u64(giant),
              s_red = warp_sum_u64(red), s_done = warp_sum_u64(done), s_sym = warp_sum_u64(sym),
              s_fb = warp_sum_u64(fb);
    const u32 s_err = __reduce_add_sync(FULL_MASK, err);
    if (lane == 0 && a.stats) {
        atomicAdd((unsigned long long *)&a.stats[ST_BABY], (unsigned long long)s_baby);
        atomicAdd((unsigned long long *)&a.stats[ST_GIANT], (unsigned long long)s_giant);
        atomicAdd((unsigned long long *)&a.stats[ST_REDUCE], (unsigned long long)s_red);
        atomicAdd((unsigned long long *)&a.stats[ST_D], (unsigned long long)s_done);
        atomicAdd((unsigned long long *)&a.stats[ST_SYM], (unsigned long long)s_sym);
        atomicAdd((unsigned long long *)&a.stats[ST_FALLBACK], (unsigned long long)s_fb);
    }
    if (lane == 0 && s_err) atomicAdd(a.err, s_err);
}

// K3a: baby steps, per-lane refill from the survivor list.
template <int KB>
__global__ void __launch_bounds__(256)
bsgs_baby_kernel(WalkArgs a, BsgsArgs B, BsgsOut o) {
    __shared__ u32 hist[NROW_MAX * HIST_CAP];
    hist_zero(a, hist);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const u32 n = *a.count;
    BabyLane ln;
    ln.phase = PH_IDLE;
    u32 off = 0, idx = 0;
    u32 *list = nullptr;
    u64 d = 0;
    bool exhausted = false;
    u64 baby = 0, done = 0, sym = 0;
    u32 err = 0;
    for (;;) {
        const u32 need = __ballot_sync(FULL_MASK, ln.phase == PH_IDLE && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            u32 base = 0;
            if (lane == leader) base = atomicAdd(a.work, (u32)__popc(need));
            base = __shfl_sync(FULL_MASK, base, leader);
            if (ln.phase == PH_IDLE && !exhausted) {
                idx = base + __popc(need & lanemask_lt());
                if (idx < n) {
                    off = __ldg(a.list + idx);
                    d = cand_d(a.i0 + (off & ~PRIME_BIT));
                    list = o.lists + (u64)idx * B.lcap;
                    baby += 1;
                    if (bsgs_begin(ln, list, B, d)) {
                        record_result(a, hist, off, d, ln.res);
                        done++;
                        sym++;
                        ln.phase = PH_IDLE;
                    }
                } else {
                    exhausted = true;
                }
            }
        }
        if (__all_sync(FULL_MASK, exhausted && ln.phase == PH_IDLE)) break;
        if (ln.phase == PH_BABY) {
            baby += bsgs_baby(ln, list, B, KB);
            if (ln.phase == PH_DONE) {
                record_result(a, hist, off, d, ln.res);
                done++;
                sym++;
                ln.phase = PH_IDLE;
            } else if (ln.phase == PH_GIANT) {
                o.brecs[idx] = baby_pack(ln, off);
                o.bqueue[atomicAdd(&o.ctr[0], 1u)] = idx;
                ln.phase = PH_IDLE;
            }
        }
    }
    flush_stats(a, baby, 0, 0, done, sym, 0, err);
    hist_flush(a, hist);
}

// K3b: each warp builds 32 stores in shared memory, then takes k = 2 for them.
__global__ void __launch_bounds__(256)
bsgs_build_kernel(WalkArgs a, BsgsArgs B, BsgsOut o) {
    extern __shared__ u32 smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int ns = 1 << B.ns_log2;
    const u32 mask = (u32)ns - 1;
    u32 *tab = smem + (size_t)wid * ns;
    const u32 nb = o.ctr[0];
    u64 giant = 0, red = 0;
    u32 err = 0;
    for (int i = lane; i < ns; i += 32) tab[i] = 0;
    __syncwarp();
    for (;;) {
        u32 base = 0;
        if (lane == 0) base = atomicAdd(&o.ctr[1], 32u);
        base = __shfl_sync(FULL_MASK, base, 0);
        if (base >= nb) break;
        const u32 cnt = min(32u, nb - base);
        const u32 myq = lane < (int)cnt ? o.bqueue[base + lane] : 0;
        for (u32 q = 0; q < cnt; q++) {
            const u32 idx = __shfl_sync(FULL_MASK, myq, q);
            const u32 ne = o.brecs[idx].n;
            const uint4 *l4 = reinterpret_cast<const uint4 *>(o.lists + (u64)idx * B.lcap);
            for (u32 jb = 0; jb < ne; jb += 512) {           // up to 4 x 16 B per lane in flight
                uint4 v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const u32 j4 = jb / 4 + (u32)u * 32 + lane;
                    v[u] = j4 * 4 < ne ? l4[j4] : make_uint4(0, 0, 0, 0);
                }
                // warp-uniform probe loops: every lane inserts its next entry and
                // the loop runs until all lanes succeeded (a per-lane while loop
                // leaves the warp split for the rest of the batch, measured
                // 2.8/32 active threads)
#pragma unroll
                for (int u = 0; u < 4; u++) {
#pragma unroll
                    for (int w = 0; w < 4; w++) {
                        const u32 j = jb + ((u32)u * 32 + lane) * 4 + w;
                        const u32 e = w == 0 ? v[u].x : (w == 1 ? v[u].y : (w == 2 ? v[u].z : v[u].w));
                        const u32 Q = e & 0xFFFFFu;
                        const u32 sv = slot_entry(Q, j, mod3(e >> 20));
                        u32 h = store_hash(Q, B.ns_log2);
                        bool todo = j < ne;
                        while (__any_sync(FULL_MASK, todo)) {
                            if (todo) {
                                if (atomicCAS(&tab[h], 0u, sv) == 0u) todo = false;
                                else h = (h + 1) & mask;
                            }
                        }
                    }
                }
            }
            __syncwarp();
            uint4 *dst = reinterpret_cast<uint4 *>(o.tables + ((u64)idx << B.ns_log2));
            uint4 *src = reinterpret_cast<uint4 *>(tab);
            for (int i = lane; i < ns / 4; i += 32) {        // write out, clear for the next d
                dst[i] = src[i];
                src[i] = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
        }
        // k = 2 (mu_2 = mu_1 * mu_1: NUDUPL) for the batch, one d per lane; the
        // lookup of mu'_2 is left to the giant kernel's pipelined probe
        bool push = false;
        u32 gidx = 0;
        const u32 kmask = __ballot_sync(FULL_MASK, lane < (int)cnt);
        if (lane < (int)cnt) {
            gidx = myq;
            const BabyRec br = o.brecs[gidx];
            GiantLane g;
            giant_init(g, B, cand_d(a.i0 + (br.off & ~PRIME_BIT)), br, &err);
            const GiantInfo gi = giant_start(g, B, &err, kmask);
            giant++;
            red += gi.nred;
            o.grecs[gidx] = giant_pack(g, br.off);
            push = true;
        }
        const u32 pm = __ballot_sync(FULL_MASK, push);
        u32 qb = 0;
        if (lane == 0 && pm) qb = atomicAdd(&o.ctr[2], (u32)__popc(pm));
        qb = __shfl_sync(FULL_MASK, qb, 0);
        if (push) o.gqueue[qb + __popc(pm & lanemask_lt())] = gidx;
    }
    flush_stats(a, 0, giant, red, 0, 0, 0, err);
}

// K3c: giant steps with per-lane refill and a pipelined lookup.
__global__ void __launch_bounds__(256)
bsgs_giant_kernel(WalkArgs a, BsgsArgs B, BsgsOut o) {
    __shared__ u32 hist[NROW_MAX * HIST_CAP];
    hist_zero(a, hist);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const u32 nq = o.ctr[2];
    const u32 *tab = nullptr, *list = nullptr;
    GiantLane g;
    g.phase = PH_IDLE;
    u32 off = 0;
    bool exhausted = false;
    u64 baby = 0, giant = 0, red = 0, done = 0, fb = 0;
    u32 err = 0;

    for (;;) {
        const u32 need = __ballot_sync(FULL_MASK, g.phase == PH_IDLE && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            u32 base = 0;
            if (lane == leader) base = atomicAdd(&o.ctr[3], (u32)__popc(need));
            base = __shfl_sync(FULL_MASK, base, leader);
            if (g.phase == PH_IDLE && !exhausted) {
                const u32 qi = base + __popc(need & lanemask_lt());
                if (qi < nq) {
                    const u32 idx = __ldg(o.gqueue + qi);
                    const GiantRec r = o.grecs[idx];
                    off = r.off;                          // (with the prime bit)
                    giant_unpack(g, r, cand_d(a.i0 + (off & ~PRIME_BIT)));
                    tab = o.tables + ((u64)idx << B.ns_log2);
                    list = o.lists + (u64)idx * B.lcap;
                } else {
                    exhausted = true;
                }
            }
        }
        if (__all_sync(FULL_MASK, exhausted && g.phase == PH_IDLE)) break;
        const u32 gmask = __ballot_sync(FULL_MASK, g.phase == PH_GIANT);
        if (g.phase == PH_GIANT) {
            // software pipeline: probe mu'_k (refills start with mu'_2, not yet
            // probed) while computing mu'_{k+1}
            const u32 pQ = g.Qc, pP = g.Pc, pt = g.tc;
            const float pdist = g.distc;
            const Probe pr = store_probe(tab, B.ns_log2, pQ);
            const GiantInfo gi = giant_advance(g, B, &err, gmask);
            giant++;
            red += gi.nred;
            u32 te, j;
            const int kind = store_resolve(tab, list, B.ns_log2, pr, g.d, (u32)g.s, pQ, pP, te, j);
            warp_reconverge(gmask);
            if (kind != HIT_NONE) {
                g.phase = giant_hit(g, kind, te, pt, pdist, pQ, g.res) ? PH_DONE : PH_HALF;
            } else if (g.k > g.kcap) {
                g.phase = PH_HALF;
            }
            if (g.phase == PH_HALF) {     // exact half walk instead
                fb++;
                g.res = half_walk_one(g.d, baby, err);
                g.phase = PH_DONE;
            }
        }
        if (g.phase == PH_DONE) {
            record_result(a, hist, off, g.d, g.res);
            done++;
            g.phase = PH_IDLE;
        }
    }
    flush_stats(a, baby, giant, red, done, 0, fb, err);
    hist_flush(a, hist);
}

// ------------------------------------------------------------- host launch --
struct BsgsScratch {
    u32 *lists = nullptr;
    size_t lists_n = 0;
    u32 *tables = nullptr;
    size_t tables_n = 0;
    BabyRec *brecs = nullptr;
    size_t brecs_n = 0;
    GiantRec *grecs = nullptr;
    size_t grecs_n = 0;
    u32 *bqueue = nullptr;
    size_t bqueue_n = 0;
    u32 *gqueue = nullptr;
    size_t gqueue_n = 0;
};

inline void bsgs_free(BsgsScratch &s) {
    cudaFree(s.lists);
    cudaFree(s.tables);
    cudaFree(s.brecs);
    cudaFree(s.grecs);
    cudaFree(s.bqueue);
    cudaFree(s.gqueue);
    s = BsgsScratch();
}

constexpr int BSGS_KB = 32;
constexpr int BSGS_THREADS = 256;

// Store sizes for a segment whose largest d is d_max: ~1.22 nats per baby step
// (SURVEY.md A.8), cap ~ the window's entry count + slack (R33: a lower cap
// only ends the window early), table load <= ~0.55.
struct BsgsSizes {
    int ns_log2, cap, lcap;
};
inline BsgsSizes bsgs_sizes(u64 d_max, float alpha) {
    BsgsSizes z;
    const double w = alpha * std::pow((double)d_max, 0.25);   // window in nats
    z.cap = std::min(2040, (int)(w / 1.22 * 1.05) + 8);
    z.ns_log2 = 6;
    while ((double)(1 << z.ns_log2) < 1.8 * z.cap && z.ns_log2 < 12) z.ns_log2++;
    z.lcap = (z.cap + 31) & ~31;
    return z;
}

template <class T>
inline int bsgs_grow(T *&p, size_t &cap, size_t n) {
    if (n <= cap && p) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return -3;
    cap = n;
    return 0;
}

struct BsgsPlan {
    BsgsArgs B;
    BsgsOut o;
    size_t build_smem;
    unsigned baby_blocks, build_blocks, giant_blocks;
};

inline size_t bsgs_bytes_per_survivor(u64 d_max, float alpha) {
    const BsgsSizes z = bsgs_sizes(d_max, alpha);
    return (size_t)4 * z.lcap + ((size_t)4 << z.ns_log2) + sizeof(BabyRec) + sizeof(GiantRec) + 8;
}

#ifdef __CUDACC__
// Size one segment buffer (seg_len candidates bound the survivors) and choose
// the launch shapes.  ctr: 4 device counters (zeroed by bsgs_launch_baby).
inline int bsgs_prepare(BsgsPlan &pl, u64 seg_len, u64 d_hi, int num_sms, int alpha_x16,
                        int giant_ctas, int two_sided, BsgsScratch &scr, u32 *ctr) {
    BsgsArgs &B = pl.B;
    B.two_sided = two_sided;
    B.alpha = alpha_x16 / 16.0f;
    const BsgsSizes z = bsgs_sizes(d_hi, B.alpha);
    B.ns_log2 = z.ns_log2;
    B.cap = z.cap;
    B.lcap = z.lcap;
    B.plain_th = 50;
    B.giant_cap_mul = 20.0f;
    const size_t n = (size_t)seg_len;
    if (bsgs_grow(scr.lists, scr.lists_n, n * (size_t)z.lcap)) return -3;
    if (bsgs_grow(scr.tables, scr.tables_n, n << z.ns_log2)) return -3;
    if (bsgs_grow(scr.brecs, scr.brecs_n, n)) return -3;
    if (bsgs_grow(scr.grecs, scr.grecs_n, n)) return -3;
    if (bsgs_grow(scr.bqueue, scr.bqueue_n, n)) return -3;
    if (bsgs_grow(scr.gqueue, scr.gqueue_n, n)) return -3;
    BsgsOut &o = pl.o;
    o.lists = scr.lists;
    o.tables = scr.tables;
    o.brecs = scr.brecs;
    o.grecs = scr.grecs;
    o.bqueue = scr.bqueue;
    o.gqueue = scr.gqueue;
    o.ctr = ctr;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsgs_baby_kernel<BSGS_KB>,
                                                      BSGS_THREADS, 0) != cudaSuccess ||
        per_sm < 1)
        return -4;
    pl.baby_blocks = (unsigned)(num_sms * per_sm);
    pl.build_smem = (size_t)(BSGS_THREADS / 32) * ((size_t)4 << z.ns_log2);
    if (cudaFuncSetAttribute(bsgs_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pl.build_smem) != cudaSuccess)
        return -4;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsgs_build_kernel, BSGS_THREADS,
                                                      pl.build_smem) != cudaSuccess ||
        per_sm < 1)
        return -4;
    pl.build_blocks = (unsigned)(num_sms * per_sm);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsgs_giant_kernel, BSGS_THREADS,
                                                      0) != cudaSuccess ||
        per_sm < 1)
        return -4;
    pl.giant_blocks = (unsigned)(num_sms * (giant_ctas > 0 ? std::min(giant_ctas, per_sm) : per_sm));
    return 0;
}

// baby + build on the main stream
inline int bsgs_launch_baby(const WalkArgs &a, const BsgsPlan &pl, cudaStream_t s) {
    if (cudaMemsetAsync(pl.o.ctr, 0, 4 * sizeof(u32), s) != cudaSuccess) return -4;
    bsgs_baby_kernel<BSGS_KB><<<pl.baby_blocks, BSGS_THREADS, 0, s>>>(a, pl.B, pl.o);
    if (cudaGetLastError() != cudaSuccess) return -4;
    bsgs_build_kernel<<<pl.build_blocks, BSGS_THREADS, pl.build_smem, s>>>(a, pl.B, pl.o);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

inline int bsgs_launch_giant(const WalkArgs &a, const BsgsPlan &pl, cudaStream_t s) {
    bsgs_giant_kernel<<<pl.giant_blocks, BSGS_THREADS, 0, s>>>(a, pl.B, pl.o);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}
#endif  // __CUDACC__ (launch)
#endif  // __CUDACC__ (kernels)
