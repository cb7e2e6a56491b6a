// walk_bsgs.cuh -- K3 in BSGS mode: the paper's Algorithm 1
// with residues in Z/3 (l.585-603): baby steps rho into a per-d store, then
// giant steps mu_k = mu_1 * mu'_{k-1} by NUCOMPchoose (forms.cuh), rho-reduction,
// and a store lookup; with the two-sided window of DESIGN.md R35.
//
// Three kernels per segment (K3 BSGS):
//   bsgs_window_kernel  one warp per wave of 32 survivors, in lockstep: every lane
//                       takes the same number nw of baby steps (the window is
//                       nw entries, ~ alpha d^(1/4) nats; R6/R29: only step
//                       counts depend on it), so the loop has no per-lane exit
//                       test besides the symmetry exit (l.553-556).  Entries are
//                       kept in registers in blocks of 8 (indices known at
//                       compile time) and written as one 32-byte store per lane
//                       into the d's list (rows or 64-entry tiles: ListRef).
//                       The same warp then builds the
//                       32 stores, one d at a time, as bucketed hash tables in
//                       shared memory from the lists (read back in groups of 256
//                       entries) and writes each out with one TMA bulk copy.
//   bsgs_prep_kernel    k = 2 for every windowed d in lockstep (mu'_2 = mu_1^2,
//                       NUDUPL, Alg. 4 l.745; R35 may make it the stride).
//   bsgs_giant_kernel   persistent lanes with per-lane refill (giant counts are
//                       heavy-tailed) and a software-pipelined lookup.
//
// The store ("dictionary of ideals", l.549, l.607).  list[j] = (Q_j >> 2) | t_j << 18
// for the j-th baby entry (theta_{j+1} <-> (Q_j, P_j); t unreduced, < 2^14).  The
// table is nb buckets of BKT = 16 slots (64 bytes, two DRAM sectors); slot =
// (Q >> 2) | (j + 1) << 18 | (t_j mod 3) << 29, 0 = empty (Q = 2 mod 4 on reduced
// ideals, so Q >> 2 identifies Q; bit 31 of a bucket's last slot is
// SLOT_PASSED).  An entry goes to the first free slot of bucket h(Q), else of
// the following buckets, and every bucket that turned it away is flagged; a
// lookup scans its bucket and follows on only past a flagged one.  P is not stored: on the principal
// cycle P_j^2 = d - Q_{j-1} Q_j with P_j > 0 (rho), so a reduced (Q*, P*)
// matches entry j >= 1 iff Q* = Q_j and P*^2 = d - Q_{j-1} Q* (exact, u64);
// entry 0 is (2, P_1), the only reduced ideal of norm 1 (R34).  The
// paper's Bloom filter plays the table's role (no false negatives; positives
// verified exactly).
//
// The guard (R14, R32): a direct hit counts if log mu'_k - log theta
// >= 1.  With log theta <= the distance of the last stored entry, a hit with
// log mu'_k - dist_last >= 1 always passes; any other hit (only possible for
// tiny d, where mu'_2 can land inside the window) sends the d to the exact half
// walk.  Conjugate hits: R35.
//
// Per-lane state machines are __host__ __device__ and are run by the CPU
// emulation harness tests/emu/kernel_emu.cu.
#pragma once
#include "common.cuh"
#include "forms.cuh"
#include "walk_half.cuh"

constexpr float LN2F = 0.69314718f;
constexpr float GUARD_LOG2 = 1.0f / LN2F;    // "log mu'_k - log theta >= 1" in log2 units
constexpr int BKT = 16;                       // slots per table bucket (64 bytes)
#ifndef BKT_LOAD_X100
#define BKT_LOAD_X100 62
#endif
constexpr float BKT_LOAD = BKT_LOAD_X100 / 100.f;   // table load factor

enum LanePhase : u32 { PH_IDLE = 0, PH_BABY = 1, PH_GIANT = 2, PH_HALF = 3, PH_DONE = 4 };

struct BsgsArgs {
    int nw;             // window entries per d (multiple of 8, <= 2040)
    int j1;             // entry index of mu_1 (= 7 mod 8: the end of a block)
    int nb;             // table buckets per d
    int lcap;           // list words per d (>= nw, multiple of 8): a wave of 32 d owns 32 lcap
    u32 lsh;            // list layout (ListRef): 6 = tiles of 64 entries, 30 = rows
    int plain_th;       // Alg. 4 plain-product threshold on Q (paper: 50; kernels: PLAIN_TH)
    float giant_cap_mul;// giant-step cap = giant_cap_mul * (d^(1/4) + 10)
    int two_sided;      // R35: conjugate hits + doubled stride (0 = the paper's one-sided Alg. 1)
};

EIS_HD u32 mod3(u32 v) { return v % 3u; }
EIS_HD int __double2loint_hd(double x) {          // the low 32 bits of x's encoding
#ifdef __CUDA_ARCH__
    return __double2loint(x);
#else
    u64 b;
    memcpy(&b, &x, sizeof b);
    return (int)(u32)b;
#endif
}
EIS_HD u32 mod3_small(u32 v) { return v - 3u * ((v * 0x5556u) >> 16); }   // v < 2^15

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
// list entry = key | t << 18 with key = Q >> 2 = (Q - 2)/4 (Q = 2 mod 4 on reduced
// ideals; Q < 2^20 so key < 2^18) and t the unreduced residue count (< 2^14)
EIS_HD u32 list_entry(u32 Q, u32 traw) { return (Q >> 2) | (traw << 18); }
EIS_HD u32 list_entry_key(u32 key, u32 traw) { return key | (traw << 18); }
EIS_HD u32 entry_Q(u32 e) { return 4u * (e & 0x3FFFFu) + 2u; }
EIS_HD u32 entry_t(u32 e) { return e >> 18; }
// key = Q >> 2 identifies Q (Q = 2 mod 4 on reduced ideals)
EIS_HD u32 entry_key(u32 e) { return e & 0x3FFFFu; }
// table slot of list entry e = key | t << 18 at index j: key (18 bits) | (j + 1) << 18
// (11 bits; 0 marks an empty slot) | (t mod 3) << 29, so a hit reads t(theta_j)
// from the slot instead of a second, dependent list load
EIS_HD u32 slot_entry(u32 e, u32 j) {
    return (e & 0x3FFFFu) | ((j + 1) << 18) | mod3_small(entry_t(e)) << 29;   // t < 2^14
}
EIS_HD u32 slot_j1(u32 slot) { return (slot >> 18) & 0x7FFu; }   // j + 1
EIS_HD u32 slot_t3(u32 slot) { return (slot >> 29) & 3u; }
// Bit 31 of a bucket's last slot: an insertion found the bucket full and went
// on to the next one, so a lookup of a key hashed here must follow it.  A full
// bucket without the flag (its own 16 entries, nothing turned away) ends the
// lookup; the flag cut the giant kernel's second-bucket scans.
constexpr u32 SLOT_PASSED = 0x80000000u;
EIS_HD u32 store_bucket(u32 key, u32 nb) {         // multiply-shift hash onto [0, nb)
#ifdef __CUDA_ARCH__
    return __umulhi(key * 0x9E3779B1u, nb);
#else
    return (u32)(((u64)(key * 0x9E3779B1u) * nb) >> 32);
#endif
}
EIS_HD u32 next_bucket(u32 b, u32 nb) { return b + 1 == nb ? 0u : b + 1; }

// List layout.  The 32 lists of a wave (32 consecutive survivors) share a
// region of 32 lcap words.  Entry j of lane l's list sits at
//   (j >> lsh) lcs + l lls + (j & (2^lsh - 1))
// from the region's base: rows (lsh = 30, lls = lcap, lcs unused: each list
// contiguous) for windows of one build group (nw <= 256), else tiles of 64
// entries (lsh = 6, lcs = 32 * 64, lls = 64: the warp's 32-byte block stores
// land in an 8 KB span instead of 32 rows across 62 KB, and a list is read back
// in 256-byte pieces).  ListRef holds a d's origin (region + l lls), lsh, lcs.
// Measured against rows: +1.8% on the bench slab, +0.5% at 5e9, +2.1% at 3e10,
// +2.4% at 1e11; tiles of 16 / 32 / 128 / 256 entries -8.6% / +0.7% / +1.6% /
// -0.6% at 1e10, and with nw = 256 (1.5e9-2.5e9) tiles lose 2%, so rows stay
// there.  The kernels are templates on the layout (LE = 0 rows, 64 tiles), so
// the baby loop's block addresses are compile-time.  DESIGN.md 4, Layout.
struct ListRef {
    const u32 *base;    // the d's lane origin: wave region + l lls
    u32 lsh, lcs;
};
EIS_HD u32 list_at(const ListRef &L, u32 j) {
    return L.base[(j >> L.lsh) * L.lcs + (j & ((1u << L.lsh) - 1u))];
}
template <int LE>
EIS_HD u32 list_off_t(u32 j) { return LE ? (j / LE) * (32u * LE) + j % LE : j; }
// a flat list (host emulation): one row
EIS_HD ListRef list_flat(const u32 *list) {
    ListRef L;
    L.base = list;
    L.lsh = 30;
    L.lcs = 0;
    return L;
}

// host/emulation build: sequential insertion into a zeroed table
EIS_HD void store_build_seq(u32 *tab, u32 nb, const u32 *list, u32 n) {
    for (u32 j = 0; j < n; j++) {
        const u32 e = list[j], key = entry_key(e);
        u32 b = store_bucket(key, nb);
        for (;;) {
            u32 i = 0;
            while (i < (u32)BKT && tab[b * BKT + i] != 0) i++;
            if (i < (u32)BKT) {
                tab[b * BKT + i] = slot_entry(e, j);
                break;
            }
            tab[b * BKT + BKT - 1] |= SLOT_PASSED;
            b = next_bucket(b, nb);
        }
    }
}

// Lookup of a reduced (Q, P) (P canonical).  Split so the giant kernel can issue
// the bucket load, compute the next giant step, then resolve.
struct Probe {
    u32 b;
    uint4 g0, g1, g2, g3;
};

EIS_HD void load_bucket(const u32 *tab, u32 b, Probe &p) {
    const uint4 *t4 = reinterpret_cast<const uint4 *>(tab + (size_t)b * BKT);
    p.b = b;
    p.g0 = t4[0];
    p.g1 = t4[1];
    p.g2 = t4[2];
    p.g3 = t4[3];
}

EIS_HD Probe store_probe(const u32 *tab, u32 nb, u32 Q) {
    Probe p;
    load_bucket(tab, store_bucket(Q >> 2, nb), p);
    return p;
}

// Hit kinds of a lookup of the reduced (Q, P): the stored ideal is (Q, P) itself
// or its conjugate (Q, -P mod Q) (R35).
enum HitKind : int { HIT_NONE = 0, HIT_DIRECT = 1, HIT_CONJ = 2 };

// P-bar: the canonical representative in (s - Q, s] of -P mod Q
EIS_HD u32 conj_P(u32 Q, u32 P, u32 s) {     // = floor((s + P)/Q) Q - P (a rho step's P)
    const float q = ffloor_div_pos((float)(s + P), (float)Q);   // exact: s + P < 2^20
    return (u32)q * Q - P;
}

// Entry jj >= 1 holds (Q_j, P_j) with P_j^2 = d - Q_{j-1} Q_j, P_j > 0 on reduced
// ideals, so Q_{j-1} identifies P_j; entry 0 is (2, P_1) = O, the only reduced
// ideal with Q = 2 (self-conjugate).
// (inline: a call ran on nearly every giant iteration, a key match in some lane)
EIS_HD int match_kind(u64 d, u32 Q, u32 P, u32 s, u32 jj, u32 Qprev) {
    if (jj == 0) return HIT_DIRECT;
    const u64 nrm = d - (u64)Qprev * Q;
    if ((u64)P * P == nrm) return HIT_DIRECT;
    const u32 Pb = conj_P(Q, P, s);
    if ((u64)Pb * Pb == nrm) return HIT_CONJ;
    return HIT_NONE;
}

EIS_HD u32 bucket_slot(const Probe &p, int i) {      // i: compile-time after unrolling
    const uint4 &g = i < 4 ? p.g0 : (i < 8 ? p.g1 : (i < 12 ? p.g2 : p.g3));
    const int k = i & 3;
    return k == 0 ? g.x : (k == 1 ? g.y : (k == 2 ? g.z : g.w));
}

// Slots before the first empty one (all 16 if the bucket is full).
EIS_HD u32 filled_mask(const Probe &p) {
    u32 em = 0;
#pragma unroll
    for (int i = 0; i < BKT; i++) em |= (u32)(bucket_slot(p, i) == 0) << i;
    return (em & (0u - em)) - 1u;
}

// Resolve a probe of (Q, P): the hit kind, t3 = t(theta) mod 3, j = the entry.
// The bucket is scanned without branches: bit i of the key-match mask is bit 31
// of ((slot_i ^ qk) & 0x3FFFF) - 1.  A bucket fills in slot order (one counter
// per bucket in the build), so it is full iff its last slot is, and an empty slot
// (0) can match only key 0 (Q = 2), which masks the empty slots off (rare).  A
// key match (about one per d) re-reads its slot and checks P (R34, R35).
// first_slots (nullable): a copy of the first probed bucket (the giant kernel's
// shared-memory buffer), read on a key match instead of global memory.
EIS_HD int store_resolve(const u32 *tab, const ListRef &list, u32 nb, Probe p, u64 d, u32 s,
                         u32 Q, u32 P, u32 &t3, u32 &j, const u32 *first_slots = nullptr) {
    const u32 qk = Q >> 2;
    for (;;) {
        u32 mm = 0;
#pragma unroll
        for (int i = BKT - 1; i >= 0; i--)
            mm = (mm << 1) | ((((bucket_slot(p, i) ^ qk) & 0x3FFFFu) - 1u) >> 31);
        const bool full = (bucket_slot(p, BKT - 1) & SLOT_PASSED) != 0;   // turned an entry away
        if (qk == 0) mm &= filled_mask(p);
        while (mm) {
            EIS_PROF(9);
            const int i = __builtin_ctz_portable(mm);
            mm &= mm - 1;
            const u32 e = first_slots ? first_slots[i] : tab[(size_t)p.b * BKT + i];
            const u32 jj = slot_j1(e) - 1;
            const u32 Qprev = jj ? entry_Q(list_at(list, jj - 1)) : 0u;
            const int k = match_kind(d, Q, P, s, jj, Qprev);
            if (k != HIT_NONE) {
                t3 = slot_t3(e);                          // t(theta_j) (0 for j = 0)
                j = jj;
                return k;
            }
        }
        if (!full) return HIT_NONE;
        EIS_PROF(10);
        load_bucket(tab, next_bucket(p.b, nb), p);       // bucket full: continue
        first_slots = nullptr;
    }
}

// ----------------------------------------------------------- window phase --
// Baby steps in the half walk's exact FP32 form (walk_half.cuh) plus the
// generator multiplier (P_j + sqrt d)/Q_{j-1}, multiplied into `prod`; its log2
// is added to the distance every 4 steps (win_flush: 4 multipliers < d^2 < 2^74).
EIS_HD bool baby_step_fd(BabyStateF &st, float sqd_m, float &prod) {
    const float num = st.Pm + st.sm;
    const float rq = rcp_approx(st.Q);
    const float rqb = rq * 1.000000476837158203125f;
    const float q = fma_rz(num, rqb, 8388608.0f) - 8388608.0f;
    const float r = fmaf(-q, st.Q, num);
    const float Pnm = st.sp - r;
    const float Qn = fmaf(q, st.Pm - Pnm, st.Qp);
    st.t2 += (f2u_bits(Pnm) & 2u) + 2u;
    prod *= (Pnm + sqd_m) * rq;
    const bool eP = (Pnm == st.Pm);
    st.Qp = st.Q;
    st.Q = Qn;
    st.Pm = Pnm;
    return (Qn == st.Qp) | eP;
}

EIS_HD u32 f_to_u(float v) { return f2u_bits(v + 8388608.0f) - 0x4B000000u; }   // v < 2^23
// key = (Q - 2)/4 of an exact float Q = 2 mod 4: Q/4 + (2^23 - 1/2) = key + 2^23 exactly
EIS_HD u32 f_to_key(float Q) { return f2u_bits(fmaf(Q, 0.25f, 8388607.5f)) - 0x4B000000u; }


struct WinLane {
    BabyStateF st;
    float dist;         // log2 theta_{j+1} of the current ideal (after win_flush)
    float prod;         // multipliers not yet in dist
    float sqd_m;        // sqrt(d) - 2^23 (P + sqrt d = Pm + sqd_m)
    u32 Q1, P1, t1;     // mu_1
    float dist1;
    u32 res;            // t at the symmetry exit
    bool live;          // no symmetry exit yet
};

struct __align__(32) BabyRec {       // window kernel -> prep kernel
    u32 off;            // survivor-list entry (offset | PRIME_BIT)
    u32 n;              // list entries
    u32 Q1, P1, t1;     // mu_1
    float dist1, dist_last;
    u32 pad;
};

// Entries 0 = theta_1 = (2, P_1) and 1 = theta_2 = (Q_1, P_1).  False if the d is
// already finished (res set).
EIS_HD bool win_begin(WinLane &w, u64 d, u32 &e0, u32 &e1) {
    BabyState b;
    u32 r1;
    w.live = false;
    if (baby_init(b, d, &r1)) {
        w.res = r1;
        return false;
    }
    w.st = baby_to_f(b);
    const float sqd = (float)sqrt((double)d);
    w.sqd_m = sqd - 8388608.0f;
    e0 = list_entry(2u, 0u);
    e1 = list_entry(b.Q, b.t2 >> 1);
    w.dist = log2_approx(((float)b.P + sqd) * 0.5f);
    w.prod = 1.f;
    w.Q1 = 0;
    w.live = true;
    return true;
}

// a harmless state for lanes without a d (the lockstep loop still steps them)
EIS_HD void win_idle(WinLane &w) {
    w.st.sm = 0.f;
    w.st.sp = 16777216.f;
    w.st.Pm = 8388609.f;
    w.st.Q = 2.f;
    w.st.Qp = 2.f;
    w.st.t2 = 0;
    w.dist = 0.f;
    w.prod = 1.f;
    w.sqd_m = -8388608.f;
    w.Q1 = w.P1 = w.t1 = 0;
    w.dist1 = 0.f;
    w.res = 0;
    w.live = false;
}

// One baby step (Alg. 1 l.549-556); returns the list entry of the new ideal.
EIS_HD u32 win_step(WinLane &w) {
    const bool ex = baby_step_fd(w.st, w.sqd_m, w.prod);
    if (ex && w.live) {
        w.res = baby_result_f(w.st);
        w.live = false;
    }
    // list_entry_key(key, t2 >> 1): t2 is even (it starts at 2 or 4 and grows by
    // 2 or 4), so (t2 >> 1) << 18 = t2 << 17 and the key (< 2^18) and t fields do
    // not overlap: one shift-add instead of shift, shift, or
    return f_to_key(w.st.Q) + (w.st.t2 << 17);
}

// fold the pending multipliers into the distance (every 4 steps: entry j = 3 mod 4)
EIS_HD void win_flush(WinLane &w) {
    w.dist += log2_approx(w.prod);
    w.prod = 1.f;
}

// mu_1 = the ideal just stored (l.559); after win_flush
EIS_HD void win_mark_mu1(WinLane &w) {
    w.Q1 = f_to_u(w.st.Q);
    w.P1 = f2u_bits(w.st.Pm) - 0x4B000000u;
    w.t1 = mod3(w.st.t2 >> 1);
    w.dist1 = w.dist;
}

EIS_HD BabyRec win_pack(const WinLane &w, u32 off, u32 n) {
    BabyRec r;
    r.off = off;
    r.n = n;
    r.Q1 = w.Q1;
    r.P1 = w.P1;
    r.t1 = w.t1;
    r.dist1 = w.dist1;
    r.dist_last = w.dist;
    r.pad = 0;
    return r;
}

// ----------------------------------------------------------- giant phase --
struct GiantLane {
    u64 d;
    u32 s, L;           // isqrt(d) < 2^19, floor(d^(1/4)) (32-bit: fewer live registers)
    float sqrtd;        // only feeds fp32 log2 distances and NUCOMP's float bound
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
    g.s = isqrt_u64_dev(d);
    g.L = isqrt_u64_dev((u64)g.s);                 // floor(d^(1/4))
    g.sqrtd = (float)sqrt((double)d);
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

// The rho reduction of a giant step's output (R18, R28), in exact fp64
// integers, carrying the third coefficient C = (d - P^2)/Q of the ideal (Q, P)
// so that no step forms d - P'^2 (|P'| reaches 2^28, so that needs int64):
// rho gives P' = qQ - P, Q' = C + q (P - P'), C' = Q, and moving P' to its
// canonical representative P' + kQ' gives C' - k (P' + P'_c).  Every result
// is an integer below 2^38 and each product is inside an fma (one rounding of
// an exact value), so all of it is exact even where k (P' + P'_c) itself
// exceeds 2^53.  The residue bit of P' is read from the low word of
// P' + 1.5 * 2^52 (no conversion), and the distance is accumulated as a
// product, with one log at the end.  (A resumable form, at most 1-3 steps per
// warp iteration with the rest parked in shared memory, measured 1.8-2.8%
// slower than running each lane's loop to the end: DESIGN.md 4, dead ends.)
struct RhoState {
    double Q, P, C, rQ, mag;   // the current ideal, 1/Q, prod |P' + sqrt d| / Q
    u32 t;                     // t(mu) (not reduced mod 3 while stepping)
    u32 nred;                  // rho steps so far
    float dist;                // log2 of the generator, without mag
};

// The output of a composition: rho state with Q, P canonical (P in (s - Q, s]).
EIS_HD RhoState rho_begin(const GiantLane &g, const GiantComp &c) {
    RhoState r;
    r.t = mod3_small(g.t1 + g.tc + 3u - c.tg);   // theta(mu_k) = theta(mu_1) theta(mu'_{k-1}) / gamma
    r.dist = g.dist1 + g.distc - c.lg;
    r.Q = c.Q;
    r.P = c.P;
    r.nred = 0;
    r.mag = 1.0;
    // C = (d - P^2)/Q for every lane, reduced or not (it is only used when the
    // output needs rho steps, 25% of lanes, but the warp ran the branch in
    // nearly every iteration: unconditional measured +0.5%).  |P| < Q + s may
    // reach 2^28, so d - P^2 in int64; the quotient is < 2^37 and the division
    // exact, so rint recovers it
    r.rQ = rcp64_1(r.Q);
    const i64 Pi = (i64)c.P;
    r.C = rint((double)((i64)g.d - Pi * Pi) * r.rQ);
    return r;
}

EIS_HD bool rho_needed(const RhoState &r, double sd) { return r.Q - r.P > sd; }

// one rho step plus the canonical shift
EIS_HD void rho_step(RhoState &r, double sd, double sqrtd) {
    EIS_PROF(3);
    const double num = r.P + sd;
    double q = floor(num * r.rQ);                // floor((P + sqrt d)/Q)
    const double rr = fma(-q, r.Q, num);
    q = rr < 0.0 ? q - 1.0 : (rr >= r.Q ? q + 1.0 : q);
    const double Pn = fma(q, r.Q, -r.P);
    double Qn = fma(q, r.P - Pn, r.C);
    const u32 plo = (u32)__double2loint_hd(Pn + 6755399441055744.0);   // P' mod 2^32
    r.t += 1u + ((plo >> 1) & 1u);               // (reduced mod 3 at rho_end)
    r.mag *= fabs(Pn + sqrtd) * r.rQ;
    double Cn = r.Q;                             // C' = Q
    if (Qn < 0.0) { Qn = -Qn; Cn = -Cn; }        // the ideal of norm |Q'|
    r.Q = Qn;
    r.rQ = rcp64_1(Qn);
    // canonical P in (s - Q, s]: P_c = P' + k Q with k = floor((s - P')/Q)
    const double a = sd - Pn;
    double k = floor(a * r.rQ);
    const double rk = fma(-k, Qn, a);
    k = rk < 0.0 ? k - 1.0 : (rk >= Qn ? k + 1.0 : k);
    r.P = fma(k, Qn, Pn);
    r.C = fma(-k, Pn + r.P, Cn);
    r.nred++;
}

// mu'_k = the reduced result: residue, distance, the exact check d = P^2 + Q C
EIS_HD void rho_end(GiantLane &g, RhoState &r, u32 *err) {
    if (r.nred) {
        r.t = mod3(r.t);
        r.dist += log2_approx((float)r.mag);
        if (fma(r.Q, r.C, r.P * r.P) != (double)g.d) *err += 1;   // exact (< 2^40)
    }
    g.k++;
    g.Qc = dlo32(r.Q);                           // (reduced: 0 < P < Q < 2^21)
    g.Pc = dlo32(r.P);
    g.tc = r.t;
    g.distc = r.dist;
}

// Advance: mu'_k = rho-reduce(NUCOMPchoose(mu_1, mu'_{k-1})) with its residue and
// distance; no lookup.  *err counts invariant violations.
// dup_fast: the step is (normally) a squaring, mu'_k = mu_1^2 (the prep kernel)
EIS_HD GiantInfo giant_advance(GiantLane &g, const BsgsArgs &B, u32 *err, u32 wmask = 0xffffffffu,
                               bool dup_fast = false) {
    GiantInfo gi;
    const GiantComp c = giant_compose(g.m1, (i64)g.Qc, (i64)g.Pc, (i64)g.d, (i64)g.s, (i64)g.L,
                                      g.sqrtd, B.plain_th, err, wmask, dup_fast);
    warp_reconverge(wmask);
    gi.kind = c.kind;
    RhoState r = rho_begin(g, c);
    const double sd = (double)g.s;
    while (rho_needed(r, sd)) {
        rho_step(r, sd, (double)g.sqrtd);
        if (r.nred > 4096) { *err += 1; break; }
    }
    warp_reconverge(wmask);
    gi.nred = r.nred;
    rho_end(g, r, err);
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
    const GiantInfo gi = giant_advance(g, B, err, wmask, true);
    const float M2 = two_sided_margin2(g.d);
    // stride shorter than the arc by >= 2M (R35), and mu''_1 = mu_1^2 beyond the
    // window by >= M (so its direct hits are never trivial)
    if (B.two_sided && g.dist_last - g.dist1 >= M2 && 2.f * g.dist1 - g.dist_last >= M2) {
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
    const int kind = store_resolve(tab, list_flat(list), B.nb, store_probe(tab, B.nb, g.Qc), g.d,
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
    u32 Pc, tk, s, L;              // tk = t1 | tc << 2 | k << 4
    float dist1, distc, dist_last;
    u32 kcap;                      // giant-step cap (giant_cap * (d^(1/4) + 10), may pass 2^16)
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
    r.L = (u32)g.L;
    r.dist1 = g.dist1;
    r.distc = g.distc;
    r.dist_last = g.dist_last;
    r.kcap = (u32)g.kcap;
    return r;
}

EIS_HD void giant_unpack(GiantLane &g, const GiantRec &r, u64 d) {
    g.d = d;
    g.s = r.s;
    g.L = r.L;
    g.kcap = (int)r.kcap;
    g.sqrtd = (float)r.sqrtd;
    g.m1.Q = r.Q1;
    g.m1.P = r.P1;
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
// (results returned by value, not through references: the out-of-line call then
// does not force the caller's counters into local memory)
struct HalfOne {
    u32 res, err, steps;
};
EIS_HD_COLD HalfOne half_walk_one(u64 d) {
    HalfOne h{0, 0, 0};
    BabyState st;
    u32 r1;
    if (baby_init(st, d, &r1)) {
        h.res = r1;
        return h;
    }
    const u32 cap = half_step_cap(st.s);
    u32 j = 0;
    bool ok;
    do { h.steps++; ok = baby_step(st); } while (!ok && ++j <= cap);
    if (ok) h.res = baby_result(st);
    else { h.err = 1; h.res = 0xFFu; }
    return h;
}

// ------------------------------------------------------------------ kernels --
struct BsgsOut {
    u32 *lists;         // [survivors][lcap] baby entries
    u32 *tables;        // [survivors][nb][BKT] store slots
    BabyRec *brecs;     // [survivors]
    GiantRec *grecs;    // [survivors]
    u32 *bqueue;        // survivor indices with a complete window
    u32 *gqueue;        // survivor indices needing giant steps
    u32 *ctr;           // device: [0] bqueue len, [1] unused, [2] gqueue len, [3] giant work
};

#ifdef __CUDACC__
__device__ __forceinline__ void record_result(const WalkArgs &a, u32 *hist, u32 le, u64 d,
                                              u32 res) {
    const u32 t = res % 3;
    if (a.flags) a.flags[le & ~PRIME_BIT] = (u8)t;
    if (a.ckpt) hist_record(a, hist, d, t, (le & PRIME_BIT) != 0);
}

__device__ __forceinline__ void flush_stats(const WalkArgs &a, u64 baby, u64 giant, u64 red,
                                            u64 done, u64 sym, u64 fb, u32 err, u64 win = 0) {
    const int lane = threadIdx.x & 31;
    const u64 s_baby = warp_sum_u64(baby), s_giant = warp_sum_u64(giant),
              s_red = warp_sum_u64(red), s_done = warp_sum_u64(done), s_sym = warp_sum_u64(sym),
              s_fb = warp_sum_u64(fb), s_win = warp_sum_u64(win);
    const u32 s_err = __reduce_add_sync(FULL_MASK, err);
    if (lane == 0 && a.stats) {
        atomicAdd((unsigned long long *)&a.stats[ST_BABY], (unsigned long long)s_baby);
        atomicAdd((unsigned long long *)&a.stats[ST_GIANT], (unsigned long long)s_giant);
        atomicAdd((unsigned long long *)&a.stats[ST_REDUCE], (unsigned long long)s_red);
        atomicAdd((unsigned long long *)&a.stats[ST_D], (unsigned long long)s_done);
        atomicAdd((unsigned long long *)&a.stats[ST_SYM], (unsigned long long)s_sym);
        atomicAdd((unsigned long long *)&a.stats[ST_FALLBACK], (unsigned long long)s_fb);
        if (s_win) atomicAdd((unsigned long long *)&a.stats[ST_WINDOWED], (unsigned long long)s_win);
    }
    if (lane == 0 && s_err) atomicAdd(a.err, s_err);
}


// K3a: baby steps for a wave of 32 survivors in lockstep, then their stores.
// Shared memory per warp: the table (nb * BKT slots) and nb fill counters.
EIS_HD u32 window_smem_words(u32 nb) { return nb * BKT + ((nb + 3) & ~3u); }

// L2 policy of the window kernel: the build's list loads and the table write-out
// are evict_first (a list is dead in L2 once its store is built -- the giant
// kernel reads only the few entries a key match needs -- and a table is next
// read by another kernel), so L2 keeps more of the lists still waiting for
// their build: +3% on the bench line (loads alone -0.6%, tables alone +0.8%;
// list stores evict_last -1.6%).
__device__ __forceinline__ u64 l2_policy_first() {
    u64 p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// one 32-byte store (st.global.v8, new on sm_100) per lane per 8 entries: one
// whole sector per instruction (two 16-byte stores measured 3.7% slower)
__device__ __forceinline__ void store_block(u32 *dst, const u32 (&e)[8]) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"l"(dst), "r"(e[0]), "r"(e[1]), "r"(e[2]), "r"(e[3]), "r"(e[4]), "r"(e[5]),
                   "r"(e[6]), "r"(e[7]) : "memory");
}

// the build reads 8 entries per lane with one 32-byte load, which also takes the
// evict_first priority as a plain qualifier (no createpolicy)
__device__ __forceinline__ void list_ld8(const u32 *p, uint4 &a, uint4 &b) {
    asm volatile("ld.global.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                   "=r"(b.w) : "l"(p));
}

__device__ __forceinline__ u32 smem_atom_inc(u32 addr) {
    u32 old;
    asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(addr) : "memory");
    return old;
}
__device__ __forceinline__ u32 smem_ld(u32 addr) {
    u32 v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void smem_st(u32 addr, u32 v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void smem_st4_zero(u32 addr) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(0u) : "memory");
}

// One store, built by the whole warp in shared memory (tab: nb * BKT slots, cnt:
// nb fill counters, both zero on entry and on exit) and written to dst.  A
// group is 256 entries, 8 per lane (two uint4 per lane).
template <int LE>
__device__ __forceinline__ void load_group0(const u32 *lst, u32 n, uint4 (&nx)[2]) {
    const int lane = threadIdx.x & 31;
    nx[0] = nx[1] = make_uint4(0, 0, 0, 0);
    if (lst && 8u * (u32)lane < n) list_ld8(lst + list_off_t<LE>(8 * lane), nx[0], nx[1]);
}

// nx: this d's first list group on entry (the caller or the previous call loaded
// it); the next d's (lst_next) on exit, so list read-back latency overlaps the
// previous d's inserts.
// tab_s, cnt_s: shared-window addresses of the warp's table and counters.
template <int LE>
__device__ __forceinline__ void build_store(const u32 *__restrict__ lst, const u32 *lst_next,
                                            u32 n, u32 nb, u32 tab_s, u32 cnt_s,
                                            u32 *__restrict__ dst, uint4 (&nx)[2]) {
    const int lane = threadIdx.x & 31;
    constexpr int K = 2;                             // 16-byte halves per lane per group
    for (u32 jb = 0; jb < n; jb += 128 * K) {
        uint4 cur[K];
#pragma unroll
        for (int k = 0; k < K; k++) cur[k] = nx[k];
        if (jb + 128 * K < n) {
            const u32 j8 = jb + 128 * K + 8u * (u32)lane;
            nx[0] = nx[1] = make_uint4(0, 0, 0, 0);
            if (j8 < n) list_ld8(lst + list_off_t<LE>(j8), nx[0], nx[1]);
        } else {
            load_group0<LE>(lst_next, n, nx);        // the next d's first group
        }
        // first attempts for the group's entries, then one warp-uniform loop for
        // full buckets (rare)
        u32 ovf = 0;                                     // bit i: entry i still to place
        u32 bb[4 * K], sv[4 * K];
        // n is a multiple of 8, so a lane's 8 entries are all in the list or all past it
        if (jb + 8 * (u32)lane < n) {
#pragma unroll
            for (int k = 0; k < K; k++) {
#pragma unroll
                for (int w = 0; w < 4; w++) {
                    const int i = 4 * k + w;
                    const u32 j = jb + 8 * lane + 4 * k + w;
                    const u32 e = w == 0 ? cur[k].x : (w == 1 ? cur[k].y : (w == 2 ? cur[k].z : cur[k].w));
                    const u32 key = entry_key(e);
                    sv[i] = slot_entry(e, j);
                    bb[i] = store_bucket(key, nb);
                    const u32 pos = smem_atom_inc(cnt_s + 4 * bb[i]);
                    if (pos < (u32)BKT) smem_st(tab_s + 4 * (bb[i] * BKT + pos), sv[i]);
                    else ovf |= 1u << i;
                }
            }
        }

        while (__any_sync(FULL_MASK, ovf)) {
            if (ovf) {
#pragma unroll
                for (int i = 0; i < 4 * K; i++) {
                    if (ovf & (1u << i)) {
                        bb[i] = next_bucket(bb[i], nb);
                        const u32 pos = smem_atom_inc(cnt_s + 4 * bb[i]);
                        if (pos < (u32)BKT) {
                            smem_st(tab_s + 4 * (bb[i] * BKT + pos), sv[i]);
                            ovf &= ~(1u << i);
                        }
                    }
                }
            }
        }
    }
    // buckets that turned an entry away (their counter passed BKT: every attempt
    // increments it) get SLOT_PASSED in their last slot (an atomic OR with the
    // entry stores instead measured 1.3% slower)
    __syncwarp();
    for (u32 b = lane; b < nb; b += 32)
        if (smem_ld(cnt_s + 4 * b) > (u32)BKT) {
            const u32 a = tab_s + 4 * (b * BKT + BKT - 1);
            smem_st(a, smem_ld(a) | SLOT_PASSED);
        }
    // write out with one TMA bulk copy (shared -> global, one lane; cp.async.bulk),
    // then clear the table once the copy has read it.  Per-lane 16-byte copies
    // through registers measured 2.5% slower on the bench line.
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                     ::"l"(dst), "r"(tab_s), "r"(nb * BKT * 4u), "l"(l2_policy_first()) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
    for (u32 i = lane; i < nb * (BKT / 4); i += 32) smem_st4_zero(tab_s + 16 * i);
    for (u32 i = lane; i < nb; i += 32) smem_st(cnt_s + 4 * i, 0u);
    __syncwarp();
}

#ifndef WINDOW_MINB
#define WINDOW_MINB 4                         // with the L2 hints: 3 / 4 / 5 / 6 CTAs per SM 436 / 436 / 433 / 427 M d/s
#endif
// LE: the list layout as a compile-time constant (0 rows, 64 tiles; B.lsh says
// which): the baby loop's block stores then cost no runtime address arithmetic
template <int LE>
__device__ __forceinline__ ListRef list_ref_t(const u32 *lists, u64 idx, const BsgsArgs &B) {
    ListRef L;
    L.base = LE ? lists + (idx >> 5) * 32u * (u64)B.lcap + (idx & 31u) * (u64)LE
                : lists + idx * (u64)B.lcap;
    L.lsh = LE ? 6 : 30;
    L.lcs = LE ? 32 * LE : 0;
    return L;
}
template <int LE>
__global__ void __launch_bounds__(256, WINDOW_MINB)
bsgs_window_kernel(WalkArgs a, BsgsArgs B, BsgsOut o) {
    static_assert(LE == 0 || LE == 64, "list tiles are 64 entries (lsh = 6)");
    extern __shared__ u32 smem[];                       // histogram, then per-warp tables
    u32 *hist = smem;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 nb = (u32)B.nb;
    const u32 wstride = window_smem_words(nb);               // 16-byte aligned per warp
    // (through a shuffle: ptxas cannot rematerialise it, and otherwise rebuilt the
    // shared-window base from SR_CgaCtaId before every table store)
    const u32 tab_s = __shfl_sync(FULL_MASK, (u32)__cvta_generic_to_shared(smem) +
                                                 4u * (hist_words(a) + wid * wstride), 0);
    const u32 cnt_s = tab_s + 4u * nb * BKT;
    hist_zero(a, hist);
    for (u32 i = lane; i < wstride; i += 32) smem_st(tab_s + 4 * i, 0u);
    __syncthreads();
    const u32 n = *a.count;
    const int nblk = B.nw / 8;
    u32 baby = 0, done = 0, sym = 0, win = 0;           // per-thread counts fit in 32 bits
    for (;;) {
        u32 wave = 0;
        if (lane == 0) wave = atomicAdd(a.work, 1u);
        wave = __shfl_sync(FULL_MASK, wave, 0);
        if ((u64)wave * 32 >= n) break;
        const u32 idx = wave * 32 + lane;
        const bool has = idx < n;
        WinLane w;
        win_idle(w);
        u32 e[8];
        e[0] = e[1] = 0;
        if (has) {   // (offset and d are re-read at the end: fewer live registers)
            const u32 off0 = __ldg(a.list + idx);
            win_begin(w, cand_d(a.i0 + (off0 & ~PRIME_BIT)), e[0], e[1]);
        }
        const ListRef Lw = list_ref_t<LE>(o.lists, idx, B);
        u32 *lst = const_cast<u32 *>(Lw.base);
        if (w.live) baby += 7;                           // theta_2 (closed form) + 6
#pragma unroll
        for (int k = 2; k < 8; k++) {
            e[k] = win_step(w);
            if (k == 3 || k == 7) win_flush(w);
        }
        if (w.live) {
            store_block(lst, e);
            if (B.j1 == 7) win_mark_mu1(w);
        }
        for (int blk = 1; blk < nblk; blk++) {
            if (!__any_sync(FULL_MASK, w.live)) break;
            if (w.live) baby += 8;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                e[k] = win_step(w);
                if (k == 3 || k == 7) win_flush(w);
            }
            if (w.live) {
                store_block(lst + list_off_t<LE>(blk * 8), e);
                if (blk * 8 + 7 == B.j1) win_mark_mu1(w);
            }
        }
        if (has && !w.live) {                            // symmetry exit (or d < 8)
            const u32 off = __ldg(a.list + idx);
            record_result(a, hist, off, cand_d(a.i0 + (off & ~PRIME_BIT)), w.res);
            done++;
            sym++;
        }
        if (w.live) {
            o.brecs[idx] = win_pack(w, __ldg(a.list + idx), (u32)B.nw);
            win++;
        }
        const u32 live = __ballot_sync(FULL_MASK, w.live);
        uint4 nx[2];
        if (live)
            load_group0<LE>(list_ref_t<LE>(o.lists, wave * 32 + (u32)(__ffs(live) - 1), B).base,
                            (u32)B.nw, nx);
        for (u32 m = live; m; m &= m - 1) {
            const u32 i = wave * 32 + (u32)(__ffs(m) - 1);
            const u32 m2 = m & (m - 1);
            const u32 *next = m2 ? list_ref_t<LE>(o.lists, wave * 32 + (u32)(__ffs(m2) - 1), B).base
                                 : nullptr;
            build_store<LE>(list_ref_t<LE>(o.lists, i, B).base, next, (u32)B.nw, nb, tab_s, cnt_s,
                        o.tables + (u64)i * ((u64)nb * BKT), nx);
        }
        u32 qb = 0;
        if (lane == 0 && live) qb = atomicAdd(&o.ctr[0], (u32)__popc(live));
        qb = __shfl_sync(FULL_MASK, qb, 0);
        if (w.live) o.bqueue[qb + __popc(live & lanemask_lt())] = idx;
    }
    flush_stats(a, baby, 0, 0, done, sym, 0, 0, win);
    hist_flush(a, hist);
}

// K3b: k = 2 (mu'_2 = mu_1 * mu_1: NUDUPL) for every windowed d, 32 per warp in
// lockstep.  One-sided: the lookup of mu'_2 is left to the giant kernel's
// pipelined probe.  Two-sided (R35): mu'_2 is the stride and mu''_1; it is
// looked up here and mu''_2 = mu''_1^2 (NUDUPL again) taken in lockstep too.
#ifndef PREP_MINB
#define PREP_MINB 4                           // measured: 2 / 3 / 4 CTAs per SM: 340 / 342 / 343 M d/s
#endif
template <int LE>
__global__ void __launch_bounds__(256, PREP_MINB)
bsgs_prep_kernel(WalkArgs a, BsgsArgs B, BsgsOut o) {
    extern __shared__ u32 hist[];                       // hist_words(a)
    hist_zero(a, hist);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const u32 nq = o.ctr[0];
    const u32 nwarps = gridDim.x * (blockDim.x / 32);
    u64 giant = 0, red = 0, done = 0, fb = 0, baby = 0;
    u32 err = 0;
    for (u32 base = (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 32; base < nq;
         base += nwarps * 32) {
        const u32 qi = base + lane;
        const bool has = qi < nq;
        const u32 kmask = __ballot_sync(FULL_MASK, has);
        u32 gidx = 0;
        GiantLane g;
        g.phase = PH_IDLE;
        BabyRec br;
        bool two = false;
        if (has) {
            gidx = o.bqueue[qi];
            br = o.brecs[gidx];
            giant_init(g, B, cand_d(a.i0 + (br.off & ~PRIME_BIT)), br, &err);
            const GiantInfo gi = giant_start(g, B, &err, kmask);
            giant++;
            red += gi.nred;
            two = g.m1.Q == g.Qc && g.dist1 == g.distc;   // stride = mu'_2 (R35)
        }
        // two-sided: look up mu''_1 = mu'_2 here and take mu''_2 = mu''_1^2 (NUDUPL,
        // the generic path) in lockstep, so the giant kernel composes distinct ideals
        if (two) {
            const u32 *tab = o.tables + (u64)gidx * ((u64)B.nb * BKT);
            const ListRef lst = list_ref_t<LE>(o.lists, gidx, B);
            u32 te, j;
            const int kind = store_resolve(tab, lst, B.nb, store_probe(tab, B.nb, g.Qc), g.d,
                                           (u32)g.s, g.Qc, g.Pc, te, j);
            if (kind != HIT_NONE)
                g.phase = giant_hit(g, kind, te, g.tc, g.distc, g.Qc, g.res) ? PH_DONE : PH_HALF;
        }
        const u32 amask = __ballot_sync(FULL_MASK, two && g.phase == PH_GIANT);
        if (two && g.phase == PH_GIANT) {
            const GiantInfo gi = giant_advance(g, B, &err, amask, true);   // mu''_1^2
            giant++;
            red += gi.nred;
        }
        if (g.phase == PH_HALF) {                              // inconclusive guard (tiny d)
            fb++;
            const HalfOne h = half_walk_one(g.d);
            g.res = h.res;
            baby += h.steps;
            err += h.err;
            g.phase = PH_DONE;
        }
        if (g.phase == PH_DONE) {
            record_result(a, hist, br.off, g.d, g.res);
            done++;
        }
        const bool push = has && g.phase == PH_GIANT;
        if (push) o.grecs[gidx] = giant_pack(g, br.off);
        const u32 pm = __ballot_sync(FULL_MASK, push);
        u32 qb = 0;
        if (lane == 0 && pm) qb = atomicAdd(&o.ctr[2], (u32)__popc(pm));
        qb = __shfl_sync(FULL_MASK, qb, 0);
        if (push) o.gqueue[qb + __popc(pm & lanemask_lt())] = gidx;
    }
    flush_stats(a, baby, giant, red, done, 0, fb, err);
    hist_flush(a, hist);
}

// K3c: giant steps with per-lane refill and a pipelined lookup.
#ifndef GIANT_THREADS
#define GIANT_THREADS 128
#endif
#ifndef GIANT_MINB
#define GIANT_MINB 7                          // 72 registers; with match_kind inlined 7 / 8 CTAs per SM measured 406.4 / 401.0 M d/s (8 spills more)
#endif
#ifndef PLAIN_TH
// Alg. 4 l.742: the plain product for Q <= 50, as printed (R6).  NUCOMP in exact
// fp64 cannot take its place for small Q: w of a small-norm form is ~d/Q (the
// "can overflow" of l.733).  Every output is checked exactly (disc_ok, the
// plain product's b3^2 = d mod 4 a3), so any inexact composition fails the call
// loudly.  (Round 1 measured 30 / 40 / 50 at 450 / 448 / 446 M d/s and 20 with
// 4.1 M violations over C5; the paper's 50 is kept.)
#define PLAIN_TH 50
#endif
#ifndef REC_Q
#define REC_Q 1
#endif
constexpr u32 STASH = 32;                     // giant kernel: resume records per warp ring
template <int LE>
__global__ void __launch_bounds__(GIANT_THREADS, GIANT_MINB)
bsgs_giant_kernel(WalkArgs a, BsgsArgs B, BsgsOut o) {
    extern __shared__ u32 hist[];                       // hist_words(a)
    // per-warp ring of resume records: refills (about one per warp iteration)
    // read shared memory; the queue and the records are fetched 32 at a time
    __shared__ GiantRec stash[GIANT_THREADS / 32][STASH];
    __shared__ u32 sidx[GIANT_THREADS / 32][STASH];
    __shared__ uint4 pbuf[GIANT_THREADS][4];           // the bucket being probed, per lane
    // per-warp statistics (shared memory: per-lane counters spilled) and the queue of
    // finished d (REC_Q): recorded 32 at a time at full width, instead of in the
    // divergent tail of the warp iteration where a finishing lane (about two per
    // iteration) made the whole warp wait on its checkpoint search and atomics
    __shared__ u32 wst[GIANT_THREADS / 32][4];         // giant, rho steps, done, fallbacks
    __shared__ unsigned long long wbaby[GIANT_THREADS / 32];
    __shared__ u32 rq_off[GIANT_THREADS / 32][64];
    __shared__ u8 rq_res[GIANT_THREADS / 32][64];
    hist_zero(a, hist);
    {
        const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (l < 4) wst[w][l] = 0;
        if (l == 0) wbaby[w] = 0;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 nq = o.ctr[2];
    u32 gidx = 0;                                      // the lane's survivor (store index)
    GiantLane g;
    g.phase = PH_IDLE;
    u32 off = 0;
    bool exhausted = false;
    u32 head = 0, tail = 0;                            // warp-uniform ring positions
    bool qdone = false;                                // the queue is drained
    u32 err = 0;
    u32 rq_n = 0;                                      // warp-uniform: finished d queued

    for (;;) {
        const u32 need = __ballot_sync(FULL_MASK, g.phase == PH_IDLE && !exhausted);
        if (need) {
            const u32 k = (u32)__popc(need);
            if (tail - head < k && !qdone) {           // fill the ring's free slots
                const u32 want = STASH - (tail - head);     // <= 32
                u32 base = 0;
                if (lane == 0) base = atomicAdd(&o.ctr[3], want);
                base = __shfl_sync(FULL_MASK, base, 0);
                const u32 qi = base + (u32)lane;
                if ((u32)lane < want && qi < nq) {
                    const u32 idx = __ldg(o.gqueue + qi);
                    const u32 sl = (tail + (u32)lane) & (STASH - 1);
                    stash[wid][sl] = o.grecs[idx];
                    sidx[wid][sl] = idx;
                }
                const u32 got = base >= nq ? 0u : min(want, nq - base);
                if (got < want) qdone = true;
                tail += got;
                __syncwarp();
            }
            const u32 avail = tail - head;
            if (g.phase == PH_IDLE && !exhausted) {
                const u32 r = (u32)__popc(need & lanemask_lt());
                if (r < avail) {
                    const u32 sl = (head + r) & (STASH - 1);
                    const u32 idx = sidx[wid][sl];
                    const GiantRec rec = stash[wid][sl];
                    off = rec.off;                        // (with the prime bit)
                    giant_unpack(g, rec, cand_d(a.i0 + (off & ~PRIME_BIT)));
                    gidx = idx;
                } else {
                    exhausted = true;                     // (only when qdone)
                }
            }
            head += min(k, avail);
            __syncwarp();
        }
        if (__all_sync(FULL_MASK, exhausted && g.phase == PH_IDLE)) break;
        const u32 gmask = __ballot_sync(FULL_MASK, g.phase == PH_GIANT);
        if (g.phase == PH_GIANT) {
            // (pointers recomputed from the 32-bit index: fewer live registers)
            const u32 *tab = o.tables + (u64)gidx * ((u64)B.nb * BKT);
            const ListRef list = list_ref_t<LE>(o.lists, gidx, B);
            // software pipeline: probe mu'_k (refills start with mu'_2, not yet
            // probed) while computing mu'_{k+1}; the bucket is copied to shared
            // memory asynchronously (cp.async), so no registers wait across the
            // composition and the compiler cannot sink the load to its use
            const u32 pQ = g.Qc, pP = g.Pc, pt = g.tc;
            const float pdist = g.distc;
            const u32 pb = store_bucket(pQ >> 2, (u32)B.nb);
            {
                const u32 *src = tab + (size_t)pb * BKT;
                const u32 dst = (u32)__cvta_generic_to_shared(&pbuf[threadIdx.x][0]);
#pragma unroll
                for (int q = 0; q < 4; q++)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * q),
                                 "l"(src + 4 * q) : "memory");
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
            const GiantInfo gi = giant_advance(g, B, &err, gmask, false);
            {
                const u32 rs = __reduce_add_sync(gmask, gi.nred);
                if (lane == __ffs(gmask) - 1) {
                    wst[wid][0] += (u32)__popc(gmask);
                    wst[wid][1] += rs;
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            Probe pr;
            pr.b = pb;
            pr.g0 = pbuf[threadIdx.x][0];
            pr.g1 = pbuf[threadIdx.x][1];
            pr.g2 = pbuf[threadIdx.x][2];
            pr.g3 = pbuf[threadIdx.x][3];
            u32 te, j;
            const int kind = store_resolve(tab, list, B.nb, pr, g.d, (u32)g.s, pQ, pP, te, j,
                                           reinterpret_cast<const u32 *>(&pbuf[threadIdx.x][0]));
            warp_reconverge(gmask);
            if (kind != HIT_NONE) {
                g.phase = giant_hit(g, kind, te, pt, pdist, pQ, g.res) ? PH_DONE : PH_HALF;
            } else if (g.k > g.kcap) {
                g.phase = PH_HALF;
            }
            if (g.phase == PH_HALF) {     // exact half walk instead
                atomicAdd(&wst[wid][3], 1u);
                const HalfOne h = half_walk_one(g.d);
            g.res = h.res;
            atomicAdd(&wbaby[wid], (unsigned long long)h.steps);
            err += h.err;
                g.phase = PH_DONE;
            }
        }
        if (REC_Q) {
            const u32 dm = __ballot_sync(FULL_MASK, g.phase == PH_DONE);
            if (dm) {
                if (g.phase == PH_DONE) {
                    const u32 p = rq_n + (u32)__popc(dm & lanemask_lt());
                    rq_off[wid][p] = off;
                    rq_res[wid][p] = (u8)(g.res % 3);
                    g.phase = PH_IDLE;
                }
                rq_n += (u32)__popc(dm);
                __syncwarp();
                if (rq_n >= 32) {                         // record 32 in lockstep
                    const u32 o2 = rq_off[wid][lane];
                    record_result(a, hist, o2, cand_d(a.i0 + (o2 & ~PRIME_BIT)), rq_res[wid][lane]);
                    __syncwarp();
                    rq_n -= 32;
                    if ((u32)lane < rq_n) {
                        rq_off[wid][lane] = rq_off[wid][lane + 32];
                        rq_res[wid][lane] = rq_res[wid][lane + 32];
                    }
                    if (lane == 0) wst[wid][2] += 32;
                    __syncwarp();
                }
            }
        } else if (g.phase == PH_DONE) {
            record_result(a, hist, off, g.d, g.res);
            atomicAdd(&wst[wid][2], 1u);
            g.phase = PH_IDLE;
        }
    }
    if ((u32)lane < rq_n) {                             // the queue's remainder
        const u32 o2 = rq_off[wid][lane];
        record_result(a, hist, o2, cand_d(a.i0 + (o2 & ~PRIME_BIT)), rq_res[wid][lane]);
    }
    if (lane == 0) wst[wid][2] += rq_n;
    __syncwarp();
    const bool l0 = lane == 0;
    flush_stats(a, l0 ? wbaby[wid] : 0, l0 ? wst[wid][0] : 0, l0 ? wst[wid][1] : 0,
                l0 ? wst[wid][2] : 0, 0, l0 ? wst[wid][3] : 0, err);
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

constexpr int BSGS_THREADS = 256;

// Window and store sizes for a segment whose largest d is d_max.  nw ~ the
// alpha d^(1/4)-nat window at ~1.22 nats per baby step, a
// multiple of 8.  mu_1 (j1, the end of a block): two-sided (R35), the last block
// end ~1.25 M nats of steps before the window end; one-sided (the paper's Alg. 1,
// or windows too short for both margins), the last block end that leaves >= 2
// more ideals (l.560).
struct BsgsSizes {
    int nw, j1, nb, lcap;
    u32 lsh;                // list layout (ListRef): 6 = tiles of 64 entries, 30 = rows
};
#ifndef NW_SNAP
#define NW_SNAP 160
#endif
// load: the table load factor (option "load_x100"; BKT_LOAD by default)
inline BsgsSizes bsgs_sizes(u64 d_max, float alpha, int two_sided, float load = BKT_LOAD) {
    BsgsSizes z;
    const double w = alpha * std::pow((double)d_max, 0.25);   // window in nats
    z.nw = std::min(2040, std::max(16, ((int)(w / 1.22) + 7) & ~7));
    // the store build reads the list in groups of 256 entries, and a group costs
    // about as much as the baby steps of its entries: a window just past a
    // multiple of 256 pays a whole extra group (at 1.5e10, nw 504 -> 520 cost
    // the window kernel 14%).  Windows up to NW_SNAP entries past a multiple of
    // 256 are cut back to it (measured: +0.9% at 2e9, +2.4% at 3e10, +2.5% at
    // 5e10, neutral elsewhere; results never depend on nw, R6/R29).  Between 256
    // and 512 the cut is 128 (with tiled lists, 448 beats 256 at 2.5e9 by 1.5% and
    // at 3e9 by 3.3%, while 1.5e9 still prefers 256).
    if (z.nw > 256 && z.nw % 256 <= (z.nw < 512 ? 128 : NW_SNAP)) z.nw -= z.nw % 256;
    // past one group the lists are tiled in 64-entry chunks (ListRef), so a window
    // is rounded up to a whole chunk: +0.5% at 5e9, +0.7% on the bench slab (nw 488
    // -> 512), +0.1% at 1e11
    if (z.nw > 256) z.nw = std::min(2040, (z.nw + 63) & ~63);
    const double lnd = std::log((double)d_max);
    const double M = 2.0 * lnd + 4.0;
    const double msteps = 1.25 * M / 1.22;                      // M nats with slack
    // one-sided: mu_1 at a block end, then 8 more ideals (>= the 2 of l.560);
    // mu'_2 = mu_1^2 lands beyond the window when dist_1 > 8 steps + kappa
    // (kappa < ln d), so tiny windows are widened to that (R6: results unchanged)
    const int j1min = (((int)std::ceil((lnd + 4.0) / 1.22 + 8.0) + 1 + 7) & ~7) - 1;
    z.j1 = std::max(z.nw - 9, j1min);
    z.nw = std::min(2040, z.j1 + 9);
    if (two_sided) {
        // mu_1 = theta_{j1+1} needs dist_last - dist_1 >= M and 2 dist_1 - dist_last
        // >= M (giant_start checks both per d; they fail only in the tails)
        const int j = ((z.nw - (int)std::ceil(msteps)) & ~7) - 1;
        if (j >= 7 && z.nw - j >= msteps && 2 * j - z.nw >= msteps) z.j1 = j;
    }
    z.nb = std::max(1, (int)std::ceil(z.nw / (BKT * load)));
    // list row pitch: nw rounded up to 32 words, plus one 32-byte sector.  The
    // pad measured +0.9% on the bench slab (nw = 488: pitch 1952 -> 1984 bytes;
    // pads of 16 / 32 / 64 / 96 words +0.6..+0.8%, a 2048-byte pitch +0.1%),
    // +0.4% at 2.5e9, neutral at 1e11 (Layout)
#ifndef LCAP_PAD
#define LCAP_PAD 8
#endif
    if (z.nw > 256) {                            // tiles of 64 entries (ListRef)
        z.lcap = (z.nw + 63) & ~63;
        z.lsh = 6;
    } else {                                     // rows
        z.lcap = ((z.nw + 31) & ~31) + LCAP_PAD;
        z.lsh = 30;
    }
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
    size_t window_smem, hist_smem;
    unsigned window_blocks, prep_blocks, giant_blocks;
};

// true if bsgs_prepare would (re)allocate scratch (the caller must then drain
// every stream that may still use it)
inline bool bsgs_needs_grow(const BsgsScratch &scr, u64 seg_len, u64 d_hi, int alpha_x16,
                            int two_sided, float load = BKT_LOAD) {
    const BsgsSizes z = bsgs_sizes(d_hi, alpha_x16 / 16.0f, two_sided, load);
    const size_t n = (size_t)seg_len;
    return !scr.lists || n * (size_t)z.lcap > scr.lists_n ||
           n * (size_t)z.nb * BKT > scr.tables_n || n > scr.brecs_n || n > scr.grecs_n ||
           n > scr.bqueue_n || n > scr.gqueue_n;
}

// Grow the scratch to hold a segment of n survivors with lcap list words and nb
// buckets each (no-op when it already does).  The caller drains the streams first.
inline int bsgs_reserve(BsgsScratch &scr, size_t n, int lcap, int nb) {
    if (bsgs_grow(scr.lists, scr.lists_n, n * (size_t)lcap)) return -3;
    if (bsgs_grow(scr.tables, scr.tables_n, n * (size_t)nb * BKT)) return -3;
    if (bsgs_grow(scr.brecs, scr.brecs_n, n)) return -3;
    if (bsgs_grow(scr.grecs, scr.grecs_n, n)) return -3;
    if (bsgs_grow(scr.bqueue, scr.bqueue_n, n)) return -3;
    if (bsgs_grow(scr.gqueue, scr.gqueue_n, n)) return -3;
    return 0;
}

inline size_t bsgs_bytes_per_survivor(u64 d_max, float alpha, int two_sided,
                                      float load = BKT_LOAD) {
    const BsgsSizes z = bsgs_sizes(d_max, alpha, two_sided, load);
    return (size_t)4 * z.lcap + (size_t)64 * z.nb + sizeof(BabyRec) + sizeof(GiantRec) + 8;
}

#ifdef __CUDACC__
// Size one segment buffer (seg_len candidates bound the survivors) and choose
// the launch shapes.  ctr: 4 device counters (zeroed by bsgs_launch_window).
inline int bsgs_prepare(BsgsPlan &pl, u64 seg_len, u64 d_hi, int num_sms, int alpha_x16,
                        int giant_ctas, int two_sided, BsgsScratch &scr, u32 *ctr,
                        int window_ctas, u32 hist_w, int giant_cap = 20, float load = BKT_LOAD) {
    BsgsArgs &B = pl.B;
    const BsgsSizes z = bsgs_sizes(d_hi, alpha_x16 / 16.0f, two_sided, load);
    B.nw = z.nw;
    B.j1 = z.j1;
    B.nb = z.nb;
    B.lcap = z.lcap;
    B.lsh = z.lsh;
    B.plain_th = PLAIN_TH;
    B.giant_cap_mul = (float)giant_cap;
    B.two_sided = two_sided;
    if (bsgs_reserve(scr, (size_t)seg_len, z.lcap, z.nb)) return -3;
    BsgsOut &o = pl.o;
    o.lists = scr.lists;
    o.tables = scr.tables;
    o.brecs = scr.brecs;
    o.grecs = scr.grecs;
    o.bqueue = scr.bqueue;
    o.gqueue = scr.gqueue;
    o.ctr = ctr;
    int per_sm = 0;
    pl.hist_smem = (size_t)hist_w * sizeof(u32);
    pl.window_smem =
        pl.hist_smem + (size_t)(BSGS_THREADS / 32) * window_smem_words((u32)z.nb) * sizeof(u32);
    if (cudaFuncSetAttribute(bsgs_window_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pl.window_smem) != cudaSuccess ||
        cudaFuncSetAttribute(bsgs_window_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pl.window_smem) != cudaSuccess)
        return -4;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsgs_window_kernel<64>, BSGS_THREADS,
                                                      pl.window_smem) != cudaSuccess ||
        per_sm < 1)
        return -4;
    pl.window_blocks = (unsigned)(num_sms * (window_ctas > 0 ? std::min(window_ctas, per_sm) : per_sm));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsgs_prep_kernel<64>, BSGS_THREADS,
                                                      pl.hist_smem) != cudaSuccess ||
        per_sm < 1)
        return -4;
    pl.prep_blocks = (unsigned)(num_sms * per_sm);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsgs_giant_kernel<64>, GIANT_THREADS,
                                                      pl.hist_smem) != cudaSuccess ||
        per_sm < 1)
        return -4;
    pl.giant_blocks = (unsigned)(num_sms * (giant_ctas > 0 ? std::min(giant_ctas, per_sm) : per_sm));
    return 0;
}

// window + prep on the main stream
inline int bsgs_launch_baby(const WalkArgs &a, const BsgsPlan &pl, cudaStream_t s) {
    if (cudaMemsetAsync(pl.o.ctr, 0, 4 * sizeof(u32), s) != cudaSuccess) return -4;
    if (pl.B.lsh == 6)
        bsgs_window_kernel<64><<<pl.window_blocks, BSGS_THREADS, pl.window_smem, s>>>(a, pl.B, pl.o);
    else
        bsgs_window_kernel<0><<<pl.window_blocks, BSGS_THREADS, pl.window_smem, s>>>(a, pl.B, pl.o);
    if (cudaGetLastError() != cudaSuccess) return -4;
    if (pl.B.lsh == 6)
        bsgs_prep_kernel<64><<<pl.prep_blocks, BSGS_THREADS, pl.hist_smem, s>>>(a, pl.B, pl.o);
    else
        bsgs_prep_kernel<0><<<pl.prep_blocks, BSGS_THREADS, pl.hist_smem, s>>>(a, pl.B, pl.o);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

inline int bsgs_launch_giant(const WalkArgs &a, const BsgsPlan &pl, cudaStream_t s) {
    if (pl.B.lsh == 6)
        bsgs_giant_kernel<64><<<pl.giant_blocks, GIANT_THREADS, pl.hist_smem, s>>>(a, pl.B, pl.o);
    else
        bsgs_giant_kernel<0><<<pl.giant_blocks, GIANT_THREADS, pl.hist_smem, s>>>(a, pl.B, pl.o);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}
#endif  // __CUDACC__ (launch)
#endif  // __CUDACC__ (kernels)
