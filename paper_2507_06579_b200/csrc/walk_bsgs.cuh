// walk_bsgs.cuh -- K3 in BSGS mode: the paper's Algorithm 1
// with residues in Z/3 (l.585-603): baby steps rho into a per-d store, then
// giant steps mu_k = mu_1 * mu'_{k-1} by NUCOMPchoose (forms.cuh), rho-reduction,
// and a store lookup.
//
// Two kernels per segment (phase-pure warps; a fused kernel measured 9/32 warp
// efficiency, K3-giant):
//   bsgs_baby_kernel   warp-synchronous batches of 32 d: bsgs_begin + baby steps
//                      (nearly constant count per d), then the k = 2 giant step
//                      (always NUDUPL, Alg. 4 l.745) for all 32 lanes at once;
//                      unfinished d go to the giant queue with their store.
//   bsgs_giant_kernel  persistent lanes with per-lane refill from the queue
//                      (giant counts are heavy-tailed).
//
// Per-lane state machine (the same functions run in the CPU emulation harness
// tests/emu/kernel_emu.cu):
//   bsgs_begin  theta_1 = 1 and the closed-form first step; store both.
//   bsgs_baby   rho steps while log theta_j < W = alpha d^(1/4) (Alg. 1 loop),
//               each stored as (Q_j, P_j) -> (t(theta_{j+1}), log theta_{j+1});
//               symmetry exit (l.553-556) ends the d; then mu_1 = theta_j and
//               two more ideals (l.559-561).
//   bsgs_giant  one giant step: NUCOMPchoose(mu_1, mu'_{k-1}), rho until reduced
//               (l.564), canonical key, lookup (l.565-569).  A hit theta with
//               log mu'_k - log theta >= 1 gives t(eps) = t(mu'_k) - t(theta)
//               (R14: the guard rejects the trivial eps^0 match).
//   HALF        fallback if the giant-step cap is hit: the half walk.
//
// Store ("dictionary of ideals", l.549, l.607): an open-addressing hash table of
// u64 entries per d in global memory, entry = Q | P<<20 | t<<40 | (2 log2 dist)<<51
// (t unreduced, < 2^11).  The baby kernel zero-fills the 32 stores of a warp
// batch with coalesced 16-byte stores (they are contiguous), so the scattered
// 8-byte slot writes that follow land in complete, L2-resident sectors (no DRAM
// read-modify-write); free slots are found through occupancy bits in shared
// memory (no global reads while inserting), and lookups stop at a zero slot.
// The paper's Bloom filter plays the same role (no false negatives; positives
// verified exactly).
#pragma once
#include "common.cuh"
#include "forms.cuh"
#include "walk_half.cuh"

constexpr float LN2F = 0.69314718f;
constexpr float GUARD_LOG2 = 1.0f / LN2F;    // "log mu'_k - log theta >= 1" in log2 units

enum LanePhase : u32 { PH_IDLE = 0, PH_BABY = 1, PH_GIANT = 2, PH_HALF = 3, PH_DONE = 4 };

struct BsgsArgs {
    int ns_log2;        // store slots per d = 1 << ns_log2
    int cap;            // max stored baby entries (load <= 1/2)
    float alpha;        // baby window factor: W = alpha d^(1/4)
    int plain_th;       // Alg. 4 plain-product threshold on Q (paper: 50)
    float giant_cap_mul;// giant-step cap = giant_cap_mul * (d^(1/4) + 10)
};

// ---------------------------------------------------------------- the store --
// Per d: a hash table of u32 slots keyed on Q, slot = (Q >> 2) | (j + 1) << 18 |
// t << 28 (Q = 2 mod 4 and Q < 2^20, so Q >> 2 < 2^18 is exact; j < 1023 is the
// entry's index in insertion order; t = t(theta) mod 3), plus a dense list
// written in insertion order, list[j] = P | (2 log2 theta) << 19 (P < 2^19).
// Same-Q entries share a probe chain and are told apart by P from the list.
struct Store {
    u32 *bm;            // occupancy bits: word w at bm[w * stride]
    int stride;
    u32 *tab;           // slots of this d
    u32 *list;          // entries of this d in insertion order
    int ns_log2;
};

EIS_HD void store_streaming(u32 *p, u32 v) {
#ifdef __CUDA_ARCH__
    __stcs(p, v);
#else
    *p = v;
#endif
}

EIS_HD u32 store_hash(u32 Q, int ns_log2) { return (Q * 0x9E3779B1u) >> (32 - ns_log2); }

EIS_HD void store_clear(Store &S) {
    for (int w = 0; w < (1 << S.ns_log2) / 32; w++) S.bm[w * S.stride] = 0;
}

EIS_HD void store_insert(Store &S, u32 j, u32 Q, u32 P, u32 t3, float dist2) {
    const u32 mask = (1u << S.ns_log2) - 1;
    u32 h = store_hash(Q, S.ns_log2);
    const float fx = dist2 * 2.0f;
    const u32 dfx = fx <= 0.f ? 0u : (fx >= 8191.f ? 8191u : (u32)fx);   // floor, 0.5 units
    store_streaming(&S.list[j], P | (dfx << 19));   // evict-first: keep the tables in L2
    const u32 e = (Q >> 2) | ((j + 1) << 18) | (t3 << 28);
    for (;;) {
        u32 *wp = &S.bm[(h >> 5) * S.stride];
        const u32 w = *wp;
        const u32 fr = ~w & (0xffffffffu << (h & 31));
        if (fr) {
            const u32 slot = (h & ~31u) | (u32)(__builtin_ctz_portable(fr));
            *wp = w | (1u << (slot & 31));
            S.tab[slot] = e;
            return;
        }
        h = ((h | 31u) + 1) & mask;
    }
}

// Look (Q, P) up.  Tables are zero-filled before use (a slot is never 0: j+1 >= 1),
// so linear probing stops at the first empty slot.  Slots are read four at a
// time (one aligned 16-byte load per group; at load <= 1/2 the chain almost
// always ends inside the first group).  Split in two so the giant kernel can
// issue the first group load, compute the next giant step, and only then
// resolve the probe (the next step does not depend on the lookup).
// Returns true with t3 and the stored log2 distance on a hit.
struct Probe {
    u32 h;              // first slot
    uint4 grp;          // the aligned group holding slot h
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

EIS_HD bool store_resolve(const u32 *tab, const u32 *list, int ns_log2, Probe p, u32 Q, u32 P,
                          u32 &t3, float &dist2) {
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
            if (e == 0) return false;
            if ((e & 0x3FFFFu) == qk) {
                const u32 le = list[((e >> 18) & 1023u) - 1];
                if ((le & 0x7FFFFu) == P) {
                    t3 = e >> 28;
                    dist2 = (float)(le >> 19) * 0.5f;
                    return true;
                }
            }
        }
        h = ((h | 3u) + 1) & mask;
        g = load_group(tab, h);
    }
}
EIS_HD bool store_lookup(const u32 *tab, const u32 *list, int ns_log2, u32 Q, u32 P, u32 &t3,
                         float &dist2) {
    return store_resolve(tab, list, ns_log2, store_probe(tab, ns_log2, Q), Q, P, t3, dist2);
}

EIS_HD u32 mod3(u32 v) { return v % 3u; }

// ------------------------------------------------------------ baby phase --
struct BsgsLane {
    u64 d;
    float sqrtd_f, W2;  // W in log2 units
    BabyState st;
    float dist;         // log2 theta_{j+1} of the current baby ideal
    int n_ent, extras;
    u32 Q1, P1, t1;     // mu_1 (t reduced mod 3)
    float dist1;
    u32 phase, res;
};

// rho step with the log2 of the generator multiplier (P_j + sqrt d)/Q_{j-1}
EIS_HD bool rho_step_dist(BabyState &st, float sqrtd_f, float &dist) {
    const u32 num = st.P + st.s;
    const float nf = u32_to_f_exact(num);
    const float rq = rcp_approx(u32_to_f_exact(st.Q));
    const u32 nq0 = 0x4B000000u - f2u_bits(fmaf(nf, rq, 8388608.0f));
    const i32 r0 = (i32)(nq0 * st.Q + num);
    const u32 m = (u32)(r0 >> 31);
    const u32 Pn = st.s - (u32)r0 - (st.Q & m);
    const u32 q = m - nq0;
    const u32 Qn = st.Qp + q * (st.P - Pn);
    st.t2 += (Pn & 2u) + 2u;
    dist += log2_approx((u32_to_f_exact(Pn) + sqrtd_f) * rq);
    const bool eP = (Pn == st.P);
    st.Qp = st.Q;
    st.Q = Qn;
    st.P = Pn;
    return (Qn == st.Qp) | eP;
}

// Start d: store theta_1 and theta_2.  Returns true if d is already finished.
EIS_HD bool bsgs_begin(BsgsLane &ln, Store &S, const BsgsArgs &B, u64 d) {
    ln.d = d;
    u32 r1;
    const bool fin = baby_init(ln.st, d, &r1);
    ln.sqrtd_f = (float)sqrt((double)d);
    ln.W2 = B.alpha * sqrtf(ln.sqrtd_f) / LN2F;
    if (fin) {
        ln.res = r1;
        ln.phase = PH_DONE;
        return true;
    }
    store_clear(S);
    // theta_1 = 1 <-> (2, P*) with P* the odd representative in (s-2, s] = P_1
    store_insert(S, 0u, 2u, ln.st.P, 0u, 0.f);
    // theta_2 = ((P_1 + sqrt d)/2) theta_1 <-> (Q_1, P_1)
    ln.dist = log2_approx(((float)ln.st.P + ln.sqrtd_f) * 0.5f);
    store_insert(S, 1u, ln.st.Q, ln.st.P, mod3(ln.st.t2 >> 1), ln.dist);
    ln.n_ent = 2;
    ln.extras = -1;
    ln.phase = PH_BABY;
    return false;
}

// Up to `kmax` baby steps.  Sets ln.phase to PH_DONE (symmetry exit) or
// PH_GIANT (window complete).  Returns the number of rho steps taken.
// Software-pipelined: the store insert of entry j (a shared-memory
// read-modify-write chain) is issued after the rho step j+1, so the two
// dependency chains overlap; the pending entry is flushed before returning.
EIS_HD int bsgs_baby(BsgsLane &ln, Store &S, const BsgsArgs &B, int kmax) {
    int k = 0;
    bool have = false;
    u32 pj = 0, pQ = 0, pP = 0, pt = 0;
    float pd = 0.f;
    for (; k < kmax; k++) {
        if (ln.extras < 0 && (ln.dist >= ln.W2 || ln.n_ent >= B.cap)) {
            ln.Q1 = ln.st.Q;                 // mu_1 = theta_j
            ln.P1 = ln.st.P;
            ln.t1 = mod3(ln.st.t2 >> 1);
            ln.dist1 = ln.dist;
            ln.extras = 2;                   // "Compute two more ideals" (l.560)
        }
        if (ln.extras == 0) {
            ln.phase = PH_GIANT;
            break;
        }
        const bool ex = rho_step_dist(ln.st, ln.sqrtd_f, ln.dist);
        if (have) store_insert(S, pj, pQ, pP, pt, pd);
        pj = (u32)ln.n_ent;
        pQ = ln.st.Q;
        pP = ln.st.P;
        pt = mod3(ln.st.t2 >> 1);
        pd = ln.dist;
        have = true;
        ln.n_ent++;
        if (ex) {
            ln.res = baby_result(ln.st);
            ln.phase = PH_DONE;
            k++;
            break;
        }
        if (ln.extras > 0) ln.extras--;
    }
    if (have) store_insert(S, pj, pQ, pP, pt, pd);
    return k;
}

// ----------------------------------------------------------- giant phase --
struct GiantLane {
    u64 d;
    i64 s, L;           // isqrt(d), floor(d^(1/4))
    double sqrtd;
    Mu1Form m1;
    u32 t1;
    float dist1;
    u32 Qc, Pc, tc;     // mu'_{k-1}
    float distc;
    int k, kcap;
    u32 phase, res;
};

// Giant-phase state from mu_1 (k = 1: mu'_1 = mu_1).
EIS_HD void giant_init(GiantLane &g, const BsgsArgs &B, u64 d, u32 Q1, u32 P1, u32 t1,
                       float dist1, u32 *err) {
    g.d = d;
    g.s = (i64)isqrt_u64_dev(d);
    g.L = (i64)isqrt_u64_dev((u64)g.s);            // floor(d^(1/4))
    g.sqrtd = sqrt((double)d);
    g.m1 = mu1_form((i64)Q1, (i64)P1, (i64)d, err);
    g.t1 = t1;
    g.dist1 = dist1;
    g.Qc = Q1;
    g.Pc = P1;
    g.tc = t1;
    g.distc = dist1;
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
EIS_HD GiantInfo giant_advance(GiantLane &g, const BsgsArgs &B, u32 *err) {
    GiantInfo gi;
    const i64 d = (i64)g.d;
    const i64 s = g.s;
    const GiantComp c = giant_compose(g.m1, (i64)g.Qc, (i64)g.Pc, d, s, g.L, (float)g.sqrtd,
                                      B.plain_th, err);
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
    gi.nred = nred;
    g.k++;
    g.Qc = (u32)Q;
    g.Pc = (u32)P;
    g.tc = t;
    g.distc = dist;
    return gi;
}

// Lookup verdict for a giant-step result (Q, P, t, dist):
// a stored theta with log mu'_k - log theta >= 1 gives t(eps) = t - t(theta).
EIS_HD bool giant_hit(u32 te, float de, u32 t, float dist, u32 &res) {
    if (dist - de >= GUARD_LOG2) {
        res = mod3(t + 3u - te);                    // eps = mu'_k / theta
        return true;
    }
    return false;
}

// One unpipelined giant step (advance + lookup): used for k = 2 in the baby
// kernel and by the CPU emulation.  Sets PH_DONE on a hit, PH_HALF past the cap.
EIS_HD GiantInfo bsgs_giant(GiantLane &g, const u32 *tab, const u32 *list, const BsgsArgs &B,
                            u32 *err) {
    const GiantInfo gi = giant_advance(g, B, err);
    u32 te;
    float de;
    if (store_lookup(tab, list, B.ns_log2, g.Qc, g.Pc, te, de) &&
        giant_hit(te, de, g.tc, g.distc, g.res)) {
        g.phase = PH_DONE;
        return gi;
    }
    if (g.k > g.kcap) g.phase = PH_HALF;
    return gi;
}

// ------------------------------------------------------------------ kernels --
// per-d record handed from the baby kernel to the giant kernel (one sector)
// Everything the giant kernel needs to resume a d, precomputed by the baby
// kernel so a refill is two 32-byte loads (no per-d square roots or divisions
// in the divergent refill path).
struct __align__(64) GiantRec {
    double sqrtd;
    i64 w1;                        // mu_1's form coefficient (P1^2 - d)/(2 Q1)
    u32 off, Q1, P1, Qc;           // P1 normalised mod Q1
    u32 Pc, tk, s, Lk;             // tk = t1 | tc << 2 | k << 4; Lk = L | kcap << 16
    float dist1, distc;
    u32 pad[2];
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
    r.pad[0] = r.pad[1] = 0;
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
    g.Qc = r.Qc;
    g.Pc = r.Pc;
    g.distc = r.distc;
    g.phase = PH_GIANT;
}

struct BsgsOut {
    u32 *tables;        // [segment survivors][ns] store slots
    u32 *lists;         // [segment survivors][lcap] store entries
    int lcap;
    GiantRec *recs;     // [segment survivors]
    u32 *queue;         // survivor indices needing giant steps
    u32 *qcount;        // device: queue length
    u32 *qwork;         // device: giant-kernel work counter
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

template <int KB>
__global__ void __launch_bounds__(256)
bsgs_baby_kernel(WalkArgs a, BsgsArgs B, BsgsOut o) {
    extern __shared__ u32 smem[];
    u32 *hist = smem;                              // NROW_MAX * HIST_CAP
    u32 *bmap = smem + NROW_MAX * HIST_CAP;        // (ns/32) words x blockDim
    hist_zero(a, hist);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const u32 n = *a.count;
    Store S;
    S.bm = bmap + threadIdx.x;
    S.stride = blockDim.x;
    S.ns_log2 = B.ns_log2;
    u64 baby = 0, giant = 0, red = 0, done = 0, sym = 0;
    u32 err = 0;

    for (;;) {
        u32 base = 0;
        if (lane == 0) base = atomicAdd(a.work, 32u);
        base = __shfl_sync(FULL_MASK, base, 0);
        if (base >= n) break;
        const u32 idx = base + lane;
        {   // zero the batch's 32 contiguous tables (coalesced, full lines)
            uint4 *z = reinterpret_cast<uint4 *>(o.tables + ((u64)base << B.ns_log2));
            const u32 nz = (min(n - base, 32u) << B.ns_log2) / 4;
            const uint4 zero = make_uint4(0, 0, 0, 0);
            for (u32 c = lane; c < nz; c += 32) z[c] = zero;
            __syncwarp();
        }
        BsgsLane ln;
        ln.phase = PH_IDLE;
        u32 off = 0;
        if (idx < n) {
            off = __ldg(a.list + idx);            // (with the prime bit)
            S.tab = o.tables + ((u64)idx << B.ns_log2);
            S.list = o.lists + (u64)idx * o.lcap;
            baby += 1;
            if (bsgs_begin(ln, S, B, cand_d(a.i0 + (off & ~PRIME_BIT)))) {
                record_result(a, hist, off, ln.d, ln.res);
                done++;
                sym++;
                ln.phase = PH_IDLE;
            }
        }
        while (__any_sync(FULL_MASK, ln.phase == PH_BABY)) {
            if (ln.phase == PH_BABY) {
                baby += bsgs_baby(ln, S, B, KB);
                if (ln.phase == PH_DONE) {
                    record_result(a, hist, off, ln.d, ln.res);
                    done++;
                    sym++;
                    ln.phase = PH_IDLE;
                }
            }
        }
        // k = 2 for all lanes together: mu_2 = mu_1 * mu_1 (NUDUPL).  Its lookup
        // is left to the giant kernel's pipelined probe (no memory wait here).
        bool push = false;
        if (ln.phase == PH_GIANT) {
            GiantLane g;
            giant_init(g, B, ln.d, ln.Q1, ln.P1, ln.t1, ln.dist1, &err);
            const GiantInfo gi = giant_advance(g, B, &err);
            giant++;
            red += gi.nred;
            const GiantRec r = giant_pack(g, off);
            o.recs[idx] = r;
            push = true;
        }
        const u32 pm = __ballot_sync(FULL_MASK, push);
        if (pm) {
            u32 qb = 0;
            const int leader = __ffs(pm) - 1;
            if (lane == leader) qb = atomicAdd(o.qcount, (u32)__popc(pm));
            qb = __shfl_sync(FULL_MASK, qb, leader);
            if (push) o.queue[qb + __popc(pm & lanemask_lt())] = idx;
        }
    }
    flush_stats(a, baby, giant, red, done, sym, 0, err);
    hist_flush(a, hist);
}

__global__ void __launch_bounds__(256)
bsgs_giant_kernel(WalkArgs a, BsgsArgs B, BsgsOut o) {
    __shared__ u32 hist[NROW_MAX * HIST_CAP];
    hist_zero(a, hist);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const u32 nq = *o.qcount;
    const u32 *tab = nullptr, *list = nullptr;
    GiantLane g;
    g.phase = PH_IDLE;
    u32 off = 0;
    bool exhausted = false, pending = false;
    u64 baby = 0, giant = 0, red = 0, done = 0, fb = 0;
    u32 err = 0;

    for (;;) {
        const u32 need = __ballot_sync(FULL_MASK, g.phase == PH_IDLE && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            u32 base = 0;
            if (lane == leader) base = atomicAdd(o.qwork, (u32)__popc(need));
            base = __shfl_sync(FULL_MASK, base, leader);
            if (g.phase == PH_IDLE && !exhausted) {
                const u32 qi = base + __popc(need & lanemask_lt());
                if (qi < nq) {
                    const u32 idx = __ldg(o.queue + qi);
                    const GiantRec r = o.recs[idx];
                    off = r.off;                          // (with the prime bit)
                    giant_unpack(g, r, cand_d(a.i0 + (off & ~PRIME_BIT)));
                    pending = true;               // mu'_2 is probed with the next advance
                    tab = o.tables + ((u64)idx << B.ns_log2);
                    list = o.lists + (u64)idx * o.lcap;
                } else {
                    exhausted = true;
                }
            }
        }
        if (__all_sync(FULL_MASK, exhausted && g.phase == PH_IDLE)) break;
        if (g.phase == PH_GIANT) {
            // software pipeline: probe mu'_k (queued on refill already checked
            // for k = 2: `pending` false) while computing mu'_{k+1}
            const u32 pQ = g.Qc, pP = g.Pc, pt = g.tc;
            const float pdist = g.distc;
            Probe pr;
            pr.h = 0;
            pr.grp = make_uint4(0, 0, 0, 0);
            if (pending) pr = store_probe(tab, B.ns_log2, pQ);
            const GiantInfo gi = giant_advance(g, B, &err);
            giant++;
            red += gi.nred;
            u32 te;
            float de;
            if (pending && store_resolve(tab, list, B.ns_log2, pr, pQ, pP, te, de) &&
                giant_hit(te, de, pt, pdist, g.res)) {
                g.phase = PH_DONE;
            } else if (g.k > g.kcap) {
                g.phase = PH_HALF;
            }
            pending = true;
            if (g.phase == PH_HALF) {     // cap exceeded: exact half walk instead
                fb++;
                BabyState st;
                u32 r1;
                if (baby_init(st, g.d, &r1)) {
                    g.res = r1;
                } else {
                    const u32 cap = half_step_cap(st.s);
                    u32 j = 0;
                    bool ok;
                    do { baby++; ok = baby_step(st); } while (!ok && ++j <= cap);
                    if (ok) g.res = baby_result(st);
                    else { err++; g.res = 0xFFu; }
                }
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
    u32 *tables = nullptr;
    size_t tables_bytes = 0;
    u32 *lists = nullptr;
    size_t lists_n = 0;
    GiantRec *recs = nullptr;
    size_t recs_n = 0;
    u32 *queue = nullptr;
    size_t queue_n = 0;
};

inline void bsgs_free(BsgsScratch &s) {
    if (s.tables) cudaFree(s.tables);
    if (s.lists) cudaFree(s.lists);
    if (s.recs) cudaFree(s.recs);
    if (s.queue) cudaFree(s.queue);
    s = BsgsScratch();
}

constexpr int BSGS_KB = 8;
constexpr int BSGS_THREADS = 256;

// store size for a segment whose largest d is d_max (load <= 1/2)
inline int bsgs_ns_log2(u64 d_max, float alpha) {
    const double w = alpha * std::pow((double)d_max, 0.25);   // window in nats
    // ~1.22 nats per baby step: the window needs ~w/1.22 entries;
    // size for load <= 1/2 at 95% of that (the cap ends the window a little
    // early for the longest walks, which only adds giant steps).
    const double need = 2.0 * 0.95 * (w / 1.22) + 8.0;
    int l = 6;
    while ((double)(1 << l) < need && l < 10) l++;
    return l;
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

// Per-segment BSGS launch plan: arguments shared by the two kernels.
struct BsgsPlan {
    BsgsArgs B;
    BsgsOut o;
    size_t baby_smem;
    unsigned baby_blocks, giant_blocks;
};

// Size the scratch of one segment buffer (`seg_len` candidates bounds its
// survivors) and choose the launch shapes.  qctr: 2 device counters.
inline int bsgs_prepare(BsgsPlan &pl, u64 seg_len, u64 d_hi, int num_sms, int alpha_x16,
                        int baby_l2_mb, int giant_ctas, BsgsScratch &scr, u32 *qctr) {
    BsgsArgs &B = pl.B;
    B.alpha = alpha_x16 / 16.0f;
    B.ns_log2 = bsgs_ns_log2(d_hi, B.alpha);
    B.cap = (1 << B.ns_log2) / 2 - 2;
    B.plain_th = 50;
    B.giant_cap_mul = 20.0f;
    const size_t n = (size_t)seg_len;
    size_t tb = scr.tables_bytes;
    if (bsgs_grow(scr.tables, tb, (n + 32) << B.ns_log2)) return -3;   // +32: batch tail
    scr.tables_bytes = tb;
    const int lcap = (B.cap + 2 + 31) & ~31;
    if (bsgs_grow(scr.lists, scr.lists_n, n * (size_t)lcap)) return -3;
    if (bsgs_grow(scr.recs, scr.recs_n, n)) return -3;
    if (bsgs_grow(scr.queue, scr.queue_n, n)) return -3;
    BsgsOut &o = pl.o;
    o.tables = scr.tables;
    o.lists = scr.lists;
    o.lcap = lcap;
    o.recs = scr.recs;
    o.queue = scr.queue;
    o.qcount = qctr;
    o.qwork = qctr + 1;
    // Baby kernel: the stores being filled are written at random slots; keep
    // the resident ones within an L2 budget (option "baby_l2_mb") so partially
    // written sectors are not evicted to DRAM (measured: 2x DRAM
    // read-modify-write traffic otherwise).
    const size_t store_bytes = (size_t)4 << B.ns_log2;
    const int bt = BSGS_THREADS;
    pl.baby_smem = (size_t)(NROW_MAX * HIST_CAP) * 4 + (size_t)(1 << B.ns_log2) / 32 * bt * 4;
    if (cudaFuncSetAttribute(bsgs_baby_kernel<BSGS_KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pl.baby_smem) != cudaSuccess)
        return -4;
    int per_sm_b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, bsgs_baby_kernel<BSGS_KB>, bt,
                                                      pl.baby_smem) != cudaSuccess ||
        per_sm_b < 1)
        return -4;
    const size_t lanes_l2 = ((size_t)baby_l2_mb << 20) / store_bytes;
    pl.baby_blocks = (unsigned)std::max<size_t>(
        1, std::min<size_t>((size_t)num_sms * per_sm_b, lanes_l2 / bt));
    int per_sm_g = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_g, bsgs_giant_kernel, BSGS_THREADS,
                                                      0) != cudaSuccess ||
        per_sm_g < 1)
        return -4;
    // giant_ctas > 0 caps the giant kernel's CTAs per SM so that the next
    // segment's baby kernel (other stream) can be resident at the same time
    pl.giant_blocks = (unsigned)(num_sms * (giant_ctas > 0 ? std::min(giant_ctas, per_sm_g) : per_sm_g));
    return 0;
}

inline int bsgs_launch_baby(const WalkArgs &a, const BsgsPlan &pl, cudaStream_t s) {
    if (cudaMemsetAsync(pl.o.qcount, 0, 2 * sizeof(u32), s) != cudaSuccess) return -4;
    bsgs_baby_kernel<BSGS_KB><<<pl.baby_blocks, BSGS_THREADS, pl.baby_smem, s>>>(a, pl.B, pl.o);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

inline int bsgs_launch_giant(const WalkArgs &a, const BsgsPlan &pl, cudaStream_t s) {
    bsgs_giant_kernel<<<pl.giant_blocks, BSGS_THREADS, 0, s>>>(a, pl.B, pl.o);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}
#endif  // __CUDACC__
