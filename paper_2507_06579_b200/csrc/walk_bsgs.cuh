// walk_bsgs.cuh -- K3 in BSGS mode: the paper's Algorithm 1
// with residues in Z/3 (l.585-603): baby steps rho into a per-d store, then
// giant steps mu_k = mu_1 * mu'_{k-1} by NUCOMPchoose (forms.cuh), rho-reduction,
// and a store lookup.  One lane per d, persistent CTAs, warp-aggregated refill.
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
// u64 entries per lane in global memory (Q | P<<20 | t<<40 | log2-dist*256 <<42)
// whose occupancy bits live in shared memory (so empty slots are never read
// and never need clearing in HBM).  The paper's Bloom filter plays the same
// role (no false negatives; positives verified exactly).
#pragma once
#include "common.cuh"
#include "forms.cuh"
#include "walk_half.cuh"

constexpr float LN2F = 0.69314718f;
constexpr float GUARD_LOG2 = 1.0f / LN2F;    // "log mu'_k - log theta >= 1" in log2 units

enum LanePhase : u32 { PH_IDLE = 0, PH_BABY = 1, PH_GIANT = 2, PH_HALF = 3, PH_DONE = 4 };

struct BsgsArgs {
    u64 *tables;        // [lanes][ns] entries
    int ns_log2;        // table slots per lane = 1 << ns_log2
    int cap;            // max stored baby entries (load <= 1/2)
    float alpha;        // baby window factor: W = alpha d^(1/4)
    int plain_th;       // Alg. 4 plain-product threshold on Q (paper: 50)
    float giant_cap_mul;// giant-step cap = giant_cap_mul * (d^(1/4) + 10)
};

struct BsgsLane {
    u64 d;
    i64 L;              // floor(d^(1/4)) for NUCOMP's partial Euclid bound
    double sqrtd;
    float sqrtd_f, W2;  // W in log2 units
    BabyState st;
    float dist;         // log2 theta_{j+1} of the current baby ideal
    int n_ent, extras;
    u32 Q1, P1, t1;     // mu_1
    float dist1;
    u32 Qc, Pc, tc;     // mu'_{k-1}
    float distc;
    int k, kcap;
    u32 phase, res;
};

// ---------------------------------------------------------------- the store --
struct Store {
    u32 *bm;            // occupancy bits: word w of this lane at bm[w * stride]
    int stride;
    u64 *tab;           // this lane's slots
    int ns_log2;
};

EIS_HD u32 store_hash(u32 Q, u32 P, int ns_log2) {
    return ((Q * 0x9E3779B1u) ^ (P * 0x85EBCA77u)) >> (32 - ns_log2);
}

EIS_HD void store_clear(Store &S) {
    for (int w = 0; w < (1 << S.ns_log2) / 32; w++) S.bm[w * S.stride] = 0;
}

EIS_HD void store_insert(Store &S, u32 Q, u32 P, u32 t, float dist2) {
    const u32 mask = (1u << S.ns_log2) - 1;
    u32 h = store_hash(Q, P, S.ns_log2);
    float fx = dist2 * 256.0f + 0.5f;
    u64 dfx = fx <= 0.f ? 0 : (fx >= 4194303.f ? 4194303ull : (u64)fx);
    const u64 e = (u64)Q | ((u64)P << 20) | ((u64)t << 40) | (dfx << 42);
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

// returns the entry or 0
EIS_HD u64 store_lookup(const Store &S, u32 Q, u32 P) {
    const u32 mask = (1u << S.ns_log2) - 1;
    const u64 key = (u64)Q | ((u64)P << 20);
    u32 h = store_hash(Q, P, S.ns_log2);
    for (;;) {
        const u32 w = S.bm[(h >> 5) * S.stride];
        if (!((w >> (h & 31)) & 1)) return 0;
        const u64 e = S.tab[h];
        if ((e & 0xFFFFFFFFFFull) == key) return e;
        h = (h + 1) & mask;
    }
}

// ------------------------------------------------------------ baby phase --
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

EIS_HD u32 mod3(u32 v) { return v % 3u; }

// Start d: store theta_1 and theta_2.  Returns true if d is already finished.
EIS_HD bool bsgs_begin(BsgsLane &ln, Store &S, const BsgsArgs &B, u64 d) {
    ln.d = d;
    u32 r1;
    const bool fin = baby_init(ln.st, d, &r1);
    ln.sqrtd = sqrt((double)d);
    ln.sqrtd_f = (float)ln.sqrtd;
    ln.L = (i64)isqrt_u64_dev((u64)ln.st.s);        // floor(d^(1/4))
    const float d14 = sqrtf(ln.sqrtd_f);
    ln.W2 = B.alpha * d14 / LN2F;
    ln.kcap = (int)(B.giant_cap_mul * (d14 + 10.f));
    if (fin) {
        ln.res = r1;
        ln.phase = PH_DONE;
        return true;
    }
    store_clear(S);
    // theta_1 = 1 <-> (2, P*) with P* the odd representative in (s-2, s] = P_1
    store_insert(S, 2u, ln.st.P, 0u, 0.f);
    // theta_2 = ((P_1 + sqrt d)/2) theta_1 <-> (Q_1, P_1)
    ln.dist = log2_approx(((float)ln.st.P + ln.sqrtd_f) * 0.5f);
    store_insert(S, ln.st.Q, ln.st.P, mod3(ln.st.t2 >> 1), ln.dist);
    ln.n_ent = 2;
    ln.extras = -1;
    ln.phase = PH_BABY;
    return false;
}

// Up to `kmax` baby steps.  Sets ln.phase to PH_DONE (symmetry exit) or
// PH_GIANT (window complete).  Returns the number of rho steps taken.
EIS_HD int bsgs_baby(BsgsLane &ln, Store &S, const BsgsArgs &B, int kmax) {
    int k = 0;
    for (; k < kmax; k++) {
        if (ln.extras < 0 && (ln.dist >= ln.W2 || ln.n_ent >= B.cap)) {
            ln.Q1 = ln.st.Q;                 // mu_1 = theta_j
            ln.P1 = ln.st.P;
            ln.t1 = mod3(ln.st.t2 >> 1);
            ln.dist1 = ln.dist;
            ln.extras = 2;                   // "Compute two more ideals" (l.560)
        }
        if (ln.extras == 0) {
            ln.Qc = ln.Q1;
            ln.Pc = ln.P1;
            ln.tc = ln.t1;
            ln.distc = ln.dist1;
            ln.k = 1;
            ln.phase = PH_GIANT;
            return k;
        }
        const bool ex = rho_step_dist(ln.st, ln.sqrtd_f, ln.dist);
        store_insert(S, ln.st.Q, ln.st.P, mod3(ln.st.t2 >> 1), ln.dist);
        ln.n_ent++;
        if (ex) {
            ln.res = baby_result(ln.st);
            ln.phase = PH_DONE;
            return k + 1;
        }
        if (ln.extras > 0) ln.extras--;
    }
    return k;
}

struct GiantInfo {
    u32 kind;       // composition kind
    u32 nred;       // rho steps in the reduction
};

// One giant step.  Sets PH_DONE on a guarded hit, PH_HALF
// when the cap is exceeded.  *err counts invariant violations.
EIS_HD GiantInfo bsgs_giant(BsgsLane &ln, const Store &S, const BsgsArgs &B, u32 *err) {
    GiantInfo gi;
    const i64 d = (i64)ln.d;
    const i64 s = (i64)ln.st.s;
    const Composed c = nucomp_choose((i64)ln.Q1, (i64)ln.P1, (i64)ln.Qc, (i64)ln.Pc, d, ln.L,
                                     ln.sqrtd, B.plain_th, err);
    gi.kind = c.kind;
    u32 t = mod3(ln.t1 + ln.tc + 3u - c.tg);       // theta(mu_k) = theta(mu_1) theta(mu'_{k-1}) / gamma
    float dist = ln.dist1 + ln.distc - c.lg;
    i64 Q = c.Q, P = c.P;
    u32 nred = 0;
    for (;;) {
        P = s - floor_mod(s - P, Q);                // canonical P in (s - Q, s]
        if (Q - P <= s) break;                      // reduced (R18)
        const i64 q = floor_div(P + s, Q);          // floor((P + sqrt d)/Q)
        const i64 Pn = q * Q - P;
        const i64 Qn = exact_div(d - Pn * Pn, Q, err);
        t = mod3(t + 1u + (u32)((Pn >> 1) & 1));
        dist += log2_approx((float)fabs((double)Pn + ln.sqrtd)) - log2_approx((float)Q);
        P = Pn;
        Q = iabs64(Qn);
        if (++nred > 4096) { *err += 1; break; }
    }
    gi.nred = nred;
    ln.k++;
    const u64 e = store_lookup(S, (u32)Q, (u32)P);
    if (e) {
        const float de = (float)(e >> 42) * (1.0f / 256.0f);
        if (dist - de >= GUARD_LOG2) {
            const u32 te = (u32)((e >> 40) & 3);
            ln.res = mod3(t + 3u - te);             // eps = mu'_k / theta
            ln.phase = PH_DONE;
            return gi;
        }
    }
    ln.Qc = (u32)Q;
    ln.Pc = (u32)P;
    ln.tc = t;
    ln.distc = dist;
    if (ln.k > ln.kcap) ln.phase = PH_HALF;
    return gi;
}

// --------------------------------------------------------------- the kernel --
#ifdef __CUDACC__
template <int KB>
__global__ void __launch_bounds__(256)
walk_bsgs_kernel(WalkArgs a, BsgsArgs B) {
    extern __shared__ u32 smem[];
    u32 *hist = smem;                              // 2 * HIST_CAP
    u32 *bmap = smem + 2 * HIST_CAP;               // (ns/32) words x blockDim
    for (int i = threadIdx.x; i < 2 * a.nb; i += blockDim.x) hist[i] = 0;
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const u32 n = *a.count;
    const u64 gtid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    Store S;
    S.bm = bmap + threadIdx.x;
    S.stride = blockDim.x;
    S.tab = B.tables + (gtid << B.ns_log2);
    S.ns_log2 = B.ns_log2;

    BsgsLane ln;
    ln.phase = PH_IDLE;
    u32 off = 0;
    bool exhausted = false;
    u32 n_done = 0, n_sym = 0, n_fb = 0;
    u64 baby = 0, giant = 0, red = 0;
    u32 err = 0;

    auto finish = [&]() {
        const u32 t = ln.res % 3;
        n_done++;
        if (a.flags) a.flags[off] = (u8)t;
        if (a.ckpt) {
            const int b = bucket_of(a.ckpt, a.b_lo, a.b_lo + a.nb - 1, ln.d) - a.b_lo;
            atomicAdd(&hist[b], 1u);
            if (t == 0) atomicAdd(&hist[a.nb + b], 1u);
        }
        ln.phase = PH_IDLE;
    };

    for (;;) {
        const u32 need = __ballot_sync(FULL_MASK, ln.phase == PH_IDLE && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            u32 base = 0;
            if (lane == leader) base = atomicAdd(a.work, (u32)__popc(need));
            base = __shfl_sync(FULL_MASK, base, leader);
            if (ln.phase == PH_IDLE && !exhausted) {
                const u32 idx = base + __popc(need & lanemask_lt());
                if (idx < n) {
                    off = __ldg(a.list + idx);
                    baby += 1;
                    if (bsgs_begin(ln, S, B, cand_d(a.i0 + off))) { n_sym++; finish(); }
                } else {
                    exhausted = true;
                }
            }
        }
        if (__all_sync(FULL_MASK, exhausted && ln.phase == PH_IDLE)) break;
        if (ln.phase == PH_BABY) {
            baby += bsgs_baby(ln, S, B, KB);
            if (ln.phase == PH_DONE) n_sym++;
        }
        if (ln.phase == PH_GIANT) {
            const GiantInfo gi = bsgs_giant(ln, S, B, &err);
            giant++;
            red += gi.nred;
            if (ln.phase == PH_HALF) {
                n_fb++;
                u32 r1;
                if (baby_init(ln.st, ln.d, &r1)) { ln.res = r1; ln.phase = PH_DONE; }
            }
        }
        if (ln.phase == PH_HALF) {
            for (int k = 0; k < KB; k++) {
                baby++;
                if (baby_step(ln.st)) { ln.res = baby_result(ln.st); ln.phase = PH_DONE; break; }
            }
        }
        if (ln.phase == PH_DONE) finish();
    }

    const u64 s_baby = warp_sum_u64(baby), s_giant = warp_sum_u64(giant),
              s_red = warp_sum_u64(red), s_done = warp_sum_u64(n_done),
              s_sym = warp_sum_u64(n_sym), s_fb = warp_sum_u64(n_fb);
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
    __syncthreads();
    if (a.ckpt) {
        for (int i = threadIdx.x; i < a.nb; i += blockDim.x) {
            if (hist[i])
                atomicAdd((unsigned long long *)&a.buckets[a.b_lo + i], (unsigned long long)hist[i]);
            if (hist[a.nb + i])
                atomicAdd((unsigned long long *)&a.buckets[a.n_ckpt + a.b_lo + i],
                          (unsigned long long)hist[a.nb + i]);
        }
    }
}

// ------------------------------------------------------------- host launch --
struct BsgsScratch {
    u64 *tables = nullptr;
    size_t bytes = 0;
};

inline void bsgs_free(BsgsScratch &s) {
    if (s.tables) cudaFree(s.tables);
    s.tables = nullptr;
    s.bytes = 0;
}

constexpr int BSGS_KB = 8;
constexpr int BSGS_THREADS = 256;

// table size for a segment whose largest d is d_max
inline int bsgs_ns_log2(u64 d_max, float alpha) {
    const double w = alpha * std::pow((double)d_max, 0.25);   // nats
    const double need = 2.0 * (w / 0.9 + 8.0);
    int l = 6;
    while ((double)(1 << l) < need && l < 10) l++;
    return l;
}

inline int launch_bsgs(const WalkArgs &a, u64 d_lo, u64 d_hi, int num_sms, int alpha_x16,
                       BsgsScratch &scr, u32 *, cudaStream_t s, int *launches) {
    (void)d_lo;
    BsgsArgs B;
    B.alpha = alpha_x16 / 16.0f;
    B.ns_log2 = bsgs_ns_log2(d_hi, B.alpha);
    B.cap = (1 << B.ns_log2) / 2 - 2;
    B.plain_th = 50;
    B.giant_cap_mul = 20.0f;
    const size_t smem = (size_t)(2 * HIST_CAP) * 4 + (size_t)(1 << B.ns_log2) / 32 * BSGS_THREADS * 4;
    if (cudaFuncSetAttribute(walk_bsgs_kernel<BSGS_KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return -4;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, walk_bsgs_kernel<BSGS_KB>,
                                                      BSGS_THREADS, smem) != cudaSuccess ||
        per_sm < 1)
        return -4;
    const unsigned blocks = (unsigned)(num_sms * per_sm);
    const size_t need = (size_t)blocks * BSGS_THREADS * ((size_t)1 << B.ns_log2) * sizeof(u64);
    if (need > scr.bytes) {
        bsgs_free(scr);
        if (cudaMalloc(&scr.tables, need) != cudaSuccess) return -3;
        scr.bytes = need;
    }
    B.tables = scr.tables;
    walk_bsgs_kernel<BSGS_KB><<<blocks, BSGS_THREADS, smem, s>>>(a, B);
    (*launches)++;
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}
#endif  // __CUDACC__
