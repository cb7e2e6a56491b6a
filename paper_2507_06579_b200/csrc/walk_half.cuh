// walk_half.cuh -- K3 in HALF mode: baby steps rho with the symmetry exit, no giant steps.
//
// For each d in D (one lane per d, persistent CTAs, warp-aggregated refill from
// a global work counter) walk the cycle of reduced principal ideals
//   (theta_{j+1}) = [Q_j/2, (P_j + sqrt d)/2],  (Q_0, P_0) = (2, 1),  theta_1 = 1,
// with rho:
//   q_j = floor((P_j + sqrt d)/Q_j), P_{j+1} = q_j Q_j - P_j, Q_{j+1} = (d - P_{j+1}^2)/Q_j,
//   theta_{j+2} = ((P_{j+1} + sqrt d)/Q_j) theta_{j+1},
// carrying theta only as its residue t in Z/3.  Since
// Q_j = 2 mod 4 and P_{j+1} is odd, (P_{j+1} + sqrt d)/Q_j = ((P-1)/2 + w)/(Q_j/2)
// has residue 1 if P_{j+1} = 1 mod 4 and 2 if P_{j+1} = 3 mod 4 (R31).
// The walk stops at the symmetry point of Algorithm 1 (PAPER.md l.553-556,
// "if Q_j = Q_{j-1} or P_j = P_{j-1}"), where (R13)
//   Q_j = Q_{j-1}:          t(eps) = t(theta_j) + t(theta_{j+1}),
//   P_j = P_{j-1}, j >= 2:  t(eps) = 2 t(theta_j).
//
// Arithmetic: all u32 (sqrt d < 2^19, Q < 2 sqrt d < 2^20 for d <= 1e11).
//  * Q_{j+1} = Q_{j-1} + q_j (P_j - P_{j+1}) in wrapping u32 (exact: the true
//    value is < 2^20), seeded with Q_{-1} = (d - 1)/2 mod 2^32.
//  * q = floor(num/Q) with num = P + s < 2^20: exact float images by the 2^23
//    magic-number trick (LOP3 + FADD instead of the narrow I2F pipe), one
//    MUFU.RCP, one FFMA that rounds num*rcp(Q) to an integer; the result is
//    floor or floor+1 (|error| < 0.27, K3), fixed by one compare.
//  * P_{j+1} = q Q - P = s - r with r = num - q Q.
#pragma once
#include "common.cuh"

struct BabyState {
    u32 s, P, Q, Qp;   // isqrt(d), P_j, Q_j, Q_{j-1}
    u32 t2;            // 2 t(theta_{j+1}) (not reduced mod 3)
};

// First rho step in closed form (PAPER.md l.541 from (Q_0, P_0) = (2, 1)):
// q_0 = floor((1 + s)/2), P_1 = 2 q_0 - 1 = s or s - 1 (the odd one),
// Q_1 = (d - P_1^2)/2, t(theta_2) = 1 + bit1(P_1).  The symmetry test at
// j = 1 is Q_1 = Q_0 = 2 only (the P test needs j >= 2).  Returns true with
// *res = t(eps) = t(theta_1) + t(theta_2) if the walk already ends here.
EIS_HD bool baby_init(BabyState &st, u64 d, u32 *res) {
    const u32 s = isqrt_u64_dev(d);
    const u32 P1 = (s - 1) | 1u;
    const u32 Q1 = (u32)((d - (u64)P1 * P1) >> 1);
    st.s = s;
    st.P = P1;
    st.Q = Q1;
    st.Qp = 2;
    st.t2 = 2 + (P1 & 2);
    *res = st.t2 >> 1;
    return Q1 == 2;
}

EIS_HD float u32_to_f_exact(u32 v) {   // v < 2^23
    return u2f_bits(v | 0x4B000000u) - 8388608.0f;
}

// One rho step j >= 2 from (Q_{j-1}, P_{j-1}) = (st.Q, st.P) with Q_{j-2} = st.Qp.
// Returns true at the symmetry point (Q_j = Q_{j-1} or P_j = P_{j-1}); the
// state is then already advanced and baby_result() reads t(eps) from it.
EIS_HD bool baby_step(BabyState &st) {
    const u32 num = st.P + st.s;
    const float nf = u32_to_f_exact(num);
    const float rq = rcp_approx(u32_to_f_exact(st.Q));
    // -q0 with q0 = round(num/Q) in {floor, floor + 1}  (|num/Q - num*rq| < 0.27)
    const u32 nq0 = 0x4B000000u - f2u_bits(fmaf(nf, rq, 8388608.0f));
    const i32 r0 = (i32)(nq0 * st.Q + num);                 // num - q0 Q in [-Q, Q)
    const u32 m = (u32)(r0 >> 31);                          // all ones iff q0 = floor + 1
    const u32 Pn = st.s - (u32)r0 - (st.Q & m);             // P_j = s - (num mod Q)
    const u32 q = m - nq0;                                  // q_{j-1} = floor(num/Q)
    const u32 Qn = st.Qp + q * (st.P - Pn);                 // Q_j (wrapping u32, exact)
    st.t2 += (Pn & 2u) + 2u;                                // residue of (P_j + sqrt d)/Q_{j-1}
    const bool eP = (Pn == st.P);
    st.Qp = st.Q;
    st.Q = Qn;
    st.P = Pn;
    return (Qn == st.Qp) | eP;
}

// t(eps) (not reduced mod 3) at the symmetry point reached by baby_step
// (R13):
//   Q_j = Q_{j-1}:  t(theta_j) + t(theta_{j+1});   P_j = P_{j-1}:  2 t(theta_j).
EIS_HD u32 baby_result(const BabyState &st) {
    const u32 inc = (st.P & 2u) + 2u;        // 2 (t(theta_{j+1}) - t(theta_j))
    const u32 t2b = st.t2 - inc;             // 2 t(theta_j)
    return (st.Q == st.Qp) ? (st.t2 + t2b) >> 1 : t2b;
}

// ---- the same step in exact FP32 integer arithmetic (the half-walk kernel's
// form).  Every value is an integer < 2^24, so FADD/FFMA on them are exact.
//  * P is kept as Pm = P + 2^23: the bits of Pm are 0x4B000000 + P, so the
//    residue bit (P & 2) is one LOP3 and P_j = P_{j-1} is a float compare.
//  * q = floor(num/Q) exactly, num = P + s < 2^20, by one FFMA rounded toward
//    zero: num * rqb + 2^23 with rqb = rcp(Q)(1 + 2^-21).  With |rel err of
//    rcp| <= 2^-22, rqb lies in [1/Q, (1/Q)(1 + 0.82 2^-20)), so num*rqb lies in
//    [num/Q, num/Q + 0.82/Q) and its floor is floor(num/Q) (the fractional part
//    of num/Q is at most 1 - 1/Q).  No correction step.
//  * r = num - q Q, P_j = s - r, Q_j = fma(q, P_{j-1} - P_j, Q_{j-2}); the FFMA
//    is exact because the true q (P_{j-1} - P_j) = Q_j - Q_{j-2} is < 2^20.
// 14 SASS instructions per step, 4 of them on the half-rate ALU pipe
// (K3 HALF).
struct BabyStateF {
    float sm, sp;       // s - 2^23, s + 2^23
    float Pm, Q, Qp;    // P_j + 2^23, Q_j, Q_{j-1}
    u32 t2;             // 2 t(theta_{j+1}) (not reduced mod 3)
};

EIS_HD BabyStateF baby_to_f(const BabyState &b) {
    BabyStateF f;
    f.sm = (float)b.s - 8388608.0f;
    f.sp = (float)b.s + 8388608.0f;
    f.Pm = (float)b.P + 8388608.0f;
    f.Q = (float)b.Q;
    f.Qp = (float)b.Qp;
    f.t2 = b.t2;
    return f;
}

EIS_HD bool baby_step_f(BabyStateF &st) {
    const float num = st.Pm + st.sm;                            // P + s
    const float rqb = rcp_approx(st.Q) * 1.000000476837158203125f;   // (1 + 2^-21)
    const float q = fma_rz(num, rqb, 8388608.0f) - 8388608.0f;  // floor(num/Q)
    const float r = fmaf(-q, st.Q, num);                        // num mod Q, exact
    const float Pnm = st.sp - r;                                // P_j + 2^23
    const float Qn = fmaf(q, st.Pm - Pnm, st.Qp);               // Q_j, exact
    st.t2 += (f2u_bits(Pnm) & 2u) + 2u;                         // residue of (P_j + sqrt d)/Q_{j-1}
    const bool eP = (Pnm == st.Pm);
    st.Qp = st.Q;
    st.Q = Qn;
    st.Pm = Pnm;
    return (Qn == st.Qp) | eP;
}

EIS_HD u32 baby_result_f(const BabyStateF &st) {
    const u32 inc = (f2u_bits(st.Pm) & 2u) + 2u;   // 2 (t(theta_{j+1}) - t(theta_j))
    const u32 t2b = st.t2 - inc;                   // 2 t(theta_j)
    return (st.Q == st.Qp) ? (st.t2 + t2b) >> 1 : t2b;
}

// Safety cap on rho steps per d: the half period is at most R/ln 2 <= ~20 sqrt(d)
// (h R < sqrt(d)(ln d + 2)/2 and two rho steps advance the distance by >= ln 2).
// A walk beyond the cap means a violated arithmetic invariant: it is counted
// as an error (the call fails with EIS_EINTERNAL) instead of looping forever.
EIS_HD u32 half_step_cap(u32 s) { return 48u * s + 64u; }

template <int KSTEPS>
__global__ void __launch_bounds__(256)
walk_half_kernel(WalkArgs a) {
    extern __shared__ u32 hist[];                  // hist_words(a)
    hist_zero(a, hist);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const u32 n = *a.count;
    BabyState st0;
    BabyStateF st;
    u64 d = 0;
    u32 off = 0;
    bool prime = false;
    bool active = false, exhausted = false;
    u32 n_done = 0, n_sym = 0, n_err = 0, dsteps = 0, cap = 0;
    u64 steps = 0;
    auto finish = [&](u32 res) {
        const u32 t = res % 3;
        steps += 1;                       // the closed-form first step
        n_done++;
        n_sym++;
        if (a.flags) a.flags[off] = (u8)t;
        if (a.ckpt) hist_record(a, hist, d, t, prime);
    };

    for (;;) {
        const u32 need = __ballot_sync(FULL_MASK, !active && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            u32 base = 0;
            if (lane == leader) base = atomicAdd(a.work, (u32)__popc(need));
            base = __shfl_sync(FULL_MASK, base, leader);
            if (!active && !exhausted) {
                const u32 idx = base + __popc(need & lanemask_lt());
                if (idx < n) {
                    const u32 le = __ldg(a.list + idx);
                    off = le & ~PRIME_BIT;
                    prime = (le & PRIME_BIT) != 0;
                    d = cand_d(a.i0 + off);
                    u32 r1;
                    if (baby_init(st0, d, &r1)) {
                        finish(r1);            // period closes at j = 1 (d = P_1^2 + 4)
                    } else {
                        st = baby_to_f(st0);
                        dsteps = 0;
                        cap = half_step_cap(st0.s);
                        active = true;
                    }
                } else {
                    exhausted = true;
                }
            }
        }
        if (__all_sync(FULL_MASK, exhausted)) break;
        if (active) {
            bool fin = false;
            int k = 0;
#pragma unroll 6
            for (; k < KSTEPS; k++) {
                if (baby_step_f(st)) { fin = true; break; }
            }
            steps += (u32)(k + fin);
            dsteps += (u32)(k + fin);
            if (fin) {
                finish(baby_result_f(st));
                active = false;
            } else if (dsteps > cap) {
                n_err++;
                finish(0xFFu);
                active = false;
            }
        }
    }

    // statistics: one atomic per warp
    u64 s_steps = warp_sum_u64(steps);
    u64 s_done = warp_sum_u64(n_done);
    u64 s_sym = warp_sum_u64(n_sym);
    const u32 s_err = __reduce_add_sync(FULL_MASK, n_err);
    if (lane == 0 && s_err) atomicAdd(a.err, s_err);
    if (lane == 0 && a.stats) {
        atomicAdd((unsigned long long *)&a.stats[ST_BABY], (unsigned long long)s_steps);
        atomicAdd((unsigned long long *)&a.stats[ST_D], (unsigned long long)s_done);
        atomicAdd((unsigned long long *)&a.stats[ST_SYM], (unsigned long long)s_sym);
    }
    if (a.ckpt) hist_flush(a, hist);
}
