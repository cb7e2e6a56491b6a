// forms.cuh -- giant-step composition of the paper's Appendix:
// NUCOMP (Alg. 2), NUDUPL (Alg. 3), NUCOMPchoose (Alg. 4) with the plain ideal
// product for small norms, on binary quadratic forms (u, v, w) of discriminant d,
// v^2 - 4uw = d.  Each returns the composed, near-reduced ideal [Q/2, (P+sqrt d)/2]
// and the relative generator gamma (I = (1/gamma) I1 I2)
// carried ONLY as
//   * its residue t(gamma) in (O_K/2O_K)^* = Z/3, and
//   * log2|gamma| (float; distances only choose the baby window and feed the
//     trivial-match guard, R14/R29).
// A, B, C of gamma = (A + B sqrt d)/C are never formed: with G odd (it divides
// u1 = Q1/2), u3 odd and v3 odd, A + B sqrt d = 2G[(x u3 + y (v3-1)/2) + y w], C = 2 u3,
// so t(gamma) = DLOG[(x + y (v3-1)/2) mod 2][y mod 2] (R12).  For the
// plain product gamma = S is odd: t = 0.
//
// Integer widths: u1, u2 < 2^20 (reduced inputs); intermediates < 2^48 at
// d <= 1e11, so int64 suffices; the plain-product numerator
// uses __int128.
#pragma once
#include "common.cuh"

EIS_HD i64 iabs64(i64 a) { return a < 0 ? -a : a; }

// ---- division helpers (no 64-bit integer divide instruction exists; nvcc's
// i64 '/' is a ~100-instruction branchy routine).  All divisors here are
// < 2^32 and all quotients < 2^50 (K3-giant).

// 1/b to full double precision: MUFU.RCP64H seed + two Newton steps.
EIS_HD double rcp64(double b) {
#ifdef __CUDA_ARCH__
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    double e = fma(-b, r, 1.0);
    r = fma(r, e, r);
    e = fma(-b, r, 1.0);
    r = fma(r, e, r);
    return r;
#else
    return 1.0 / b;
#endif
}

// 1/b with one Newton step from the MUFU.RCP64H seed.  Measured on B200
// (bench_tools/rcp64_accuracy.cu, 1.6e8 samples): seed 2^-19.9, one step
// 2^-39.9, two steps exact.  One step suffices wherever the quotient stays
// below 2^38.8 (rint of an exact quotient: error < 0.5) or a floor is
// corrected by one exact remainder test (quotient below 2^39.8): the rho loop,
// w2, the divisions by By, x, G, H, u1 and the canonical shift below.  Their
// bounds at d <= 1e11 (Q2 > 50): |w2| < d/100 < 2^30, |cx| < 2^21,
// |dx| < 2^33, |dy| < 2^34, (b m + l By)/H < 2^38; every quotient is checked
// by its remainder (dexact_div) anyway, so a violation fails the call.
// Only cy = Q2/bx keeps the two-step reciprocal (no small bound on it).
EIS_HD double rcp64_1(double b) {
#ifdef __CUDA_ARCH__
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    const double e = fma(-b, r, 1.0);
    return fma(r, e, r);
#else
    return 1.0 / b;
#endif
}

// floor(a / b) for b > 0, |a| < 2^62, |a/b| < 2^50: double estimate, one
// integer correction each way.
EIS_HD i64 floor_div(i64 a, i64 b) {
    i64 q = (i64)floor((double)a * rcp64((double)b));
    i64 r = a - q * b;
    if (r < 0) { q -= 1; r += b; }
    if (r >= b) { q += 1; }
    return q;
}
EIS_HD i64 floor_mod(i64 a, i64 b) {   // b > 0, result in [0, b)
    return a - floor_div(a, b) * b;
}

// exact floor-mod of fp64 integers, |a| < 2^52, 0 < b < 2^52 (rb ~ 1/b)
EIS_HD double dfloor_mod(double a, double b, double rb) {   // b > 0, result in [0, b)
    const double q = floor(a * rb);
    double r = fma(-q, b, a);
    r = r < 0.0 ? r + b : r;                  // selects, not branches
    r = r >= b ? r - b : r;
    return r;
}

// a symmetric residue of a mod b (fp64 integers, b > 0, |a / b| < 2^38, rb ~ 1/b
// to 2^-39.9): a - rint(a rb) b, in [-b/2 - b 2^-2, b/2 + b 2^-2]; exact (fma)
EIS_HD double smod(double a, double b, double rb) { return fma(-rint(a * rb), b, a); }

// 32-bit floor division for 0 <= a < 2^23, 0 < b < 2^23 (same float trick as
// the baby step: round(a/b) by one FFMA, then one correction).
EIS_HD u32 udiv23(u32 a, u32 b) {
    const float af = u2f_bits(a | 0x4B000000u) - 8388608.0f;
    const float rb = rcp_approx(u2f_bits(b | 0x4B000000u) - 8388608.0f);
    u32 q = f2u_bits(fmaf(af, rb, 8388608.0f)) - 0x4B000000u;
    if ((i32)(a - q * b) < 0) q -= 1;
    return q;
}

// Extended Euclid for 0 <= a, b < 2^23: returns g = gcd(a, b) = x a + y b
// (|x|, |y| <= max(a, b), so 32-bit cofactors suffice).
EIS_HD i32 xgcd32(i32 a, i32 b, i32 &x, i32 &y) {
    i32 x0 = 1, y0 = 0, x1 = 0, y1 = 1;
    while (b != 0) {
        const i32 q = (i32)udiv23((u32)a, (u32)b);
        i32 t = a - q * b; a = b; b = t;
        t = x0 - q * x1; x0 = x1; x1 = t;
        t = y0 - q * y1; y0 = y1; y1 = t;
    }
    x = x0;
    y = y0;
    return a;
}
EIS_HD i64 xgcd(i64 a, i64 b, i64 &x, i64 &y) {   // a, b in [0, 2^23)
    i32 xx, yy;
    const i32 g = xgcd32((i32)a, (i32)b, xx, yy);
    x = xx;
    y = yy;
    return g;
}
// signed variant: g = gcd(|a|, |b|) = x a + y b
EIS_HD i64 xgcd_s(i64 a, i64 b, i64 &x, i64 &y) {
    i64 g = xgcd(iabs64(a), iabs64(b), x, y);
    if (a < 0) x = -x;
    if (b < 0) y = -y;
    return g;
}

// ---- Euclid in exact FP32 integer arithmetic.  Every value below is an
// integer of magnitude < 2^24, so FFMA/FADD on them are exact.  No
// integer<->float conversion inside the loops (the XU pipe is narrow).
constexpr float FMAGIC = 8388608.0f;   // 2^23

// floor(a/b) for integers 0 <= a < 2^20, 0 < b, with no correction step (the
// baby step's rule, walk_bsgs.cuh baby_step_fd): rqb = rcp(b)(1 + 2^-21) lies in
// [1/b, (1 + 2^-20)/b) (rcp error <= 2^-23), so a rqb - a/b < a 2^-20 / b < 1/b,
// which is at most the gap between a/b and the next integer; the
// round-toward-zero FFMA then truncates a rqb to floor(a/b).
EIS_HD float ffloor_div_pos(float a, float b) {
    const float rqb = rcp_approx(b) * 1.000000476837158203125f;
    return fma_rz(a, rqb, FMAGIC) - FMAGIC;
}

// g = gcd(a, b) and x with x a = g (mod b), for 0 <= a, b < 2^20 (exact floats).
// Nearest-integer Euclid with signed remainders: q = round(a * rcp(b)) is
// within 1/2 + 1/4 of a/b (|a/b| < 2^20, relative rcp error < 2^-22), so
// |r| <= 3/4 |b| and no correction step is needed.  About 30% fewer iterations than the
// floor-quotient loop (R36).  x is correct modulo b/g, which is all
// NUCOMP uses (Alg. 2 l.626-634: b enters only through b u2 = F (mod u1)).
constexpr float RMAGIC = 12582912.0f;  // 1.5 * 2^23: round to nearest for |v| < 2^22
#ifndef EUCLID_UNROLL
#define EUCLID_UNROLL 2                 // Euclid loops unrolled twice: +0.5% (4: +0.3%)
#endif
constexpr int kEuclidUnroll = EUCLID_UNROLL;
// Stopping bound of the fast paths' partial Euclid (nucomp_d, nudupl_d) as a
// multiple of the paper's L = d^(1/4) (R38): 1.6 L
// leaves fewer rho steps for the slowest lane of a warp (1.96 vs 2.89 at 1e10)
// and fewer Euclid iterations; measured +1.5% at 1e10, +2% at 1e11 (1.4 / 1.8 /
// 2.0 / 2.4 / 3.0: +1.4 / +1.5 / +1.4 / +0.9 / -0.1%)
#ifndef EUCLID_BOUND_X10
#define EUCLID_BOUND_X10 16
#endif
constexpr float kEuclidBound = EUCLID_BOUND_X10 / 10.f;

EIS_HD float fxgcd_x(float a, float b, float &x) {
    float x0 = 1.f, x1 = 0.f;
#pragma unroll kEuclidUnroll
    while (b != 0.f) {
        EIS_PROF(0);
        const float q = fmaf(a, rcp_approx(b), RMAGIC) - RMAGIC;
        const float r = fmaf(-q, b, a);
        a = b;
        b = r;
        const float t = fmaf(-q, x1, x0);
        x0 = x1;
        x1 = t;
    }
    x = a < 0.f ? -x0 : x0;
    return fabsf(a);
}

// exact division of small integers: |a| < 2^23, 0 < b < 2^23, b | a
EIS_HD i64 sdiv_exact23(i64 a, i64 b) {
    const u32 q = udiv23((u32)iabs64(a), (u32)b);
    return a < 0 ? -(i64)q : (i64)q;
}
// does b divide a?  |a| < 2^23, 0 < b < 2^23
EIS_HD bool divides23(i64 b, i64 a) {
    const u32 ua = (u32)iabs64(a);
    return ua - udiv23(ua, (u32)b) * (u32)b == 0;
}

// Exact division (the "without remainder" divisions of Algs. 2-3), |n/dv| < 2^50:
// the rounded double quotient is exact; *err++ if the remainder is not 0.
EIS_HD i64 exact_div_r(i64 n, i64 dv, double rdv, u32 *err) {
    const i64 q = (i64)rint((double)n * rdv);
    if (q * dv != n) *err += 1;
    return q;
}
EIS_HD i64 exact_div(i64 n, i64 dv, u32 *err) {
    return exact_div_r(n, dv, rcp64((double)dv), err);
}

struct Composed {
    i64 Q, P;      // the ideal [Q/2, (P + sqrt d)/2], Q > 0 (not necessarily reduced)
    u32 tg;        // t(gamma) in {0,1,2}
    float lg;      // log2 |gamma|
    u32 kind;      // 0 plain product, 1 NUCOMP, 2 NUDUPL
    u32 nerr;      // invariant violations (returned, not through a pointer: the out-of-line
                   // caller's counter then stays in a register)
};

// residue of gamma from the final Euclid cofactors (R12)
EIS_HD u32 t_gamma(i64 x, i64 y, i64 v3) {
    const u32 a = (u32)((x + (y * ((v3 - 1) >> 1))) & 1);
    const u32 b = (u32)(y & 1);
    return a ? (b ? 2u : 0u) : 1u;    // (1,0)->0, (0,1)->1, (1,1)->2; (0,0) impossible
}

// log2|gamma|, gamma = G (a + y sqrt d)/(2 u3), a = 2 x u3 + y v3.  If a and y
// have opposite signs the sum cancels; then use |N(gamma)| = (Q1/2)(Q2/2)/|u3|
// (norms of the ideals, R29) and the conjugate, which does not cancel.
EIS_HD float log2_gamma(i64 G, i64 x, i64 y, i64 u3, i64 v3, float sqrtd_f, i64 Q1, i64 Q2) {
    const i64 a = 2 * x * u3 + y * v3;
    const float mag = fabsf((float)a) + fabsf((float)y) * sqrtd_f;   // |a| + |y| sqrt d
    const float au3 = fabsf((float)u3);
    if ((a >= 0) == (y >= 0) || a == 0 || y == 0)                    // no cancellation
        return log2_approx((float)G * mag / (2.f * au3));
    // log|gamma| = log|N(gamma)| - log|conj gamma|, |N| = (Q1/2)(Q2/2)/|u3|
    return log2_approx(2.f * (float)(Q1 >> 1) * (float)(Q2 >> 1) / ((float)G * mag));
}

// Partial Euclid of Algs. 2-3, in exact FP32
// (0 <= bx < by < 2^19 on entry: bx = Bx mod By, By = u1/G, u1 = Q1/2 < 2^19).
EIS_HD void partial_euclid(i64 &bx, i64 &by, i64 &x, i64 &y, int &z, i64 L) {
    float fbx = (float)bx, fby = (float)by, fx = 1.f, fy = 0.f;
    const float fL = (float)L;
    z = 0;
    while (fby > fL && fbx != 0.f) {
        const float q = ffloor_div_pos(fby, fbx);
        const float t = fmaf(-q, fbx, fby);
        fby = fbx;
        fbx = t;
        const float u = fmaf(-q, fx, fy);
        fy = fx;
        fx = u;
        z++;
    }
    if (z & 1) { fby = -fby; fy = -fy; }
    bx = (i64)fbx; by = (i64)fby; x = (i64)fx; y = (i64)fy;
}

// Algorithm 2 NUCOMP on forms (u1,v1,w1), (u2,v2,w2).
EIS_HD void nucomp(i64 u1, i64 v1, i64 w1, i64 u2, i64 v2, i64 w2, i64 L, i64 &u3, i64 &v3,
                   i64 &w3, i64 &G, i64 &xo, i64 &yo, u32 *err) {
    if (w1 < w2) {
        i64 t;
        t = u1; u1 = u2; u2 = t;
        t = v1; v1 = v2; v2 = t;
        t = w1; w1 = w2; w2 = t;
    }
    const i64 s = (v1 + v2) / 2;    // exact: v1, v2 odd
    const i64 m = v2 - s;
    float fb;
    const i64 F = (i64)fxgcd_x((float)u2, (float)u1, fb);   // b u2 + c u1 = F
    const i64 b = (i64)fb;
    i64 Bx, By, Cy, Dy;
    if (F == 1 || divides23(F, s)) {
        G = F;
        Bx = m * b;
        if (F == 1) { By = u1; Cy = u2; Dy = s; }
        else {
            By = sdiv_exact23(u1, G);
            Cy = sdiv_exact23(u2, G);
            Dy = sdiv_exact23(s, G);
        }
    } else {
        const i64 c = exact_div(F - b * u2, u1, err);
        i64 xx, yy;
        G = xgcd_s(F, s, xx, yy);       // xx F + yy s = G
        const i64 H = sdiv_exact23(F, G);
        By = sdiv_exact23(u1, G);
        Cy = sdiv_exact23(u2, G);
        Dy = sdiv_exact23(s, G);
        const i64 inner = floor_mod(b * floor_mod(w1, H) + c * floor_mod(w2, H), H);
        const i64 l = floor_mod(floor_mod(yy, H) * inner, H);
        Bx = exact_div(b * m + l * By, H, err);
    }
    i64 bx = floor_mod(Bx, By), by = By, x, y;
    int z;
    partial_euclid(bx, by, x, y, z, L);
    const i64 ay = G * y;
    if (z != 0) {
        const double rBy = rcp64((double)By);
        const i64 cx = exact_div_r(Cy * bx - m * x, By, rBy, err);
        const i64 Q1 = by * cx;
        const i64 Q2 = Q1 + m;
        const i64 dx = exact_div_r(Dy * bx - w2 * x, By, rBy, err);
        const i64 Q3 = y * dx;
        const i64 Q4 = Q3 + Dy;
        const i64 dy = exact_div(Q4, x, err);
        i64 cy;
        if (bx != 0) cy = exact_div(Q2, bx, err);
        else cy = exact_div(cx * dy - w1, dx, err);
        u3 = by * cy - ay * dy;
        w3 = bx * cx - G * x * dx;         // ax = G x
        v3 = G * (Q3 + Q4) - Q1 - Q2;
    } else {
        const double rBy = rcp64((double)By);
        const i64 Q1 = Cy * bx;
        const i64 cx = exact_div_r(Q1 - m, By, rBy, err);
        const i64 dx = exact_div_r(bx * Dy - w2, By, rBy, err);
        u3 = by * Cy;
        w3 = bx * cx - G * dx;
        v3 = v2 - 2 * Q1;
    }
    xo = x;
    yo = y;
}

// Algorithm 3 NUDUPL on the form (u, v, w).
EIS_HD void nudupl(i64 u, i64 v, i64 w, i64 L, i64 &u3, i64 &v3, i64 &w3, i64 &G, i64 &xo,
                   i64 &yo, u32 *err) {
    i64 xx, yy;
    G = xgcd_s(u, v, xx, yy);     // xx u + yy v = G
    const i64 By = sdiv_exact23(u, G);
    const i64 Dy = sdiv_exact23(v, G);
    const i64 Bx = floor_mod(floor_mod(yy, By) * floor_mod(w, By), By);
    i64 bx = Bx, by = By, x, y;
    int z;
    partial_euclid(bx, by, x, y, z, L);
    const i64 ay = G * y;
    if (z == 0) {
        const i64 dx = exact_div(bx * Dy - w, By, err);
        u3 = by * by;
        w3 = bx * bx;
        v3 = v - (bx + by) * (bx + by) + u3 + w3;
        w3 = w3 - G * dx;
    } else {
        const i64 dx = exact_div(bx * Dy - w * x, By, err);
        const i64 Q1 = dx * y;
        i64 dy = Q1 + Dy;
        v3 = G * (dy + Q1);
        dy = exact_div(dy, x, err);
        u3 = by * by;
        w3 = bx * bx;
        v3 = v3 - (bx + by) * (bx + by) + u3 + w3;
        u3 = u3 - ay * dy;
        w3 = w3 - G * x * dx;                            // ax = G x
    }
    xo = x;
    yo = y;
}

// Plain ideal product (the small-norm branch of Alg. 4, PAPER.md l.733, l.742-744;
// the J-W Sec. 5.4 procedure is not reproduced in the paper: Dirichlet
// composition, R20).  Inputs a_i = Q_i/2, b_i = P_i (odd).
EIS_HD i64 mulmod(i64 a, i64 b, i64 M) {   // |a|, |b| < M < 2^31: (a b) mod M in [0, M)
    return floor_mod(a * b, M);
}
EIS_HD Composed plain_product(i64 Q1, i64 P1, i64 Q2, i64 P2, i64 d, u32 *err) {
    const i64 a1 = Q1 >> 1, a2 = Q2 >> 1;
    i64 x, y;
    const i64 e = xgcd(a1, a2, x, y);         // x a1 + y a2 = e
    Composed r;
    r.tg = 0;                                  // gamma = S odd
    r.kind = 0;
    if (e == 1) {
        // coprime norms (the usual case): S = 1 with (X, Y) = (1, 0), so
        // b3 = x a1 P2 + y a2 P1 mod 2 a1 a2 (the CRT lift).  min(a1, a2) <= 25
        // bounds |x a1|, |y a2| by 25 * 2^19 and P1, P2 < 2^20, so the sum is an
        // exact fp64 integer < 2^45 and one exact floor-mod finishes it.
        const double M = 2.0 * (double)a1 * (double)a2;
        const double v = fma((double)(x * a1), (double)P2, (double)(y * a2) * (double)P1);
        r.Q = 2 * a1 * a2;
        r.P = (i64)dfloor_mod(v, M, rcp64(M));
        r.lg = 0.f;
        if (floor_mod(r.P * r.P - d, 2 * r.Q) != 0) *err += 1;   // b3^2 = d mod 4 a3 (R20)
        return r;
    }
    const i64 n = (P1 + P2) / 2;
    i64 X, Y;
    const i64 S = xgcd_s(e, n, X, Y);         // X e + Y n = S
    const i64 a3 = sdiv_exact23(a1, S) * sdiv_exact23(a2, S);
    // b3 = num / S mod 2 a3 with num = X x a1 P2 + X y a2 P1 + Y (P1 P2 + d)/2;
    // S | num, so reduce num modulo M = 2 a3 S (< 2^31: a1 <= 25) and divide.
    const i64 M = 2 * a3 * S;
    const i64 t1 = mulmod(mulmod(floor_mod(X, M), floor_mod(x, M), M),
                          mulmod(a1, floor_mod(P2, M), M), M);
    const i64 t2 = mulmod(mulmod(floor_mod(X, M), floor_mod(y, M), M),
                          mulmod(a2, floor_mod(P1, M), M), M);
    const i64 h = floor_mod(((P1 * P2) >> 1) + ((d >> 1) + 1) , M);   // (P1 P2 + d)/2, both odd
    const i64 t3 = mulmod(floor_mod(Y, M), h, M);
    const i64 num = floor_mod(t1 + t2 + t3, M);
    if (num % S != 0) *err += 1;
    r.Q = 2 * a3;
    r.P = num / S;                             // in [0, 2 a3)
    r.lg = log2_approx((float)S);
    if (floor_mod(r.P * r.P - d, 2 * r.Q) != 0) *err += 1;       // b3^2 = d mod 4 a3 (R20)
    return r;
}

// The fixed left operand of every giant step (mu_1), normalised as in Alg. 4
// (P mod Q, w = (P^2 - d)/(2Q)) once per d.
struct Mu1Form {
    u32 Q, P;           // < 2^20 (reduced); 32-bit to keep the giant lane state small
    i64 w;
};
EIS_HD Mu1Form mu1_form(i64 Q1, i64 P1, i64 d, u32 *err) {
    Mu1Form f;
    f.Q = Q1;
    f.P = floor_mod(P1, Q1);
    f.w = exact_div((i64)f.P * f.P - d, 2 * Q1, err);
    return f;
}

// Algorithm 4 NUCOMPchoose for reduced ideals
// I1 = mu_1 = [Q1/2, (P1+sqrt d)/2] (pre-normalised) and I2 = [Q2/2, (P2+sqrt d)/2].
EIS_HD_COLD Composed nucomp_choose(Mu1Form m1, i64 Q2, i64 P2, i64 d, i64 L, double sqrtd,
                                   int plain_th) {
    u32 nerr = 0, *err = &nerr;
    const i64 Q1 = m1.Q, P1 = m1.P;
    P2 = P2 < Q2 ? P2 : floor_mod(P2, Q2);
    if (Q1 <= plain_th || Q2 <= plain_th) {
        Composed r = plain_product(Q1, P1, Q2, P2, d, err);
        r.nerr = nerr;
        return r;
    }
    i64 u3, v3, w3, G, x, y;
    Composed r;
    if (Q1 == Q2 && P1 == P2) {
        nudupl(Q1 >> 1, -P1, m1.w, L, u3, v3, w3, G, x, y, err);
        r.kind = 2;
    } else {
        const i64 w2 = exact_div(P2 * P2 - d, 2 * Q2, err);
        nucomp(Q1 >> 1, -P1, m1.w, Q2 >> 1, -P2, w2, L, u3, v3, w3, G, x, y, err);
        r.kind = 1;
    }
    // the output form's discriminant (l.622, l.687), exact in 128 bits
    if ((__int128)v3 * v3 - 4 * (__int128)u3 * w3 != (__int128)d) *err += 1;
    r.Q = iabs64(2 * u3);
    r.P = floor_mod(-v3, r.Q);
    r.tg = t_gamma(x, y, v3);
    r.lg = log2_gamma(G, x, y, u3, v3, (float)sqrtd, Q1, Q2);
    if ((r.Q & 3) != 2 || (r.P & 1) != 1 || (G & 1) == 0) *err += 1;   // Thm A.1 / 2 inert
    r.nerr = nerr;
    return r;
}

// ---------------------------------------------------------------------------
// NUCOMP, hot path of the giant kernel, in exact fp64 integer arithmetic.
// Every quantity is an integer of magnitude < 2^53 at d <= 1e11 (<= 47 bits
// measured), so DFMA/DMUL/DADD on them are exact; each
// "without remainder" division is rint(n * rcp(dv)) with its remainder checked
// by one exact DFMA (*err++ otherwise).  The Euclid loops run in exact FP32.
// Same steps and variable names as nucomp() above (Alg. 2),
// including the branch F not | s (second xgcd, products reduced mod H first).
EIS_HD double dexact_div(double n, double dv, double rdv, u32 *err) {
    const double q = rint(n * rdv);
    if (fma(-q, dv, n) != 0.0) *err += 1;
    return q;
}

struct CompD {
    double u3, v3, w3, x, y, G;
};

// Exact check of the output form's discriminant, v3^2 - 4 u3 w3 = d (Alg. 2/3
// output phi_3 "whose discriminant is d"), on fp64
// integers that may exceed 2^53 in the squares: p = v3^2 and q = 4 u3 w3 are
// split into rounded value + exact FMA error.  If the form is right, p and q
// agree to within d, so p - q is exact (Sterbenz) and the rest are small exact
// integers; if p and q differ by more than a factor 2, |p - q| > 2^52 > d and
// the test fails as it should.
EIS_HD bool disc_ok(double u3, double v3, double w3, double d) {
    const double p = v3 * v3, e1 = fma(v3, v3, -p);
    const double t = 4.0 * u3;
    const double q = t * w3, e2 = fma(t, w3, -q);
    return ((p - q) - d) + (e1 - e2) == 0.0;
}

EIS_HD bool nucomp_d(double u1, double v1, double w1, double u2, double v2, double w2, float L,
                     CompD &o, u32 *err, u32 wmask) {
    if (w1 < w2) {
        double t;
        t = u1; u1 = u2; u2 = t;
        t = v1; v1 = v2; v2 = t;
        t = w1; w1 = w2; w2 = t;
    }
    const double s = (v1 + v2) * 0.5;          // exact: v1, v2 odd
    const double m = v2 - s;
    float fb;
    const float F = fxgcd_x((float)u2, (float)u1, fb);   // b u2 = F (mod u1)
    warp_reconverge(wmask);
    double G = 1.0, By = u1, Cy = u2, Dy = s, rBy;
    float fbx0;
    EIS_PROF(4);
    {
        // Alg. 2 l.626-634 as one straight path for every lane (all reduced mod H
        // first).  The branches F = 1 / F | s / F not | s ran one after another
        // whenever any lane of the warp needed them (27% of lanes have F != 1);
        // F = 1 gives G = H = 1, l = 0 and Bx = m b, F | s gives G = F, H = 1 (the
        // same), a symmetric residue mod 1 is 0.  l = yy (b w1 + c w2) mod H in
        // symmetric residues (|r| <= H/2; any representative of l makes b m + l By
        // divisible by H, which dexact_div checks): |b|, |c|, |yy| < 2^19, H < 2^19,
        // so every product is exact (< 2^38).  One path measured +0.75% on the bench
        // slab, +1.2% at 3e10, +0.9% at 1e11 (giant kernel).
        const float fs = fabsf((float)s);
        float fyy;
        const float Gf = fxgcd_x(fs, F, fyy);  // yy |s| = G (mod F); F = 1: one iteration
        warp_reconverge(wmask);
        G = (double)Gf;
        const double rG = rcp64_1(G);
        By = rint(u1 * rG);
        Cy = rint(u2 * rG);
        Dy = rint(s * rG);
        rBy = rcp64_1(By);
        const double H = rint((double)F * rG), rH = rcp64_1(H);
        if (F != 1.f) EIS_PROF(5);
        if (H != 1.0) EIS_PROF(1);
        const double b = fb;
        const double c = dexact_div(fma(-b, u2, (double)F), u1, rcp64_1(u1), err);
        const double yy = s < 0.0 ? -(double)fyy : (double)fyy;
        const double inner = smod(fma(b, smod(w1, H, rH), c * smod(w2, H, rH)), H, rH);
        const double l = smod(yy * inner, H, rH);
        const double Bx = dexact_div(fma(b, m, l * By), H, rH, err);
        fbx0 = (float)dfloor_mod(Bx, By, rBy);
    }
    // partial Euclid (Alg. 2 l.637-643) in exact FP32
    float fbx = fbx0, fby = (float)By, fx = 1.f, fy = 0.f;
    int z = 0;
    const float Lb = L * kEuclidBound;
#pragma unroll kEuclidUnroll
    while (fby > Lb && fbx != 0.f) {
        EIS_PROF(2);
        const float q = ffloor_div_pos(fby, fbx);
        const float t = fmaf(-q, fbx, fby);
        fby = fbx;
        fbx = t;
        const float u = fmaf(-q, fx, fy);
        fy = fx;
        fx = u;
        z++;
    }
    if (z & 1) { fby = -fby; fy = -fy; }
    warp_reconverge(wmask);
    const double bx = fbx, by = fby, x = fx, y = fy;
    if (z == 0) EIS_PROF(6);
    if (bx == 0.0) EIS_PROF(7);
    // Alg. 2 l.644-660 as one path: with no Euclid step (z = 0: x = 1, y = 0,
    // by = By) the general formulas give cy = Cy, u3 = By Cy, v3 = v2 - 2 Cy bx,
    // the z = 0 branch's values (Dy G + m = v2), and for bx = 0 the paper's
    // alternative cy = (cx dy - w1)/dx is taken by a select (m Dy + w1 By = Cy w2
    // from v_i^2 - 4 u_i w_i = d makes it Cy too when z = 0).  The warp used to
    // run both branches whenever one lane needed the rare one.
    const double cx = dexact_div(fma(Cy, bx, -m * x), By, rBy, err);
    const double Q1 = by * cx;
    const double Q2 = Q1 + m;
    const double dx = dexact_div(fma(Dy, bx, -w2 * x), By, rBy, err);
    const double Q3 = y * dx;
    const double Q4 = Q3 + Dy;
    const double dy = dexact_div(Q4, x, rcp64_1(x), err);
    const bool bz = bx == 0.0;
    const double cn = bz ? fma(cx, dy, -w1) : Q2, cd = bz ? dx : bx;
    const double cy = dexact_div(cn, cd, rcp64(cd), err);
    o.u3 = fma(by, cy, -G * y * dy);
    o.w3 = fma(bx, cx, -G * x * dx);              // w3 = bx cx - ax dx, ax = G x
    o.v3 = G * (Q3 + Q4) - Q1 - Q2;
    o.x = x;
    o.y = y;
    o.G = G;
    return true;
}

// NUDUPL (Alg. 3) in the same exact fp64/FP32 arithmetic as
// nucomp_d: the prep kernel's two doublings per d (mu_1^2, then mu''_1^2 when
// two-sided).  Same steps and names as nudupl() above.  yy comes from the
// nearest-integer xgcd (R36): yy v = G (mod u); Bx needs it only mod By = u/G.
EIS_HD bool nudupl_d(double u, double v, double w, float L, CompD &o, u32 *err, u32 wmask) {
    float fyy;
    const float Gf = fxgcd_x(fabsf((float)v), (float)u, fyy);   // fyy |v| = G (mod u)
    warp_reconverge(wmask);
    const double G = (double)Gf;
    const double rG = rcp64_1(G);
    const double By = rint(u * rG), Dy = rint(v * rG);
    const double rBy = rcp64_1(By);
    const double yy = v < 0.0 ? -(double)fyy : (double)fyy;
    const double Bx = dfloor_mod(smod(yy, By, rBy) * smod(w, By, rBy), By, rBy);   // (< 2^38)
    // partial Euclid (Alg. 3 l.694-700) in exact FP32, as in nucomp_d
    float fbx = (float)Bx, fby = (float)By, fx = 1.f, fy = 0.f;
    int z = 0;
    const float Lb = L * kEuclidBound;
    while (fby > Lb && fbx != 0.f) {
        const float q = ffloor_div_pos(fby, fbx);
        const float t = fmaf(-q, fbx, fby);
        fby = fbx;
        fbx = t;
        const float uu = fmaf(-q, fx, fy);
        fy = fx;
        fx = uu;
        z++;
    }
    if (z & 1) { fby = -fby; fy = -fy; }
    warp_reconverge(wmask);
    const double bx = fbx, by = fby, x = fx, y = fy;
    const double sq = (bx + by) * (bx + by) - bx * bx;   // exact: < 2^40
    // one path (Alg. 3 l.701-711): with no Euclid step (x = 1, y = 0) it gives
    // u3 = by^2, v3 = G Dy - sq + by^2 = v - sq + u3, w3 = bx^2 - G dx: the z = 0 values
    const double dx = dexact_div(fma(bx, Dy, -w * x), By, rBy, err);
    const double Q1 = dx * y;
    const double dy0 = Q1 + Dy;
    const double dy = dexact_div(dy0, x, rcp64_1(x), err);
    o.v3 = G * (dy0 + Q1) - sq + by * by;
    o.u3 = fma(by, by, -G * y * dy);
    o.w3 = fma(bx, bx, -G * x * dx);              // w3 = bx^2 - ax dx
    o.x = x;
    o.y = y;
    o.G = G;
    return true;
}

// The giant step's composition (NUCOMPchoose, Alg. 4, for I1 = mu_1 and a reduced
// I2 != mu_1) followed by the canonical representative (R17): returns
// Q = |2 u3| and P* = s - ((s + v3) mod Q) in (s - Q, s] (P = -v3 mod Q, l.753).
struct GiantComp {
    double Q, P;       // integers (|P| < 2^29): the rho state works in fp64
    u32 tg, kind;
    float lg;
};

// dup_fast (a compile-time constant at each call site): squarings take the fp64
// NUDUPL; otherwise (the giant kernel, where mu_1^2 is rare) the generic path.
EIS_HD GiantComp giant_compose(const Mu1Form &m1, i64 Q2, i64 P2, i64 d, i64 s, i64 L,
                               float sqrtd_f, int plain_th, u32 *err, u32 wmask,
                               bool dup_fast = false) {
    GiantComp r;
    const i64 Q1 = m1.Q, P1 = m1.P;
    if (P2 >= Q2) P2 -= Q2 * (i64)ffloor_div_pos((float)P2, (float)Q2);   // Alg. 4 l.739
    const bool dup = Q1 == Q2 && P1 == P2;
    const bool rare = Q1 <= plain_th || Q2 <= plain_th || (dup && !dup_fast);
    const bool fdup = dup_fast && dup && !rare;
    // lanes of `wmask` that run the NUCOMP / NUDUPL fast paths (their
    // reconvergence points must be reached by exactly these lanes)
    const u32 fmask = warp_ballot(wmask, !rare && !fdup);
    const u32 dmask = dup_fast ? warp_ballot(wmask, fdup) : 0u;
    if (rare) {
        EIS_PROF(8);
        const Composed c = nucomp_choose(m1, Q2, P2, d, L, (double)sqrtd_f, plain_th);
        *err += c.nerr;
        r.Q = (double)c.Q;
        r.P = (double)(s - floor_mod(s - c.P, c.Q));
        r.tg = c.tg;
        r.lg = c.lg;
        r.kind = c.kind;
        return r;
    }
    CompD o;
    bool ok;
    if (fdup) {
        ok = nudupl_d((double)(Q1 >> 1), -(double)P1, (double)m1.w, (float)L, o, err, dmask);
    } else {
        const double dd = (double)d;
        const double w2 = rint(((double)P2 * (double)P2 - dd) * rcp64_1(2.0 * (double)Q2));   // exact
        ok = nucomp_d((double)(Q1 >> 1), -(double)P1, (double)m1.w, (double)(Q2 >> 1),
                      -(double)P2, w2, (float)L, o, err, fmask);
    }
    if (!ok) {
        const Composed c = nucomp_choose(m1, Q2, P2, d, L, (double)sqrtd_f, plain_th);
        *err += c.nerr;
        r.Q = (double)c.Q;
        r.P = (double)(s - floor_mod(s - c.P, c.Q));
        r.tg = c.tg;
        r.lg = c.lg;
        r.kind = c.kind;
        return r;
    }
    const double Qd = fabs(2.0 * o.u3);
    const double sd = (double)s;
    const double Ps = sd - dfloor_mod(sd + o.v3, Qd, rcp64_1(Qd));
    r.Q = Qd;
    r.P = Ps;
    // t(gamma) = DLOG[(x + y (v3-1)/2) mod 2][y mod 2] (R12), from the
    // low bits of x, y, v3 (dlo32: no conversions)
    r.tg = t_gamma(dlo32(o.x), dlo32(o.y), dlo32(o.v3));
    // log2|gamma|, gamma = G (a + y sqrt d)/(2 u3), a = 2 x u3 + y v3
    const double a = fma(2.0 * o.x, o.u3, o.y * o.v3);
    const float mag = fabsf((float)a) + fabsf((float)o.y) * sqrtd_f;
    // |N(gamma)| = (Q1/2)(Q2/2)/|u3|: where a and y sqrt d cancel, the conjugate
    // (no cancellation) gives log|gamma| = log|N| - log|conj gamma| (one log either way)
    const bool direct = (a >= 0.0) == (o.y >= 0.0) || a == 0.0 || o.y == 0.0;
    // (an approximate reciprocal: an IEEE float division is a subroutine with a
    // slow path, and distances are float estimates anyway)
    const float gm = (float)o.G * mag;
    const float num = direct ? gm : 2.f * (float)(Q1 >> 1) * (float)(Q2 >> 1);
    r.lg = log2_approx(num * rcp_approx(direct ? (float)Qd : gm));
    r.kind = fdup ? 2u : 1u;
    if (((dlo32(Qd) & 3) != 2) | ((dlo32(Ps) & 1) != 1) | ((dlo32(o.G) & 1) == 0) |
        !disc_ok(o.u3, o.v3, o.w3, (double)d))
        *err += 1;
    return r;
}

