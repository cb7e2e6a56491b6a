/*
 * oracle/eis_oracle.c -- CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the Eisenstein
 * classification of Breuer & Punch, "Quadratic units and cubic fields"
 * (arXiv 2507.06579).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA path in
 * paper_2507_06579_b200/ and never calls it.
 *
 * What it computes (the plain definition, not the paper's fast method):
 *
 *   PAPER.md l.52-55 (Sec. 1): d = 5 mod 8 squarefree, O_K = Z[w], w=(1+sqrt d)/2,
 *     fundamental unit eps_d = (x0 + y0 sqrt d)/2.
 *   PAPER.md l.95-103 (Sec. 1): D = squarefree d = 5 mod 8;
 *     E = { d in D : eps_d = 1 mod 2 O_K }.
 *   pi_E(x) = #{d in E, d <= x}, pi_D(x) = #{d in D, d <= x}.
 *
 * Steps (one function each, in this order):
 *   1. squarefree test by trial division: d is squarefree iff no odd m >= 3
 *      with m^2 | d (4 never divides d = 5 mod 8).            [eo_is_squarefree]
 *   2. eps_d from the regular continued fraction of w = (1+sqrt d)/2 with
 *      exact big-integer convergents p/q: complete quotients (P_k+sqrt d)/Q_k,
 *      P_0=1, Q_0=2, a_k = floor((P_k + isqrt d)/Q_k), P_{k+1} = a_k Q_k - P_k,
 *      Q_{k+1} = (d - P_{k+1}^2)/Q_k; stop at the first k>=1 with Q_k = 2
 *      (end of the first period).  Then eps = p - q*conj(w) =
 *      ((2p-q) + q sqrt d)/2, i.e. x0 = 2p-q, y0 = q.               [eo_unit]
 *      The result is CERTIFIED per d: x0^2 - d y0^2 = +-4 is checked exactly
 *      with big integers; a failure aborts with EO_ECERT.
 *   3. residue class in (O_K/2O_K)^* = F_4^* = Z/3:
 *      eps = (p-q)*1 + q*w in the basis [1,w]; the parity pair
 *      ((p-q) mod 2, q mod 2) maps (1,0)->0, (0,1)->1, (1,1)->2.  t = 0 iff
 *      eps = 1 mod 2O_K iff d in E.                               [eo_residue]
 *
 * Parity pins (tests/test_oracle.py): brute-force smallest solution of
 * x^2 - d y^2 = +-4 for tiny d; Lemma 1.1(2) by brute-force
 * search for odd solutions of x^2 - d y^2 = 4; the paper's examples 1901, 7053
 * in E; the Moebius closed form for pi_D; Table 1 totals
 * (PAPER.md l.419-464).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle/eis_oracle.c -o oracle/liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EO_OK 0
#define EO_EINVAL (-1)   /* d not = 5 mod 8, or not squarefree where required */
#define EO_ECERT (-2)    /* norm certificate failed: a bug, never expected */
#define EO_ENOMEM (-3)
#define EO_NOT_IN_D 0xFF

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- bigint -- */
/* Non-negative big integer, little-endian 64-bit limbs. Deliberately minimal. */
typedef struct {
    uint64_t *w;
    int n;    /* used limbs (no leading zero limbs; n==0 means value 0) */
    int cap;
} big;

static int big_init(big *a, int cap) {
    a->w = (uint64_t *)calloc((size_t)cap, sizeof(uint64_t));
    a->n = 0;
    a->cap = cap;
    return a->w ? 0 : -1;
}
static void big_free(big *a) { free(a->w); a->w = NULL; a->n = a->cap = 0; }
static int big_reserve(big *a, int cap) {
    if (cap <= a->cap) return 0;
    int nc = a->cap * 2 > cap ? a->cap * 2 : cap;
    uint64_t *w = (uint64_t *)realloc(a->w, (size_t)nc * sizeof(uint64_t));
    if (!w) return -1;
    memset(w + a->cap, 0, (size_t)(nc - a->cap) * sizeof(uint64_t));
    a->w = w;
    a->cap = nc;
    return 0;
}
static void big_set_u64(big *a, uint64_t v) {
    a->w[0] = v;
    a->n = v ? 1 : 0;
}
static void big_trim(big *a) { while (a->n > 0 && a->w[a->n - 1] == 0) a->n--; }
static int big_copy(big *r, const big *a) {
    if (big_reserve(r, a->n + 1)) return -1;
    memcpy(r->w, a->w, (size_t)a->n * sizeof(uint64_t));
    r->n = a->n;
    return 0;
}
/* r = a*m + b   (m a machine word; r aliases neither a nor b) */
static int big_muladd(big *r, const big *a, uint64_t m, const big *b) {
    int na = a->n, nb = b->n;
    int n = na > nb ? na : nb;
    if (big_reserve(r, n + 2)) return -1;
    u128 carry = 0;
    int i = 0;
    for (; i < na && i < nb; i++) {
        u128 s = (u128)a->w[i] * m + b->w[i] + carry;
        r->w[i] = (uint64_t)s;
        carry = s >> 64;
    }
    for (; i < na; i++) {
        u128 s = (u128)a->w[i] * m + carry;
        r->w[i] = (uint64_t)s;
        carry = s >> 64;
    }
    for (; i < nb; i++) {
        u128 s = (u128)b->w[i] + carry;
        r->w[i] = (uint64_t)s;
        carry = s >> 64;
    }
    r->w[n] = (uint64_t)carry;
    r->n = n + 1;
    big_trim(r);
    return 0;
}
/* r = a - b, requires a >= b */
static int big_sub(big *r, const big *a, const big *b) {
    if (big_reserve(r, a->n + 1)) return -1;
    uint64_t borrow = 0;
    for (int i = 0; i < a->n; i++) {
        uint64_t bi = i < b->n ? b->w[i] : 0;
        u128 s = (u128)a->w[i] - bi - borrow;
        r->w[i] = (uint64_t)s;
        borrow = (uint64_t)(s >> 64) ? 1 : 0;
    }
    r->n = a->n;
    big_trim(r);
    return 0;
}
static int big_cmp(const big *a, const big *b) {
    if (a->n != b->n) return a->n < b->n ? -1 : 1;
    for (int i = a->n - 1; i >= 0; i--)
        if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
    return 0;
}
/* r = a*b, schoolbook (r must not alias a or b) */
static int big_mul(big *r, const big *a, const big *b) {
    int n = a->n + b->n;
    if (big_reserve(r, n + 1)) return -1;
    memset(r->w, 0, (size_t)(n + 1) * sizeof(uint64_t));
    for (int i = 0; i < a->n; i++) {
        u128 carry = 0;
        for (int j = 0; j < b->n; j++) {
            u128 s = (u128)a->w[i] * b->w[j] + r->w[i + j] + carry;
            r->w[i + j] = (uint64_t)s;
            carry = s >> 64;
        }
        int k = i + b->n;
        while (carry) {
            u128 s = (u128)r->w[k] + carry;
            r->w[k] = (uint64_t)s;
            carry = s >> 64;
            k++;
        }
    }
    r->n = n;
    big_trim(r);
    return 0;
}

/* ------------------------------------------------------------- integers -- */
static uint64_t isqrt_u64(uint64_t n) {
    /* exact floor(sqrt(n)) by bisection: obviously correct, n < 2^62 */
    uint64_t lo = 0, hi = (uint64_t)1 << 32;
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (mid * mid <= n) lo = mid; else hi = mid;
    }
    return lo;
}

/* Step 1. PAPER.md l.97: D requires d squarefree. Trial division by every
 * odd m >= 3 with m^2 <= d (composite m are redundant but harmless). */
int eo_is_squarefree(uint64_t d) {
    if (d == 0) return 0;
    if (d % 4 == 0) return 0;
    for (uint64_t m = 3; m * m <= d; m += 2)
        if (d % (m * m) == 0) return 0;
    return 1;
}

/* Step 2. The fundamental unit by the continued fraction of (1+sqrt d)/2.
 * On return p, q hold the last convergent before the period closes.
 * *period receives the period length l.  Returns EO_OK or EO_ECERT. */
static int eo_unit_pq(uint64_t d, big *p, big *q, int64_t *period, int *norm_sign) {
    const uint64_t s = isqrt_u64(d);
    int64_t P = 1, Q = 2;           /* complete quotient (P + sqrt d)/Q */
    big p1, p2, q1, q2, t;          /* p_{k-1}, p_{k-2}, q_{k-1}, q_{k-2} */
    if (big_init(&p1, 4) || big_init(&p2, 4) || big_init(&q1, 4) || big_init(&q2, 4) ||
        big_init(&t, 4))
        return EO_ENOMEM;
    big_set_u64(&p1, 1); big_set_u64(&p2, 0);   /* p_{-1}=1, p_{-2}=0 */
    big_set_u64(&q1, 0); big_set_u64(&q2, 1);   /* q_{-1}=0, q_{-2}=1 */
    int64_t k = 0;
    int rc = EO_OK;
    for (;;) {
        uint64_t a = ((uint64_t)P + s) / (uint64_t)Q;      /* a_k */
        /* p_k = a_k p_{k-1} + p_{k-2}; q_k likewise */
        if (big_muladd(&t, &p1, a, &p2)) { rc = EO_ENOMEM; break; }
        { big sw = p2; p2 = p1; p1 = t; t = sw; }
        if (big_muladd(&t, &q1, a, &q2)) { rc = EO_ENOMEM; break; }
        { big sw = q2; q2 = q1; q1 = t; t = sw; }
        int64_t Pn = (int64_t)a * Q - P;
        int64_t Qn = ((int64_t)d - Pn * Pn) / Q;           /* exact */
        if (((int64_t)d - Pn * Pn) % Q != 0) { rc = EO_ECERT; break; }
        P = Pn; Q = Qn;
        k++;
        if (Q == 2) break;
    }
    if (rc == EO_OK) {
        /* x0 = 2p - q, y0 = q; certify x0^2 - d*y0^2 = +-4 exactly. */
        big x0, two_p, zero, x2, y2, dy2, diff;
        big_init(&x0, 4); big_init(&two_p, 4); big_init(&zero, 1);
        big_init(&x2, 4); big_init(&y2, 4); big_init(&dy2, 4); big_init(&diff, 4);
        big_set_u64(&zero, 0);
        big_muladd(&two_p, &p1, 2, &zero);
        big_sub(&x0, &two_p, &q1);
        big_mul(&x2, &x0, &x0);
        big_mul(&y2, &q1, &q1);
        big_muladd(&dy2, &y2, d, &zero);
        int c = big_cmp(&x2, &dy2);
        int sign = 0;
        if (c > 0) { big_sub(&diff, &x2, &dy2); sign = +1; }
        else if (c < 0) { big_sub(&diff, &dy2, &x2); sign = -1; }
        if (!(diff.n == 1 && diff.w[0] == 4)) rc = EO_ECERT;
        if (norm_sign) *norm_sign = sign;
        big_free(&x0); big_free(&two_p); big_free(&zero); big_free(&x2);
        big_free(&y2); big_free(&dy2); big_free(&diff);
        if (rc == EO_OK) {
            big_copy(p, &p1);
            big_copy(q, &q1);
        }
    }
    if (period) *period = k;
    big_free(&p1); big_free(&p2); big_free(&q1); big_free(&q2); big_free(&t);
    return rc;
}

/* Step 3. Residue of eps = (p-q)*1 + q*w in F_4^* = Z/3.
 * DLOG: (1,0)->0, (0,1)->1, (1,1)->2 on ((p-q) mod 2, q mod 2). */
static int dlog_parity(int a_odd, int b_odd) {
    if (a_odd && !b_odd) return 0;
    if (!a_odd && b_odd) return 1;
    if (a_odd && b_odd) return 2;
    return -1; /* (0,0): element in 2O_K, impossible for a unit */
}

/* Residue t in {0,1,2} of eps_d for d in D; negative EO_* code on error.
 * Requires d = 5 mod 8 and squarefree. */
int eo_residue(uint64_t d, int64_t *period) {
    if (d % 8 != 5 || !eo_is_squarefree(d)) return EO_EINVAL;
    big p, q;
    if (big_init(&p, 4) || big_init(&q, 4)) return EO_ENOMEM;
    int rc = eo_unit_pq(d, &p, &q, period, NULL);
    int t = rc;
    if (rc == EO_OK) {
        int p_odd = p.n ? (int)(p.w[0] & 1) : 0;
        int q_odd = q.n ? (int)(q.w[0] & 1) : 0;
        t = dlog_parity(p_odd ^ q_odd, q_odd);
        if (t < 0) t = EO_ECERT;
    }
    big_free(&p); big_free(&q);
    return t;
}

/* eps_d = (x0 + y0 sqrt d)/2 as decimal-free little-endian 64-bit limb arrays.
 * Writes up to cap limbs of x0 and y0; *nx, *ny receive the limb counts
 * (if larger than cap the arrays are truncated and EO_ENOMEM is returned).
 * *norm receives +1 or -1 (the sign of x0^2 - d y0^2). */
int eo_unit(uint64_t d, uint64_t *x0, int *nx, uint64_t *y0, int *ny, int cap, int *norm,
            int64_t *period) {
    if (d % 8 != 5 || !eo_is_squarefree(d)) return EO_EINVAL;
    big p, q, x, two_p, zero;
    big_init(&p, 4); big_init(&q, 4); big_init(&x, 4); big_init(&two_p, 4); big_init(&zero, 1);
    big_set_u64(&zero, 0);
    int rc = eo_unit_pq(d, &p, &q, period, norm);
    if (rc == EO_OK) {
        big_muladd(&two_p, &p, 2, &zero);
        big_sub(&x, &two_p, &q);
        *nx = x.n;
        *ny = q.n;
        if (x.n > cap || q.n > cap) rc = EO_ENOMEM;
        else {
            memcpy(x0, x.w, (size_t)x.n * 8);
            memcpy(y0, q.w, (size_t)q.n * 8);
        }
    }
    big_free(&p); big_free(&q); big_free(&x); big_free(&two_p); big_free(&zero);
    return rc;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

/* One byte per candidate d_i = first + 8 i (first = smallest d >= lo with
 * d = 5 mod 8), d_i <= hi: out[i] = t(eps) in {0,1,2}, or 0xFF if d_i is not
 * squarefree.  Returns the number of candidates, or a negative EO_* code. */
int64_t eo_classify_range(uint64_t lo, uint64_t hi, uint8_t *out, int64_t out_len,
                          int nthreads) {
    if (lo > hi) return 0;
    uint64_t first = lo + ((5 + 8 - lo % 8) % 8);
    if (first > hi) return 0;
    int64_t n = (int64_t)((hi - first) / 8 + 1);
    if (n > out_len) return EO_EINVAL;
    set_threads(nthreads);
    int err = 0;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; i++) {
        uint64_t d = first + 8 * (uint64_t)i;
        if (!eo_is_squarefree(d)) { out[i] = EO_NOT_IN_D; continue; }
        int t = eo_residue(d, NULL);
        if (t < 0) {
#pragma omp atomic write
            err = t;
            out[i] = 0xFE;
        } else {
            out[i] = (uint8_t)t;
        }
    }
    return err ? err : n;
}

/* Classify an explicit list of d (each must be = 5 mod 8): out[i] as above. */
int eo_classify_list(const uint64_t *d, int64_t n, uint8_t *out, int nthreads) {
    set_threads(nthreads);
    int err = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; i++) {
        if (d[i] % 8 != 5) { out[i] = 0xFE; err = EO_EINVAL; continue; }
        if (!eo_is_squarefree(d[i])) { out[i] = EO_NOT_IN_D; continue; }
        int t = eo_residue(d[i], NULL);
        if (t < 0) {
#pragma omp atomic write
            err = t;
            out[i] = 0xFE;
        } else {
            out[i] = (uint8_t)t;
        }
    }
    return err;
}

/* Window counts: for strictly ascending x[0..n-1] with
 * lo < x[0]: cnt_D[i] = #{d in D: lo < d <= x[i]}, cnt_E[i] likewise for E. */
int eo_count_window(uint64_t lo, const uint64_t *x, int64_t n, uint64_t *cnt_D,
                    uint64_t *cnt_E, int nthreads) {
    if (n <= 0) return 0;
    for (int64_t i = 0; i < n; i++) {
        if (x[i] <= lo) return EO_EINVAL;
        if (i && x[i] <= x[i - 1]) return EO_EINVAL;
    }
    uint64_t hi = x[n - 1];
    uint64_t first = (lo + 1) + ((5 + 8 - (lo + 1) % 8) % 8);
    int64_t m = first > hi ? 0 : (int64_t)((hi - first) / 8 + 1);
    uint8_t *f = (uint8_t *)malloc(m ? (size_t)m : 1);
    if (!f) return EO_ENOMEM;
    int64_t r = m ? eo_classify_range(first, hi, f, m, nthreads) : 0;
    if (r < 0) { free(f); return (int)r; }
    int64_t j = 0;
    uint64_t cD = 0, cE = 0;
    for (int64_t i = 0; i < n; i++) {
        for (; j < m && first + 8 * (uint64_t)j <= x[i]; j++) {
            if (f[j] != EO_NOT_IN_D) cD++;
            if (f[j] == 0) cE++;
        }
        cnt_D[i] = cD;
        cnt_E[i] = cE;
    }
    free(f);
    return 0;
}
