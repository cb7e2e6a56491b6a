// regulator_sample.c -- design-analysis helper (not on the product path, not a
// test oracle): for each d on stdin that is squarefree, print
//   d  R  steps  omega  omega_B  log L_B
// R = the principal-cycle distance in nats (sum of log((P + sqrt d)/Q) over one
// period of the continued fraction of (1 + sqrt d)/2, in double), steps = the
// period length, omega = the number of prime factors of d, omega_B = the number
// below B (argv[1], default 100), log L_B = the truncated Euler product
// log prod_{p <= B} (1 - (d/p)/p)^-1 (with chi(2) = -1 for d = 5 mod 8).
// Used by scripts/class_window_model.py (per-class windows).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

typedef unsigned long long u64;
typedef long long i64;

static int primes[4000], nprimes;

int main(int argc, char **argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 100;
    for (int p = 3; p < 20000; p += 2) {
        int ok = 1;
        for (int q = 3; q * q <= p; q += 2)
            if (p % q == 0) { ok = 0; break; }
        if (ok) primes[nprimes++] = p;
    }
    u64 d;
    while (scanf("%llu", &d) == 1) {
        u64 m = d;
        int sf = 1;
        for (u64 p = 3; p * p <= m; p += 2)
            if (m % p == 0) {
                m /= p;
                if (m % p == 0) { sf = 0; break; }
            }
        if (!sf) continue;
        int omega = 0;
        m = d;
        for (u64 p = 3; p * p <= m; p += 2)
            if (m % p == 0) { omega++; m /= p; }
        if (m > 1) omega++;
        int omB = 0;
        double logL = log(2.0 / 3.0);
        for (int i = 0; i < nprimes && primes[i] <= B; i++) {
            const u64 p = (u64)primes[i], r = d % p;
            if (r == 0) { omB++; continue; }
            u64 e = (p - 1) / 2, b = r, res = 1;
            while (e) {
                if (e & 1) res = res * b % p;
                b = b * b % p;
                e >>= 1;
            }
            logL += -log(1.0 - (res == 1 ? 1.0 : -1.0) / (double)p);
        }
        const double sq = sqrt((double)d);
        u64 s = (u64)sq;
        while (s * s > d) s--;
        while ((s + 1) * (s + 1) <= d) s++;
        i64 P = (s & 1) ? (i64)s : (i64)s - 1, Q = 2;
        const i64 P0 = P;
        double R = 0;
        long steps = 0;
        do {
            const i64 a = (P + (i64)s) / Q, Pn = a * Q - P, Qn = ((i64)d - Pn * Pn) / Q;
            R += log((P + sq) / Q);
            P = Pn;
            Q = Qn;
            steps++;
        } while (!(Q == 2 && P == P0) && steps < 100000000);
        printf("%llu %.4f %ld %d %d %.5f\n", d, R, steps, omega, omB, logL);
    }
    return 0;
}
