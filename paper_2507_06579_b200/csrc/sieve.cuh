// sieve.cuh -- K1 segmented p^2 sieve + K2 compaction.
//
// D = { d = 5 mod 8, squarefree }.  In candidate-index space
// (d = 8 i + 5) the multiples of p^2 (p odd prime; p^2 = 1 mod 8) are the i with
// i = (5 p^2 - 5)/8 (mod p^2): 8 (5p^2-5)/8 + 5 = 5 p^2.  4 never divides d.
//
// One CTA owns SIEVE_CHUNK candidates as a bitmap in shared memory:
//  * small primes (p^2 <= SIEVE_CHUNK) are struck cooperatively by the whole CTA,
//  * large primes are taken one per thread (at most one strike per chunk),
//  * survivors are compacted with popc + a CTA scan and ONE global atomic per
//    CTA into the segment's survivor list (u32 offsets within the segment).
// Non-survivor flags (EIS_NOT_IN_D = 0xFF) are written with 16-byte stores.
//
// With `primes` set (the prime subsequence, Sec. 3.2 l.501-522), a
// second bitmap marks the prime candidates: every odd prime p <= sqrt(d_max)
// strikes its multiples d = p m >= p^2 (d = 5 mod 8 <=> i = r_p mod p with
// r_p = -5/8 mod p), and survivors carry PRIME_BIT in their list entry.
#pragma once
#include "common.cuh"

constexpr int SIEVE_CHUNK = 1 << 18;          // candidates per CTA (32 KB bitmap)
constexpr int SIEVE_WORDS = SIEVE_CHUNK / 32;
constexpr int SIEVE_THREADS = 512;
constexpr int SIEVE_WPT = SIEVE_WORDS / SIEVE_THREADS;   // bitmap words per thread

__global__ void __launch_bounds__(SIEVE_THREADS)
sieve_compact_kernel(u64 i0, u64 len, const u32 *__restrict__ primes, int n_small, int n_primes,
                     u32 *__restrict__ list, u32 *__restrict__ count, u8 *__restrict__ flags,
                     int with_primes, int n_small1) {
    extern __shared__ u32 bm[];
    u32 *pm = bm + SIEVE_WORDS;                   // primality bitmap (with_primes)
    __shared__ u32 warp_tot[SIEVE_THREADS / 32];
    __shared__ u32 blk_base;
    const int tid = threadIdx.x;
    const u64 c0 = (u64)blockIdx.x * SIEVE_CHUNK;
    const u32 clen = (u32)min((u64)SIEVE_CHUNK, len - c0);
    const u64 base = i0 + c0;   // candidate index of bit 0

    for (int w = tid; w < SIEVE_WORDS; w += SIEVE_THREADS) {
        u32 lo = (u32)w * 32;
        u32 v = 0;
        if (lo + 32 <= clen) v = FULL_MASK;
        else if (lo < clen) v = (1u << (clen - lo)) - 1;
        bm[w] = v;
        if (with_primes) pm[w] = v;
    }
    __syncthreads();

    // small primes: the whole CTA strides over the multiples
    for (int k = 0; k < n_small; k++) {
        u64 p = primes[k];
        u64 p2 = p * p;
        u64 r = (5 * p2 - 5) / 8;
        u64 off = (r + p2 - base % p2) % p2;
        for (u64 j = off + (u64)tid * p2; j < clen; j += (u64)SIEVE_THREADS * p2)
            atomicAnd(&bm[j >> 5], ~(1u << (j & 31)));
    }
    // large primes (p^2 > SIEVE_CHUNK): at most one strike each
    for (int k = n_small + tid; k < n_primes; k += SIEVE_THREADS) {
        u64 p = primes[k];
        u64 p2 = p * p;
        u64 r = (5 * p2 - 5) / 8;
        u64 off = (r + p2 - base % p2) % p2;
        if (off < clen) atomicAnd(&bm[off >> 5], ~(1u << (off & 31)));
    }
    if (with_primes) {
        // multiples d = p m, m >= p (so p itself stays prime), of every odd
        // prime p <= sqrt(d_max): i = r_p (mod p), i >= (p^2 - 1)/8
        auto first_strike = [&](u32 p) -> u64 {      // offset of the first strike, or >= clen
            const u32 inv8 = (u32)((1 + (u64)p * ((8 - p % 8) % 8)) / 8);   // 8^-1 mod p
            u32 r5 = 5 * inv8;                                               // < 5p
            while (r5 >= p) r5 -= p;
            const u32 rp = r5 ? p - r5 : 0;                                  // -5/8 mod p
            const u64 i_min = ((u64)p * p - 1) / 8;
            const u64 f0 = base > i_min ? base : i_min;
            u64 q = (u64)((double)f0 / (double)p);                           // f0 < 2^34: exact
            while (q * p > f0) q--;
            while ((q + 1) * p <= f0) q++;
            const u32 fm = (u32)(f0 - q * p);                                // f0 mod p
            const u64 first = f0 + (rp >= fm ? rp - fm : rp + p - fm);
            return first - base;
        };
        for (int k = 0; k < n_small1; k++) {          // many strikes per chunk: whole CTA
            const u32 p = primes[k];
            const u64 j0 = first_strike(p);
            for (u64 j = j0 + (u64)tid * p; j < clen; j += (u64)SIEVE_THREADS * p)
                atomicAnd(&pm[j >> 5], ~(1u << (j & 31)));
        }
        for (int k = n_small1 + tid; k < n_primes; k += SIEVE_THREADS) {   // few strikes each
            const u32 p = primes[k];
            for (u64 j = first_strike(p); j < clen; j += p) atomicAnd(&pm[j >> 5], ~(1u << (j & 31)));
        }
    }
    __syncthreads();

    // compaction: each thread owns SIEVE_WPT consecutive words
    const int w0 = tid * SIEVE_WPT;
    u32 mine = 0;
#pragma unroll 4
    for (int w = 0; w < SIEVE_WPT; w++) mine += __popc(bm[w0 + w]);
    // CTA exclusive scan of `mine`
    const int lane = tid & 31, wid = tid >> 5;
    u32 incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 v = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        u32 v = lane < SIEVE_THREADS / 32 ? warp_tot[lane] : 0;
        u32 iv = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 t = __shfl_up_sync(FULL_MASK, iv, o);
            if (lane >= o) iv += t;
        }
        if (lane < SIEVE_THREADS / 32) warp_tot[lane] = iv - v;   // exclusive
        if (lane == 31) blk_base = atomicAdd(count, iv);          // CTA total
    }
    __syncthreads();
    u32 pos = blk_base + warp_tot[wid] + (incl - mine);
    for (int w = 0; w < SIEVE_WPT; w++) {
        u32 bits = bm[w0 + w];
        u32 o = (u32)(c0 + (u64)(w0 + w) * 32);
        while (bits) {
            int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const u32 pb = with_primes ? ((pm[w0 + w] >> b) & 1u) << 31 : 0u;
            list[pos++] = (o + b) | pb;
        }
    }
    if (flags) {
        // 0xFF for struck candidates, 0x00 placeholder for survivors (the walk
        // overwrites them).  Bytes beyond clen are not written.
        for (int w = 0; w < SIEVE_WPT; w++) {
            u32 wi = w0 + w;
            u32 lo = wi * 32;
            if (lo >= clen) break;
            u32 bits = bm[wi];
            u8 *dst = flags + c0 + lo;
            if (lo + 32 <= clen && ((uintptr_t)dst & 15) == 0) {
                uint4 v[2];
                u32 *vw = reinterpret_cast<u32 *>(v);
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    u32 nib = (bits >> (4 * q)) & 0xF;
                    // byte k of word q <- 0xFF if bit (4q+k) is clear
                    u32 x = 0;
#pragma unroll
                    for (int k = 0; k < 4; k++) x |= ((nib >> k) & 1) ? 0u : (0xFFu << (8 * k));
                    vw[q] = x;
                }
                reinterpret_cast<uint4 *>(dst)[0] = v[0];
                reinterpret_cast<uint4 *>(dst)[1] = v[1];
            } else {
                for (u32 k = 0; k < 32 && lo + k < clen; k++)
                    dst[k] = ((bits >> k) & 1) ? 0 : 0xFF;
            }
        }
    }
}
