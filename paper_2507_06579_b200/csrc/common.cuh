// common.cuh -- shared device helpers of the sm_100a Eisenstein classifier.
// (No code is shared with oracle/: this is the product path only.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cmath>
#include <cstring>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;
typedef int32_t i32;
typedef uint8_t u8;
typedef uint16_t u16;

#define FULL_MASK 0xffffffffu

// Device step functions are also compiled for the host by the CPU emulation
// harness in tests/ (tests/emu/kernel_emu.cu), which runs the same per-d state
// machine lane by lane against the oracle.  The product library never calls
// them on the host.
#define EIS_HD __host__ __device__ __forceinline__
// rare paths kept out of line (smaller hot loops, fewer instruction-cache misses)
#define EIS_HD_COLD __host__ __device__ __noinline__

// Host-only event counters for the CPU emulation's per-step profile
// (tests/emu, -DEIS_HOST_PROFILE); compiled out everywhere else.
#if defined(EIS_HOST_PROFILE) && !defined(__CUDA_ARCH__)
extern unsigned eis_prof[16];
#define EIS_PROF(i) (void)(eis_prof[i]++)
#else
#define EIS_PROF(i) (void)0
#endif

// fast reciprocal: MUFU.RCP on the device; IEEE 1/x in the host emulation
// (both are within the 2^-22 relative error the quotient proofs assume)
EIS_HD float rcp_approx(float x) {
#ifdef __CUDA_ARCH__
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
#else
    return 1.0f / x;
#endif
}

EIS_HD float u2f_bits(u32 v) {
#ifdef __CUDA_ARCH__
    return __uint_as_float(v);
#else
    float f;
    memcpy(&f, &v, 4);
    return f;
#endif
}
EIS_HD u32 f2u_bits(float f) {
#ifdef __CUDA_ARCH__
    return __float_as_uint(f);
#else
    u32 v;
    memcpy(&v, &f, 4);
    return v;
#endif
}

// the low 32 bits of an integer-valued double v, |v| < 2^51, without a
// conversion (the XU pipe is narrow): v + 1.5 * 2^52 holds v in its low mantissa
// bits, two's complement for v < 0
EIS_HD u32 dlo32(double v) {
#ifdef __CUDA_ARCH__
    return (u32)__double2loint(v + 6755399441055744.0);
#else
    return (u32)(long long)v;
#endif
}

// fma rounded toward zero (FFMA.RZ).  The host emulation computes the exact
// product-sum in double (a 20-bit x 24-bit product plus 2^23 is exact there)
// and truncates, which equals RZ to float for results in [2^23, 2^24).
EIS_HD float fma_rz(float a, float b, float c) {
#ifdef __CUDA_ARCH__
    return __fmaf_rz(a, b, c);
#else
    return (float)trunc((double)a * (double)b + (double)c);
#endif
}

// Explicit reconvergence point for the lanes in `mask` after a loop with a
// data-dependent trip count (otherwise the warp may stay split for the rest of
// the step: measured 2.8/32 active threads in a probe loop).  No-op on the host.
EIS_HD void warp_reconverge(u32 mask) {
#ifdef __CUDA_ARCH__
    __syncwarp(mask);
#else
    (void)mask;
#endif
}

// ballot over the lanes in `mask` (all of them must execute it); host: 1 lane
EIS_HD u32 warp_ballot(u32 mask, bool pred) {
#ifdef __CUDA_ARCH__
    return __ballot_sync(mask, pred);
#else
    (void)mask;
    return pred ? 1u : 0u;
#endif
}

// clamp to [0, 1] (FADD.SAT / FMUL.SAT modifier on the device)
EIS_HD float sat01(float x) {
#ifdef __CUDA_ARCH__
    return __saturatef(x);
#else
    return fminf(fmaxf(x, 0.f), 1.f);
#endif
}

// index of the lowest set bit (x != 0)
EIS_HD int __builtin_ctz_portable(u32 x) {
#ifdef __CUDA_ARCH__
    return __ffs(x) - 1;
#else
    return __builtin_ctz(x);
#endif
}

EIS_HD float log2_approx(float x) {
#ifdef __CUDA_ARCH__
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
#else
    return log2f(x);
#endif
}

// Candidate index i <-> d = 8 i + 5 (every d in D is = 5 mod 8).
__host__ __device__ __forceinline__ u64 cand_d(u64 i) { return 8 * i + 5; }

// floor(sqrt(d)) exactly for d < 2^53 (fp64 sqrt is within 1 ulp; two fixes).
EIS_HD u32 isqrt_u64_dev(u64 d) {
    u64 s = (u64)sqrt((double)d);
    while (s * s > d) --s;
    while ((s + 1) * (s + 1) <= d) ++s;
    return (u32)s;
}

// Segment-local checkpoint histogram capacity (buckets per segment).
constexpr int HIST_CAP = 1024;

// Count rows of the checkpoint histogram (eis_count_window_ext):
//   0 D, 1 E (t = 0), 2 t = 1, 3 D cap P (prime d), 4 E cap P.
// The basic counting functions use rows 0-1 only.
constexpr int NROW_MAX = 5;
// Survivor-list entries: bit 31 flags a prime d (set only when the sieve
// was asked for primality); the low 31 bits are the segment offset.
constexpr u32 PRIME_BIT = 0x80000000u;

// Arguments shared by the walk kernels.
struct WalkArgs {
    u64 i0;              // candidate index of segment offset 0
    const u32 *list;     // survivor offsets (d in D) within the segment
    const u32 *count;    // device: number of survivors
    u32 *work;           // device: work counter (zeroed before launch)
    u8 *flags;           // nullable: flags[off] = t for survivors
    const u64 *ckpt;     // nullable: checkpoints x[0..n_ckpt)
    int b_lo, nb;        // bucket range of this segment: [b_lo, b_lo+nb)
    int n_ckpt;
    int nrow;            // count rows (2 or NROW_MAX)
    u32 hist_w;          // hist_words_of(ckpt, nrow, nb), set on the host
    u64 ck_x0, ck_step;  // ck_step > 0: x[b_lo + i] = ck_x0 + i ck_step on this segment's
    double ck_rstep;     // buckets (checkpoints in arithmetic progression), 1 / ck_step
    u64 *buckets;        // device: [nrow][n_ckpt] counts (row order above)
    u64 *stats;          // device: EisStatSlot counters
    u32 *err;            // device: invariant-violation counter
};

enum EisStatSlot {
    ST_D = 0, ST_BABY = 1, ST_GIANT = 2, ST_REDUCE = 3, ST_SYM = 4, ST_FALLBACK = 5,
    ST_WINDOWED = 6,     // d whose BSGS window (list + table) was stored
    ST_NSLOTS = 8
};

// least b in [lo, hi] with d <= x[b]  (caller guarantees d <= x[hi])
__device__ __forceinline__ int bucket_of(const u64 *x, int lo, int hi, u64 d) {
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (d <= __ldg(x + mid)) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// shared-memory words of a walk kernel's histogram (dynamic shared memory, a
// multiple of 4 so that what follows stays 16-byte aligned)
inline __host__ __device__ u32 hist_words_of(const void *ckpt, int nrow, int nb) {
    return ckpt ? ((u32)(nrow * nb) + 3u) & ~3u : 0u;
}
// (a precomputed field: the compiler rematerialises it inside hot loops, where
// a single constant load is much cheaper than the expression)
inline __host__ __device__ u32 hist_words(const WalkArgs &a) { return a.hist_w; }

#ifdef __CUDACC__
__device__ __forceinline__ void hist_zero(const WalkArgs &a, u32 *hist) {
    for (int i = threadIdx.x; i < a.nrow * a.nb; i += blockDim.x) hist[i] = 0;
}
// K4: one finished d into the CTA's shared-memory histogram
// the bucket when the segment's checkpoints are an arithmetic progression: the
// least i with d <= x0 + i step, from one fp64 quotient and exact integer
// corrections (d - x0 < 2^53), instead of a binary search of dependent loads
__device__ __forceinline__ int bucket_arith(const WalkArgs &a, u64 d) {
    if (d <= a.ck_x0) return 0;
    const u64 t = d - a.ck_x0;
    u64 i = (u64)ceil((double)t * a.ck_rstep);
    if (i * a.ck_step < t) i++;
    else if (i > 0 && (i - 1) * a.ck_step >= t) i--;
    return i < (u64)(a.nb - 1) ? (int)i : a.nb - 1;
}
__device__ __forceinline__ void hist_record(const WalkArgs &a, u32 *hist, u64 d, u32 t,
                                            bool prime) {
    const int b = a.ck_step ? bucket_arith(a, d)
                            : bucket_of(a.ckpt, a.b_lo, a.b_lo + a.nb - 1, d) - a.b_lo;
    atomicAdd(&hist[b], 1u);
    if (t == 0) atomicAdd(&hist[a.nb + b], 1u);
    if (a.nrow > 2) {
        if (t == 1) atomicAdd(&hist[2 * a.nb + b], 1u);
        if (prime) {
            atomicAdd(&hist[3 * a.nb + b], 1u);
            if (t == 0) atomicAdd(&hist[4 * a.nb + b], 1u);
        }
    }
}
// one global atomic per CTA per nonzero bucket
__device__ __forceinline__ void hist_flush(const WalkArgs &a, u32 *hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < a.nrow * a.nb; i += blockDim.x) {
        if (hist[i]) {
            const int r = i / a.nb, b = i - r * a.nb;
            atomicAdd((unsigned long long *)&a.buckets[(size_t)r * a.n_ckpt + a.b_lo + b],
                      (unsigned long long)hist[i]);
        }
    }
}
#endif

__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    return v;
}
