// eis_api.cu -- C ABI (include/eis.h) of the B200 Eisenstein classifier.
//
// Host runtime: validates arguments, owns device scratch, splits the candidate
// range into segments, and launches per segment
//   K1+K2 sieve_compact_kernel  (sieve.cuh)       -> survivor list
//   K3+K4 walk kernel            (walk_*.cuh)     -> flags and/or bucket counts
// and finally the prefix kernel for the counting functions.  Everything the
// method computes runs in these kernels; the host only does index arithmetic.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types and prototypes only: libnccl is dlopen'ed by eis_comm_init

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/eis.h"
#include "common.cuh"
#include "sieve.cuh"
#include "walk_half.cuh"
#include "walk_bsgs.cuh"

namespace {

// One of two segment buffers: consecutive segments alternate, so the giant
// kernel of segment i (aux stream) overlaps the sieve and baby kernel of
// segment i+1 (main stream); events order the reuse of a buffer.
struct SegBuf {
    u32 *list = nullptr;
    size_t list_cap = 0;
    u32 *ctr = nullptr;              // [0] survivors, [1] work, [2..3] BSGS queue counters
    BsgsScratch bsgs;
    cudaEvent_t baby_done = nullptr, giant_done = nullptr;
};

struct Ctx {
    bool inited = false;
    int device = -1;
    int num_sms = 0;
    std::vector<u32> h_primes;       // odd primes p <= isqrt(EIS_MAX_D)
    u32 *d_primes = nullptr;
    SegBuf buf[2];
    u32 *d_err = nullptr;            // in-kernel invariant violations of the current call
    u8 *d_flags = nullptr;
    size_t flags_cap = 0;
    u64 *d_x = nullptr;
    size_t x_cap = 0;
    u64 *d_buckets = nullptr;
    size_t buckets_cap = 0;
    u64 *d_stats = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;      // giant kernels
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    bool walk_open = false;          // ev[2] marks the start of an unfinished run_range sequence
    // eis_classify_range: two flag buffers, their D2H copies on a copy stream
    u8 *d_flags2[2] = {nullptr, nullptr};
    size_t flags2_cap = 0;
    cudaStream_t cpy = nullptr;
    cudaEvent_t fl_ready[2] = {nullptr, nullptr}, fl_free[2] = {nullptr, nullptr};
    // whole box (eis_comm_init): NCCL communicator over one process per GPU
    ncclComm_t comm = nullptr;
    int comm_world = 1, comm_rank = 0;
    // options
    int mode = EIS_MODE_AUTO;
    u64 crossover = 750000000ULL;    // AUTO: HALF below, BSGS at/above (measured on B200, end of
                                     // round 2, 1e8-wide windows: HALF 1.01x faster at 7e8, BSGS
                                     // 1.02x at 8e8, 1.07x at 1e9, 1.09x at 1.1e9)
    int alpha_x16 = 0;               // BSGS baby window W = alpha d^(1/4); 0 = by d (alpha_for)
    int segment_log2 = 25;
    int blocks_per_sm = 4;           // measured: 4 >= 6 >= 8 (K3 HALF)
    int threads = 256;
    int giant_ctas = 0;
    int window_ctas = 0;             // BSGS window kernel CTAs per SM (0 = occupancy maximum)
    int giant_cap = 20;              // BSGS giant steps per d before the exact half walk takes
                                     // over: giant_cap * (d^(1/4) + 10) (tests force it to 0)
    int bsgs_gb = 48;                // BSGS store memory per segment buffer in GiB (two buffers;
                                     // a range within 2 bsgs_gb GiB runs as one segment)
    int half_ksteps = 0;             // 0: chosen per segment from d
    int two_sided = 1;               // BSGS: two-sided window (R35); 0 = paper's Alg. 1
    int load_x100 = BKT_LOAD_X100;   // BSGS table load factor x 100 (tests stress chains with it)
    // instrumentation of the last call
    eis_stats last{};
    float walk_ms_acc = 0.f;
    int last_nw = 0, last_nb = 0;    // window entries / table buckets per d of the last BSGS segment
    int launches = 0;
    // per-kernel device time: event pairs around each launch, summed at the end
    // of run_range (the events are complete then)
    std::vector<cudaEvent_t> kev;
    std::vector<std::pair<int, int>> kspan[3];     // [0] sieve, [1] window+prep / half, [2] giant
    int kev_used = 0;
    double kms[3] = {0, 0, 0};
};

Ctx g;
thread_local std::string g_err;

// next event of the per-kernel timing pool (created on first use)
cudaEvent_t kev_next(int &idx) {
    if (g.kev_used == (int)g.kev.size()) {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        g.kev.push_back(e);
    }
    idx = g.kev_used++;
    return g.kev[idx];
}

const char *eis_last_error_internal();
int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(e_ == cudaErrorMemoryAllocation ? EIS_ENOMEM : EIS_EDEVICE,        \
                        "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                         \
    } while (0)

const char *eis_last_error_internal() {
    static thread_local std::string copy;
    copy = g_err;
    return copy.c_str();
}

u64 isqrt_host(u64 n) {
    u64 s = (u64)std::sqrt((double)n);
    while (s * s > n) --s;
    while ((s + 1) * (s + 1) <= n) ++s;
    return s;
}

void build_primes(std::vector<u32> &out) {
    const u32 M = (u32)isqrt_host(EIS_MAX_D);
    std::vector<uint8_t> comp(M + 1, 0);
    out.clear();
    for (u32 i = 2; i <= M; i++) {
        if (comp[i]) continue;
        if (i != 2) out.push_back(i);
        for (u64 j = (u64)i * i; j <= M; j += i) comp[j] = 1;
    }
}

template <class T>
int ensure(T *&ptr, size_t &cap, size_t n) {
    if (n <= cap && ptr) return 0;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    size_t want = std::max(n, (size_t)1);
    CUDA_TRY(cudaMalloc(&ptr, want * sizeof(T)));
    cap = want;
    return 0;
}

int do_init(int device) {
    if (g.inited && (device < 0 || device == g.device)) return 0;
    if (g.inited) eis_finalize();
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(EIS_EDEVICE, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device >= 0) CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaGetDevice(&g.device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, g.device));
    if (prop.major < 10)
        return fail(EIS_EDEVICE, "device %d is sm_%d%d; this library is built for sm_100a",
                    g.device, prop.major, prop.minor);
    g.num_sms = prop.multiProcessorCount;
    build_primes(g.h_primes);
    CUDA_TRY(cudaMalloc(&g.d_primes, g.h_primes.size() * sizeof(u32)));
    CUDA_TRY(cudaMemcpy(g.d_primes, g.h_primes.data(), g.h_primes.size() * sizeof(u32),
                        cudaMemcpyHostToDevice));
    for (auto &b : g.buf) {
        CUDA_TRY(cudaMalloc(&b.ctr, 8 * sizeof(u32)));
        CUDA_TRY(cudaEventCreateWithFlags(&b.baby_done, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&b.giant_done, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaMalloc(&g.d_err, sizeof(u32)));
    CUDA_TRY(cudaMalloc(&g.d_stats, ST_NSLOTS * sizeof(u64)));
    CUDA_TRY(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&g.aux, cudaStreamNonBlocking));
    for (auto &ev : g.ev) CUDA_TRY(cudaEventCreate(&ev));
    CUDA_TRY(cudaStreamCreateWithFlags(&g.cpy, cudaStreamNonBlocking));
    for (int k = 0; k < 2; k++) {
        CUDA_TRY(cudaEventCreateWithFlags(&g.fl_ready[k], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&g.fl_free[k], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaFuncSetAttribute(sieve_compact_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  2 * SIEVE_WORDS * (int)sizeof(u32)));
    g.inited = true;
    return 0;
}

// number of odd primes p with p^2 <= v
int primes_upto_sq(u64 v) {
    u64 r = isqrt_host(v);
    return (int)(std::upper_bound(g.h_primes.begin(), g.h_primes.end(), (u32)std::min<u64>(r, 0xFFFFFFFFull)) -
                 g.h_primes.begin());
}
int primes_small() {   // p^2 <= SIEVE_CHUNK
    return primes_upto_sq((u64)SIEVE_CHUNK);
}

// candidate index range [i_first, i_last] for lo <= d <= hi; false if empty
bool cand_range(u64 lo, u64 hi, u64 &i_first, u64 &i_last) {
    if (lo > hi || hi < 5) return false;
    const u64 L = lo < 5 ? 5 : lo;
    const u64 first = L + (13 - L % 8) % 8;   // least d >= L with d = 5 mod 8
    if (first > hi) return false;
    i_first = (first - 5) / 8;
    i_last = (hi - 5) / 8;
    return true;
}

// BSGS window factor (x16) for a segment ending at d: the option, or (0) the
// measured optimum log-interpolated over d (2.25 up to 2e9, 1.875
// at 1e10, 1.625 at 1e11); results never depend on it (R6, R29)
int alpha_for(u64 d) {
    if (g.alpha_x16 > 0) return g.alpha_x16;
    const double x = std::log10((double)d);
    double a;
    if (x <= 9.3) a = 36;                                  // 2.25
    else if (x <= 10.0) a = 36 + (30 - 36) * (x - 9.3) / 0.7;
    else if (x <= 11.0) a = 30 + (26 - 30) * (x - 10.0);
    else a = 26;
    return (int)std::lround(a);
}

bool want_bsgs(u64 d_lo) {
    if (g.mode == EIS_MODE_HALF) return false;
    if (g.mode == EIS_MODE_BSGS) return true;
    return d_lo >= g.crossover;
}

// Process candidates [i_first, i_last].  flags_dev (nullable) is indexed by
// candidate index - i_first.  x_host/x_dev/n/buckets_dev (nullable) receive counts.
// The end of a sequence of run_range(..., finish = false) calls: wait for the
// streams, add the segment loop's and the kernels' device times to the call's
// statistics, and fail the call if any kernel counted an invariant violation.
int finish_range(cudaStream_t s) {
    if (g.walk_open) {
        CUDA_TRY(cudaEventRecord(g.ev[3], s));
        CUDA_TRY(cudaEventSynchronize(g.ev[3]));
        float ms = 0;
        cudaEventElapsedTime(&ms, g.ev[2], g.ev[3]);
        g.walk_ms_acc += ms;
        g.walk_open = false;
    }
    for (int k = 0; k < 3; k++) {
        for (auto &pr : g.kspan[k]) {
            float t = 0;
            if (cudaEventElapsedTime(&t, g.kev[pr.first], g.kev[pr.second]) == cudaSuccess)
                g.kms[k] += t;
        }
        g.kspan[k].clear();
    }
    g.kev_used = 0;
    u32 err = 0;
    CUDA_TRY(cudaMemcpy(&err, g.d_err, sizeof(u32), cudaMemcpyDeviceToHost));
    if (err) return fail(EIS_EINTERNAL, "%u in-kernel invariant violations", err);
    return 0;
}

// Process candidates [i_first, i_last].  flags_dev (nullable) is indexed by
// candidate index - i_first.  x_host/x_dev/n/buckets_dev (nullable) receive counts.
// finish = false leaves the kernels queued (no host wait); the caller then
// calls finish_range.
int run_range(u64 i_first, u64 i_last, u8 *flags_dev, const u64 *x_host, const u64 *x_dev,
              int n, u64 *buckets_dev, cudaStream_t s, int nrow = 2, bool finish = true) {
    // AUTO: a range that spans the crossover runs as two ranges (HALF below, BSGS
    // at and above it)
    if (g.mode == EIS_MODE_AUTO && cand_d(i_first) < g.crossover && cand_d(i_last) >= g.crossover) {
        const u64 i_cross = (g.crossover - 5 + 7) / 8;     // least i with 8i + 5 >= crossover
        if (int rc = run_range(i_first, i_cross - 1, flags_dev, x_host, x_dev, n, buckets_dev, s,
                               nrow, false))
            return rc;
        if (int rc = run_range(i_cross, i_last, flags_dev ? flags_dev + (i_cross - i_first) : nullptr,
                               x_host, x_dev, n, buckets_dev, s, nrow, false))
            return rc;
        return finish ? finish_range(s) : 0;
    }
    const int with_primes = nrow > 2;
    const u64 SEG = 1ull << g.segment_log2;
    const int n_small = primes_small();
    const int n_small1 = primes_upto_sq((u64)SIEVE_CHUNK * SIEVE_CHUNK / (64 * 64));   // p <= chunk/64
    // BSGS keeps one store per candidate slot of the segment, in two segment
    // buffers of at most bsgs_gb GiB each -- or, when the whole range fits in
    // 2 bsgs_gb GiB, as ONE segment in one buffer: fewer segments, fewer
    // giant-kernel tails (the bench slab as one segment instead of two measured
    // +1.5%, Layout).
    const bool bsgs = want_bsgs(cand_d(i_first));
    u64 seg_cap = SEG;
    if (bsgs) {
        const u64 per = bsgs_bytes_per_survivor(cand_d(i_last), alpha_for(cand_d(i_last)) / 16.0f,
                                                g.two_sided, g.load_x100 / 100.f);
        const u64 total = i_last - i_first + 1;
        const u64 cap_bytes = (u64)g.bsgs_gb << 30;
        seg_cap = total * per <= 2 * cap_bytes ? total
                                               : std::max<u64>(cap_bytes / per, 1ull << 16);
        seg_cap = std::min<u64>(SEG, seg_cap);
    }
    // equal segments: a short remainder segment would be all giant-kernel tail
    {
        const u64 total = i_last - i_first + 1;
        const u64 nseg = (total + seg_cap - 1) / seg_cap;
        seg_cap = (total + nseg - 1) / nseg;
    }
    // BSGS scratch: reserved once per range, for a full segment at the larger of
    // the two ends' window sizes (growing it segment by segment drained both
    // streams and reallocated tens of GiB on most segments of a prefix run)
    if (bsgs) {
        const u64 d_a = cand_d(i_first), d_b = cand_d(i_last);
        const BsgsSizes za = bsgs_sizes(d_a, alpha_for(d_a) / 16.0f, g.two_sided, g.load_x100 / 100.f);
        const BsgsSizes zb = bsgs_sizes(d_b, alpha_for(d_b) / 16.0f, g.two_sided, g.load_x100 / 100.f);
        const int lcap = std::max(za.lcap, zb.lcap), nbk = std::max(za.nb, zb.nb);
        // if the device cannot hold two buffers of bsgs_gb, halve the segment
        // (results do not depend on it) down to 2^16 candidates
        for (;;) {
            bool ok = true;
            // a range of one segment needs one buffer (the other may be freed to make room)
            const int nbuf = i_last - i_first + 1 > seg_cap ? 2 : 1;   // one segment: one buffer
            for (int ib = 0; ib < nbuf; ib++) {
                SegBuf &b = g.buf[ib];
                if (b.bsgs.lists && b.bsgs.lists_n >= seg_cap * (size_t)lcap &&
                    b.bsgs.tables_n >= seg_cap * (size_t)nbk * BKT && b.bsgs.brecs_n >= seg_cap)
                    continue;
                CUDA_TRY(cudaStreamSynchronize(g.aux));
                CUDA_TRY(cudaStreamSynchronize(s));
                if (bsgs_reserve(b.bsgs, (size_t)seg_cap, lcap, nbk)) {
                    ok = false;
                    break;
                }
            }
            if (ok) break;
            (void)cudaGetLastError();                    // clear the allocation failure
            for (SegBuf &b : g.buf) bsgs_free(b.bsgs);
            if (seg_cap <= (1ull << 16)) return fail(EIS_ENOMEM, "BSGS scratch allocation failed");
            const u64 total = i_last - i_first + 1;
            const u64 nseg = (total + seg_cap / 2 - 1) / (seg_cap / 2);
            seg_cap = std::max<u64>((total + nseg - 1) / nseg, 1ull << 16);
        }
    }
    if (!g.walk_open) {
        CUDA_TRY(cudaEventRecord(g.ev[2], s));
        g.walk_open = true;
    }
    int iseg = 0;
    bool used_aux = false;
    for (u64 seg = i_first; seg <= i_last; iseg++) {
        SegBuf &bf = g.buf[iseg & 1];
        u64 len = std::min(seg_cap, i_last - seg + 1);
        int b_lo = 0, nb = 0;
        if (x_host) {
            // bucket span of [d(seg), d(seg+len-1)] must fit HIST_CAP
            u64 d0 = cand_d(seg);
            b_lo = (int)(std::lower_bound(x_host, x_host + n, d0) - x_host);
            if (b_lo >= n) break;   // beyond the last checkpoint
            u64 dlast = cand_d(seg + len - 1);
            int b_hi = (int)(std::lower_bound(x_host, x_host + n, dlast) - x_host);
            if (b_hi >= n) {   // clip to the last checkpoint
                b_hi = n - 1;
                if (x_host[n - 1] < d0) break;
                len = (x_host[n - 1] - 5) / 8 - seg + 1;
            }
            if (b_hi - b_lo + 1 > HIST_CAP) {
                b_hi = b_lo + HIST_CAP - 1;
                u64 lim = x_host[b_hi];            // last d allowed: <= x[b_hi]
                len = (lim - 5) / 8 - seg + 1;
            }
            nb = b_hi - b_lo + 1;
        }
        const u64 d_last = cand_d(seg + len - 1);
        const int n_primes = primes_upto_sq(d_last);
        // the buffer is free once the giant kernel that last used it is done
        if (bsgs) CUDA_TRY(cudaStreamWaitEvent(s, bf.giant_done, 0));
        if (bf.list_cap < (size_t)len) {
            CUDA_TRY(cudaStreamSynchronize(s));
            if (ensure(bf.list, bf.list_cap, (size_t)len)) return EIS_ENOMEM;
        }
        CUDA_TRY(cudaMemsetAsync(bf.ctr, 0, 8 * sizeof(u32), s));
        const unsigned sblocks = (unsigned)((len + SIEVE_CHUNK - 1) / SIEVE_CHUNK);
        u8 *fseg = flags_dev ? flags_dev + (seg - i_first) : nullptr;
        int e0, e1;
        CUDA_TRY(cudaEventRecord(kev_next(e0), s));
        sieve_compact_kernel<<<sblocks, SIEVE_THREADS,
                               (with_primes ? 2 : 1) * SIEVE_WORDS * sizeof(u32), s>>>(
            seg, len, g.d_primes, std::min(n_small, n_primes), n_primes, bf.list, bf.ctr, fseg,
            with_primes, std::min(n_small1, n_primes));
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaEventRecord(kev_next(e1), s));
        g.kspan[0].push_back({e0, e1});
        g.launches++;

        WalkArgs a;
        a.i0 = seg;
        a.list = bf.list;
        a.count = bf.ctr;
        a.work = bf.ctr + 1;
        a.err = g.d_err;
        a.flags = fseg;
        a.ckpt = x_host ? x_dev : nullptr;
        a.b_lo = b_lo;
        // checkpoints of this segment in arithmetic progression: bucket by division
        a.ck_x0 = 0;
        a.ck_step = 0;
        a.ck_rstep = 0.0;
        if (x_host && nb >= 1) {
            const u64 x0 = x_host[b_lo], step = nb > 1 ? x_host[b_lo + 1] - x0 : 1;
            bool ar = step > 0;
            for (int i = 2; ar && i < (int)nb; i++) ar = x_host[b_lo + i] == x0 + (u64)i * step;
            if (ar) {
                a.ck_x0 = x0;
                a.ck_step = step;
                a.ck_rstep = 1.0 / (double)step;
            }
        }
        a.nb = nb;
        a.n_ckpt = n;
        a.nrow = nrow;
        a.hist_w = hist_words_of(a.ckpt, nrow, nb);
        a.buckets = buckets_dev;
        a.stats = g.d_stats;
        if (bsgs) {
            BsgsPlan pl;
            // scratch is (re)allocated only when it must grow: drain both streams then
            // (otherwise the giant kernel of the previous segment keeps running on aux)
            if (bsgs_needs_grow(bf.bsgs, len, d_last, alpha_for(d_last), g.two_sided,
                                g.load_x100 / 100.f)) {
                CUDA_TRY(cudaStreamSynchronize(g.aux));
                CUDA_TRY(cudaStreamSynchronize(s));
            }
            int rc = bsgs_prepare(pl, len, d_last, g.num_sms, alpha_for(d_last), g.giant_ctas, g.two_sided, bf.bsgs,
                                  bf.ctr + 2, g.window_ctas, hist_words(a), g.giant_cap,
                                  g.load_x100 / 100.f);
            if (rc) return rc == EIS_ENOMEM ? fail(EIS_ENOMEM, "BSGS scratch allocation failed")
                              : fail(EIS_EDEVICE, "BSGS setup failed: %s",
                                     cudaGetErrorString(cudaGetLastError()));
            g.last_nw = pl.B.nw;
            g.last_nb = pl.B.nb;
            CUDA_TRY(cudaEventRecord(kev_next(e0), s));
            if (bsgs_launch_baby(a, pl, s))
                return fail(EIS_EDEVICE, "BSGS baby launch failed: %s",
                            cudaGetErrorString(cudaGetLastError()));
            g.launches += 2;                            // window + prep
            CUDA_TRY(cudaEventRecord(kev_next(e1), s));
            g.kspan[1].push_back({e0, e1});
            CUDA_TRY(cudaEventRecord(bf.baby_done, s));
            CUDA_TRY(cudaStreamWaitEvent(g.aux, bf.baby_done, 0));
            CUDA_TRY(cudaEventRecord(kev_next(e0), g.aux));
            if (bsgs_launch_giant(a, pl, g.aux))
                return fail(EIS_EDEVICE, "BSGS giant launch failed: %s",
                            cudaGetErrorString(cudaGetLastError()));
            g.launches++;
            CUDA_TRY(cudaEventRecord(kev_next(e1), g.aux));
            g.kspan[2].push_back({e0, e1});
            CUDA_TRY(cudaEventRecord(bf.giant_done, g.aux));
            used_aux = true;
        } else {
            const unsigned wblocks = (unsigned)(g.num_sms * g.blocks_per_sm);
            // chunk length: ~1/8 of the expected half period (~0.07 sqrt d steps),
            // so lanes rarely idle after an exit (option half_ksteps = 0: auto)
            int ks = g.half_ksteps;
            if (ks == 0) {
                const double exp_steps = 0.07 * std::sqrt((double)cand_d(seg));
                ks = exp_steps >= 8 * 144 ? 144 : exp_steps >= 8 * 72 ? 72 : exp_steps >= 8 * 36 ? 36 : 18;
            }
            const size_t hb = (size_t)hist_words(a) * sizeof(u32);
            CUDA_TRY(cudaEventRecord(kev_next(e0), s));
            switch (ks) {
                case 18: walk_half_kernel<18><<<wblocks, 256, hb, s>>>(a); break;
                case 72: walk_half_kernel<72><<<wblocks, 256, hb, s>>>(a); break;
                case 144: walk_half_kernel<144><<<wblocks, 256, hb, s>>>(a); break;
                default: walk_half_kernel<36><<<wblocks, 256, hb, s>>>(a); break;
            }
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaEventRecord(kev_next(e1), s));
            g.kspan[1].push_back({e0, e1});
            g.launches++;
        }
        seg += len;
    }
    if (used_aux) {                                   // join the aux stream back into s
        CUDA_TRY(cudaEventRecord(g.ev[4], g.aux));
        CUDA_TRY(cudaStreamWaitEvent(s, g.ev[4], 0));
    }
    if (!finish) return 0;
    if (int rc = finish_range(s))
        return rc == EIS_EINTERNAL
                   ? fail(EIS_EINTERNAL, "%s in [%llu, %llu]", eis_last_error_internal(),
                          (unsigned long long)cand_d(i_first), (unsigned long long)cand_d(i_last))
                   : rc;
    return 0;
}

__global__ void prefix_kernel(const u64 *in, u64 *out, int n, int nrow) {
    // one CTA of 1024 threads: nrow independent inclusive scans of length n
    __shared__ u64 part[1024];
    for (int arr = 0; arr < nrow; arr++) {
        const u64 *src = in + (size_t)arr * n;
        u64 *dst = out + (size_t)arr * n;
        const int per = (n + 1023) / 1024;
        const int b = threadIdx.x * per, e = min(n, b + per);
        u64 acc = 0;
        for (int i = b; i < e; i++) acc += src[i];
        part[threadIdx.x] = acc;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            u64 v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
            __syncthreads();
            part[threadIdx.x] += v;
            __syncthreads();
        }
        u64 run = part[threadIdx.x] - acc;
        __syncthreads();
        for (int i = b; i < e; i++) { run += src[i]; dst[i] = run; }
        __syncthreads();
    }
}

int begin_call(cudaStream_t s) {
    g.walk_ms_acc = 0;
    g.walk_open = false;
    g.last_nw = g.last_nb = 0;
    g.launches = 0;
    g.kms[0] = g.kms[1] = g.kms[2] = 0;
    CUDA_TRY(cudaMemsetAsync(g.d_stats, 0, ST_NSLOTS * sizeof(u64), s));
    CUDA_TRY(cudaMemsetAsync(g.d_err, 0, sizeof(u32), s));
    CUDA_TRY(cudaEventRecord(g.ev[0], s));
    return 0;
}

int end_call(cudaStream_t s) {
    CUDA_TRY(cudaEventRecord(g.ev[1], s));
    CUDA_TRY(cudaEventSynchronize(g.ev[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, g.ev[0], g.ev[1]);
    u64 st[ST_NSLOTS];
    CUDA_TRY(cudaMemcpy(st, g.d_stats, sizeof st, cudaMemcpyDeviceToHost));
    g.last.d_classified = st[ST_D];
    g.last.baby_steps = st[ST_BABY];
    g.last.giant_steps = st[ST_GIANT];
    g.last.reduce_steps = st[ST_REDUCE];
    g.last.sym_exits = st[ST_SYM];
    g.last.fallbacks = st[ST_FALLBACK];
    g.last.kernel_launches = (u64)g.launches;
    g.last.walk_ms = g.walk_ms_acc;
    g.last.total_ms = ms;
    g.last.sieve_ms = g.kms[0];
    g.last.window_ms = g.kms[1];
    g.last.giant_ms = g.kms[2];
    g.last.windowed = st[ST_WINDOWED];
    g.last.window_nw = (u64)g.last_nw;
    g.last.window_nb = (u64)g.last_nb;
    return 0;
}

int check_x(const u64 *x, size_t n, u64 lo) {
    if (n == 0) return 0;
    if (!x) return fail(EIS_EINVAL, "x is NULL");
    if (x[0] <= lo) return fail(EIS_EINVAL, "x[0]=%llu must exceed lo=%llu",
                                (unsigned long long)x[0], (unsigned long long)lo);
    for (size_t i = 1; i < n; i++)
        if (x[i] <= x[i - 1]) return fail(EIS_EINVAL, "x must be strictly ascending (x[%zu])", i);
    if (x[n - 1] > EIS_MAX_D)
        return fail(EIS_ERANGE, "x[n-1]=%llu exceeds EIS_MAX_D", (unsigned long long)x[n - 1]);
    if (n > (size_t)1 << 30) return fail(EIS_EINVAL, "too many checkpoints");
    return 0;
}

int count_buckets(u64 lo, u64 hi, const u64 *x, size_t n, u64 *buckets_dev, cudaStream_t s,
                  int nrow = 2) {
    if (n == 0 || hi <= lo) return 0;
    if (ensure(g.d_x, g.x_cap, n)) return EIS_ENOMEM;
    CUDA_TRY(cudaMemcpyAsync(g.d_x, x, n * sizeof(u64), cudaMemcpyHostToDevice, s));
    u64 top = std::min(hi, x[n - 1]);
    u64 i_first, i_last;
    if (!cand_range(lo + 1, top, i_first, i_last)) return 0;
    return run_range(i_first, i_last, nullptr, x, g.d_x, (int)n, buckets_dev, s, nrow);
}

// counts over (lo, x[n-1]] into host out[nrow][n] (prefix sums at checkpoints)
int count_window_rows(u64 lo, const u64 *x, size_t n, int nrow, u64 *out) {
    if (n == 0) return 0;
    if (int rc = check_x(x, n, lo)) return rc;
    if (!out) return fail(EIS_EINVAL, "NULL output");
    if (int rc = do_init(-1)) return rc;
    cudaStream_t s = g.stream;
    if (int rc = begin_call(s)) return rc;
    const size_t m = (size_t)nrow * n;
    if (ensure(g.d_buckets, g.buckets_cap, m)) return EIS_ENOMEM;
    CUDA_TRY(cudaMemsetAsync(g.d_buckets, 0, m * sizeof(u64), s));
    if (int rc = count_buckets(lo, x[n - 1], x, n, g.d_buckets, s, nrow)) return rc;
    prefix_kernel<<<1, 1024, 0, s>>>(g.d_buckets, g.d_buckets, (int)n, nrow);
    CUDA_TRY(cudaGetLastError());
    g.launches++;
    CUDA_TRY(cudaMemcpyAsync(out, g.d_buckets, m * sizeof(u64), cudaMemcpyDeviceToHost, s));
    return end_call(s);
}

// ---- whole box: contiguous shards, one all-reduce ----------

// Relative device time per candidate at d of the AUTO path (measured on one
// B200): HALF below the crossover, rate ~ 2.68e8 (1e10/d)^(1/2)
// d/s; BSGS at and above it, rate ~ 5.0e8 (1e10/d)^0.224 d/s (fitted to 8e8-1e11
// at the end of round 2, within 7%).  Only the
// shape matters for splitting.
double auto_cost_density(double d) {
    d = std::max(d, 1.0);
    return d < (double)g.crossover ? std::pow(d / 1e10, 0.5) / 2.68e8
                                   : std::pow(d / 1e10, 0.224) / 5.0e8;
}

// cut point g of (lo, hi] into `world` contiguous shards, a multiple of 8
// (never = 5 mod 8, so no candidate is split) clamped to [lo, hi]
u64 shard_cut(u64 lo, u64 hi, int world, int gi, int balance, const std::vector<double> &cum,
              const std::vector<double> &xs) {
    if (gi <= 0) return lo;
    if (gi >= world) return hi;
    u64 v;
    const double f = (double)gi / world;
    if (balance == EIS_BALANCE_PREFIX) {
        v = lo + (u64)((double)(hi - lo) * std::pow(f, 0.8));   // x_g = X (g/G)^(4/5)
    } else if (balance == EIS_BALANCE_AUTO) {
        size_t k = (size_t)(std::lower_bound(cum.begin(), cum.end(), f) - cum.begin());
        k = std::min(std::max<size_t>(k, 1), cum.size() - 1);
        const double t = cum[k] > cum[k - 1] ? (f - cum[k - 1]) / (cum[k] - cum[k - 1]) : 0.0;
        v = (u64)(xs[k - 1] + t * (xs[k] - xs[k - 1]));
    } else {
        v = lo + (hi - lo) / (u64)world * (u64)gi + (hi - lo) % (u64)world * (u64)gi / (u64)world;
    }
    v -= v % 8;
    return std::min(hi, std::max(lo, v));
}

int shard_bounds(u64 lo, u64 hi, int world, int rank, int balance, u64 &a, u64 &b) {
    if (world < 1 || rank < 0 || rank >= world)
        return fail(EIS_EINVAL, "need 0 <= rank < world (rank %d, world %d)", rank, world);
    if (balance < EIS_BALANCE_FLAT || balance > EIS_BALANCE_AUTO)
        return fail(EIS_EINVAL, "unknown balance %d", balance);
    if (lo > hi) return fail(EIS_EINVAL, "lo > hi");
    if (world == 1) { a = lo; b = hi; return 0; }
    std::vector<double> cum, xs;
    if (balance == EIS_BALANCE_AUTO) {
        // cumulative modelled cost on 4096 equal intervals (trapezoids), normalised
        const int K = 4096;
        xs.resize(K + 1);
        cum.resize(K + 1);
        double prev = 0;
        for (int i = 0; i <= K; i++) {
            xs[i] = (double)lo + (double)(hi - lo) * i / K;
            const double c = auto_cost_density(xs[i]);
            cum[i] = i ? cum[i - 1] + 0.5 * (c + prev) * (xs[i] - xs[i - 1]) : 0.0;
            prev = c;
        }
        if (cum[K] > 0) for (double &v : cum) v /= cum[K];
    }
    a = shard_cut(lo, hi, world, rank, balance, cum, xs);
    b = shard_cut(lo, hi, world, rank + 1, balance, cum, xs);
    return 0;
}

// NCCL, resolved at run time (the library does not link it: a process that
// never calls eis_comm_init never loads it, and one that already holds
// libnccl.so.2, e.g. through torch, shares that copy)
struct NcclApi {
    void *h = nullptr;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};
NcclApi nccl;

int nccl_load() {
    if (nccl.h) return 0;
    const char *name = getenv("EIS_NCCL_LIB");
    void *h = dlopen(name && *name ? name : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(EIS_EDEVICE, "cannot load NCCL: %s", dlerror());
    nccl.get_unique_id = (decltype(&ncclGetUniqueId))dlsym(h, "ncclGetUniqueId");
    nccl.comm_init_rank = (decltype(&ncclCommInitRank))dlsym(h, "ncclCommInitRank");
    nccl.all_reduce = (decltype(&ncclAllReduce))dlsym(h, "ncclAllReduce");
    nccl.comm_destroy = (decltype(&ncclCommDestroy))dlsym(h, "ncclCommDestroy");
    nccl.error_string = (decltype(&ncclGetErrorString))dlsym(h, "ncclGetErrorString");
    if (!nccl.get_unique_id || !nccl.comm_init_rank || !nccl.all_reduce || !nccl.comm_destroy ||
        !nccl.error_string) {
        dlclose(h);
        return fail(EIS_EDEVICE, "libnccl lacks a required symbol");
    }
    nccl.h = h;
    return 0;
}

#define NCCL_TRY(expr)                                                                     \
    do {                                                                                   \
        ncclResult_t r_ = (expr);                                                          \
        if (r_ != ncclSuccess)                                                             \
            return fail(EIS_EDEVICE, "%s failed: %s", #expr, nccl.error_string(r_));       \
    } while (0)

void comm_release() {
    if (g.comm && nccl.comm_destroy) nccl.comm_destroy(g.comm);
    g.comm = nullptr;
    g.comm_world = 1;
    g.comm_rank = 0;
}

}  // namespace

extern "C" {

int eis_init(int device) { return do_init(device); }

void eis_finalize(void) {
    comm_release();
    if (!g.inited) return;
    cudaFree(g.d_primes);
    for (auto &b : g.buf) {
        cudaFree(b.list);
        cudaFree(b.ctr);
        bsgs_free(b.bsgs);
        if (b.baby_done) cudaEventDestroy(b.baby_done);
        if (b.giant_done) cudaEventDestroy(b.giant_done);
    }
    cudaFree(g.d_err);
    cudaFree(g.d_flags);
    cudaFree(g.d_x);
    cudaFree(g.d_buckets);
    cudaFree(g.d_stats);
    for (auto &ev : g.ev) if (ev) cudaEventDestroy(ev);
    for (int k = 0; k < 2; k++) {
        cudaFree(g.d_flags2[k]);
        if (g.fl_ready[k]) cudaEventDestroy(g.fl_ready[k]);
        if (g.fl_free[k]) cudaEventDestroy(g.fl_free[k]);
    }
    if (g.cpy) cudaStreamDestroy(g.cpy);
    for (auto &ev : g.kev) cudaEventDestroy(ev);
    if (g.stream) cudaStreamDestroy(g.stream);
    if (g.aux) cudaStreamDestroy(g.aux);
    Ctx fresh;
    fresh.mode = g.mode;
    fresh.crossover = g.crossover;
    fresh.alpha_x16 = g.alpha_x16;
    fresh.segment_log2 = g.segment_log2;
    fresh.blocks_per_sm = g.blocks_per_sm;
    fresh.giant_ctas = g.giant_ctas;
    fresh.window_ctas = g.window_ctas;
    fresh.bsgs_gb = g.bsgs_gb;
    fresh.giant_cap = g.giant_cap;
    fresh.half_ksteps = g.half_ksteps;
    fresh.two_sided = g.two_sided;
    fresh.load_x100 = g.load_x100;
    g = fresh;
}

const char *eis_last_error(void) { return g_err.c_str(); }

int eis_set_option(const char *key, int64_t v) {
    if (!key) return fail(EIS_EINVAL, "NULL key");
    std::string k(key);
    if (k == "mode") {
        if (v < 0 || v > 2) return fail(EIS_EINVAL, "mode must be 0..2");
        g.mode = (int)v;
    } else if (k == "crossover") {
        if (v < 0) return fail(EIS_EINVAL, "crossover must be >= 0");
        g.crossover = (u64)v;
    } else if (k == "alpha_x16") {
        if (v != 0 && (v < 4 || v > 64))
            return fail(EIS_EINVAL, "alpha_x16 must be 0 (by d) or in [4, 64]");
        g.alpha_x16 = (int)v;
    } else if (k == "segment_log2") {
        if (v < 18 || v > 31) return fail(EIS_EINVAL, "segment_log2 must be in [18, 31]");
        g.segment_log2 = (int)v;
    } else if (k == "giant_cap") {
        if (v < 0 || v > 1000) return fail(EIS_EINVAL, "giant_cap must be in [0, 1000]");
        g.giant_cap = (int)v;
    } else if (k == "bsgs_gb") {
        if (v < 1 || v > 160) return fail(EIS_EINVAL, "bsgs_gb must be in [1, 160]");
        g.bsgs_gb = (int)v;
    } else if (k == "window_ctas") {
        if (v < 0 || v > 32) return fail(EIS_EINVAL, "window_ctas must be in [0, 32]");
        g.window_ctas = (int)v;
    } else if (k == "giant_ctas") {
        if (v < 0 || v > 32) return fail(EIS_EINVAL, "giant_ctas must be in [0, 32]");
        g.giant_ctas = (int)v;
    } else if (k == "half_ksteps") {
        if (v != 0 && v != 18 && v != 36 && v != 72 && v != 144)
            return fail(EIS_EINVAL, "half_ksteps must be 0 (auto), 18, 36, 72 or 144");
        g.half_ksteps = (int)v;
    } else if (k == "blocks_per_sm") {
        if (v < 1 || v > 32) return fail(EIS_EINVAL, "blocks_per_sm must be in [1, 32]");
        g.blocks_per_sm = (int)v;
    } else if (k == "two_sided") {
        if (v != 0 && v != 1) return fail(EIS_EINVAL, "two_sided must be 0 or 1");
        g.two_sided = (int)v;
    } else if (k == "load_x100") {
        if (v < 30 || v > 90) return fail(EIS_EINVAL, "load_x100 must be in [30, 90]");
        g.load_x100 = (int)v;
    } else {
        return fail(EIS_EINVAL, "unknown option '%s'", key);
    }
    return 0;
}

int64_t eis_get_option(const char *key) {
    if (!key) return fail(EIS_EINVAL, "NULL key");
    std::string k(key);
    if (k == "mode") return g.mode;
    if (k == "crossover") return (int64_t)g.crossover;
    if (k == "alpha_x16") return g.alpha_x16;
    if (k == "segment_log2") return g.segment_log2;
    if (k == "blocks_per_sm") return g.blocks_per_sm;
    if (k == "giant_ctas") return g.giant_ctas;
    if (k == "window_ctas") return g.window_ctas;
    if (k == "bsgs_gb") return g.bsgs_gb;
    if (k == "giant_cap") return g.giant_cap;
    if (k == "half_ksteps") return g.half_ksteps;
    if (k == "two_sided") return g.two_sided;
    if (k == "load_x100") return g.load_x100;
    return fail(EIS_EINVAL, "unknown option '%s'", key);
}

size_t eis_num_candidates(uint64_t lo, uint64_t hi) {
    u64 a, b;
    if (!cand_range(lo, hi, a, b)) return 0;
    return (size_t)(b - a + 1);
}

int eis_classify_range_dev(uint64_t lo, uint64_t hi, uint8_t *out_dev, size_t out_len,
                           void *stream) {
    if (lo > hi) return fail(EIS_EINVAL, "lo > hi");
    if (hi > EIS_MAX_D) return fail(EIS_ERANGE, "hi exceeds EIS_MAX_D");
    size_t n = eis_num_candidates(lo, hi);
    if (n == 0) return 0;
    if (!out_dev) return fail(EIS_EINVAL, "out is NULL");
    if (out_len < n) return fail(EIS_EINVAL, "out_len %zu < %zu candidates", out_len, n);
    if (int rc = do_init(-1)) return rc;
    cudaStream_t s = stream ? (cudaStream_t)stream : 0;
    if (int rc = begin_call(s)) return rc;
    u64 a, b;
    cand_range(lo, hi, a, b);
    if (int rc = run_range(a, b, out_dev, nullptr, nullptr, 0, nullptr, s)) return rc;
    return end_call(s);
}

int eis_classify_range(uint64_t lo, uint64_t hi, uint8_t *out, size_t out_len) {
    if (lo > hi) return fail(EIS_EINVAL, "lo > hi");
    if (hi > EIS_MAX_D) return fail(EIS_ERANGE, "hi exceeds EIS_MAX_D");
    size_t n = eis_num_candidates(lo, hi);
    if (n == 0) return 0;
    if (!out) return fail(EIS_EINVAL, "out is NULL");
    if (out_len < n) return fail(EIS_EINVAL, "out_len %zu < %zu candidates", out_len, n);
    if (int rc = do_init(-1)) return rc;
    cudaStream_t s = g.stream;
    if (int rc = begin_call(s)) return rc;
    u64 a, b;
    cand_range(lo, hi, a, b);
    // Flags of slice k go to device buffer k & 1; its D2H copy (copy stream)
    // overlaps slice k+1's kernels: slice k+1 is queued before the host issues
    // (and, for pageable `out`, waits for) slice k's copy.
    const u64 SEG = 1ull << g.segment_log2;
    const size_t cap = (size_t)std::min<u64>(SEG, n);
    if (g.flags2_cap < cap) {
        CUDA_TRY(cudaDeviceSynchronize());
        for (auto &p : g.d_flags2) { cudaFree(p); p = nullptr; }
        g.flags2_cap = 0;
        for (auto &p : g.d_flags2) CUDA_TRY(cudaMalloc(&p, cap));
        g.flags2_cap = cap;
    }
    u64 prev = ~0ull, prev_e = 0;
    int k = 0;
    auto copy_out = [&](u64 seg, u64 e, int buf) -> int {
        CUDA_TRY(cudaStreamWaitEvent(g.cpy, g.fl_ready[buf], 0));
        CUDA_TRY(cudaMemcpyAsync(out + (seg - a), g.d_flags2[buf], (size_t)(e - seg + 1),
                                 cudaMemcpyDeviceToHost, g.cpy));
        CUDA_TRY(cudaEventRecord(g.fl_free[buf], g.cpy));
        return 0;
    };
    for (u64 seg = a; seg <= b; seg += SEG, k++) {
        const u64 e = std::min(b, seg + SEG - 1);
        const int buf = k & 1;
        if (k >= 2) CUDA_TRY(cudaStreamWaitEvent(s, g.fl_free[buf], 0));   // its last copy is done
        if (int rc = run_range(seg, e, g.d_flags2[buf], nullptr, nullptr, 0, nullptr, s, 2, false))
            return rc;
        CUDA_TRY(cudaEventRecord(g.fl_ready[buf], s));
        if (prev != ~0ull)
            if (int rc = copy_out(prev, prev_e, buf ^ 1)) return rc;
        prev = seg;
        prev_e = e;
    }
    if (int rc = copy_out(prev, prev_e, (k - 1) & 1)) return rc;
    CUDA_TRY(cudaStreamSynchronize(g.cpy));
    if (int rc = finish_range(s)) return rc;
    return end_call(s);
}

int eis_count_buckets_dev(uint64_t lo, uint64_t hi, const uint64_t *x, size_t n,
                          uint64_t *bucket_dev, void *stream) {
    if (int rc = check_x(x, n, 0)) return rc;
    if (n && !bucket_dev) return fail(EIS_EINVAL, "bucket_dev is NULL");
    if (hi > EIS_MAX_D) return fail(EIS_ERANGE, "hi exceeds EIS_MAX_D");
    if (lo > hi) return fail(EIS_EINVAL, "lo > hi");
    if (int rc = do_init(-1)) return rc;
    cudaStream_t s = stream ? (cudaStream_t)stream : 0;
    if (int rc = begin_call(s)) return rc;
    if (int rc = count_buckets(lo, hi, x, n, bucket_dev, s)) return rc;
    return end_call(s);
}

int eis_prefix_dev(const uint64_t *bucket_dev, size_t n, uint64_t *out_dev, void *stream) {
    if (n == 0) return 0;
    if (!bucket_dev || !out_dev) return fail(EIS_EINVAL, "NULL pointer");
    if (int rc = do_init(-1)) return rc;
    cudaStream_t s = stream ? (cudaStream_t)stream : 0;
    prefix_kernel<<<1, 1024, 0, s>>>(bucket_dev, out_dev, (int)n, 2);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int eis_count_window(uint64_t lo, const uint64_t *x, size_t n, uint64_t *cnt_D,
                     uint64_t *cnt_E) {
    if (n == 0) return 0;
    if (!cnt_D || !cnt_E) return fail(EIS_EINVAL, "NULL output");
    std::vector<u64> h(2 * n);
    if (int rc = count_window_rows(lo, x, n, 2, h.data())) return rc;
    std::memcpy(cnt_D, h.data(), n * sizeof(u64));
    std::memcpy(cnt_E, h.data() + n, n * sizeof(u64));
    return 0;
}

int eis_count_window_ext(uint64_t lo, const uint64_t *x, size_t n, uint64_t *out) {
    return count_window_rows(lo, x, n, EIS_NROWS, out);
}

int eis_count(const uint64_t *x, size_t n, uint64_t *pi_D, uint64_t *pi_E) {
    return eis_count_window(0, x, n, pi_D, pi_E);
}

int eis_shard_bounds(uint64_t lo, uint64_t hi, int world, int rank, int balance, uint64_t *a,
                     uint64_t *b) {
    if (!a || !b) return fail(EIS_EINVAL, "NULL output");
    u64 aa = 0, bb = 0;
    if (int rc = shard_bounds(lo, hi, world, rank, balance, aa, bb)) return rc;
    *a = aa;
    *b = bb;
    return 0;
}

int eis_comm_unique_id(void *id) {
    if (!id) return fail(EIS_EINVAL, "NULL id");
    if (int rc = nccl_load()) return rc;
    ncclUniqueId u;
    NCCL_TRY(nccl.get_unique_id(&u));
    std::memcpy(id, &u, sizeof u);
    return 0;
}

int eis_comm_init(const void *id, int world, int rank) {
    if (!id) return fail(EIS_EINVAL, "NULL id");
    if (world < 1 || rank < 0 || rank >= world)
        return fail(EIS_EINVAL, "need 0 <= rank < world (rank %d, world %d)", rank, world);
    if (int rc = do_init(-1)) return rc;
    if (int rc = nccl_load()) return rc;
    comm_release();
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    NCCL_TRY(nccl.comm_init_rank(&g.comm, world, u, rank));
    g.comm_world = world;
    g.comm_rank = rank;
    return 0;
}

void eis_comm_finalize(void) { comm_release(); }

int eis_count_window_comm(uint64_t lo, const uint64_t *x, size_t n, uint64_t *cnt_D,
                          uint64_t *cnt_E) {
    if (!g.comm) return eis_count_window(lo, x, n, cnt_D, cnt_E);
    if (n == 0) return 0;
    if (!cnt_D || !cnt_E) return fail(EIS_EINVAL, "NULL output");
    if (int rc = check_x(x, n, lo)) return rc;
    if (int rc = do_init(-1)) return rc;
    u64 a, b;
    if (int rc = shard_bounds(lo, x[n - 1], g.comm_world, g.comm_rank, EIS_BALANCE_AUTO, a, b))
        return rc;
    cudaStream_t s = g.stream;
    if (int rc = begin_call(s)) return rc;
    if (ensure(g.d_buckets, g.buckets_cap, 2 * n)) return EIS_ENOMEM;
    CUDA_TRY(cudaMemsetAsync(g.d_buckets, 0, 2 * n * sizeof(u64), s));
    if (int rc = count_buckets(a, b, x, n, g.d_buckets, s)) return rc;
    // the path's one exchange step: sum the 2n buckets over all ranks (NVLink)
    NCCL_TRY(nccl.all_reduce(g.d_buckets, g.d_buckets, 2 * n, ncclUint64, ncclSum, g.comm, s));
    prefix_kernel<<<1, 1024, 0, s>>>(g.d_buckets, g.d_buckets, (int)n, 2);
    CUDA_TRY(cudaGetLastError());
    g.launches++;
    std::vector<u64> h(2 * n);
    CUDA_TRY(cudaMemcpyAsync(h.data(), g.d_buckets, 2 * n * sizeof(u64), cudaMemcpyDeviceToHost, s));
    if (int rc = end_call(s)) return rc;
    std::memcpy(cnt_D, h.data(), n * sizeof(u64));
    std::memcpy(cnt_E, h.data() + n, n * sizeof(u64));
    return 0;
}

int eis_get_stats(eis_stats *out) {
    if (!out) return fail(EIS_EINVAL, "NULL out");
    *out = g.last;
    return 0;
}

}  // extern "C"
