/*
 * eis.h -- C ABI of the B200 Eisenstein-discriminant classifier.
 *
 * Breuer & Punch, "Quadratic units and cubic fields", arXiv 2507.06579.
 * Citations are /root/reference/PAPER.md line numbers (the paper's LaTeX).
 *
 * The problem (Sec. 1):
 *   D = { d > 0 : d = 5 (mod 8), d squarefree },
 *   E = { d in D : eps_d = 1 (mod 2 O_K) },  eps_d the fundamental unit of Q(sqrt d),
 *   pi_D(x) = #{d in D : d <= x},  pi_E(x) = #{d in E : d <= x}.
 * The paper computes pi_E(x) for x <= 1e11 with the
 * residue-tracking infrastructure method of its Appendix (PAPER.md
 * l.535-756): the generator of each reduced principal ideal is carried only
 * as its class in (O_K/2O_K)^* = F_4^* = Z/3 (l.601-603), with continued-
 * fraction baby steps rho (l.541), and NUCOMP/NUDUPL giant steps (l.617-756).
 *
 * Residue labelling (one fixed choice, reading R30): an element
 * a*1 + b*w of O_K, w = (1+sqrt d)/2, with (a mod 2, b mod 2) = (1,0), (0,1),
 * (1,1) has residue t = 0, 1, 2.  d in E  <=>  t(eps_d) = 0.
 *
 * Conventions for every entry point:
 *  - Return 0 (EIS_OK) on success or a negative EIS_E* code; no exception or
 *    abort crosses the ABI.  eis_last_error() then describes the failure.
 *  - Candidates are the integers d = 5 (mod 8); candidate index i <-> d = 8i+5.
 *  - Host pointers are owned by the caller and only read/written during the
 *    call (the call is synchronous).  Device pointers (the *_dev variants) are
 *    owned by the caller, must be device memory on the library's current
 *    device, and are written by kernels on `stream` (a cudaStream_t passed as
 *    void*; NULL = the legacy default stream).  eis_count_buckets_dev and
 *    eis_classify_range_dev return only after their kernels have finished
 *    (they read back an invariant-violation counter); eis_prefix_dev is
 *    asynchronous (the caller synchronises).
 *  - The library owns its device scratch (prime table, survivor lists,
 *    counters) until eis_finalize().
 *  - Calls are NOT reentrant and not thread-safe: serialise them per process.
 *  - Every computation runs in the library's CUDA kernels for sm_100a; there
 *    is no CPU fallback.  Without a usable device every compute call fails
 *    with EIS_EDEVICE.
 */
#ifndef EIS_H
#define EIS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define EIS_API __attribute__((visibility("default")))
#else
#define EIS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Largest d accepted.  The 32-bit baby-step and float-quotient bounds
 * (sqrt d < 2^19, Q < 2 sqrt d < 2^20) and the int64 giant-step bounds were
 * validated up to here ("at least for d <= 10^11"). */
#define EIS_MAX_D 100000000000ULL

/* flag value of a candidate d = 5 (mod 8) that is not squarefree (d not in D) */
#define EIS_NOT_IN_D 0xFF

enum {
    EIS_OK = 0,
    EIS_EINVAL = -1,     /* bad argument: lo > hi, unsorted x, short buffer, NULL */
    EIS_ERANGE = -2,     /* d > EIS_MAX_D requested */
    EIS_ENOMEM = -3,     /* device allocation failed */
    EIS_EDEVICE = -4,    /* no CUDA device / CUDA error / kernel fault */
    EIS_EINTERNAL = -5   /* an in-kernel invariant failed (a bug; never expected) */
};

/* Walk modes (eis_set_option("mode", m)).
 *  EIS_MODE_HALF: baby steps rho from (1) with the symmetry
 *    exit of Algorithm 1 (l.553-556) and no giant steps: half a period.
 *  EIS_MODE_BSGS: the paper's Algorithm 1 (l.543-574) with NUCOMPchoose
 *    giant steps (l.733-756), residues in Z/3 (l.585-603).
 *  EIS_MODE_AUTO: HALF for d below the crossover (option "crossover"), else BSGS.
 * All modes return identical results (tests/test_gpu_parity.py). */
enum { EIS_MODE_AUTO = 0, EIS_MODE_HALF = 1, EIS_MODE_BSGS = 2 };

/* Select the CUDA device this process uses (device < 0: keep the current
 * one) and build the prime table.  Idempotent; called implicitly by the
 * compute entry points.  Returns EIS_EDEVICE if no device is usable. */
EIS_API int eis_init(int device);

/* Release all library-owned device memory and streams. */
EIS_API void eis_finalize(void);

/* Human-readable description of the last failure in this process; owned by
 * the library, valid until the next call. */
EIS_API const char *eis_last_error(void);

/* Tunables; unknown key or bad value -> EIS_EINVAL.  None changes a result.
 *  "mode"          EIS_MODE_* (default AUTO)
 *  "crossover"     AUTO: HALF for segments starting below this d, else BSGS
 *  "alpha_x16"     BSGS baby window W = (alpha_x16/16) d^(1/4), in [4, 64]; 0 (default) =
 *                  chosen per segment from d (measured optimum)
 *  "segment_log2"  candidates per segment (HALF; BSGS caps it by store memory)
 *  "blocks_per_sm" HALF walk kernel CTAs per SM
 *  "giant_ctas"    BSGS giant kernel CTAs per SM (0 = occupancy maximum)
 *  "window_ctas"   BSGS window kernel CTAs per SM (0 = occupancy maximum)
 *  "bsgs_gb"       BSGS store memory per segment buffer in GiB, [1, 160], default 48: two
 *                  buffers; a range whose stores fit in 2 bsgs_gb GiB runs as one segment
 *  "giant_cap"     BSGS giant steps per d before the exact half walk takes over:
 *                  giant_cap * (d^(1/4) + 10), in [0, 1000] (default 20; 0 sends
 *                  every d past k = 2 to the half walk, a test of that path)
 *  "half_ksteps"   HALF walk: rho steps per lane between refills (0 = auto, 18/36/72/144)
 *  "two_sided"     BSGS: 1 (default) = the store is also matched against conjugates and
 *                  the giant stride is mu_1^2 (R35); 0 = the paper's one-sided
 *                  Algorithm 1
 *  "load_x100"     BSGS store table load factor x 100, in [30, 90] (default 62, the
 *                  measured optimum); results never depend on it (tests raise it to
 *                  force overflow chains) */
EIS_API int eis_set_option(const char *key, int64_t value);
EIS_API int64_t eis_get_option(const char *key);

/* Number of candidates d = 5 (mod 8) with lo <= d <= hi (0 if lo > hi). */
EIS_API size_t eis_num_candidates(uint64_t lo, uint64_t hi);

/* Per-d classification.  Slices of 2^segment_log2
 * candidates are classified in turn; each slice's device-to-host copy overlaps
 * the next slice's kernels (two device buffers, a copy stream).
 * out[i] describes d_i = first + 8 i, first = least d >= lo with d = 5 mod 8,
 * for every d_i <= hi: out[i] = t(eps_{d_i}) in {0,1,2} (d_i in E iff 0),
 * or EIS_NOT_IN_D if d_i is not squarefree.
 * out_len must be >= eis_num_candidates(lo, hi) (EIS_EINVAL otherwise);
 * hi > EIS_MAX_D -> EIS_ERANGE; lo > hi -> EIS_EINVAL.  out may be NULL only
 * if the range holds no candidate. */
EIS_API int eis_classify_range(uint64_t lo, uint64_t hi, uint8_t *out, size_t out_len);

/* Counting functions at checkpoints.
 * x[0..n-1] strictly ascending, 0 < x[0], x[n-1] <= EIS_MAX_D.
 * pi_D[i] = #{d in D : d <= x[i]},  pi_E[i] = #{d in E : d <= x[i]}.
 * Equivalent to eis_count_window(0, x, n, pi_D, pi_E).  n == 0 is a no-op. */
EIS_API int eis_count(const uint64_t *x, size_t n, uint64_t *pi_D, uint64_t *pi_E);

/* Window form (Table 1's windows; the d ~ 1e10 metric):
 * lo < x[0] < ... < x[n-1] <= EIS_MAX_D,
 * cnt_D[i] = #{d in D : lo < d <= x[i]},  cnt_E[i] likewise for E. */
EIS_API int eis_count_window(uint64_t lo, const uint64_t *x, size_t n, uint64_t *cnt_D,
                     uint64_t *cnt_E);

/* Extended counts: the prime subsequence (Sec. 3.2, l.501-522) and
 * the residue classes.  out is a row-major [EIS_NROWS][n] host array:
 *   out[0*n+i] = #{d in D : lo < d <= x[i]}
 *   out[1*n+i] = #{d in E : ...}                      (t(eps_d) = 0)
 *   out[2*n+i] = #{d in D with t(eps_d) = 1 : ...}    (t = 2 is row 0 - row 1 - row 2)
 *   out[3*n+i] = #{d in D, d prime : ...}             (pi_{D cap P})
 *   out[4*n+i] = #{d in E, d prime : ...}             (pi_{E cap P}, l.503-507)
 * Same argument rules as eis_count_window; primality is decided by the
 * sieve kernel (every odd prime p <= sqrt(x[n-1])). */
#define EIS_NROWS 5
EIS_API int eis_count_window_ext(uint64_t lo, const uint64_t *x, size_t n, uint64_t *out);

/* ---- device-resident variants (multi-GPU path: one process per GPU) ---- */

/* Accumulate per-bucket counts of d in (lo, hi] into bucket_dev[0..2n-1]:
 * bucket_dev[b] += #{d in D, lo < d <= hi, bucket(d) = b} and
 * bucket_dev[n+b] += the same for E, where bucket(d) = least b with
 * d <= x[b].  d > x[n-1] are not counted.  x: n uint64 checkpoints in HOST
 * memory, strictly ascending, x[n-1] <= EIS_MAX_D (the library copies them;
 * the host needs them to cut segments).  bucket_dev (device memory, 2n
 * uint64) is NOT zeroed.  Kernels run on `stream`; the call returns after
 * they finish (it reads back an invariant-violation counter per segment).
 * Buckets of disjoint (lo, hi] shards sum (e.g. by an NCCL allreduce) to the
 * buckets of their union. */
EIS_API int eis_count_buckets_dev(uint64_t lo, uint64_t hi, const uint64_t *x, size_t n,
                                  uint64_t *bucket_dev, void *stream);

/* Inclusive prefix sums of 2 arrays of n buckets: out_dev[k] =
 * sum_{b<=k} bucket_dev[b], out_dev[n+k] = sum_{b<=k} bucket_dev[n+b].
 * Async on `stream`; out_dev may equal bucket_dev. */
EIS_API int eis_prefix_dev(const uint64_t *bucket_dev, size_t n, uint64_t *out_dev, void *stream);

/* eis_classify_range into device memory out_dev (out_len bytes), on `stream`;
 * returns after the kernels finished (host-blocking, like eis_count_buckets_dev). */
EIS_API int eis_classify_range_dev(uint64_t lo, uint64_t hi, uint8_t *out_dev, size_t out_len,
                           void *stream);

/* ---- the whole box: one process per GPU ----
 *
 * Every d is independent, so the range is cut into contiguous shards, one per
 * process/GPU, and the only exchange is ONE sum-all-reduce of the 2n
 * checkpoint buckets (NCCL over NVLink/NVSwitch), followed by the prefix
 * kernel.  Two ways to run it:
 *  (a) inside the library: rank 0 calls eis_comm_unique_id, the caller
 *      broadcasts the EIS_COMM_ID_BYTES bytes by any means (a file, MPI,
 *      torch.distributed), every rank calls eis_init(its device) and
 *      eis_comm_init(id, world, rank), then eis_count_window_comm with the
 *      same arguments on every rank; each rank receives the whole result.
 *      NCCL is loaded at eis_comm_init (dlopen "libnccl.so.2", or the path in
 *      the environment variable EIS_NCCL_LIB); the library does not link it.
 *  (b) with the caller's own collective: per rank, eis_shard_bounds ->
 *      eis_count_buckets_dev over its shard into zeroed device buckets ->
 *      all-reduce(sum, uint64, 2n) on the same stream -> eis_prefix_dev ->
 *      copy out.  (paper_2507_06579_b200/dist.py does this with
 *      torch.distributed; examples/count_box.c does (a) from C.)
 * Per-d flags need no collective: rank r classifies its own slice
 * (eis_shard_bounds of (lo - 1, hi], then eis_classify_range(a + 1, b)); the
 * slices of all ranks, concatenated in rank order, are eis_classify_range(lo, hi).
 * Results never depend on the number of ranks or on the split. */
enum { EIS_BALANCE_FLAT = 0, EIS_BALANCE_PREFIX = 1, EIS_BALANCE_AUTO = 2 };

/* Contiguous shard (*a, *b] of (lo, hi] for `rank` of `world`:
 *  FLAT   equal widths (windows, where the cost per d is flat);
 *  PREFIX equal cost under a d^(1/4) cost model: cut points lo + (hi-lo)(g/G)^(4/5);
 *  AUTO   equal cost under the measured cost model of EIS_MODE_AUTO (HALF ~ d^(1/2)
 *         below option "crossover", BSGS ~ d^0.224 above), integrated numerically.
 * Interior cut points are multiples of 8 (never a candidate), so no candidate
 * is split; the shards of ranks 0..world-1 are disjoint and cover (lo, hi].
 * Host-only (no device needed).  Bad world/rank/balance, lo > hi -> EIS_EINVAL. */
EIS_API int eis_shard_bounds(uint64_t lo, uint64_t hi, int world, int rank, int balance,
                             uint64_t *a, uint64_t *b);

#define EIS_COMM_ID_BYTES 128
/* Write a new NCCL unique id (EIS_COMM_ID_BYTES bytes, caller-owned) into id.
 * Called by rank 0 only.  EIS_EDEVICE if NCCL cannot be loaded. */
EIS_API int eis_comm_unique_id(void *id);
/* Join the world-rank communicator named by id as `rank` on this process's
 * device (eis_init's).  Collective: every rank must call it.  Replaces any
 * previous communicator.  EIS_EINVAL on bad rank/world, EIS_EDEVICE on NCCL
 * failure. */
EIS_API int eis_comm_init(const void *id, int world, int rank);
/* Destroy the communicator (also done by eis_finalize). */
EIS_API void eis_comm_finalize(void);
/* eis_count_window over the whole communicator: same arguments on every rank;
 * rank r walks its EIS_BALANCE_AUTO shard of (lo, x[n-1]], the buckets are
 * summed by ncclAllReduce on the library's stream, and every rank receives
 * the full cnt_D, cnt_E.  Collective.  Without a communicator it is
 * eis_count_window. */
EIS_API int eis_count_window_comm(uint64_t lo, const uint64_t *x, size_t n, uint64_t *cnt_D,
                                  uint64_t *cnt_E);

/* ---- instrumentation ---- */
typedef struct {
    uint64_t d_classified;   /* d in D walked by the last compute call */
    uint64_t baby_steps;     /* rho steps, all modes */
    uint64_t giant_steps;    /* NUCOMPchoose calls (BSGS) */
    uint64_t reduce_steps;   /* rho steps reducing giant-step results */
    uint64_t sym_exits;      /* d finished by the symmetry exit */
    uint64_t fallbacks;      /* d re-walked by the half-walk after a BSGS bail-out */
    uint64_t kernel_launches;/* kernels launched by the last call */
    double walk_ms;          /* device time of the segment loop: sieve + walk kernels (CUDA events) */
    double total_ms;         /* device time of the whole call */
    double sieve_ms;         /* summed device time of the sieve kernels (events on their stream) */
    double window_ms;        /* ... of the HALF walk kernels, or of the BSGS window + prep kernels */
    double giant_ms;         /* ... of the BSGS giant kernels (aux stream; overlaps the others) */
    uint64_t windowed;       /* d whose BSGS window (list + hash table) was stored */
    uint64_t window_nw;      /* window entries per d of the last BSGS segment (0: none) */
    uint64_t window_nb;      /* table buckets (64 bytes each) per d of the last BSGS segment */
} eis_stats;

/* Counters of the most recent compute call (a copy of host-side values the
 * call recorded when it finished; no device work). */
EIS_API int eis_get_stats(eis_stats *out);

#ifdef __cplusplus
}
#endif
#endif /* EIS_H */
