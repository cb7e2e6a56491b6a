// pipe_peaks.cu -- measured per-pipe issue peaks of one B200 (sm_100a), the
// denominators of the walk kernels' per-pipe roofline.
//
// For each op, every thread of a full-occupancy grid (148 SMs x 2048 threads)
// runs ILP = 8 independent dependency chains of one PTX instruction whose SASS
// is the pipe's (checked by cuobjdump in tests/test_pipe_peaks.py):
//   IADD3 (add.u32), LOP3 (lop3.b32), ISETP+SEL-free SHF (shf), IMAD (mad.lo.u32),
//   FFMA (fma.rn.f32), FADD (add.f32), DFMA (fma.rn.f64), MUFU.RCP (rcp.approx.f32),
//   MUFU.LG2 (lg2.approx.f32), the conversions (cvt), and a 1:1 IADD3 + FFMA mix.
// The issue ceiling (one warp-instruction per clock per SMSP, 4 per SM) is
// shown by FFMA alone (3.93 measured); the mix stays below it (2.7: a
// dependent IADD3 chain per ILP slot occupies the half-rate ALU pipe).
// Time is taken on the device: per SM, (max end - min start) of its CTAs'
// clock64 (SM cycles) and globaltimer (ns), so ops/clk/SM does not depend on
// the clock and the clock itself is measured (cycles / ns).
// Output: one JSON object on stdout.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int ILP = 8, ITERS = 2048, THREADS = 256, CTAS_PER_SM = 8;

struct Span { unsigned long long c0, c1, t0, t1; unsigned smid; };

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

#define KERNEL(NAME, T, INIT, BODY)                                                        \
    __global__ void __launch_bounds__(THREADS) NAME(T *sink, Span *spans, T seed) {        \
        T v[ILP];                                                                          \
        _Pragma("unroll") for (int i = 0; i < ILP; i++) v[i] = INIT;                       \
        T a = seed, b = seed + (T)1;                                                       \
        __syncthreads();                                                                   \
        unsigned long long c0 = clock64(), t0 = gtimer();                                  \
        for (int it = 0; it < ITERS; it++) {                                               \
            _Pragma("unroll") for (int i = 0; i < ILP; i++) { BODY; }                      \
        }                                                                                  \
        __syncthreads();                                                                   \
        unsigned long long c1 = clock64(), t1 = gtimer();                                  \
        T acc = v[0];                                                                      \
        _Pragma("unroll") for (int i = 1; i < ILP; i++) acc += v[i];                       \
        if (acc == (T)12345) sink[threadIdx.x] = acc;                                      \
        if (threadIdx.x == 0) spans[blockIdx.x] = Span{c0, c1, t0, t1, smid()};            \
    }

// three-input adds (v_i + v_{i^1} + a): ptxas folds plain add chains into IMAD/LEA
KERNEL(k_iadd3, uint32_t, (uint32_t)(threadIdx.x + i),
       asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(v[i]) : "r"(v[i ^ 1]), "r"(a)))
KERNEL(k_lop3, uint32_t, (uint32_t)(threadIdx.x + i),
       asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[i]) : "r"(a), "r"(b)))
KERNEL(k_shf, uint32_t, (uint32_t)(threadIdx.x + i),
       asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(a), "r"(b)))
KERNEL(k_imad, uint32_t, (uint32_t)(threadIdx.x + i),
       asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(a), "r"(b)))
KERNEL(k_ffma, float, (float)(threadIdx.x + i),
       asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(a), "f"(b)))
KERNEL(k_fadd, float, (float)(threadIdx.x + i),
       asm volatile("add.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(a)))
KERNEL(k_dfma, double, (double)(threadIdx.x + i),
       asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(v[i]) : "d"(a), "d"(b)))
// rcp(v + a): one FADD per MUFU (the FMA pipe is 8x wider, so MUFU binds)
KERNEL(k_rcp, float, (float)(threadIdx.x + i + 1),
       asm volatile("{.reg .f32 t; add.f32 t, %0, %1; rcp.approx.ftz.f32 %0, t;}" : "+f"(v[i]) : "f"(a)))
KERNEL(k_lg2, float, (float)(threadIdx.x + i + 2),
       asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(v[i])))
// I2F and F2I alternate on one chain (both conversion ops): 2 ops per body
KERNEL(k_cvt, uint32_t, (uint32_t)(threadIdx.x + i),
       asm volatile("{.reg .f32 f; cvt.rn.f32.u32 f, %0; add.f32 f, f, 0f3F800000; cvt.rzi.u32.f32 %0, f;}"
                    : "+r"(v[i])))
// int <-> double conversions (I2F.F64 / F2I.F64), with one DADD
KERNEL(k_cvt64, uint32_t, (uint32_t)(threadIdx.x + i),
       asm volatile("{.reg .f64 f; cvt.rn.f64.u32 f, %0; add.f64 f, f, 0d3FF0000000000000; cvt.rzi.u32.f64 %0, f;}"
                    : "+r"(v[i])))
// double <-> float conversions (F2F), with one DADD
KERNEL(k_f2f, double, (double)(threadIdx.x + i),
       asm volatile("{.reg .f32 f; cvt.rn.f32.f64 f, %0; cvt.f64.f32 %0, f; add.f64 %0, %0, %1;}"
                    : "+d"(v[i]) : "d"(a)))
// issue limit: one IADD3 (ALU pipe) and one FFMA (FMA pipe) per body, 2 ops
// on two pipes, so only the issue slot (1 warp-instruction/clk/SMSP) binds
__global__ void __launch_bounds__(THREADS) k_mix(float *sink, Span *spans, float seed) {
    float f[ILP];
    uint32_t u[ILP];
#pragma unroll
    for (int i = 0; i < ILP; i++) { f[i] = (float)(threadIdx.x + i); u[i] = threadIdx.x + i; }
    float a = seed, b = seed + 1.f;
    uint32_t ua = (uint32_t)seed;
    __syncthreads();
    unsigned long long c0 = clock64(), t0 = gtimer();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < ILP; i++) {
            asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(a), "f"(b));
            asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}"
                         : "+r"(u[i]) : "r"(u[i ^ 1]), "r"(ua));
        }
    }
    __syncthreads();
    unsigned long long c1 = clock64(), t1 = gtimer();
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < ILP; i++) acc += f[i] + (float)u[i];
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) spans[blockIdx.x] = Span{c0, c1, t0, t1, smid()};
}

template <class T, class K>
void run(const char *name, const char *pipe, K kern, int ops_per_body, int nsm, bool last) {
    const int nblk = nsm * CTAS_PER_SM;
    T *sink;
    Span *dsp;
    cudaMalloc(&sink, THREADS * sizeof(T));
    cudaMalloc(&dsp, nblk * sizeof(Span));
    std::vector<Span> sp(nblk);
    double best_opc = 0, best_clk = 0;
    for (int rep = 0; rep < 5; rep++) {
        kern<<<nblk, THREADS>>>(sink, dsp, (T)3);
        cudaDeviceSynchronize();
        cudaMemcpy(sp.data(), dsp, nblk * sizeof(Span), cudaMemcpyDeviceToHost);
        // per SM: ops over its CTAs' union span
        std::vector<unsigned long long> c0(nsm, ~0ull), c1(nsm, 0), t0(nsm, ~0ull), t1(nsm, 0);
        std::vector<int> cnt(nsm, 0);
        for (auto &s : sp) {
            if (s.smid >= (unsigned)nsm) continue;
            c0[s.smid] = std::min(c0[s.smid], s.c0);
            c1[s.smid] = std::max(c1[s.smid], s.c1);
            t0[s.smid] = std::min(t0[s.smid], s.t0);
            t1[s.smid] = std::max(t1[s.smid], s.t1);
            cnt[s.smid]++;
        }
        double opc = 0, clk = 0;
        int used = 0;
        for (int m = 0; m < nsm; m++) {
            if (!cnt[m]) continue;
            const double ops = (double)cnt[m] * THREADS * ITERS * ILP * ops_per_body;
            opc += ops / (double)(c1[m] - c0[m]);
            clk += (double)(c1[m] - c0[m]) / (double)(t1[m] - t0[m]) * 1e3;   // MHz
            used++;
        }
        opc /= used;   // mean over SMs of thread-ops per SM cycle
        clk /= used;
        if (opc > best_opc) { best_opc = opc; best_clk = clk; }
    }
    printf("    \"%s\": {\"pipe\": \"%s\", \"thread_ops_per_clk_per_sm\": %.2f, "
           "\"warp_inst_per_clk_per_sm\": %.3f, \"sm_mhz_measured\": %.0f, "
           "\"chip_tops_at_measured_clock\": %.3f, \"chip_tops_at_1965mhz\": %.3f}%s\n",
           name, pipe, best_opc, best_opc / 32, best_clk, best_opc * nsm * best_clk * 1e6 / 1e12,
           best_opc * nsm * 1965e6 / 1e12, last ? "" : ",");
    cudaFree(sink);
    cudaFree(dsp);
}

int main() {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) { fprintf(stderr, "no device\n"); return 1; }
    const int nsm = p.multiProcessorCount;
    printf("{\n  \"gpu\": \"%s\", \"sm_count\": %d, \"threads_per_sm\": %d, \"ilp\": %d,\n",
           p.name, nsm, THREADS * CTAS_PER_SM, ILP);
    printf("  \"method\": \"per SM: thread-ops / (max clock64 end - min clock64 start) over its CTAs, best of 5; clock = cycles / globaltimer ns\",\n");
    printf("  \"ops\": {\n");
    run<uint32_t>("IADD3", "alu", k_iadd3, 1, nsm, false);
    run<uint32_t>("LOP3", "alu", k_lop3, 1, nsm, false);
    run<uint32_t>("SHF", "alu", k_shf, 1, nsm, false);
    run<uint32_t>("IMAD", "fma(imad)", k_imad, 1, nsm, false);
    run<float>("FFMA", "fma", k_ffma, 1, nsm, false);
    run<float>("FADD", "fma", k_fadd, 1, nsm, false);
    run<double>("DFMA", "fp64", k_dfma, 1, nsm, false);
    run<float>("MUFU.RCP", "xu", k_rcp, 1, nsm, false);
    run<float>("MUFU.LG2", "xu", k_lg2, 1, nsm, false);
    run<uint32_t>("I2FP+F2I", "cvt f32", k_cvt, 2, nsm, false);
    run<uint32_t>("I2F.F64+F2I.F64", "cvt f64", k_cvt64, 2, nsm, false);
    run<double>("F2F.F32.F64+F2F.F64.F32", "cvt f2f", k_f2f, 2, nsm, false);
    run<float>("IADD3+FFMA", "alu+fma mix", k_mix, 2, nsm, true);
    printf("  }\n}\n");
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
