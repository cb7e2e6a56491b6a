// walk_bsgs.cuh -- K3 in BSGS mode (placeholder until the giant-step kernels land).
#pragma once
#include "common.cuh"

struct BsgsScratch {
    void *p = nullptr;
};

inline void bsgs_free(BsgsScratch &s) {
    if (s.p) cudaFree(s.p);
    s.p = nullptr;
}

inline int launch_bsgs(const WalkArgs &, u64, u64, int, int, BsgsScratch &, u32 *, cudaStream_t,
                       int *) {
    return -4;   // EIS_EDEVICE: not built yet
}
