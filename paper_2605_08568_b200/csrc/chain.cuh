// chain.cuh -- parameter block of the single-launch decode chain (decode.cu).
#pragma once

#include "pg_common.cuh"

namespace pg {

constexpr int kChainThreads = 512;
constexpr int kChainWarps = kChainThreads / 32;
constexpr int kMaxLin = 3;
constexpr int kMaxPhase = 2;

struct ChainLin {
    const void* bt;
    int64_t ldb;
    const void* a;
    int64_t lda;
    SlotMap sm;
    int cap;      // slots upper bound (smem / partial sizing)
    int n, m;
    void* zpart;  // [cap * split] accumulator partials
    void* y;      // output (epilogue 0)
};

struct ChainPhase {
    int nlin;
    ChainLin lin[kMaxLin];
    const void* x;  // [n] input shared by the phase's linears (W dtype)
    int epilogue;   // 0: y_l per linear (ydt); 1: act = silu(y_1) * y_0 -> act (W dtype)
    int ydt;
    void* act;
    int split;      // warps per slot row in stage 1
};

struct ChainParams {
    int nphase;
    ChainPhase ph[kMaxPhase];
    unsigned long long* bar;
    int prefetch;
};

void launch_chain(pg_dtype wdt, const ChainParams& P, size_t smem, cudaStream_t st);
int chain_grid();
int chain_split(int total_slots);

}  // namespace pg
