// union_wm.cuh -- host interface of the weights-on-M stream-K union GEMM
// (union_wm.cu), the config-4 heterogeneous decode batch path.
#pragma once

#include <vector>

#include "pg_common.cuh"

namespace pg {

// One GEMM of a launch: out[t, i] = sum_k W[i, k] x[t, k] for t < T, i < R
// (bf16 operands, K-major, f32 accumulation), stored token-major into out
// [T, ldo] as bf16 or f32; with `mask`, out[t, i] = 0 unless
// mask[tok_pat[t] * mask_ld + i] != 0 (the stage-1 selection mask).
struct WmSpec {
    const void* w;      // [R, ldw] weights (B^T for stage 1, A for stage 2)
    long long ldw;
    int R, K;
    const void* x;      // [T, ldx] tokens (x for stage 1, Z for stage 2)
    long long ldx;
    void* out;
    long long ldo;
    int out_bf16;
    const uint8_t* mask = nullptr;
    long long mask_ld = 0;
    int tok_off = 0;   // union program: this GEMM's token 0 is token tok_off of the launch's pattern table
    int w_hint = 1;    // union program: L2 policy of the weight loads (1 evict-first, 0 evict-normal)
};

bool union_wm_enabled();                                 // PG_UNION_WM (default 1)
bool union_wm_ok(int T, const std::vector<WmSpec>& specs);  // T <= 256, <= 4 GEMMs, alignment
// All specs as one launch (one persistent CTA pair per TPC, stream-K split),
// async on st; a per-(stream, grid) workspace holds the split tiles' partials.
void launch_union_wm(const std::vector<WmSpec>& specs, int T, const int32_t* tok_pat, cudaStream_t st);
void union_wm_release(cudaStream_t st);
int union_wm_debug_dump(unsigned long long* out, size_t n);  // PG_WM_DBG=1: [grid][8] stamps

}  // namespace pg
