// umma.cuh -- host interface of the tcgen05 grouped GEMM (umma.cu).
#pragma once

#include <cuda.h>

#include <vector>

#include "pg_common.cuh"

namespace pg {

// One GEMM C[M, N] = A[M, K] . B[N, K]^T, bf16 operands (both K-major, rows
// 16-byte aligned), f32 accumulation, bf16 or f32 output.
struct UmmaSpec {
    const void* a;
    long long lda;
    const void* b;
    long long ldb;
    void* out;
    long long ldo;
    int M, N, K;
    int out_bf16;
    // optional per-row column mask applied in the epilogue (union-masked
    // heterogeneous batches): C[i, j] = 0 unless mask[row_pat[i] * mask_ld + j]
    const uint8_t* mask = nullptr;
    long long mask_ld = 0;
    const int32_t* row_pat = nullptr;
    int b_rows = 0;  // rows of the B operand in memory (0: N); rows in [b_rows, N) read as zero
    int bn = 0;      // tile width override (0: chosen by launch_umma)
    int a_hint = 0, b_hint = 0;  // L2 policy of the operand loads: 0 default, 1 evict-first, 2 evict-last
    int direct_epi = 0;  // CTA-pair kernel: store from registers instead of the TMA-store epilogue
    // optional gathered B rows (CTA-pair kernel): row j of the B operand is row
    // b_idx[j] of `b` for j < b_idx_n, zero for j >= b_idx_n (TMA gather4 straight
    // from the unpacked arena; b_idx_rows = rows of `b` in memory)
    const int32_t* b_idx = nullptr;
    int b_idx_n = 0, b_idx_rows = 0;
};

// C = A . B^T with K split across CTAs when the M x N tiles cannot cover the
// SMs without re-reading the A operand once per narrow N tile (small-batch
// GEMMs with long K): S K-slices run as one grouped launch into f32 partials
// (register-store epilogue: the tiles are short), then one kernel sums them in
// slice order (deterministic), applies the row mask and converts.  Returns
// false (and launches nothing) when splitting does not pay; workspace bytes
// from umma_splitk_bytes.
size_t umma_splitk_bytes(const UmmaSpec& s);
bool launch_umma_splitk(const UmmaSpec& s, void* workspace, cudaStream_t st);
bool launch_umma_splitk_multi(const std::vector<UmmaSpec>& specs, void* workspace, cudaStream_t st);



// 2-D bf16 K-major TMA operand map [rows, K] (row stride ld elements), box
// {64, box_rows}, 128-byte swizzle (the UMMA K-major SW128 layout).
CUtensorMap make_map(const void* ptr, int rows, int K, long long ld, int box_rows);
// 2-D output map [rows, cols] (row stride ld elements), box {box_cols, box_rows},
// no swizzle: TMA-store epilogues (rows / columns past the bounds are clipped).
CUtensorMap make_store_map(void* ptr, int rows, int cols, long long ld, bool bf16, int box_cols, int box_rows);

// All specs run as grouped launches (<= 32 groups per launch), async on st.
void launch_umma(const std::vector<UmmaSpec>& specs, cudaStream_t st);

}  // namespace pg
