// umma.cuh -- host interface of the tcgen05 grouped GEMM (umma.cu).
#pragma once

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
};



// All specs run as grouped launches (<= 32 groups per launch), async on st.
void launch_umma(const std::vector<UmmaSpec>& specs, cudaStream_t st);

}  // namespace pg
