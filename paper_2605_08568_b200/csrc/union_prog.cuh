// union_prog.cuh -- host interface of the persistent union program
// (union_prog.cu): a sequence of weights-on-M union GEMM phases (WmSpec, as
// union_wm.cuh) executed as ONE launch, phases chained by per-tile ready
// counters instead of kernel boundaries.
#pragma once

#include <memory>
#include <vector>

#include "union_wm.cuh"

namespace pg {

class UnionProgram {
   public:
    explicit UnionProgram(int T);  // T <= 256 tokens per launch
    ~UnionProgram();
    // Append a phase (<= 4 GEMMs sharing nothing but the launch).  A GEMM whose
    // X is exactly an earlier phase's output (same base and stride) waits for
    // that output tile by tile; any other X is an external input, ready at
    // launch.  Buffers are written once per program and never after being read.
    void add_phase(const std::vector<WmSpec>& specs);
    // Allocates the workspace on first use (not capturable); then one launch.
    void run(const int32_t* tok_pat, cudaStream_t st);
    int phases() const;
    int grid() const;
    int debug_dump(unsigned long long* out, size_t n) const;  // PG_PROG_DBG=1: [grid][16] stamps

   private:
    void finalize(cudaStream_t st);
    struct Impl;
    std::unique_ptr<Impl> d;
};

}  // namespace pg
