// chain.cuh -- parameter block of the single-launch decode chain (decode.cu).
#pragma once

#include "pg_common.cuh"

namespace pg {

constexpr int kChainThreads = 384;
constexpr int kChainWarps = kChainThreads / 32;
constexpr int kConsumerWarps = kChainWarps - 1;  // warp 15 is the TMA producer
constexpr int kMaxLin = 3;
constexpr int kMaxPhase = 16;  // 2 per MLP block: up to 8 chained blocks per launch
constexpr int kLinSBytes = 128;  // shared-memory table entry per (phase, linear)
constexpr int kRingStages = 8;
constexpr int kMaxChunkItems = 16;
constexpr int kMaxPeers = 8;

struct ChainLin {
    const void* bt;  // B^T arena [.., ldb] (storage dtype)
    int64_t ldb;
    const void* a;   // A arena [m, lda]
    int64_t lda;
    SlotMap sm;      // runs + activity mask (no gather lists), resolved on device
    int cap;         // slots upper bound
    int n, m;
    void* zpart;     // [cap * (f64 ? 2 : 1)] tagged z words (cross-CTA exchange)
    void* y;         // output (epilogue 0)
};

struct ChainPhase {
    int nlin;
    ChainLin lin[kMaxLin];
    const void* x;  // [n] phase input (storage dtype): the block input, the block's act, or the previous block's y
    int epilogue;   // 0: y_l per linear (ydt); 1: act = silu(y_1) * y_0 -> act (storage dtype)
    int ydt;
    void* act;
};

struct ChainParams {
    int nphase;
    int tab_bytes;  // shared-memory tables: nphase * kMaxLin * kLinSBytes (>= 1024)
    ChainPhase ph[kMaxPhase];
    unsigned long long* bar;    // grid-barrier counter (act hand-over between MLP phases)
    unsigned long long* epoch;  // launch counter (each CTA adds 1 per launch): z-word tags
    int ztag;                   // 1: z exchanged as tagged words (MLP); 0: plain z + grid barrier
    int xs_bytes;             // shared-memory x region (max over phases)
    int zs_bytes;             // shared-memory z region (max over phases)
    int chunk_bytes;          // ring stage size
    int max_stages;           // ring depth cap (<= kRingStages)
    unsigned long long* dbg;  // optional per-CTA %globaltimer stamps [grid][16]
    // expert-sharded peer reduction (single linear, single phase): the stage-2
    // epilogue pushes each row's partial as a tagged word into every rank's
    // receive buffer (peer memory over NVLink; [2 parity][npeer][m] words), then
    // each CTA sums its own rows over the ranks in rank order -- compute and
    // all-reduce in one kernel, no fence (the tag is in the data word)
    int throttle;  // >= 0: after a stage-1 segment, at most this many chunks until the z exchange is done
    int l2hint;    // 1: weight copies carry an L2 evict-first policy
    int npeer, prank;
    int peer_words;     // receive-buffer words per (parity, rank): m, or 2 m_ff + d for an MLP block
    int peer_last_off;  // offset of the last phase's words (0, or 2 m_ff: up and gate come first)
    unsigned long long* peer_recv[kMaxPeers];
};

void launch_chain(pg_dtype wdt, const ChainParams& P, size_t smem, cudaStream_t st, int grid = 0);
int chain_grid();

}  // namespace pg
