// Bulk-copy (cp.async.bulk) completion latency at kernel start, back-to-back
// launches in a CUDA graph (the decode chain's producer pattern): 148 CTAs, one
// thread issues NCOPY copies of SZ bytes (distinct global ranges per CTA and per
// launch replica) into shared memory on one mbarrier per copy; thread 0 stamps
// %globaltimer at kernel start, after issuing, and at each copy's completion.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_latency bulk_latency.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NCOPY>
__global__ void k(const char* src, size_t per_cta, int sz, uint64_t* out, int pdl) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t bar[NCOPY];
    const uint64_t t0 = gt();
    if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int i = 0; i < NCOPY; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const char* s = src + blockIdx.x * per_cta;
        for (int i = 0; i < NCOPY; ++i) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[i])), "r"(sz) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su(sm + (size_t)i * sz)), "l"(s + (size_t)i * sz), "r"(sz), "r"(su(&bar[i])) : "memory");
        }
        const uint64_t t1 = gt();
        uint64_t tc[NCOPY];
        for (int i = 0; i < NCOPY; ++i) {
            asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}"
                         ::"r"(su(&bar[i])) : "memory");
            tc[i] = gt();
        }
        if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
        const uint64_t t2 = gt();
        uint64_t* o = out + blockIdx.x * 8;
        o[0] = t0; o[1] = t1; o[2] = tc[0]; o[3] = tc[NCOPY / 2]; o[4] = tc[NCOPY - 1]; o[5] = t2;
    }
    __syncthreads();
}

int main(int argc, char** argv) {
    const int sz = argc > 1 ? atoi(argv[1]) : 24576;
    const int pdl = argc > 2 ? atoi(argv[2]) : 1;

    constexpr int NC = 4;
    const int G = 148, R = 16;  // 16 replicas of every CTA's range (> L2 when large)
    const size_t per_cta = (size_t)NC * sz;
    char* src; cudaMalloc(&src, per_cta * G * R);
    cudaMemset(src, 1, per_cta * G * R);
    uint64_t* out; cudaMalloc(&out, (size_t)R * G * 8 * 8);
    cudaFuncSetAttribute(k<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    auto launch = [&](int r) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = G; cfg.blockDim = 128; cfg.dynamicSmemBytes = 200 * 1024; cfg.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl; cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k<NC>, (const char*)(src + (size_t)r * per_cta * G), per_cta, sz, out + (size_t)r * G * 8, pdl);
    };
    for (int r = 0; r < R; ++r) launch(r);
    cudaStreamSynchronize(st);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < R; ++r) launch(r);
    cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(e0, st);
    for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<uint64_t> h((size_t)R * G * 8);
    cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    // per launch (replica 8): medians over CTAs relative to the earliest CTA start
    const uint64_t* b = h.data() + (size_t)8 * G * 8;
    uint64_t t0 = ~0ull; for (int c = 0; c < G; ++c) t0 = std::min(t0, b[c * 8]);
    auto med = [&](int j) { std::vector<double> v; for (int c = 0; c < G; ++c) v.push_back((b[c * 8 + j] - t0) / 1e3); std::sort(v.begin(), v.end()); return v[G / 2]; };
    const uint64_t* bn = h.data() + (size_t)9 * G * 8;
    uint64_t t0n = ~0ull; for (int c = 0; c < G; ++c) t0n = std::min(t0n, bn[c * 8]);
    printf("copy %6d B x %d per CTA, pdl %d: %.2f us/launch | start %.2f issued %.2f first %.2f mid %.2f last %.2f done %.2f | next launch start +%.2f | %.0f GB/s\n",
           sz, NC, pdl, ms * 1e3 / 20 / R, med(0), med(1), med(2), med(3), med(4), med(5), (t0n - t0) / 1e3,
           per_cta * G / (ms * 1e-3 / 20 / R) / 1e9);
    return 0;
}
