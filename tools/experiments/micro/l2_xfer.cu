// L2 exchange microbenchmark (the union program's split-tile tail pattern):
// every CTA writes 128 KB of f32 partials, then reads 128 KB written by other
// CTAs.  Prints per-kernel device time and the aggregate rate.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_xfer l2_xfer.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kBytes = 128 * 1024;
constexpr int kF4 = kBytes / 16;

__global__ void __launch_bounds__(128) k_write(float4* buf, int reps) {
    float4* dst = buf + (size_t)blockIdx.x * kF4;
    for (int r = 0; r < reps; ++r) {
        const float4 v = make_float4(threadIdx.x, r, 2.f, 3.f);
#pragma unroll 8
        for (int i = threadIdx.x; i < kF4; i += blockDim.x) __stcg(dst + i, v);
    }
}

template <int U>
__global__ void __launch_bounds__(1024) k_read(const float4* buf, float* out, int shift, int reps) {
    // read the slab of CTA (blockIdx + shift) mod grid: another SM's partial
    const int src = (blockIdx.x + shift) % gridDim.x;
    const float4* s = buf + (size_t)src * kF4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < kF4; i += blockDim.x * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = (i + u * blockDim.x < kF4) ? __ldcg(s + i + u * blockDim.x) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    if (acc.x == -1.f) out[0] = acc.y + acc.z + acc.w;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 20 * 1e3f;  // us
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float4* buf;
    float* out;
    cudaMalloc(&buf, (size_t)sms * kBytes);
    cudaMalloc(&out, 16);
    const double tot = (double)sms * kBytes;
    const int reps = 20;
    float us = timeit([&] { k_write<<<sms, 128>>>(buf, reps); });
    printf("write 128 thr: %7.2f us  %6.2f TB/s\n", us, reps * tot / us / 1e6);
    for (int thr : {128, 256, 512, 1024}) {
        float u1 = timeit([&] { k_read<1><<<sms, thr>>>(buf, out, 1, reps); });
        float u2 = timeit([&] { k_read<2><<<sms, thr>>>(buf, out, 1, reps); });
        float u4 = timeit([&] { k_read<4><<<sms, thr>>>(buf, out, 1, reps); });
        printf("read %4d thr: U1 %6.2f TB/s | U2 %6.2f | U4 %6.2f\n", thr, reps * tot / u1 / 1e6, reps * tot / u2 / 1e6,
               reps * tot / u4 / 1e6);
    }
    // the same bytes from HBM (slabs far larger than L2): 8 MB per CTA
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
