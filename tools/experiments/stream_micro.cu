// read_micro.cu -- achievable HBM read bandwidth by load flavour / access shape
#include <cuda_bf16.h>
#include <cstdio>

template <int MODE>
__device__ __forceinline__ int4 ld(const int4* p) {
    int4 r;
    if (MODE == 0) r = *p;
    else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (MODE == 3) asm volatile("ld.global.cs.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else asm volatile("ld.global.L1::no_allocate.L2::128B.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int MODE, int U>
__global__ void rd(const int4* __restrict__ a, size_t n, int* out) {
    int acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld<MODE>(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n; i += stride) { int4 v = ld<MODE>(a + i); acc ^= v.x ^ v.w; }
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    const size_t bytes = 108273664;  // one MLP decode step
    const int R = 4;
    char* A; int* o;
    cudaMalloc(&A, bytes * R); cudaMalloc(&o, 4);
    cudaMemset(A, 1, bytes * R);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto k, int grid, int block) {
        const size_t n = bytes / 16;
        for (int i = 0; i < 10; ++i) k<<<grid, block>>>((const int4*)(A + (i % R) * bytes), n, o);
        cudaEventRecord(e0);
        for (int i = 0; i < 100; ++i) k<<<grid, block>>>((const int4*)(A + (i % R) * bytes), n, o);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double us = ms * 10;
        printf("%-34s grid %5d x %4d: %7.2f us %6.0f GB/s %s\n", name, grid, block, us, bytes / us / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("plain U4", rd<0, 4>, 148 * 4, 512);
    run("nc.noalloc U4", rd<1, 4>, 148 * 4, 512);
    run("nc.noalloc.L2::256B U4", rd<2, 4>, 148 * 4, 512);
    run("cs U4", rd<3, 4>, 148 * 4, 512);
    run("noalloc.L2::128B U4", rd<4, 4>, 148 * 4, 512);
    run("plain U8", rd<0, 8>, 148 * 4, 512);
    run("plain U8 1/SM", rd<0, 8>, 148, 1024);
    run("plain U16 2/SM", rd<0, 16>, 296, 512);
    run("nc.noalloc U8 big grid", rd<1, 8>, 148 * 16, 256);
    // 1 GiB read to compare with the driver's copy peak
    const size_t big = (size_t)1 << 30;
    char* B; cudaMalloc(&B, big); cudaMemset(B, 1, big);
    {
        auto k = rd<0, 8>;
        for (int i = 0; i < 3; ++i) k<<<148 * 4, 512>>>((const int4*)B, big / 16, o);
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) k<<<148 * 4, 512>>>((const int4*)B, big / 16, o);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("1 GiB read plain U8: %.0f GB/s\n", big / (ms / 10 * 1e-3) / 1e9);
    }
    return 0;
}
