// gemv_micro.cu -- stage-2 structure experiments: y[i] = sum_s A[i,s] z[s],
// A [m, ns] bf16 row-major (one contiguous row per output), z f32 in smem.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gemv_micro gemv_micro.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ int4 ldg_nc(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ float wsum(float v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ void unpack8(const int4& v, float* o) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    for (int q = 0; q < 4; ++q) { float2 f = __bfloat1622float2(h[q]); o[2*q] = f.x; o[2*q+1] = f.y; }
}

// RB rows per warp iteration, all loads of the RB rows issued before use
template <int RB, int MAXV>
__global__ void gemv_rows(const __nv_bfloat16* __restrict__ A, const float* __restrict__ z, int m, int ns,
                          float* __restrict__ y) {
    extern __shared__ float zs[];
    for (int s = threadIdx.x; s < ns; s += blockDim.x) zs[s] = z[s];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x / 32);
    const int gw = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int nv = ns / 8;
    for (int r0 = gw * RB; r0 < m; r0 += nw * RB) {
        int4 w[RB][MAXV];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int k = 0; k < MAXV; ++k) {
                const int v = lane + 32 * k;
                if (r0 + r < m && v < nv) w[r][k] = ldg_nc(A + (size_t)(r0 + r) * ns + v * 8);
            }
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < MAXV; ++k) {
                const int v = lane + 32 * k;
                if (v < nv) {
                    float f[8];
                    unpack8(w[r][k], f);
                    const float4 z0 = *reinterpret_cast<const float4*>(zs + v * 8);
                    const float4 z1 = *reinterpret_cast<const float4*>(zs + v * 8 + 4);
                    acc += f[0]*z0.x + f[1]*z0.y + f[2]*z0.z + f[3]*z0.w + f[4]*z1.x + f[5]*z1.y + f[6]*z1.z + f[7]*z1.w;
                }
            }
            acc = wsum(acc);
            if (lane == 0 && r0 + r < m) y[r0 + r] = acc;
        }
    }
}

int main() {
    const int m = 11008, ns = 1216, R = 8;  // R replicas to defeat L2
    const size_t bytes = (size_t)m * ns * 2;
    __nv_bfloat16* A; float *z, *y;
    cudaMalloc(&A, bytes * R); cudaMalloc(&z, ns * 4); cudaMalloc(&y, m * 4);
    cudaMemset(A, 0, bytes * R); cudaMemset(z, 0, ns * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern, int grid, int block) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        for (int i = 0; i < 20; ++i) kern<<<grid, block, ns * 4>>>(A + (size_t)(i % R) * m * ns, z, m, ns, y);
        cudaEventRecord(e0);
        const int it = 200;
        for (int i = 0; i < it; ++i) kern<<<grid, block, ns * 4>>>(A + (size_t)(i % R) * m * ns, z, m, ns, y);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / it;
        printf("%-28s grid %5d block %4d: %7.2f us  %6.0f GB/s  (%s)\n", name, grid, block, us,
               bytes / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    run("rows RB=1 persistent", gemv_rows<1, 5>, 148, 512);
    run("rows RB=2 persistent", gemv_rows<2, 5>, 148, 512);
    run("rows RB=4 persistent", gemv_rows<4, 5>, 148, 512);
    run("rows RB=1 148x2 cta", gemv_rows<1, 5>, 296, 512);
    run("rows RB=1 1024thr", gemv_rows<1, 5>, 148, 1024);
    run("rows RB=2 1024thr", gemv_rows<2, 5>, 148, 1024);
    run("rows RB=1 grid m/8", gemv_rows<1, 5>, (m + 7) / 8, 256);
    run("rows RB=2 grid m/16", gemv_rows<2, 5>, (m + 15) / 16, 256);
    run("rows RB=4 grid m/32", gemv_rows<4, 5>, (m + 31) / 32, 256);
    run("rows RB=2 4/SM", gemv_rows<2, 5>, 148 * 4, 256);
    return 0;
}
