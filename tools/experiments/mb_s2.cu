// Microbenchmark: stage-2 MLP row GEMV (A rows 1216 bf16, up+gate), variants.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ int4 ldw(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ int4 ldp(const void* p) { return __ldg(reinterpret_cast<const int4*>(p)); }
__device__ __forceinline__ float2 bf2(uint32_t h) { return make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u)); }
__device__ __forceinline__ void dot(float& a, const int4& w, const float* z) {
    const float4 z0 = *reinterpret_cast<const float4*>(z), z1 = *reinterpret_cast<const float4*>(z + 4);
    float2 p;
    p = bf2(w.x); a = fmaf(p.x, z0.x, a); a = fmaf(p.y, z0.y, a);
    p = bf2(w.y); a = fmaf(p.x, z0.z, a); a = fmaf(p.y, z0.w, a);
    p = bf2(w.z); a = fmaf(p.x, z1.x, a); a = fmaf(p.y, z1.y, a);
    p = bf2(w.w); a = fmaf(p.x, z1.z, a); a = fmaf(p.y, z1.w, a);
}
__device__ __forceinline__ float wsum(float v) { for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o); return v; }
constexpr int M = 11008, NS = 1216, NV = NS / 8;
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(const __nv_bfloat16* __restrict__ up, const __nv_bfloat16* __restrict__ gt,
                                            const float* __restrict__ zg, __nv_bfloat16* act) {
    __shared__ __align__(16) float zs[2 * NS];
    for (int i = threadIdx.x; i < 2 * NS; i += 512) zs[i] = zg[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = (int)((long long)M * blockIdx.x / gridDim.x), r1 = (int)((long long)M * (blockIdx.x + 1) / gridDim.x);
    for (int r = r0 + warp; r < r1; r += 16) {
        const char* ru = reinterpret_cast<const char*>(up + (size_t)r * NS);
        const char* rg = reinterpret_cast<const char*>(gt + (size_t)r * NS);
        int4 wu[5], wg[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int v = j * 32 + lane;
            if (MODE == 0) { wu[j] = v < NV ? ldw(ru + v * 16) : make_int4(0,0,0,0); wg[j] = v < NV ? ldw(rg + v * 16) : make_int4(0,0,0,0); }
            else { const int vv = min(v, NV - 1); wu[j] = ldp(ru + vv * 16); wg[j] = ldp(rg + vv * 16); }
        }
        float au = 0, ag = 0;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int v = min(j * 32 + lane, NV - 1);
            if (MODE == 1 && j * 32 + lane >= NV) continue;
            dot(au, wu[j], zs + v * 8);
            dot(ag, wg[j], zs + NS + v * 8);
        }
        au = wsum(au); ag = wsum(ag);
        if (lane == 0) act[r] = __float2bfloat16_rn(ag / (1.f + __expf(-ag)) * au);
    }
}
int main() {
    const int R = 4;
    const size_t mb = (size_t)M * NS * 2;
    char* buf; cudaMalloc(&buf, 2 * mb * R); cudaMemset(buf, 0, 2 * mb * R);
    float* z; cudaMalloc(&z, 2 * NS * 4); cudaMemset(z, 0, 2 * NS * 4);
    __nv_bfloat16* act; cudaMalloc(&act, M * 2);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* nm, auto kern, int grid) {
        for (int i = 0; i < 10; ++i) kern<<<grid, 512>>>((__nv_bfloat16*)(buf + (i % R) * 2 * mb), (__nv_bfloat16*)(buf + (i % R) * 2 * mb + mb), z, act);
        cudaEventRecord(e0);
        for (int i = 0; i < 100; ++i) kern<<<grid, 512>>>((__nv_bfloat16*)(buf + (i % R) * 2 * mb), (__nv_bfloat16*)(buf + (i % R) * 2 * mb + mb), z, act);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s grid %4d: %7.2f us  %6.0f GB/s  %s\n", nm, grid, ms * 10, 2 * mb / (ms * 10) / 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    run("mode0 predicated ldw", k<0>, 148);
    run("mode1 clamped ldg", k<1>, 148);
    run("mode0 predicated ldw x2", k<0>, 296);
    run("mode1 clamped ldg x2", k<1>, 296);
    run("mode1 clamped ldg x4", k<1>, 592);
    return 0;
}
