// host_utils.cu -- the reference's seeded generators, re-implemented for the
// product side (synthetic inputs for bench/tests), and a device normal fill.
//
//  * pg_rng_fill_gaussian: Rng (include/parse/rng.hpp:10-41) -- splitmix64 and
//    Box-Muller without a cached spare, so fixtures match the reference bits.
//  * pg_make_patterns: the prefix-biased K-subset generator of
//    tests/test_acceptance.cpp:412-425 (pick = below(2) ? 0 : below(pool.size()),
//    pool.erase(pick)).  pool stays sorted, so pool[pick] is the pick-th
//    smallest remaining id: a Fenwick tree gives O(log r) select + erase
//    instead of the reference's O(r) vector::erase, same ids.
#include <algorithm>
#include <cmath>
#include <vector>

#include "pg_common.cuh"

namespace {

struct Rng {
    uint64_t state;
    uint64_t next_u64() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }
    uint64_t below(uint64_t n) { return next_u64() % n; }
    double gaussian() {
        double u1 = uniform();
        double u2 = uniform();
        while (u1 <= 0) u1 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

struct Fenwick {
    std::vector<int> t;
    int n, logn;
    explicit Fenwick(int n_) : t(n_ + 1, 0), n(n_) {
        for (int i = 1; i <= n; ++i) {
            t[i] += 1;
            int j = i + (i & -i);
            if (j <= n) t[j] += t[i];
        }
        logn = 1;
        while ((1 << logn) <= n) ++logn;
    }
    void remove(int pos0) {
        for (int i = pos0 + 1; i <= n; i += i & -i) t[i] -= 1;
    }
    // 0-based position of the (k+1)-th present element
    int select(int k) {
        int pos = 0;
        for (int b = logn; b >= 0; --b) {
            const int nx = pos + (1 << b);
            if (nx <= n && t[nx] <= k) {
                pos = nx;
                k -= t[nx];
            }
        }
        return pos;  // pos is the 1-based index of the last prefix with count <= k -> element pos (0-based)
    }
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void k_fill_normal(T* out, size_t count, uint64_t seed, double scale) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint64_t a = mix64(seed * 0x9e3779b97f4a7c15ULL + 2 * i + 1);
        const uint64_t b = mix64(a ^ 0xd1342543de82ef95ULL);
        const float u1 = ((a >> 40) + 1) * (1.0f / 16777217.0f);
        const float u2 = (b >> 40) * (1.0f / 16777216.0f);
        const float g = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
        const float v = (float)scale * g;
        if constexpr (sizeof(T) == 2) out[i] = __float2bfloat16_rn(v);
        else out[i] = (T)v;
    }
}

}  // namespace

#include <mutex>
#include <set>
#include <utility>

namespace pg {

int current_device() {
    int dev = 0;
    PG_CUDA_THROW(cudaGetDevice(&dev));
    return dev;
}

int device_sms() {
    static std::atomic<int> sms[128];
    const int dev = current_device();
    if (dev < 0 || dev >= 128) throw Error{PG_CUDA_ERROR, "device index out of range"};
    int v = sms[dev].load(std::memory_order_relaxed);
    if (!v) {
        PG_CUDA_THROW(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        sms[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

void once_per_device(const void* tag, void (*fn)()) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({tag, dev})) return;
    fn();
    done.insert({tag, dev});
}

void launch_fill_normal(void* out, pg_dtype dt, size_t count, uint64_t seed, double scale,
                        cudaStream_t st) {
    const int blocks = kNumSMs * 8;
    if (dt == PG_F64) k_fill_normal<double><<<blocks, 256, 0, st>>>(static_cast<double*>(out), count, seed, scale);
    else if (dt == PG_F32) k_fill_normal<float><<<blocks, 256, 0, st>>>(static_cast<float*>(out), count, seed, scale);
    else k_fill_normal<__nv_bfloat16><<<blocks, 256, 0, st>>>(static_cast<__nv_bfloat16*>(out), count, seed, scale);
    PG_LAUNCH_CHECK();
}
// Step I/O as a kernel: copies between device-accessible buffers (device
// memory or pinned host memory, which UVA maps at the same address), so a
// decode step's input / output transfers chain with the step's kernels under
// programmatic dependent launch instead of splitting the stream with copy-engine
// nodes.  16-byte vectors when both ends allow it.
__global__ void __launch_bounds__(256) k_copy_io(const unsigned char* __restrict__ src,
                                                 unsigned char* __restrict__ dst, size_t bytes) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the predecessor may produce src
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        const size_t n16 = bytes / 16;
        for (size_t i = tid; i < n16; i += nt)
            reinterpret_cast<int4*>(dst)[i] = reinterpret_cast<const int4*>(src)[i];
        for (size_t i = n16 * 16 + tid; i < bytes; i += nt) dst[i] = src[i];
    } else {
        for (size_t i = tid; i < bytes; i += nt) dst[i] = src[i];
    }
}

void launch_copy_io(const void* src, void* dst, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    const int blocks = (int)std::min<size_t>(64, (bytes / 16 + 255) / 256 + 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_copy_io, static_cast<const unsigned char*>(src),
                                     static_cast<unsigned char*>(dst), bytes));
    count_launch();
}
}  // namespace pg

extern "C" {

void pg_rng_fill_gaussian(uint64_t seed, double* out, size_t count) {
    Rng r{seed};
    for (size_t i = 0; i < count; ++i) out[i] = r.gaussian();
}

void pg_make_patterns(uint64_t seed, size_t n_patterns, const size_t* r_stores, const size_t* ks,
                      size_t n_layers, uint32_t* out) {
    Rng rng{seed};
    size_t w = 0;
    for (size_t p = 0; p < n_patterns; ++p) {
        for (size_t l = 0; l < n_layers; ++l) {
            const int r = (int)r_stores[l];
            Fenwick fw(r);
            size_t remaining = (size_t)r;
            uint32_t* sel = out + w;
            for (size_t i = 0; i < ks[l]; ++i) {
                const size_t pick = rng.below(2) ? 0 : (size_t)rng.below(remaining);
                const int pos = fw.select((int)pick);
                sel[i] = (uint32_t)pos;
                fw.remove(pos);
                --remaining;
            }
            std::sort(sel, sel + ks[l]);
            w += ks[l];
        }
    }
}

}  // extern "C"
