// Max co-resident clusters for a 1-CTA-per-SM kernel shaped like k_union_prog
// (224 threads, ~227 KB dynamic shared memory) at cluster sizes 2, 4, 8, 16.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_occ cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dummy(int* p) {
    extern __shared__ int s[];
    if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 232448 - 1024;
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3((unsigned)(sms / cs * cs));
        q.blockDim = dim3(224);
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        q.attrs = a;
        q.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &q);
        printf("cluster %2d: max active clusters %3d -> %3d SMs busy of %d (%s)\n", cs, n, n * cs, sms,
               cudaGetErrorString(e));
    }
    return 0;
}
