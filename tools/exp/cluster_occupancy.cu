// How many clusters of 2 / 4 / 8 CTAs with the GEMM's per-CTA footprint (230 KB of shared memory,
// 320 threads) can be co-resident on this GPU?  (TMA multicast needs 8-CTA clusters.)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe() { extern __shared__ char s[]; if (threadIdx.x == 9999) s[0] = 0; }
int main() {
    const int smem = 230656;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("{\"sms\": %d", sms);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(320);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
        printf(", \"cluster_%d\": {\"max_active_clusters\": %d, \"sms_used\": %d, \"err\": \"%s\"}", cs, n, n * cs,
               cudaGetErrorString(e));
    }
    printf("}\n");
    return 0;
}
