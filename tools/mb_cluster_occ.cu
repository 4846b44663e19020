// Dev probe: how many thread-block clusters of size 2/4/8 are co-resident on
// this GPU with one 320-thread, ~220 KB CTA per SM (the megakernel's shape)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mb_cluster_occ.cu -o tools/mb_cluster_occ
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() {}
int main() {
    int dev = 0, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 220 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nsm / cs * cs);
        cfg.blockDim = dim3(320);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
        printf("cluster %2d: max active clusters %3d (= %3d CTAs of %d SMs) %s\n", cs, nc, nc * cs, nsm,
               e ? cudaGetErrorString(e) : "");
    }
    return 0;
}
