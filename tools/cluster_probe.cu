// How many clusters of size C (1 CTA/SM via ~225 KB dynamic smem) can be co-resident on this GPU?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int* x) { extern __shared__ int s[]; if (threadIdx.x == 0 && x) x[0] = s[0]; }
int main() {
    int smem = 225 * 1024;
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c = 1; c <= 16; ++c) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(c * 64); cfg.blockDim = dim3(768); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = c; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr; cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d SMs %s\n", c, n, n * c, e ? cudaGetErrorString(e) : "");
    }
    return 0;
}
