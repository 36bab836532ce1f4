// Microbenchmark: cost of cluster barriers on B200 (16- and 8-CTA clusters, 1024 threads,
// 227 KB dynamic smem, as k_csort).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(1024, 1) k_sync(int iters, int mode, unsigned long long* out)
{
    extern __shared__ unsigned sm[];
    cg::cluster_group cl = cg::this_cluster();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (mode == 1) {  // DSMEM store to the next CTA then sync
            unsigned* r = cl.map_shared_rank(sm + threadIdx.x, (cl.block_rank() + 1) % cl.num_blocks());
            *r = i;
        }
        if (mode == 2) {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
            asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
        } else if (mode == 3) {
            __syncthreads();
        } else {
            cl.sync();
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && cl.block_rank() == 0) *out = (t1 - t0) / (iters ? iters : 1);
}

int main()
{
    unsigned long long* d;
    cudaMalloc(&d, 8);
    int smem = 227 * 1024;
    cudaFuncSetAttribute(k_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {16, 8, 2}) {
        for (int mode : {0, 1, 2, 3}) {
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(cs);
            lc.blockDim = dim3(1024);
            lc.dynamicSmemBytes = smem;
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = cs; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
            lc.attrs = &at; lc.numAttrs = 1;
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaLaunchKernelEx(&lc, k_sync, 1000, mode, d);
            cudaEventRecord(a);
            cudaLaunchKernelEx(&lc, k_sync, 1000, mode, d);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
            cudaEventRecord(a);
            cudaLaunchKernelEx(&lc, k_sync, 0, mode, d);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms0; cudaEventElapsedTime(&ms0, a, b);
            printf("cluster %2d mode %d: %llu cycles/iter, %.2f us per 1000 iters, empty launch %.2f us  (%s)\n", cs, mode, cyc,
                   ms * 1000, ms0 * 1000, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
