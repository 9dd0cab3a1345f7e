// Can a cooperative (grid-sync) kernel also be launched with thread-block
// clusters on B200?  Measures grid.sync and cluster.sync costs.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int mode, unsigned long long *out) {
    cg::grid_group g = cg::this_grid();
    cg::cluster_group cl = cg::this_cluster();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { if (mode == 0) g.sync(); else cl.sync(); }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[mode] = clock64() - t0;
}
int main() {
    unsigned long long *d; cudaMalloc(&d, 16);
    int iters = 2000;
    for (int csize : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg = {};
        int grid = 148 * 4;
        grid -= grid % csize;
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension; at[1].val.clusterDim.x = csize; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 2;
        for (int mode = 0; mode < 2; ++mode) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaError_t e = cudaLaunchKernelEx(&cfg, k, iters, mode, d);
            cudaEventRecord(a);
            if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, k, iters, mode, d);
            cudaEventRecord(b);
            cudaError_t e2 = cudaDeviceSynchronize();
            float ms = 0; cudaEventElapsedTime(&ms, a, b);
            printf("cluster %d grid %d %s: launch=%s sync=%s  %.3f us per barrier\n", csize, grid, mode ? "cluster.sync" : "grid.sync",
                   cudaGetErrorString(e), cudaGetErrorString(e2), ms * 1e3 / iters);
            cudaGetLastError();
        }
    }
}
