// Microbenchmark: cost of a cooperative grid barrier vs CTA count / size.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned long long *out) {
    cg::grid_group g = cg::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}
// hand-rolled: one atomic per CTA on a sense-reversing counter
__device__ unsigned int bar_count = 0;
__device__ volatile unsigned int bar_gen = 0;
__global__ void k2(int iters, unsigned long long *out) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned gen = bar_gen;
            __threadfence();
            if (atomicAdd(&bar_count, 1) == gridDim.x - 1) {
                bar_count = 0;
                __threadfence();
                bar_gen = gen + 1;
            } else {
                while (bar_gen == gen) {}
            }
            __threadfence();
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}
int main() {
    unsigned long long *d, h;
    cudaMalloc(&d, 8);
    int iters = 2000;
    int cfg[][2] = {{148 * 6, 256}, {148 * 3, 512}, {148 * 2, 768}, {148, 1024}, {148 * 8, 256}};
    for (auto &c : cfg) {
        void *args[] = {&iters, &d};
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void *)k, c[0], c[1], args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)k, c[0], c[1], args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        cudaLaunchCooperativeKernel((void *)k2, c[0], c[1], args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)k2, c[0], c[1], args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms2; cudaEventElapsedTime(&ms2, a, b);
        printf("grid %d x %d: cg.sync %.3f us/barrier, hand %.3f us/barrier (%s)\n", c[0], c[1], ms * 1e3 / iters,
               ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
