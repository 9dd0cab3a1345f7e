// Dependent-access latencies on B200 (one thread; the megakernel's solo-level
// chain is a sequence of these): ld.global (L2 hit / DRAM), ld.global.nc,
// returning atomicOr / atomicAdd, red, cluster barrier.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __cluster_dims__(8, 1, 1) k(uint32_t *buf, uint32_t n, int mode, int iters,
                                             unsigned long long *out) {
    cg::cluster_group cl = cg::this_cluster();
    uint32_t idx = 0;
    unsigned long long t0 = 0, c0 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // warm
        if (n <= (1u << 21))   // L2 case: touch the chain's lines first
            for (int i = 0; i < iters; ++i) idx = buf[idx];
        idx = 0;
        t0 = gt();
        c0 = clock64();
        for (int i = 0; i < iters; ++i) {
            switch (mode) {
            case 0: idx = buf[idx]; break;                               // L2-resident chase
            case 1: idx = __ldg(buf + idx); break;
            case 2: idx = atomicOr(buf + idx, 0u); break;
            case 3: idx = atomicAdd(buf + idx, 0u); break;
            case 4: idx = __ldcg(buf + idx); break;
            case 5: idx = *(volatile uint32_t *)(buf + idx); break;
            }
        }
        out[0] = gt() - t0;
        out[1] = clock64() - c0;
        out[2] = idx;
    }
    if (mode == 6) {
        cl.sync();
        unsigned long long a = 0, b = 0;
        if (blockIdx.x == 0 && threadIdx.x == 0) { a = gt(); b = clock64(); }
        for (int i = 0; i < iters; ++i) cl.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = gt() - a; out[1] = clock64() - b; }
    }
    if (mode == 7) {   // globaltimer resolution: distinct consecutive values
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long last = gt(), steps = 0, s0 = last;
            for (int i = 0; i < iters; ++i) { unsigned long long x = gt(); if (x != last) { ++steps; last = x; } }
            out[0] = last - s0; out[1] = steps;
        }
    }
}

int main() {
    const char *names[] = {"ld L2 (stride, 8MB set)", "ld.nc", "atomicOr ret", "atomicAdd ret", "ld.cg",
                           "ld.volatile", "cluster.sync (8 CTAs)", "globaltimer ticks"};
    for (int big = 0; big < 2; ++big) {
        const uint32_t n = big ? (1u << 28) : (1u << 21);   // 8 MB (L2) / 1 GB (DRAM)
        uint32_t *buf, *h = (uint32_t *)malloc((size_t)n * 4);
        cudaMalloc(&buf, (size_t)n * 4);
        // random cyclic permutation with 4 KB+ jumps
        uint32_t stride = big ? 1000003u : 4099u;
        for (uint32_t i = 0; i < n; ++i) h[i] = (uint32_t)(((uint64_t)i * 0 + i + stride) % n);
        cudaMemcpy(buf, h, (size_t)n * 4, cudaMemcpyHostToDevice);
        unsigned long long *out;
        cudaMalloc(&out, 32);
        for (int mode = 0; mode < 8; ++mode) {
            if (big && mode >= 6) continue;
            const int iters = 2000;
            k<<<16, 256>>>(buf, n, mode, iters, out);
            unsigned long long o[3];
            cudaDeviceSynchronize();
            cudaMemcpy(o, out, 24, cudaMemcpyDeviceToHost);
            if (mode == 7)
                printf("%-28s %llu ns over %llu ticks (%.1f ns/tick)\n", names[mode], o[0], o[1], (double)o[0] / o[1]);
            else
                printf("%-28s %s %.1f ns  %.0f cyc per op\n", names[mode], big ? "DRAM" : "L2  ",
                       (double)o[0] / iters, (double)o[1] / iters);
        }
        cudaFree(buf);
        free(h);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
