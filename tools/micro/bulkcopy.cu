// Minimal check of the cp.async.bulk + mbarrier stream pipeline used by
// edge_stream_body (sums a u32 array through 2 shared-memory stages).
#include <cstdio>
#include <cstdint>
constexpr int kStages = 2;
constexpr uint32_t kChunk = 2048;
struct SS { uint32_t buf[kStages][kChunk]; unsigned long long bar[kStages]; };
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <bool FP>
__device__ void issue(SS *ss, int st, const uint32_t *src, uint32_t bytes) {
    if (FP) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&ss->bar[st])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(sa(ss->buf[st])), "l"(src), "r"(bytes), "r"(sa(&ss->bar[st])) : "memory");
}
__device__ void waitp(SS *ss, int st, uint32_t par, unsigned long long *spins) {
    uint32_t done = 0;
    unsigned long long n = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(sa(&ss->bar[st])), "r"(par) : "memory");
        if (++n > 100000000ull) { if (threadIdx.x == 0) atomicAdd(spins, 1ull); return; }
    }
}
template <bool FP, bool FI>
__global__ void k(const uint32_t *a, uint64_t m, unsigned long long *sum, unsigned long long *timeouts) {
    __shared__ __align__(16) SS ss;
    const uint64_t nch = (m + kChunk - 1) / kChunk;
    auto bytes = [&](uint64_t ch) { uint64_t s = m - ch * kChunk; if (s > kChunk) s = kChunk; return (uint32_t)((s * 4 + 15) & ~15ull); };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&ss.bar[s])) : "memory");
        if (FI) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < kStages; ++s) { uint64_t ch = blockIdx.x + (uint64_t)s * gridDim.x; if (ch < nch) issue<FP>(&ss, s, a + ch * kChunk, bytes(ch)); }
    }
    __syncthreads();
    unsigned long long loc = 0;
    uint32_t kk = 0;
    for (uint64_t ch = blockIdx.x; ch < nch; ch += gridDim.x, ++kk) {
        const int st = kk % kStages;
        waitp(&ss, st, (kk / kStages) & 1u, timeouts);
        for (uint32_t i = threadIdx.x; i < kChunk; i += blockDim.x) if (ch * kChunk + i < m) loc += ss.buf[st][i];
        __syncthreads();
        if (threadIdx.x == 0) { uint64_t nx = ch + (uint64_t)kStages * gridDim.x; if (nx < nch) issue<FP>(&ss, st, a + nx * kChunk, bytes(nx)); }
    }
    // block reduce, one atomic per CTA (a per-thread atomic on one address
    // would dominate the kernel)
    __shared__ unsigned long long part[32];
    for (int o = 16; o > 0; o >>= 1) loc += __shfl_down_sync(0xffffffffu, loc, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        atomicAdd(sum, t);
    }
}
int main() {
    for (uint64_t m : {1000ull, 2048ull, 100000ull, 1ull << 27}) {
        uint32_t *a; unsigned long long *d;
        cudaMalloc(&a, m * 4 + 16); cudaMalloc(&d, 16);
        cudaMemset(a, 0, m * 4 + 16); cudaMemset(d, 0, 16);
        // a[i] = 1
        uint32_t *h = new uint32_t[m]; for (uint64_t i = 0; i < m; ++i) h[i] = 1; cudaMemcpy(a, h, m * 4, cudaMemcpyHostToDevice);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int var = 0; var < 4; ++var) {
            auto run = [&](auto kern) { kern<<<148 * 5, 256>>>(a, m, d, d + 1); cudaEventRecord(e0); kern<<<148 * 5, 256>>>(a, m, d, d + 1); cudaEventRecord(e1); };
            cudaMemset(d, 0, 16);
            if (var == 0) run(k<true, true>); else if (var == 1) run(k<false, true>); else if (var == 2) run(k<true, false>); else run(k<false, false>);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long r[2]; cudaMemcpy(r, d, 16, cudaMemcpyDeviceToHost);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("var=%d m=%llu err=%s ok=%d timeouts=%llu  %.1f us %.1f GB/s\n", var, (unsigned long long)m, cudaGetErrorString(e), (int)(r[0] == 2 * m), r[1], ms * 1e3, m * 4 / (ms * 1e-3) / 1e9);
        }
        delete[] h; cudaFree(a); cudaFree(d);
    }
}
