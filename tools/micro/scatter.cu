// Scattered-access throughput per SM: each thread issues independent random
// 8-byte accesses (ld.cg / st.cg / red.min) into an array; one 768-thread CTA per SM.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int MODE>
__global__ void __launch_bounds__(768, 1) k(unsigned long long *a, unsigned mask, int iters, unsigned long long *out) {
    unsigned s = blockIdx.x * 768 + threadIdx.x;
    unsigned long long acc = 0;
    for (int it = 0; it < iters; it++) {
        unsigned long long v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            unsigned idx = hash(s * 8 + u + it * 0x9e3779b9u) & mask;
            if (MODE == 0) v[u] = __ldcg(a + idx * 4);
            else if (MODE == 1) __stcg(a + idx * 4, (unsigned long long)it);
            else asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(a + idx * 4), "l"((unsigned long long)it) : "memory");
        }
        if (MODE == 0) {
#pragma unroll
            for (int u = 0; u < 8; u++) acc += v[u];
        }
    }
    if (acc == 12345) out[0] = acc;
}
int main() {
    for (size_t mb : {16, 256, 2048}) {
        size_t n = mb << 20 >> 3;   // u64 elements
        unsigned long long *a, *o;
        cudaMalloc(&a, n * 8); cudaMalloc(&o, 64);
        cudaMemset(a, 0, n * 8);
        unsigned mask = (unsigned)(n / 4 - 1);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        const char *names[3] = {"ld.cg", "st.cg", "red.min"};
        for (int mode = 0; mode < 3; mode++) {
            int iters = 200;
            for (int rep = 0; rep < 2; rep++) {
                cudaEventRecord(e0);
                if (mode == 0) k<0><<<148, 768>>>(a, mask, iters, o);
                if (mode == 1) k<1><<<148, 768>>>(a, mask, iters, o);
                if (mode == 2) k<2><<<148, 768>>>(a, mask, iters, o);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
            }
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double acc = 148.0 * 768 * iters * 8;
            printf("%5zu MB %-8s: %.2f G acc/s total, %.3f acc/cycle/SM @1.965GHz, %.0f GB/s of sectors\n", mb, names[mode],
                   acc / ms / 1e6, acc / (ms * 1e-3) / 148 / 1.965e9, acc * 32 / ms / 1e6);
        }
        cudaFree(a); cudaFree(o);
    }
}
