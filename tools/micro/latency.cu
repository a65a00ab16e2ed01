// Dependent-load latency probe: one warp chases a random cycle with ld.global.cg
// over arrays of various sizes; prints ns per dependent load.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
__global__ void chase(const unsigned *next, int steps, unsigned *out, long long *ns) {
    unsigned i = threadIdx.x * 97;
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int s = 0; s < steps; s++) i = __ldcg(next + i);
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[threadIdx.x] = i;
    if (threadIdx.x == 0) *ns = t1 - t0;
}
int main() {
    for (size_t mb : {1, 16, 64, 256, 1024, 4096}) {
        size_t n = mb * 1024 * 1024 / 4;
        std::vector<unsigned> h(n);
        // random permutation cycle with stride of 8 words (32B sectors)
        size_t m = n / 8;
        std::vector<unsigned> perm(m);
        for (size_t k = 0; k < m; k++) perm[k] = (unsigned)k;
        std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
        for (size_t k = 0; k < m; k++) for (int j = 0; j < 8; j++) h[perm[k] * 8 + j] = perm[(k + 1) % m] * 8 + j;
        unsigned *d, *o; long long *t;
        cudaMalloc(&d, n * 4); cudaMalloc(&o, 4096); cudaMalloc(&t, 8);
        cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
        int steps = 20000;
        chase<<<1, 1>>>(d, 1000, o, t);
        chase<<<1, 1>>>(d, steps, o, t);
        long long ns; cudaMemcpy(&ns, t, 8, cudaMemcpyDeviceToHost);
        printf("%5zu MB: %.1f ns per dependent load\n", mb, (double)ns / steps);
        cudaFree(d); cudaFree(o); cudaFree(t);
    }
}
