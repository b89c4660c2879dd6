// Is instruction fetch a bottleneck for straight-line code executed once per SM?
// Same arithmetic (N dependent-free FFMA groups) as one unrolled body vs a loop.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
template <int N, bool UNROLL>
__global__ void __launch_bounds__(512) k(float* out, unsigned long long* tt, float s) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    unsigned long long t0 = gt();
    if (UNROLL) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            a0 = fmaf(a0, s, 1.0f + i); a1 = fmaf(a1, s, 2.0f + i); a2 = fmaf(a2, s, 3.0f + i); a3 = fmaf(a3, s, 4.0f + i);
        }
    } else {
#pragma unroll 1
        for (int i = 0; i < N; ++i) {
            a0 = fmaf(a0, s, 1.0f + i); a1 = fmaf(a1, s, 2.0f + i); a2 = fmaf(a2, s, 3.0f + i); a3 = fmaf(a3, s, 4.0f + i);
        }
    }
    unsigned long long t1 = gt();
    if (threadIdx.x == 0) tt[blockIdx.x] = t1 - t0;
    out[blockIdx.x * 512 + threadIdx.x] = a0 + a1 + a2 + a3;
}
template <int N, bool U>
void run(float* o, unsigned long long* d) {
    unsigned long long h[64];
    for (int it = 0; it < 3; ++it) k<N, U><<<64, 512>>>(o, d, 0.999f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * 64, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 64; ++i) s += h[i];
    printf("N=%5d %s: %.2f us  (%.2f ns per group of 4 FFMA)\n", N, U ? "unrolled" : "loop    ", s / 64 / 1000, s / 64 / N);
}
int main() {
    float* o;
    unsigned long long* d;
    cudaMalloc(&o, 64 * 512 * 4);
    cudaMalloc(&d, 8 * 64);
    run<500, true>(o, d);
    run<500, false>(o, d);
    run<2000, true>(o, d);
    run<2000, false>(o, d);
    run<8000, true>(o, d);
    run<8000, false>(o, d);
    return 0;
}
