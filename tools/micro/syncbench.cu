// Micro-benchmark: cost of block-wide phases (smem + __syncthreads) in a 64-CTA x
// 1024-thread kernel, and of dependent smem chains by one warp, on B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_sync(int phases, int* out) {
    __shared__ int s[1024];
    int v = threadIdx.x;
    for (int p = 0; p < phases; ++p) {
        s[threadIdx.x] = v;
        __syncthreads();
        v += s[(threadIdx.x + 37) & 1023];
        __syncthreads();
    }
    if (v == -1) out[blockIdx.x] = v;
}

__global__ void k_warpchain(int n, int* out) {  // warp 0 walks a dependent smem chain, others wait
    __shared__ int s[1024];
    s[threadIdx.x] = (threadIdx.x * 7 + 1) & 1023;
    __syncthreads();
    int v = 0;
    if (threadIdx.x < 32)
        for (int i = 0; i < n; ++i) v = s[(v + threadIdx.x) & 1023];
    __syncthreads();
    if (v == -1) out[blockIdx.x] = v;
}

__global__ void k_empty(int* out) {
    if (threadIdx.x == 12345) out[0] = 1;
}

__global__ void sleepk(long long cyc) {
    long long t0 = clock64();
    while (clock64() - t0 < cyc) {}
}

template <class F>
float timeit(F f, int reps = 20) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int r = 0; r < reps; ++r) {
        sleepk<<<1, 1>>>(2000000);
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    return best * 1000.0f;
}

int main() {
    int* out;
    cudaMalloc(&out, 1 << 20);
    printf("empty 64x1024: %.2f us\n", timeit([&] { k_empty<<<64, 1024>>>(out); }));
    printf("empty 148x128: %.2f us\n", timeit([&] { k_empty<<<148, 128>>>(out); }));
    for (int ph : {0, 1, 5, 10, 20, 40})
        printf("sync phases %2d (x2 barriers) 64x1024: %.2f us\n", ph, timeit([&] { k_sync<<<64, 1024>>>(ph, out); }));
    for (int ph : {10, 40})
        printf("sync phases %2d 64x512: %.2f us\n", ph, timeit([&] { k_sync<<<64, 512>>>(ph, out); }));
    for (int n : {0, 100, 1000})
        printf("warp chain %4d 64x1024: %.2f us\n", n, timeit([&] { k_warpchain<<<64, 1024>>>(n, out); }));
    return 0;
}
