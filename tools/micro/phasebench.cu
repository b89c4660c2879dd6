// Calibrate the select kernel's phase costs on B200 (64 CTAs x 1024 threads, %globaltimer
// inside the kernel): butterflies, block barriers, smem round trips.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int MODE>
__global__ void k(int reps, unsigned long long* out, float* sink) {
    __shared__ float red[32][4];
    float v[4] = {threadIdx.x * 1.0f, 2.0f, 3.0f, 4.0f};
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    unsigned long long t0 = gt();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0) {  // butterfly max over 4 heads, 5 levels
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int g = 0; g < 4; ++g) v[g] = fmaxf(v[g], __shfl_xor_sync(0xffffffffu, v[g], o));
        } else if (MODE == 1) {  // block barrier + smem round trip (cross-warp reduce like the select)
            if (lane == 0)
#pragma unroll
                for (int g = 0; g < 4; ++g) red[warp][g] = v[g];
            __syncthreads();
#pragma unroll
            for (int g = 0; g < 4; ++g) v[g] += red[lane][g];
            __syncthreads();
        } else if (MODE == 2) {  // full max phase: butterfly + smem + barrier + butterfly
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int g = 0; g < 4; ++g) v[g] = fmaxf(v[g], __shfl_xor_sync(0xffffffffu, v[g], o));
            if (lane == 0)
#pragma unroll
                for (int g = 0; g < 4; ++g) red[warp][g] = v[g];
            __syncthreads();
#pragma unroll
            for (int g = 0; g < 4; ++g) v[g] = red[lane][g] + v[g] * 0.5f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int g = 0; g < 4; ++g) v[g] = fmaxf(v[g], __shfl_xor_sync(0xffffffffu, v[g], o));
            __syncthreads();
        }
    }
    unsigned long long t1 = gt();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (v[0] == -1.0f) sink[0] = v[1] + v[2] + v[3];
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&sink, 64);
    unsigned long long h[148];
    const char* names[] = {"butterfly 5x4", "barrier+smem x2", "max phase"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int reps : {1, 100}) {
            for (int it = 0; it < 3; ++it) {
                if (mode == 0) k<0><<<64, 1024>>>(reps, d, sink);
                if (mode == 1) k<1><<<64, 1024>>>(reps, d, sink);
                if (mode == 2) k<2><<<64, 1024>>>(reps, d, sink);
            }
            cudaDeviceSynchronize();
            cudaMemcpy(h, d, 8 * 64, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0, sum = 0;
            for (int i = 0; i < 64; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
            printf("%-18s reps %3d: mean %.1f ns per rep (max CTA %.1f)\n", names[mode], reps, sum / 64.0 / reps, mx / (double)reps);
        }
    }
    return 0;
}
