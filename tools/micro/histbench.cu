// Cost of the select kernel's radix histogram pass pieces (512 threads, 2 keys per thread,
// 4096 bins), %globaltimer inside the kernel, 64 CTAs.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
template <int MODE>
__global__ void __launch_bounds__(512) k(unsigned long long* out, int* sink, int reps) {
    __shared__ __align__(16) int h[4096];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned key[2];
    for (int l = 0; l < 2; ++l) {  // keys with few distinct top bits (like pooled probabilities)
        unsigned x = (tid * 2 + l) * 2654435761u;
        key[l] = 0x3b000000u + ((x >> 8) & 0x00ffffffu) % 0x03000000u;
    }
    for (int i = tid; i < 4096; i += 512) h[i] = 0;
    __syncthreads();
    unsigned long long t0 = gt();
    int acc = 0;
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int l = 0; l < 2; ++l) {
                const int dg = (int)((key[l] >> 20) & 4095u);
                if (MODE == 0) {
                    const unsigned grp = __match_any_sync(0xffffffffu, dg);
                    if (lane == __ffs(grp) - 1) atomicAdd(&h[dg], __popc(grp));
                } else {
                    atomicAdd(&h[dg], 1);
                }
            }
            __syncthreads();
        }
        if (MODE == 1) {  // warp 0 scans 4096 bins: int4 sums + suffix scan
            if (warp == 0) {
                int lsum = 0;
                for (int i = 0; i < 128; i += 4) {
                    const int4 h4 = *reinterpret_cast<const int4*>(&h[lane * 128 + i]);
                    lsum += h4.x + h4.y + h4.z + h4.w;
                }
                int suf = lsum;
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_down_sync(0xffffffffu, suf, o);
                    if (lane + o < 32) suf += y;
                }
                acc += suf;
            }
            __syncthreads();
        }
    }
    unsigned long long t1 = gt();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345) sink[0] = h[5];
}
int main() {
    unsigned long long* d;
    int* sink;
    cudaMalloc(&d, 8 * 64);
    cudaMalloc(&sink, 64);
    unsigned long long hst[64];
    const char* names[] = {"hist match_any+atomic", "warp0 scan 4096", "hist atomic only"};
    for (int mode = 0; mode < 3; ++mode)
        for (int reps : {1, 20}) {
            for (int it = 0; it < 3; ++it) {
                if (mode == 0) k<0><<<64, 512>>>(d, sink, reps);
                if (mode == 1) k<1><<<64, 512>>>(d, sink, reps);
                if (mode == 2) k<2><<<64, 512>>>(d, sink, reps);
            }
            cudaDeviceSynchronize();
            cudaMemcpy(hst, d, 8 * 64, cudaMemcpyDeviceToHost);
            double s = 0;
            for (int i = 0; i < 64; ++i) s += hst[i];
            printf("%-24s reps %2d: %.1f ns per rep\n", names[mode], reps, s / 64 / reps);
        }
    return 0;
}
