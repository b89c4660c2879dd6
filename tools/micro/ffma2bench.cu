// FFMA vs FFMA2 (fma.rn.f32x2) vs LOP3+FFMA throughput/latency on one SM: W warps, each with
// C independent accumulator chains, N iterations.  Prints cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cstdint>
__global__ void k_ffma(float* out, float a, float b, int n, int chains) {
    float acc[8];
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 0.001f + i;
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(acc[i], a, b);
    }
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) out[1 << 20] = (float)(t1 - t0);
}
__global__ void k_ffma2(float* out, float a, float b, int n, int chains) {
    unsigned long long acc[8];
    unsigned long long a2, b2;
    asm("mov.b64 %0, {%1, %1};" : "=l"(a2) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(b2) : "f"(b));
    for (int i = 0; i < 8; ++i) { float x = threadIdx.x * 0.001f + i; asm("mov.b64 %0, {%1, %1};" : "=l"(acc[i]) : "f"(x)); }
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(a2), "l"(b2));
    }
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i])); s += lo + hi; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) out[1 << 20] = (float)(t1 - t0);
}
// select + FFMA: sel = (mx & m) | (mn & ~m)  (LOP3) then FFMA
__global__ void k_selfma(float* out, float a, uint32_t mx, uint32_t mn, int n, int chains) {
    float acc[8];
    uint32_t m[8];
    for (int i = 0; i < 8; ++i) { acc[i] = threadIdx.x * 0.001f + i; m[i] = (threadIdx.x >> i) & 1 ? 0xffffffffu : 0u; }
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t s = (mx & m[i]) | (mn & ~m[i]);
            acc[i] = __fmaf_rn(a, __uint_as_float(s), acc[i]);
            m[i] ^= it;
        }
    }
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) out[1 << 20] = (float)(t1 - t0);
}
int main() {
    float* d; cudaMalloc(&d, (1 << 20) * 4 + 64);
    const int n = 4096;
    for (int w : {1, 4, 8, 16}) {
        float c;
        k_ffma<<<1, 32 * w>>>(d, 1.0001f, 0.5f, n, 8); cudaDeviceSynchronize();
        cudaMemcpy(&c, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
        printf("FFMA   warps=%2d  cycles/instr/SMSP = %.2f\n", w, c / (n * 8.0) / ((w + 3) / 4));
        k_ffma2<<<1, 32 * w>>>(d, 1.0001f, 0.5f, n, 8); cudaDeviceSynchronize();
        cudaMemcpy(&c, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
        printf("FFMA2  warps=%2d  cycles/instr/SMSP = %.2f\n", w, c / (n * 8.0) / ((w + 3) / 4));
        k_selfma<<<1, 32 * w>>>(d, 1.0001f, 0x3f800000u, 0x3f000000u, n, 8); cudaDeviceSynchronize();
        cudaMemcpy(&c, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
        printf("LOP3+FFMA warps=%2d cycles/(lop3+ffma)/SMSP = %.2f\n", w, c / (n * 8.0) / ((w + 3) / 4));
    }
    return 0;
}
