// Device cost of a chain of dependent kernels in one CUDA graph (launch + boundary latency).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0 && p[0] == 12345) p[1] = 1; }
__global__ void k_touch(int* p, int n) {  // every CTA reads + writes one word (one round trip)
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = p[i] + 1;
}
int main() {
    int* d; cudaMalloc(&d, 1 << 24); cudaMemset(d, 0, 1 << 24);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const int N = 200;
    for (int variant = 0; variant < 4; ++variant) {
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < N; ++i) {
            if (variant == 0) k_empty<<<1, 32, 0, s>>>(d);
            else if (variant == 1) k_empty<<<148 * 4, 128, 0, s>>>(d);
            else if (variant == 2) k_touch<<<64, 512, 0, s>>>(d, 64 * 512);
            else k_touch<<<148 * 8, 256, 0, s>>>(d, 148 * 8 * 256);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const char* names[] = {"empty 1x32", "empty 592x128", "touch 64x512", "touch 1184x256"};
        printf("{\"%s_us_per_kernel\": %.3f}\n", names[variant], ms * 1e3 / (10 * N));
    }
    return 0;
}
