// FP64 latency / throughput and smem + __syncthreads costs on this B200.
#include <cstdio>
__global__ void k_lat(double* out, int n) {
    double a = threadIdx.x * 1e-3, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = a * b + 1e-9;  // dependent DFMA chain
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / n;
    out[1 + threadIdx.x] = a;
}
__global__ void k_tput(double* out, int n) {
    double a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = a[j] * 1.0000001 + 1e-9;
    double s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_bar(double* out, int n) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (double)(t1 - t0) / n;
}
int main() {
    double* d;
    cudaMalloc(&d, 1 << 26);
    double h[4];
    k_lat<<<1, 32>>>(d, 1 << 16);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("dependent DFMA latency: %.1f cycles\n", h[0]);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int n = 4096;
    k_tput<<<148 * 8, 256>>>(d, n);
    cudaEventRecord(a);
    k_tput<<<148 * 8, 256>>>(d, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * n * 148.0 * 8 * 256;
    printf("DFMA throughput: %.2f TFLOP/s\n", flops / ms / 1e9);
    for (int t : {256, 1024}) {
        k_bar<<<148, t>>>(d, 10000);
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("__syncthreads with %d threads: %.1f cycles\n", t, h[0]);
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock rate attr %d kHz\n", clk);
    return 0;
}
