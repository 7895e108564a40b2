// Microbenchmark: 64-bit atomicMin (no return) throughput in the fused
// aggregation+WTA pattern: nd slices x (w x h) pixels, warp = 32 consecutive
// pixels of one slice, every slice hitting the same w x h key array.
#include <cstdio>
#include <cstdint>

__global__ void k_red(unsigned long long* keys, int n, int nd, int per_thread) {
    const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    for (int j = 0; j < per_thread; ++j) {
        const size_t e = tid * per_thread + j;
        const int k = static_cast<int>(e / n);
        const int p = static_cast<int>(e - static_cast<size_t>(k) * n);
        if (k >= nd) return;
        const unsigned v = (static_cast<unsigned>(p) * 2654435761u) ^ (static_cast<unsigned>(k) * 40503u);
        atomicMin(keys + p, (static_cast<unsigned long long>(v >> 2) << 32) | static_cast<unsigned>(k));
    }
}
__global__ void k_store(float* vol, int n, int nd) {
    const size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (e < static_cast<size_t>(n) * nd) vol[e] = static_cast<float>(e & 1023);
}

int main() {
    const int w = 640, h = 360, nd = 128, n = w * h;
    unsigned long long* keys;
    float* vol;
    cudaMalloc(&keys, n * 8);
    cudaMalloc(&vol, static_cast<size_t>(n) * nd * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(keys, 0xff, n * 8);
        const size_t tot = static_cast<size_t>(n) * nd;
        cudaEventRecord(a);
        k_red<<<(tot + 255) / 256, 256>>>(keys, n, nd, 1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventRecord(a);
        k_store<<<(tot + 255) / 256, 256>>>(vol, n, nd);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms2;
        cudaEventElapsedTime(&ms2, a, b);
        printf("29.5M red.min.u64 over 230K keys: %.1f us (%.0f G atomics/s); the same count of float stores: %.1f us\n",
               ms * 1e3, tot / (ms * 1e-3) / 1e9, ms2 * 1e3);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
