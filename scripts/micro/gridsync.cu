// Microbenchmark: cost of one grid-wide barrier on B200 (148 SMs x 1 block).
// cg::grid_group::sync() vs a hand-rolled sense-reversing barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* sink) {
    cg::grid_group g = cg::this_grid();
    double acc = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        acc = acc * 1.0000001 + 1.0;
        g.sync();
    }
    if (acc == -1.0) sink[0] = acc;
}

__device__ __forceinline__ void my_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks, unsigned& local_gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g = local_gen;
        __threadfence();
        unsigned arrived = atomicAdd(count, 1u);
        if (arrived == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicExch((unsigned*)gen, g + 1);
        } else {
            unsigned cur;
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(gen));
            } while (cur == g);
        }
        local_gen = g + 1;
    }
    __syncthreads();
}

__global__ void k_mine(int iters, double* sink, unsigned* count, unsigned* gen) {
    __shared__ unsigned lg;
    if (threadIdx.x == 0) lg = *((volatile unsigned*)gen);
    __syncthreads();
    unsigned local_gen = lg;
    double acc = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        acc = acc * 1.0000001 + 1.0;
        my_barrier(count, gen, gridDim.x, local_gen);
    }
    if (acc == -1.0) sink[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    unsigned *count, *gen;
    cudaMalloc(&sink, 8);
    cudaMalloc(&count, 4);
    cudaMalloc(&gen, 4);
    cudaMemset(count, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int threads : {256, 512, 1024}) {
        int iters = 2000;
        void* args[] = {&iters, &sink};
        cudaLaunchCooperativeKernel((void*)k_cg, sms, threads, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_cg, sms, threads, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cg grid.sync   blocks=%d threads=%d: %.3f us/sync\n", sms, threads, 1000.0 * ms / iters);
        void* args2[] = {&iters, &sink, &count, &gen};
        cudaLaunchCooperativeKernel((void*)k_mine, sms, threads, args2, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_mine, sms, threads, args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("custom barrier blocks=%d threads=%d: %.3f us/sync  (%s)\n", sms, threads, 1000.0 * ms / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
