// Microbenchmark: monotonic-counter grid barrier + fixed-order all-reduce of K
// doubles (the PCG's barrier_reduce), 148 x 1024 threads, with and without a
// burst of global stores before each barrier.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;

#include "../../paper_2203_02300_b200/csrc/grid_reduce.cuh"
using namespace dco_gpu;

template <int K>
__global__ void __launch_bounds__(1024, 1) k_bar(int iters, int stores, GridBar* count, double* part, double* buf,
                                                  double* sink) {
    __shared__ double sm[32 * 16];
    unsigned gen = 0;
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
        for (int s = 0; s < stores; ++s)
            __stcg(buf + (static_cast<size_t>(blockIdx.x) * stores + s) * 1024 + threadIdx.x, v[0]);
        double res[K];
        barrier_reduce<K>(v, count, part, gen, sm, res);
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = res[k] * 1e-9 + k;
    }
    if (threadIdx.x == 0 && v[0] == -1.0) sink[0] = v[0];
}

template <int K>
void run(int stores, GridBar* count, double* part, double* buf, double* sink) {
    int nb = 0;
    cudaDeviceGetAttribute(&nb, cudaDevAttrMultiProcessorCount, 0);
    if (const char* e = getenv("NB")) nb = atoi(e);  // fewer blocks (e.g. one per cluster of 2)
    int iters = 2000;
    void* params[] = {&iters, &stores, &count, &part, &buf, &sink};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(count, 0, sizeof(GridBar));
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_bar<K>, dim3(nb), dim3(1024), params, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("K=%2d stores/thread=%d: %.3f us per barrier_reduce\n", K, stores, ms * 1e3 / iters);
}

int main() {
    GridBar* count;
    double *part, *buf, *sink;
    cudaMalloc(&count, sizeof(GridBar));
    cudaMalloc(&part, 2 * 1024 * 16 * 8);
    cudaMalloc(&buf, 148ull * 8 * 1024 * 8);
    cudaMalloc(&sink, 8);
    for (int st : {0, 2, 8}) {
        run<1>(st, count, part, buf, sink);
        run<2>(st, count, part, buf, sink);
        run<3>(st, count, part, buf, sink);
        run<5>(st, count, part, buf, sink);
        run<10>(st, count, part, buf, sink);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
