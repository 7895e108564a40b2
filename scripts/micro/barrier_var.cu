// Microbenchmark: variants of the grid barrier-reduce (grid_reduce.cuh) at
// 148 blocks x {640, 1024} threads, K = 10 values: the arrival-stripe count S
// and the poll (ld.acquire per poll, or relaxed polls + one fence).
#include <cstdio>

#include "../../paper_2203_02300_b200/csrc/grid_reduce.cuh"
using namespace dco_gpu;

struct Bar16 {
    unsigned count[16][32];
};

template <int K, int S, bool RELAXED>
__device__ __forceinline__ void bar_var(double (&v)[K], Bar16* bar, double* partials, unsigned& gen, double* sm,
                                        double (&res)[K]) {
    constexpr int P = ReducePad<K>::P;
    const int nb = gridDim.x, bid = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* table = partials + (gen & 1u) * (static_cast<size_t>(nb) * 16);
    {
        double u[P];
#pragma unroll
        for (int k = 0; k < P; ++k) u[k] = k < K ? v[k] : 0.0;
        warp_halving_reduce<P>(u, lane);
        constexpr int low = 32 / P;
        if ((lane & (low - 1)) == 0) sm[warp * P + grid_reduce_index<P>(lane)] = u[0];
    }
    __syncthreads();
    if (warp == 0) {
        constexpr int groups = 32 / P;
        const int k = lane % P, g = lane / P;
        double s = 0.0;
        for (int w = g; w < nw; w += groups) s += sm[w * P + k];
#pragma unroll
        for (int off = 16; off >= P; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane < K) __stcg(table + static_cast<size_t>(lane) * nb + bid, s);
        __syncwarp();
        if (lane == 0)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&bar->count[bid % S][0]) : "memory");
        if (lane < S) {
            const unsigned members = static_cast<unsigned>((nb - lane + S - 1) / S);
            const unsigned target = members * (gen + 1u);
            unsigned c;
            if (RELAXED) {
                do {
                    asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(c) : "l"(&bar->count[lane][0]) : "memory");
                } while (c < target);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else {
                do {
                    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(c) : "l"(&bar->count[lane][0]) : "memory");
                } while (c < target);
            }
        }
        __syncwarp();
    }
    __syncthreads();
    double* sres = sm + 32 * 16 - 16;
    if (warp < K) {
        double s = 0.0;
        for (int b = lane; b < nb; b += 32) s += __ldcg(table + static_cast<size_t>(warp) * nb + b);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) sres[warp] = s;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) res[k] = sres[k];
    ++gen;
    __syncthreads();
}

template <int K, int S, bool RELAXED, int T>
__global__ void __launch_bounds__(T, 1) k_bar(int iters, Bar16* count, double* part, double* sink) {
    __shared__ double sm[32 * 16];
    unsigned gen = 0;
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
        double res[K];
        bar_var<K, S, RELAXED>(v, count, part, gen, sm, res);
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = res[k] * 1e-9 + k;
    }
    if (threadIdx.x == 0 && v[0] == -1.0) sink[0] = v[0];
}

template <int S, bool RELAXED, int T>
void run(Bar16* count, double* part, double* sink) {
    int nb = 0;
    cudaDeviceGetAttribute(&nb, cudaDevAttrMultiProcessorCount, 0);
    int iters = 2000;
    void* params[] = {&iters, &count, &part, &sink};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(count, 0, sizeof(Bar16));
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_bar<10, S, RELAXED, T>, dim3(nb), dim3(T), params, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    printf("threads %4d stripes %2d %s: %.3f us per barrier_reduce (K=10)\n", T, S, RELAXED ? "relaxed+fence" : "acquire      ",
           best * 1e3 / iters);
}

int main() {
    Bar16* count;
    double *part, *sink;
    cudaMalloc(&count, sizeof(Bar16));
    cudaMalloc(&part, 2 * 1024 * 16 * 8);
    cudaMalloc(&sink, 8);
    run<8, false, 1024>(count, part, sink);
    run<8, false, 640>(count, part, sink);
    run<8, true, 640>(count, part, sink);
    run<1, false, 640>(count, part, sink);
    run<2, false, 640>(count, part, sink);
    run<4, false, 640>(count, part, sink);
    run<16, false, 640>(count, part, sink);
    run<16, true, 640>(count, part, sink);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
