// Throughput of the cost kernel's non-FP64 per-element operations on one B200:
// float->double and double->float conversions (F2F, XU pipe), 64-bit POPC, and
// integer restatements of the two conversions. Each thread runs 8 independent
// chains; the result is lane-operations per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu_pipe xu_pipe.cu
#include <cstdint>
#include <cstdio>

constexpr int kIters = 4096, kChains = 8;

__global__ void k_f2d(float* out, float seed) {
    float v[kChains];
    double acc[kChains];
    for (int c = 0; c < kChains; ++c) v[c] = seed + threadIdx.x * 1e-7f + c, acc[c] = 0;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            const double d = static_cast<double>(v[c]);
            v[c] = __int_as_float(__float_as_int(v[c]) ^ static_cast<int>(__double2hiint(d)));
        }
    float s = 0;
    for (int c = 0; c < kChains; ++c) s += v[c] + static_cast<float>(acc[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_d2f(float* out, double seed) {
    double v[kChains];
    for (int c = 0; c < kChains; ++c) v[c] = seed + threadIdx.x * 1e-9 + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            const float f = __double2float_rn(v[c]);
            v[c] = __hiloint2double(__double2hiint(v[c]), __double2loint(v[c]) ^ __float_as_int(f));
        }
    float s = 0;
    for (int c = 0; c < kChains; ++c) s += static_cast<float>(v[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_popc(float* out, uint64_t seed) {
    uint64_t v[kChains];
    for (int c = 0; c < kChains; ++c) v[c] = seed * (threadIdx.x + 1) + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) v[c] ^= static_cast<uint64_t>(__popcll(v[c]));
    float s = 0;
    for (int c = 0; c < kChains; ++c) s += static_cast<float>(v[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// integer float->double for 0 or normal |x|
__device__ __forceinline__ double f2d_int(uint32_t b) {
    const uint32_t hi = b ? (b >> 3) + 0x38000000u : 0u;
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(b << 29));
}
// integer RN double->float for v = 0, a denormal double, or v >= 2^-126 (finite, positive)
__device__ __forceinline__ float d2f_int(double v) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    const uint64_t t = b + 0x0FFFFFFFull + ((b >> 29) & 1u);
    const uint32_t f = static_cast<uint32_t>(t >> 29) - (896u << 23);
    return __uint_as_float(static_cast<uint32_t>(b >> 32) ? f : 0u);
}

__global__ void k_f2d_int(float* out, float seed) {
    float v[kChains];
    for (int c = 0; c < kChains; ++c) v[c] = seed + threadIdx.x * 1e-7f + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            const double d = f2d_int(__float_as_uint(v[c]));
            v[c] = __int_as_float(__float_as_int(v[c]) ^ (__double2hiint(d) & 0x7));
        }
    float s = 0;
    for (int c = 0; c < kChains; ++c) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_d2f_int(float* out, double seed) {
    double v[kChains];
    for (int c = 0; c < kChains; ++c) v[c] = seed + threadIdx.x * 1e-9 + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            const float f = d2f_int(v[c]);
            v[c] = __hiloint2double(__double2hiint(v[c]), __double2loint(v[c]) ^ (__float_as_int(f) & 0xff));
        }
    float s = 0;
    for (int c = 0; c < kChains; ++c) s += static_cast<float>(v[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 8, threads = 256;
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = 5.0 * blocks * threads * kIters * kChains;
        const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
        printf("%-10s %8.3f ms  %7.1f ops/clk/SM (at the %d MHz max clock)\n", name, ms, per_clk_sm, clk / 1000);
    };
    run("f2d", [&] { k_f2d<<<blocks, threads>>>(out, 0.5f); });
    run("d2f", [&] { k_d2f<<<blocks, threads>>>(out, 0.5); });
    run("popc64", [&] { k_popc<<<blocks, threads>>>(out, 0x9E3779B97F4A7C15ull); });
    run("f2d_int", [&] { k_f2d_int<<<blocks, threads>>>(out, 0.5f); });
    run("d2f_int", [&] { k_d2f_int<<<blocks, threads>>>(out, 0.5); });
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
