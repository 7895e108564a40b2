// common.cuh — context, error plumbing and launch helpers shared by every
// translation unit of libdco_gpu.so. Host code is C++17; device code targets
// sm_100a only and is compiled with --fmad=false so that every float/double
// expression rounds exactly like the reference's x86-64 build (no FMA
// contraction there). Where the reference's libm is involved
// the glibc replicas in dco_libm.h are used.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "dco_gpu.h"

namespace dco_gpu {

// Status-carrying exception: thrown by host code, converted to the C status
// (and the context's last_error) at the C-ABI edge.
struct Failure : std::runtime_error {
    int status;
    Failure(int st, const std::string& msg) : std::runtime_error(msg), status(st) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Failure(status, msg); }
inline void require(bool ok, const std::string& msg) {
    if (!ok) fail(DCO_INPUT, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(DCO_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Grow-only device buffer: the context keeps one per scratch slot so the
// steady-state frame loop performs no allocation.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
};

enum Slot : int {
    S_ARM_RAW = 0,
    S_REGION,
    S_CENSUS,
    S_HSUM,
    S_COST,
    S_AGG,
    S_DISP0,
    S_DISP1,
    S_ARMS,
    S_SCALAR,
    S_FLOW_PYR,
    S_FLOW_PATCH,
    S_FLOW_ACC,
    S_FLOW_TMP,
    S_CONTOUR0,
    S_CONTOUR1,
    S_CONTOUR2,
    S_CONTOUR3,
    S_SAT,
    S_LABELS,
    S_CG,
    S_RED,
    S_STATS,
    S_TMP0,
    S_TMP1,
    S_FLAG_FLOW,
    S_FLAG_ARM,
    S_FLAG_BIN,
    S_FLAG_PEAK,
    S_FLAG_ASM,
    S_FLAG_SLICE,
    S_FLAG_DIV,
    S_RENDER,
    S_RENDER_LIST,
    S_HIST,
    S_STAGE,
    S_FIXLIST,
    S_BADROW,
    S_EXPORT,
    S_RUNS,
    S_COUNT
};

}  // namespace dco_gpu

struct dco_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    dco_gpu::DevBuf slots[dco_gpu::S_COUNT];
    void* pinned = nullptr;  // small pinned host staging area for scalar readbacks
    size_t pinned_bytes = 0;
    const char* last_solver = "";  // kernel instance of the last dense solve
};

namespace dco_gpu {

void* scratch(dco_ctx* ctx, Slot s, size_t bytes);
void* pinned_host(dco_ctx* ctx, size_t bytes);

// Raises fn's dynamic shared-memory cap to `bytes` (and the shared-memory
// carveout to 100 % when `carveout`) on the context's device, once per
// (device, kernel, size): function attributes are per device, so a process
// holding contexts on several GPUs sets them on each.
void smem_attr(dco_ctx* ctx, const void* fn, int bytes, bool carveout = false);
template <typename K>
inline void smem_attr(dco_ctx* ctx, K* fn, int bytes, bool carveout = false) {
    smem_attr(ctx, reinterpret_cast<const void*>(fn), bytes, carveout);
}
// Multiprocessor count of the context's device (cached per device).
int sm_count(dco_ctx* ctx);

// Counts and error-checks every launch made through it.
inline void launched(dco_ctx* ctx, const char* name) {
    ++ctx->launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(DCO_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
}

inline unsigned blocks_for(size_t n, unsigned threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

#ifdef __CUDACC__
// One global atomic per BLOCK instead of one per warp: same-address atomics
// serialise at their L2 slice, so a per-warp atomic over a full-frame grid
// (28 800 warps at 1280x720) costs more than the kernel's own work. Every
// thread of the block must call these (they contain __syncthreads); v is the
// thread's value, `skip` the identity the global update is not issued for.
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce_lane(T v, Op op, T ident) {
    __shared__ T s_red[32];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nw = (blockDim.x * blockDim.y * blockDim.z + 31) >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, off));
    if ((tid & 31) == 0) s_red[tid >> 5] = v;
    __syncthreads();
    T r = ident;
    if (tid < 32) {
        r = tid < nw ? s_red[tid] : ident;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) r = op(r, __shfl_xor_sync(0xffffffffu, r, off));
    }
    __syncthreads();  // s_red reusable
    return r;  // valid in thread 0
}
struct OpMax {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a > b ? a : b; }
};
struct OpMin {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a < b ? a : b; }
};
struct OpAdd {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a + b; }
};
__device__ __forceinline__ bool block_leader() { return (threadIdx.x | threadIdx.y | threadIdx.z) == 0; }
__device__ __forceinline__ void block_atomic_max(unsigned* g, unsigned v) {
    const unsigned r = block_reduce_lane(v, OpMax{}, 0u);
    if (block_leader() && r) atomicMax(g, r);
}
__device__ __forceinline__ void block_atomic_max(int* g, int v) {
    const int r = block_reduce_lane(v, OpMax{}, 0);
    if (block_leader() && r > 0) atomicMax(g, r);
}
__device__ __forceinline__ void block_atomic_min(int* g, int v, int ident) {
    const int r = block_reduce_lane(v, OpMin{}, ident);
    if (block_leader() && r != ident) atomicMin(g, r);
}
__device__ __forceinline__ void block_atomic_add(unsigned long long* g, unsigned long long v) {
    const unsigned long long r = block_reduce_lane(v, OpAdd{}, 0ull);
    if (block_leader() && r) atomicAdd(g, r);
}
#endif

// The C-ABI edge: runs fn, maps Failure/std::exception to status codes.
template <typename F>
int guarded(dco_ctx* ctx, F&& fn) {
    try {
        if (!ctx) return DCO_INPUT;
        // every entry point runs on the context's device, whatever the
        // calling thread's current device is
        cuda_check(cudaSetDevice(ctx->device), "set device");
        fn();
        return DCO_OK;
    } catch (const Failure& f) {
        ctx->err = f.what();
        return f.status;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return DCO_CUDA;
    }
}

void validate_config(const dco_config* cfg);  // PipelineConfig::validate, config.cpp:10-36

// Host-side precomputed tables (computed with the host libm exactly as the
// reference computes them, then uploaded):
//   alpha[l]   = adaptive_alpha(l)            stereo.cpp:102-104, l in 0..255
//   census[h]  = 1 - exp(-h/lambda_census)    stereo.cpp:125-127, h in 0..64
struct StereoTables {
    double alpha[256];
    double census[65];
};
void make_stereo_tables(const dco_config* cfg, StereoTables* t);

}  // namespace dco_gpu
