// Deterministic grid-wide barrier + all-reduce of K doubles for persistent
// cooperative kernels (one block per SM). Every block ends with bit-identical
// sums: the reduction tree has a fixed shape that does not depend on arrival
// order.
//
//  1. warp level: recursive halving. With P = K rounded up to a power of two,
//     each butterfly level exchanges half of the remaining values, so a warp
//     reduces P values with P/2 + P/4 + ... + 1 shuffles (not 5 K).
//  2. block level: warp 0 sums the per-warp rows in shared memory and writes
//     the block's row into a transposed partial table partials[k][block].
//  3. arrival on monotonic counters (never reset inside a launch: barrier g
//     completes when every stripe's count reaches members * (g + 1));
//     release / acquire at gpu scope.
//     Two partial tables alternate, so a block one barrier ahead never
//     overwrites a row still being read.
//  4. every block sums all rows itself, value k on warp k, coalesced loads.
#pragma once

namespace dco_gpu {

// Arrival counters striped over kGridBarStripes cache lines: same-address
// atomics serialise at their L2 slice, so block b arrives on stripe b % S.
constexpr int kGridBarStripes = 8;
struct GridBar {
    unsigned count[kGridBarStripes][32];  // one 128 B line per stripe
};

template <int K>
struct ReducePad {
    static constexpr int P = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : 16;
};

// Recursive-halving warp reduction: on return v[0] of lane L holds the warp
// total of value index grid_reduce_index<P>(L).
template <int P>
__device__ __forceinline__ void warp_halving_reduce(double (&v)[P], int lane) {
    int cnt = P;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        if (cnt > 1) {
            const bool up = (lane & off) != 0;
            const int half = cnt >> 1;
#pragma unroll
            for (int i = 0; i < P / 2; ++i) {
                if (i < half) {
                    const double send = up ? v[i] : v[i + half];
                    const double keep = up ? v[i + half] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
            }
            cnt = half;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
        }
    }
}

template <int P>
__device__ __forceinline__ int grid_reduce_index(int lane) {
    int idx = 0, cnt = P;
#pragma unroll
    for (int off = 16; off > 0 && cnt > 1; off >>= 1) {
        cnt >>= 1;
        if (lane & off) idx += cnt;
    }
    return idx;
}

// sm: >= 32 * 16 doubles of shared scratch. partials: 2 * 16 * gridDim.x doubles.
// kTailSync = false skips the closing CTA barrier: the caller guarantees a
// __syncthreads() before sm is written again.
// nb / bid: the participating blocks and this block's index among them (the
// whole grid, or one rank's group of blocks in the row-band solver).
template <int K, bool kTailSync = true>
__device__ __forceinline__ void barrier_reduce_of(double (&v)[K], GridBar* bar, double* partials, unsigned& gen,
                                                  double* sm, double (&res)[K], int nb, int bid) {
    constexpr int P = ReducePad<K>::P;
    static_assert(K <= 16, "at most 16 values per reduction");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* table = partials + (gen & 1u) * (static_cast<size_t>(nb) * 16);
    // 1. warp level
    {
        double u[P];
#pragma unroll
        for (int k = 0; k < P; ++k) u[k] = k < K ? v[k] : 0.0;
        warp_halving_reduce<P>(u, lane);
        constexpr int low = 32 / P;  // lanes sharing one index
        if ((lane & (low - 1)) == 0) sm[warp * P + grid_reduce_index<P>(lane)] = u[0];
    }
    __syncthreads();
    // 2. block level (warp 0): lane l sums index l % P over warps l / P, l / P + 32 / P, ...
    if (warp == 0) {
        constexpr int groups = 32 / P;
        const int k = lane % P, g = lane / P;
        double s = 0.0;
        for (int w = g; w < nw; w += groups) s += sm[w * P + k];
#pragma unroll
        for (int off = 16; off >= P; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane < K) __stcg(table + static_cast<size_t>(lane) * nb + bid, s);
        __syncwarp();
        // 3. arrive on this block's stripe; lanes 0..S-1 each wait for one stripe
        if (lane == 0)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&bar->count[bid % kGridBarStripes][0])
                         : "memory");
        if (lane < kGridBarStripes) {
            const unsigned members = static_cast<unsigned>((nb - lane + kGridBarStripes - 1) / kGridBarStripes);
            const unsigned target = members * (gen + 1u);
            unsigned c;
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(c) : "l"(&bar->count[lane][0]) : "memory");
            } while (c < target);
        }
        __syncwarp();
    }
    __syncthreads();
    // 4. value k on warp k: coalesced loads of row k, fixed-order tree
    // step 2's reads finished before the barrier; the top 16 slots stay clear
    // of a following K <= 2 step 1 when kTailSync = false
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
    if (kTailSync) __syncthreads();  // sm reused by the next reduction
}

template <int K, bool kTailSync = true>
__device__ __forceinline__ void barrier_reduce(double (&v)[K], GridBar* bar, double* partials, unsigned& gen,
                                               double* sm, double (&res)[K]) {
    barrier_reduce_of<K, kTailSync>(v, bar, partials, gen, sm, res, static_cast<int>(gridDim.x),
                                    static_cast<int>(blockIdx.x));
}

}  // namespace dco_gpu
