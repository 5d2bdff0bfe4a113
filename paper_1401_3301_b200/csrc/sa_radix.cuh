// sa_radix.cuh -- stable LSD radix sort of (uint64 key, uint32 value) pairs.
//
// Hand-written (no CUB/Thrust).  One pass per 8-bit digit:
//   k_radix_hist     per-block digit histograms, bin-major [256][nblocks]
//   exclusive scan   over the flattened histogram -> global scatter offsets
//   k_radix_scatter  stable ranking: each warp walks its contiguous slice of
//                    the block's tile 32 keys at a time; __match_any_sync
//                    groups equal digits, the rank inside the group is the
//                    popcount of lower lanes, per-warp running bin counters
//                    live in shared memory, warps are combined in order.
// Used by the symbolic phase to group (chunk, entry) records by chunk.
#pragma once
#include "sa_common.cuh"

namespace sa {
namespace radix {
namespace {  // internal linkage: included by every per-dimension unit

constexpr int BLOCK = 256;
constexpr int WARPS = BLOCK / 32;
constexpr int ITEMS = 16;                      // keys per thread per tile
constexpr int TILE = BLOCK * ITEMS;            // 4096 keys per block
constexpr int WARP_TILE = TILE / WARPS;        // 512 keys per warp, in order

__global__ void __launch_bounds__(BLOCK) k_radix_hist(const uint64_t *__restrict__ keys, int64_t n, int shift,
                                                      int64_t nblocks, int64_t *__restrict__ hist)
{
    __shared__ unsigned cnt[256];
    for (int i = threadIdx.x; i < 256; i += BLOCK) cnt[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * TILE;
    for (int i = threadIdx.x; i < TILE; i += BLOCK) {
        const int64_t idx = base + i;
        if (idx < n) atomicAdd(&cnt[(keys[idx] >> shift) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += BLOCK) hist[(int64_t)i * nblocks + blockIdx.x] = cnt[i];
}

__global__ void __launch_bounds__(BLOCK) k_radix_scatter(const uint64_t *__restrict__ kin,
                                                         const uint32_t *__restrict__ vin, int64_t n, int shift,
                                                         int64_t nblocks, const int64_t *__restrict__ offs,
                                                         uint64_t *__restrict__ kout, uint32_t *__restrict__ vout)
{
    __shared__ unsigned wcnt[WARPS][256];   // per-warp digit counts, then per-warp bases
    __shared__ int64_t gbase[256];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < WARPS * 256; i += BLOCK) (&wcnt[0][0])[i] = 0;
    for (int i = threadIdx.x; i < 256; i += BLOCK) gbase[i] = offs[(int64_t)i * nblocks + blockIdx.x];
    __syncthreads();
    const int64_t wbase = (int64_t)blockIdx.x * TILE + (int64_t)wid * WARP_TILE;
    const unsigned lt = (1u << lane) - 1u;
    // pass 1: per-warp counts
    for (int j = 0; j < WARP_TILE; j += 32) {
        const int64_t idx = wbase + j + lane;
        const bool ok = idx < n;
        const unsigned dg = ok ? (unsigned)((kin[idx] >> shift) & 0xff) : 256u + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        if (ok && (peers & lt) == 0) wcnt[wid][dg] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps per digit (warps are in tile order)
    for (int d = threadIdx.x; d < 256; d += BLOCK) {
        unsigned run = 0;
        for (int w = 0; w < WARPS; ++w) {
            const unsigned c = wcnt[w][d];
            wcnt[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
    // pass 2: stable ranks and scatter
    for (int j = 0; j < WARP_TILE; j += 32) {
        const int64_t idx = wbase + j + lane;
        const bool ok = idx < n;
        const uint64_t k = ok ? kin[idx] : 0;
        const unsigned dg = ok ? (unsigned)((k >> shift) & 0xff) : 256u + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        if (ok) {
            const unsigned r = __popc(peers & lt);
            const int64_t pos = gbase[dg] + wcnt[wid][dg] + r;
            kout[pos] = k;
            vout[pos] = vin[idx];
        }
        __syncwarp();
        if (ok && (peers & lt) == 0) wcnt[wid][dg] += __popc(peers);
        __syncwarp();
    }
}

// Sort n pairs by the key bits [0, key_bits).  Returns the buffer index (0 or
// 1) that holds the result: (k0, v0) or (k1, v1).
inline int sort_pairs(uint64_t *k0, uint32_t *v0, uint64_t *k1, uint32_t *v1, int64_t n, int key_bits,
                      cudaStream_t st, int *which)
{
    *which = 0;
    if (n <= 1) return SA_OK;
    const int64_t nblocks = (n + TILE - 1) / TILE;
    const int64_t nh = 256 * nblocks;
    int64_t *hist = nullptr, *tmp = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&hist, (nh + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&tmp, (scan_tmp_elems(nh) + 1) * sizeof(int64_t), st));
    uint64_t *ki = k0, *ko = k1;
    uint32_t *vi = v0, *vo = v1;
    for (int shift = 0; shift < key_bits; shift += 8) {
        SA_LAUNCH(k_radix_hist, (unsigned)nblocks, BLOCK, 0, st, ki, n, shift, nblocks, hist);
        SA_TRY(exclusive_scan_i64(hist, hist, nh, tmp, st));
        SA_LAUNCH(k_radix_scatter, (unsigned)nblocks, BLOCK, 0, st, ki, vi, n, shift, nblocks, hist, ko, vo);
        std::swap(ki, ko);
        std::swap(vi, vo);
        *which ^= 1;
    }
    SA_CUDA_TRY(cudaFreeAsync(hist, st));
    SA_CUDA_TRY(cudaFreeAsync(tmp, st));
    return SA_OK;
}

}  // namespace
}  // namespace radix
}  // namespace sa
