// sa_scan.cu -- device-wide exclusive scan (int64) and error plumbing.
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sa_common.cuh"

namespace sa {

ErrState &err_state()
{
    static thread_local ErrState s;
    return s;
}

static const char *tune_find(const char *key, size_t *len)
{
    const char *t = getenv("SA_TUNE");
    if (!t) return nullptr;
    const size_t kl = strlen(key);
    for (const char *p = t; *p;) {
        const char *e = strchr(p, ',');
        const size_t n = e ? (size_t)(e - p) : strlen(p);
        if (n > kl && strncmp(p, key, kl) == 0 && p[kl] == '=') {
            *len = n - kl - 1;
            return p + kl + 1;
        }
        p += n + (e ? 1 : 0);
    }
    return nullptr;
}

int tune_int(const char *key, int dflt)
{
    size_t n = 0;
    const char *v = tune_find(key, &n);
    return v && n ? atoi(v) : dflt;
}

bool tune_is(const char *key, const char *value)
{
    size_t n = 0;
    const char *v = tune_find(key, &n);
    return v && n == strlen(value) && strncmp(v, value, n) == 0;
}

static void readback_drop_pending();

int set_error(int status, const char *fmt, ...)
{
    readback_drop_pending();   // an error return must not leave read-backs aimed at a dead frame
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err_state().msg = buf;
    return status;
}

// ---- read-backs through mapped pinned memory (sa_common.cuh) ---------------
namespace {
__global__ void k_readback(const unsigned long long *__restrict__ src, unsigned long long *__restrict__ dst, int nwords)
{
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = src[i];
}

struct ReadbackState {
    unsigned char *staging = nullptr;   // mapped pinned, RB_BYTES
    size_t used = 0;
    struct Item { void *dst; size_t off, n; };
    Item items[64];
    int nitems = 0;
};
constexpr size_t RB_BYTES = 4096;
ReadbackState &rb_state()
{
    static thread_local ReadbackState s;
    return s;
}
}  // namespace

static void readback_drop_pending()
{
    ReadbackState &r = rb_state();
    r.nitems = 0;
    r.used = 0;
}

int readback(void *host_dst, const void *dev_src, size_t bytes, cudaStream_t st)
{
    ReadbackState &r = rb_state();
    if (!r.staging) {
        void *p = nullptr;
        if (cudaHostAlloc(&p, RB_BYTES, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        r.staging = (unsigned char *)p;
    }
    if (!r.staging || bytes == 0 || bytes % 8 != 0 || ((uintptr_t)dev_src & 7) || r.used + bytes > RB_BYTES ||
        r.nitems == 64) {
        SA_CUDA_TRY(cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, st));
        return SA_OK;
    }
    k_readback<<<1, 32, 0, st>>>((const unsigned long long *)dev_src, (unsigned long long *)(r.staging + r.used),
                                 (int)(bytes / 8));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(SA_ERR_CUDA, "read-back launch failed: %s", cudaGetErrorString(e));
    r.items[r.nitems++] = {host_dst, r.used, bytes};
    r.used += bytes;
    return SA_OK;
}

int sync_stream(cudaStream_t st)
{
    ReadbackState &r = rb_state();
    cudaError_t e = cudaStreamSynchronize(st);
    // (delivered even after an error: the caller reports it)
    for (int i = 0; i < r.nitems; ++i) memcpy(r.items[i].dst, r.staging + r.items[i].off, r.items[i].n);
    r.nitems = 0;
    r.used = 0;
    if (e != cudaSuccess)
        return set_error(SA_ERR_CUDA, "cudaStreamSynchronize failed: %s", cudaGetErrorString(e));
    return SA_OK;
}

namespace {
constexpr int SCAN_BLOCK = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int64_t SCAN_TILE = (int64_t)SCAN_BLOCK * SCAN_ITEMS;

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// exclusive block scan of one value per thread; returns the block total in *total
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *total)
{
    __shared__ int64_t warp_sums[SCAN_BLOCK / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t inc = warp_incl_scan(v);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int64_t s = lane < SCAN_BLOCK / 32 ? warp_sums[lane] : 0;
        s = warp_incl_scan(s);
        if (lane < SCAN_BLOCK / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    int64_t base = wid ? warp_sums[wid - 1] : 0;
    *total = warp_sums[SCAN_BLOCK / 32 - 1];
    __syncthreads();
    return base + inc - v;
}

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_reduce(const int64_t *__restrict__ in, int64_t n,
                                                            int64_t *__restrict__ sums)
{
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        int64_t idx = base + (int64_t)i * SCAN_BLOCK + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    int64_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// each thread owns SCAN_ITEMS consecutive items of the tile
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_tiles(const int64_t *in, int64_t *out, int64_t n,
                                                           const int64_t *__restrict__ offs)
{
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        s += v[i];
    }
    int64_t tot;
    int64_t run = block_excl_scan(s, &tot) + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = (offs ? offs[blockIdx.x] : 0) + tot;
}
}  // namespace

int64_t scan_tmp_elems(int64_t n)
{
    if (n <= SCAN_TILE) return 1;
    int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    return (nb + 1) + scan_tmp_elems(nb);
}

int exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, int64_t *tmp, cudaStream_t st)
{
    if (n <= 0) {
        SA_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
        return SA_OK;
    }
    if (n <= SCAN_TILE) {
        SA_LAUNCH(k_scan_tiles, 1, SCAN_BLOCK, 0, st, in, out, n, (const int64_t *)nullptr);
        return SA_OK;
    }
    int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    int64_t *sums = tmp;
    SA_LAUNCH(k_scan_reduce, (unsigned)nb, SCAN_BLOCK, 0, st, in, n, sums);
    SA_TRY(exclusive_scan_i64(sums, sums, nb, tmp + nb + 1, st));
    SA_LAUNCH(k_scan_tiles, (unsigned)nb, SCAN_BLOCK, 0, st, in, out, n, (const int64_t *)sums);
    return SA_OK;
}

}  // namespace sa
