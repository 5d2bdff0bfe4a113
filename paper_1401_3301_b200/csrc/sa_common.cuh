// sa_common.cuh -- error plumbing, launch accounting and a small device scan.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/simplex_asm_b200.h"

namespace sa {

// thread-local error state behind sa_last_error() / sa_bad_index()
struct ErrState {
    std::string msg;
    int64_t bad = -1;
    int64_t launches = 0;
};
ErrState &err_state();

int set_error(int status, const char *fmt, ...);

#define SA_CUDA_TRY(expr)                                                                   \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return ::sa::set_error(SA_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,             \
                                   cudaGetErrorString(_e), __FILE__, __LINE__);            \
    } while (0)

#define SA_TRY(expr)                        \
    do {                                    \
        int _s = (expr);                    \
        if (_s != SA_OK) return _s;         \
    } while (0)

// launch + accounting; checks the launch error immediately
#define SA_LAUNCH(kernel, grid, block, smem, stream, ...)                                   \
    do {                                                                                    \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                         \
        ::sa::err_state().launches++;                                                       \
        cudaError_t _e = cudaGetLastError();                                                \
        if (_e != cudaSuccess)                                                              \
            return ::sa::set_error(SA_ERR_CUDA, "launch of %s failed: %s", #kernel,         \
                                   cudaGetErrorString(_e));                                 \
    } while (0)

// SA_TUNE="key=value,..." -- the library's single developer/test switch
// (keys: kernel=rowgather|twopass, symfast=0|1, winc=0|1); unset in
// production, every default is the measured best
int tune_int(const char *key, int dflt);
bool tune_is(const char *key, const char *value);

// Small device->host read-backs (sizes, counters, flags) that do not go
// through the copy engines: a one-warp kernel writes the words into mapped
// pinned host memory, and sync_stream() -- cudaStreamSynchronize plus the
// delivery of this thread's pending read-backs -- hands them over.  A
// cudaMemcpyAsync of 8 bytes queues behind every device->host copy submitted
// before it on ANY stream (measured: the library's plan construction stalled
// 20 ms behind a 1 GB pattern download running on another stream).
int readback(void *host_dst, const void *dev_src, size_t bytes, cudaStream_t st);
int sync_stream(cudaStream_t st);

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// Device-wide exclusive scan of int64 (in place allowed): out[i] = sum_{j<i} in[j],
// out[n] = total.  Three-phase reduce/scan/add, recursive on the block sums.
// `tmp` must hold scan_tmp_elems(n) int64.
int64_t scan_tmp_elems(int64_t n);
int exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, int64_t *tmp, cudaStream_t st);

}  // namespace sa
