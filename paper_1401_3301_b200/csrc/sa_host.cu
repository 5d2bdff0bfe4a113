// sa_host.cu -- host side of the transfers: a small persistent thread pool
// and the two passes that run on it.
//
// The reference API hands over me as int64 (mesh.py:54-58) and takes column
// indices as int64 (sparse.py:53-55); the device keeps int32 (sa_mesh_create
// range-checks against nq < 2^31).  Crossing PCIe as int64 costs twice the
// bytes (C5: 3.2 GB of the 5.8 GB a call uploads), so
//  * sa_host_narrow_upload narrows rows of me to int32 -- checking the index
//    range in the same pass, since the narrowing would hide a bad high word --
//    into a pinned staging buffer, chunk by chunk; the thread that finishes a
//    chunk last enqueues its host->device copy, so the copies overlap the
//    narrowing of the later chunks (and the int64 upload of the rows the
//    caller sends as they are);
//  * sa_host_widen_i32 widens downloaded int32 indices to int64.
// The pool threads park on a condition variable between jobs (no spinning:
// they must not compete with the caller's own threads).
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "sa_common.cuh"

using namespace sa;

namespace {

class HostPool {
public:
    // run fn(t, T) on T threads (the caller is thread 0); returns when all are done
    void run(int T, const std::function<void(int, int)> &fn)
    {
        std::lock_guard<std::mutex> serial(run_mu_);   // one job at a time
        T = std::max(1, std::min(T, 64));
        grow(T - 1);
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            nthreads_ = T;
            pending_ = T - 1;
            ++generation_;
        }
        cv_.notify_all();
        fn(0, T);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }
    ~HostPool()
    {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++generation_;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }

private:
    void grow(int n)
    {
        while ((int)workers_.size() < n) {
            const int id = (int)workers_.size() + 1;
            uint64_t seen;
            {
                std::lock_guard<std::mutex> lk(mu_);
                seen = generation_;
            }
            workers_.emplace_back([this, id, seen]() mutable {
                for (;;) {
                    const std::function<void(int, int)> *fn;
                    int T;
                    {
                        std::unique_lock<std::mutex> lk(mu_);
                        cv_.wait(lk, [&] { return generation_ != seen; });
                        seen = generation_;
                        if (stop_) return;
                        fn = fn_;
                        T = nthreads_;
                    }
                    if (id < T) {
                        (*fn)(id, T);
                        std::lock_guard<std::mutex> lk(mu_);
                        if (--pending_ == 0) done_cv_.notify_one();
                    }
                }
            });
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> workers_;
    const std::function<void(int, int)> *fn_ = nullptr;
    int nthreads_ = 0, pending_ = 0;
    uint64_t generation_ = 0;
    bool stop_ = false;
};

HostPool &pool()
{
    static HostPool *p = new HostPool();   // never destroyed: no join at process exit
    return *p;
}

}  // namespace

extern "C" int sa_host_narrow_upload(const int64_t *src, int64_t n, int64_t nq, int32_t *staging, int32_t *dst_dev,
                                     int nthreads, int device, void *stream, int64_t *first_bad)
{
    if (first_bad) *first_bad = -1;
    if (n <= 0) return SA_OK;
    if (!src || !staging || !dst_dev) return set_error(SA_ERR_ARG, "sa_host_narrow_upload: NULL argument");
    const int64_t CH = (int64_t)4 << 20;   // entries per chunk (16 MB of int32)
    const int64_t nch = (n + CH - 1) / CH;
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(nthreads, 64), (n + (1 << 16) - 1) >> 16));
    std::unique_ptr<std::atomic<int>[]> done(new std::atomic<int>[nch]);
    for (int64_t c = 0; c < nch; ++c) done[c].store(0, std::memory_order_relaxed);
    std::atomic<int64_t> bad(INT64_MAX);
    std::atomic<int> cuda_err(0);
    cudaStream_t st = (cudaStream_t)stream;
    pool().run(T, [&](int t, int TT) {
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess || (cur != device && cudaSetDevice(device) != cudaSuccess)) cuda_err.store(1);
        for (int64_t c = 0; c < nch; ++c) {
            const int64_t c0 = c * CH, len = std::min(CH, n - c0);
            const int64_t i0 = c0 + len * t / TT, i1 = c0 + len * (t + 1) / TT;
            unsigned long long any = 0;
            for (int64_t i = i0; i < i1; ++i) {
                const int64_t x = src[i];
                staging[i] = (int32_t)x;
                any |= (unsigned long long)((uint64_t)x >= (uint64_t)nq);
            }
            if (any) {   // rare: locate the first bad entry of this slice
                for (int64_t i = i0; i < i1; ++i)
                    if ((uint64_t)src[i] >= (uint64_t)nq) {
                        int64_t cur_bad = bad.load();
                        while (i < cur_bad && !bad.compare_exchange_weak(cur_bad, i)) {}
                        break;
                    }
            }
            if (done[c].fetch_add(1, std::memory_order_acq_rel) == TT - 1) {
                if (cudaMemcpyAsync(dst_dev + c0, staging + c0, (size_t)len * sizeof(int32_t), cudaMemcpyHostToDevice, st) !=
                    cudaSuccess)
                    cuda_err.store(1);
            }
        }
    });
    if (cuda_err.load()) return set_error(SA_ERR_CUDA, "sa_host_narrow_upload: %s", cudaGetErrorString(cudaGetLastError()));
    if (bad.load() != INT64_MAX && first_bad) *first_bad = bad.load();
    return SA_OK;
}

extern "C" int sa_host_widen_i32(const int32_t *src, int64_t n, int64_t offset, int64_t *dst, int nthreads)
{
    if (n <= 0) return SA_OK;
    if (!src || !dst) return set_error(SA_ERR_ARG, "sa_host_widen_i32: NULL argument");
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(nthreads, 64), (n + (1 << 16) - 1) >> 16));
    pool().run(T, [&](int t, int TT) {
        const int64_t i0 = n * t / TT, i1 = n * (t + 1) / TT;
        for (int64_t i = i0; i < i1; ++i) dst[i] = (int64_t)src[i] + offset;
    });
    return SA_OK;
}
