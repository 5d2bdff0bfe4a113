// sa_pk.cuh -- Pk mass matrix on the B200, included by
// the C-ABI translation unit (sa_core.cu with SA_ABI).
//
// Reference: assemble_mass_pk (assembly.py:265-292): every local entry is
// (d! C[a][b]) * |K| with an element-independent table C, triplets
// element-major, canonicalised by sparse_from_triplets (sparse.py:85-133).
// Same contract as the P1 path: each CSR entry is the left-to-right sum of
// its contributions in ascending element order (bitwise optv2-style), exact
// zero sums dropped by sa_pk_compact.  ndfe = (d+k)!/(d!k!) lattice nodes
// per element (<= 84), at most 255 distinct neighbours per node.
//
// Symbolic (once per lattice mesh): node -> (element, local node) incidences
// sorted by element, sorted unique neighbour nodes per node, and per
// incidence the 8-bit column rank of each of the element's nodes.
// Numeric: one thread per node row, private shared-memory accumulators
// indexed by rank, (d! C[a][b]) * vol folded per incidence.

struct sa_pk_plan {
    int device = 0;
    int ndfe = 0;
    int64_t nq = 0, nme = 0, n_inc = 0, nnz = 0, max_deg = 0;
    int32_t *me = nullptr;        // (ndfe, nme) int32
    int64_t *inc_ptr = nullptr;   // (nq+1)
    uint2 *inc = nullptr;         // (n_inc): x = element, y = local node
    int64_t *colptr = nullptr;    // (nq+1) == CSR indptr (one dof per node)
    int32_t *cols = nullptr;      // (nnz) sorted neighbour nodes == CSR indices
    uint8_t *rank = nullptr;      // (n_inc * ndfe)
    int64_t *counters = nullptr;  // [0] zero count, [1] capacity flag, [2] max degree, [3] bad index
    int64_t *scan_tmp = nullptr;
};

namespace {

__global__ void k_pk_pack(const int64_t *__restrict__ me, int64_t n, int64_t nq, int32_t *__restrict__ out,
                          unsigned long long *bad)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = me[i];
        if (v < 0 || v >= nq) atomicMin(bad, (unsigned long long)i);
        out[i] = (int32_t)v;
    }
}

__global__ void k_pk_count(const int32_t *__restrict__ me, int ndfe, int64_t nme, unsigned long long *__restrict__ cnt)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= nme) return;
    for (int a = 0; a < ndfe; ++a) atomicAdd(cnt + me[a * nme + e], 1ull);
}

__global__ void k_pk_fill(const int32_t *__restrict__ me, int ndfe, int64_t nme, const int64_t *__restrict__ inc_ptr,
                          unsigned long long *__restrict__ cursor, uint2 *__restrict__ inc)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= nme) return;
    for (int a = 0; a < ndfe; ++a) {
        const int v = me[a * nme + e];
        inc[inc_ptr[v] + (int64_t)atomicAdd(cursor + v, 1ull)] = make_uint2((unsigned)e, (unsigned)a);
    }
}

// ascending element order per node (insertion sort; few incidences per node)
__global__ void k_pk_sort(const int64_t *__restrict__ inc_ptr, int64_t nq, uint2 *__restrict__ inc)
{
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= nq) return;
    const int64_t t0 = inc_ptr[v], t1 = inc_ptr[v + 1];
    for (int64_t t = t0 + 1; t < t1; ++t) {
        const uint2 x = inc[t];
        int64_t u = t - 1;
        while (u >= t0 && inc[u].x > x.x) { inc[u + 1] = inc[u]; --u; }
        inc[u + 1] = x;
    }
}

// sorted unique neighbours of node v (cols == nullptr: count only); then
// (ranks != nullptr) the column rank of every node of every incidence
__global__ void k_pk_cols(const int32_t *__restrict__ me, int ndfe, int64_t nme, const int64_t *__restrict__ inc_ptr,
                          const uint2 *__restrict__ inc, int64_t nq, int64_t *__restrict__ ncol,
                          const int64_t *__restrict__ colptr, int32_t *__restrict__ cols, uint8_t *__restrict__ rank,
                          unsigned long long *cap)
{
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= nq) return;
    int buf[255];
    int n = 0;
    const int64_t t0 = inc_ptr[v], t1 = inc_ptr[v + 1];
    for (int64_t t = t0; t < t1; ++t) {
        const int64_t e = inc[t].x;
        for (int a = 0; a < ndfe; ++a) {
            const int x = me[a * nme + e];
            int lo = 0, hi = n;
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (buf[mid] < x) lo = mid + 1; else hi = mid; }
            if (lo < n && buf[lo] == x) continue;
            if (n == 255) { atomicOr(cap, 1ull); return; }
            for (int u = n; u > lo; --u) buf[u] = buf[u - 1];
            buf[lo] = x;
            ++n;
        }
    }
    if (!cols) { ncol[v] = n; return; }
    const int64_t c0 = colptr[v];
    for (int u = 0; u < n; ++u) cols[c0 + u] = buf[u];
    for (int64_t t = t0; t < t1; ++t) {
        const int64_t e = inc[t].x;
        for (int a = 0; a < ndfe; ++a) {
            const int x = me[a * nme + e];
            int lo = 0, hi = n;
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (buf[mid] < x) lo = mid + 1; else hi = mid; }
            rank[t * ndfe + a] = (uint8_t)lo;
        }
    }
}

// one thread per node row, accumulators acc[k][thread] in shared memory
__global__ void k_pk_mass(const int64_t *__restrict__ inc_ptr, const uint2 *__restrict__ inc,
                          const uint8_t *__restrict__ rank, const int64_t *__restrict__ colptr, int ndfe, int64_t nq,
                          const double *__restrict__ cs, const double *__restrict__ vols, double *__restrict__ vals,
                          unsigned long long *zeros)
{
    extern __shared__ double acc[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t v = blockIdx.x * (int64_t)nt + tid;
    int nz = 0;
    if (v < nq) {
        const int64_t c0 = colptr[v];
        const int deg = (int)(colptr[v + 1] - c0);
        for (int k = 0; k < deg; ++k) acc[k * nt + tid] = 0.0;
        const int64_t t0 = inc_ptr[v], t1 = inc_ptr[v + 1];
        for (int64_t t = t0; t < t1; ++t) {
            const uint2 r = __ldg(inc + t);
            const double vol = __ldg(vols + r.x);
            const double *row = cs + (int64_t)r.y * ndfe;
            const uint8_t *rk = rank + t * ndfe;
            for (int b = 0; b < ndfe; ++b) {
                double &s = acc[(int)__ldg(rk + b) * nt + tid];
                s = __dadd_rn(s, __dmul_rn(__ldg(row + b), vol));   // (d! C[a][b]) * |K|, folded in element order
            }
        }
        for (int k = 0; k < deg; ++k) {
            const double x = acc[k * nt + tid];
            vals[c0 + k] = x;
            nz += x == 0.0;
        }
    }
    for (int s = 16; s > 0; s >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, s);
    if ((tid & 31) == 0 && nz) atomicAdd(zeros, (unsigned long long)nz);
}

}  // namespace

extern "C" {

int sa_pk_plan_destroy(sa_pk_plan *P)
{
    if (!P) return SA_OK;
    free_all({P->me, P->inc_ptr, P->inc, P->colptr, P->cols, P->rank, P->counters, P->scan_tmp});
    delete P;
    return SA_OK;
}

int sa_pk_plan_create(int ndfe, int64_t nq, int64_t nme, const int64_t *me_dev, int device, void *stream,
                      sa_pk_plan **out)
{
    err_state().msg.clear();
    err_state().bad = -1;
    if (!out) return set_error(SA_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (ndfe < 2 || ndfe > 84) return set_error(SA_ERR_ARG, "ndfe must be in [2, 84], got %d", ndfe);
    if (nq < 0 || nme < 0) return set_error(SA_ERR_ARG, "negative sizes");
    if (nq >= ((int64_t)1 << 31) || nme >= ((int64_t)1 << 31) || (int64_t)ndfe * nme >= ((int64_t)1 << 40))
        return set_error(SA_ERR_CAPACITY, "lattice mesh nq=%lld nme=%lld exceeds the index range", (long long)nq,
                         (long long)nme);
    SA_TRY(set_device(device));
    pool_keep_memory(device);
    cudaStream_t st = (cudaStream_t)stream;
    sa_pk_plan *P = new sa_pk_plan();
    P->device = device; P->ndfe = ndfe; P->nq = nq; P->nme = nme;
    auto fail = [&](int r) {
        std::string msg = err_state().msg;
        cudaStreamSynchronize(st);
        sa_pk_plan_destroy(P);
        err_state().msg = msg;
        return r;
    };
    const int64_t nm = (int64_t)ndfe * nme;
    if (cudaMallocAsync((void **)&P->me, std::max<int64_t>(nm, 1) * sizeof(int32_t), st) != cudaSuccess ||
        cudaMallocAsync((void **)&P->counters, 8 * sizeof(int64_t), st) != cudaSuccess ||
        cudaMallocAsync((void **)&P->inc_ptr, (nq + 1) * sizeof(int64_t), st) != cudaSuccess ||
        cudaMallocAsync((void **)&P->colptr, (nq + 1) * sizeof(int64_t), st) != cudaSuccess ||
        cudaMallocAsync((void **)&P->scan_tmp, (scan_tmp_elems(nq + 1) + 1) * sizeof(int64_t), st) != cudaSuccess)
        return fail(set_error(SA_ERR_NOMEM, "device allocation failed"));
    int64_t *cnt = nullptr;
    if (cudaMallocAsync((void **)&cnt, (nq + 1) * sizeof(int64_t), st) != cudaSuccess)
        return fail(set_error(SA_ERR_NOMEM, "device allocation failed"));
    auto run = [&]() -> int {
        unsigned long long *c = (unsigned long long *)P->counters;
        SA_CUDA_TRY(cudaMemsetAsync(P->counters, 0, 8 * sizeof(int64_t), st));
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 3, 0xff, sizeof(int64_t), st));
        if (nm) SA_LAUNCH(k_pk_pack, std::min<int64_t>(grid_for(nm, 256), 148 * 32), 256, 0, st, me_dev, nm, nq, P->me,
                          c + 3);
        int64_t h[4];
        SA_TRY(readback(h, P->counters, 4 * sizeof(int64_t), st));
        SA_TRY(sync_stream(st));
        if (h[3] != -1) {
            err_state().bad = h[3];
            return set_error(SA_ERR_INDEX_RANGE, "connectivity entry me[%lld, %lld] out of range [0, %lld)",
                             (long long)(h[3] / nme), (long long)(h[3] % nme), (long long)nq);
        }
        SA_CUDA_TRY(cudaMemsetAsync(cnt, 0, (nq + 1) * sizeof(int64_t), st));
        if (nme) SA_LAUNCH(k_pk_count, grid_for(nme, 128), 128, 0, st, P->me, ndfe, nme, (unsigned long long *)cnt);
        SA_TRY(exclusive_scan_i64(cnt, P->inc_ptr, nq, P->scan_tmp, st));
        SA_TRY(readback(&P->n_inc, P->inc_ptr + nq, sizeof(int64_t), st));
        SA_TRY(sync_stream(st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->inc, std::max<int64_t>(P->n_inc, 1) * sizeof(uint2), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->rank, std::max<int64_t>(P->n_inc * ndfe, 1), st));
        SA_CUDA_TRY(cudaMemsetAsync(cnt, 0, (nq + 1) * sizeof(int64_t), st));
        if (nme) SA_LAUNCH(k_pk_fill, grid_for(nme, 128), 128, 0, st, P->me, ndfe, nme, P->inc_ptr,
                           (unsigned long long *)cnt, P->inc);
        if (nq) {
            SA_LAUNCH(k_pk_sort, grid_for(nq, 128), 128, 0, st, P->inc_ptr, nq, P->inc);
            SA_LAUNCH(k_pk_cols, grid_for(nq, 128), 128, 0, st, P->me, ndfe, nme, P->inc_ptr, P->inc, nq, cnt,
                      (const int64_t *)nullptr, (int32_t *)nullptr, (uint8_t *)nullptr, c + 1);
        }
        SA_TRY(exclusive_scan_i64(cnt, P->colptr, nq, P->scan_tmp, st));
        if (nq) SA_LAUNCH(k_max_diff, std::min<int64_t>(grid_for(nq, 256), 148 * 8), 256, 0, st, P->colptr, nq, c + 2);
        SA_TRY(readback(h, P->counters, 4 * sizeof(int64_t), st));
        SA_TRY(readback(&P->nnz, P->colptr + nq, sizeof(int64_t), st));
        SA_TRY(sync_stream(st));
        if (h[1]) return set_error(SA_ERR_CAPACITY, "a lattice node has more than 255 distinct neighbours");
        if (P->nnz >= ((int64_t)1 << 31)) return set_error(SA_ERR_CAPACITY, "int32 column indices overflow");
        P->max_deg = h[2];
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->cols, std::max<int64_t>(P->nnz, 1) * sizeof(int32_t), st));
        if (nq) SA_LAUNCH(k_pk_cols, grid_for(nq, 128), 128, 0, st, P->me, ndfe, nme, P->inc_ptr, P->inc, nq, cnt,
                          (const int64_t *)P->colptr, P->cols, P->rank, c + 1);
        SA_CUDA_TRY(cudaFreeAsync(cnt, st));
        SA_TRY(sync_stream(st));
        return SA_OK;
    };
    const int rc = run();
    if (rc != SA_OK) return fail(rc);
    *out = P;
    return SA_OK;
}

int sa_pk_plan_info(const sa_pk_plan *P, int64_t *nnz, int64_t *max_row_nodes)
{
    if (!P) return set_error(SA_ERR_ARG, "plan is NULL");
    if (nnz) *nnz = P->nnz;
    if (max_row_nodes) *max_row_nodes = P->max_deg;
    return SA_OK;
}

int sa_pk_plan_pattern(const sa_pk_plan *P, int64_t *indptr_dev, int32_t *indices_dev, void *stream)
{
    if (!P) return set_error(SA_ERR_ARG, "plan is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    if (indptr_dev)
        SA_CUDA_TRY(cudaMemcpyAsync(indptr_dev, P->colptr, (P->nq + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    if (indices_dev && P->nnz)
        SA_CUDA_TRY(cudaMemcpyAsync(indices_dev, P->cols, P->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    return SA_OK;
}

int sa_pk_mass(sa_pk_plan *P, const double *cs_dev, const double *vols_dev, double *vals_dev, int64_t *n_zero_out,
               void *stream)
{
    if (!P || !cs_dev || !vols_dev || !vals_dev) return set_error(SA_ERR_ARG, "NULL argument");
    SA_TRY(set_device(P->device));
    cudaStream_t st = (cudaStream_t)stream;
    SA_CUDA_TRY(cudaMemsetAsync(P->counters, 0, sizeof(int64_t), st));
    int block = 128;
    while ((size_t)std::max<int64_t>(P->max_deg, 1) * block * sizeof(double) > 100 * 1024 && block > 32) block /= 2;
    const size_t smem = (size_t)std::max<int64_t>(P->max_deg, 1) * block * sizeof(double);
    SA_CUDA_TRY(cudaFuncSetAttribute(k_pk_mass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (P->nq)
        SA_LAUNCH(k_pk_mass, grid_for(P->nq, block), block, smem, st, P->inc_ptr, P->inc, P->rank, P->colptr,
                  P->ndfe, P->nq, cs_dev, vols_dev, vals_dev, (unsigned long long *)P->counters);
    if (n_zero_out) {
        SA_TRY(readback(n_zero_out, P->counters, sizeof(int64_t), st));
        SA_TRY(sync_stream(st));
    }
    return SA_OK;
}

int sa_pk_compact(const sa_pk_plan *P, const double *vals_dev, int64_t *indptr_out, int32_t *indices_out,
                  double *vals_out, void *stream)
{
    if (!P) return set_error(SA_ERR_ARG, "plan is NULL");
    SA_TRY(set_device(P->device));
    cudaStream_t st = (cudaStream_t)stream;
    return compact_csr(P->colptr, P->cols, vals_dev, P->nq, P->nnz, P->scan_tmp, indptr_out, indices_out, vals_out, st);
}

}  // extern "C"
