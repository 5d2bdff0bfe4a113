// sa_core.cu -- device mesh, symbolic phase (K3) and numeric phase (K1+K2+K4+K5)
// behind the C ABI of include/simplex_asm_b200.h.
//
// Numeric design ("row gather"): one thread owns one mesh node, i.e. the m
// dof rows m*i+l of the block.  It walks the node's incident elements in
// ascending element order (the order the symbolic phase sorted them in),
// recomputes each element's geometry in registers (K1: bit-exact OpenBLAS
// LU/solve), forms the element row(s) it needs (K2) and folds them into its
// row accumulators.  Because every CSR entry is summed left to right in
// ascending element index, the values are bitwise those of the reference's
// assemble_optv2 (sparse.py:97-106: stable lexsort + sequential bincount),
// and the value-dependent pattern (sparse.py:108-111) follows exactly.
// No atomics touch values: the output is deterministic by construction.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sa_common.cuh"
#include "sa_geometry.cuh"

using namespace sa;

struct sa_mesh {
    int d = 0;
    int64_t nq = 0, nme = 0;
    int core = 0;
    int device = 0;
    void *qv = nullptr;   // VecT<d>[nq]   (AoS, padded: one 32 B sector per 3D vertex)
    void *me = nullptr;   // IdxT<d>[nme]  (int32 AoS, one 16 B load per element)
    double *vols = nullptr;
    int64_t *scratch = nullptr;  // [0] bad index
};

struct sa_plan {
    const sa_mesh *mesh = nullptr;
    int m = 1;
    int64_t row_begin = 0, row_end = 0, nrows = 0;
    int64_t node_begin = 0, node_end = 0, nnodes = 0;
    int64_t n_inc = 0, n_colnodes = 0, nnz = 0, max_deg = 0;
    int64_t *inc_ptr = nullptr;   // (nnodes+1)
    uint2 *inc = nullptr;         // (n_inc): x = e | alpha<<30, y = 4 x 8-bit column ranks
    int64_t *colptr = nullptr;    // (nnodes+1) node-level
    int32_t *cols = nullptr;      // (n_colnodes) node-level sorted columns
    int64_t *indptr = nullptr;    // (nrows+1) dof-level, block relative
    int32_t *indices = nullptr;   // (nnz) global column dofs
    int64_t *counters = nullptr;  // [0..3] zero counts per output, [4] bad element, [5] capacity flag
    int64_t *scan_tmp = nullptr;
};

namespace {

constexpr int MAXC = 255;  // 8-bit ranks: at most 255 distinct neighbour nodes per node

inline int set_device(int dev)
{
    int cur = -1;
    SA_CUDA_TRY(cudaGetDevice(&cur));
    if (cur != dev) SA_CUDA_TRY(cudaSetDevice(dev));
    return SA_OK;
}

// ---------------------------------------------------------------------------
// mesh upload: q (d,nq) SoA -> padded AoS, me (d+1,nme) int64 -> int32 AoS

template <int D>
__global__ void k_pack_q(const double *__restrict__ q, int64_t nq, typename VecT<D>::type *__restrict__ qv)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
        typename VecT<D>::type t;
        if constexpr (D == 1) t = q[i];
        else if constexpr (D == 2) t = make_double2(q[i], q[nq + i]);
        else t = make_double4(q[i], q[nq + i], q[2 * nq + i], 0.0);
        qv[i] = t;
    }
}

template <int D>
__global__ void k_pack_me(const int64_t *__restrict__ me, int64_t nq, int64_t nme,
                          typename IdxT<D>::type *__restrict__ out, unsigned long long *bad)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nme; k += (int64_t)gridDim.x * blockDim.x) {
        int v[4] = {0, 0, 0, 0};
#pragma unroll
        for (int a = 0; a <= D; ++a) {
            int64_t x = me[a * nme + k];
            if (x < 0 || x >= nq) atomicMin(bad, (unsigned long long)(a * nme + k));
            v[a] = (int)x;
        }
        typename IdxT<D>::type t;
        if constexpr (D == 1) t = make_int2(v[0], v[1]);
        else t = make_int4(v[0], v[1], v[2], v[3]);
        out[k] = t;
    }
}

template <int D, int CORE>
__global__ void k_volumes(const typename VecT<D>::type *__restrict__ qv, const typename IdxT<D>::type *__restrict__ me,
                          int64_t nme, double *__restrict__ vols, unsigned long long *bad)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nme; k += (int64_t)gridDim.x * blockDim.x) {
        int v[D + 1];
        load_element<D>(me, k, v);
        double x[D + 1][D];
#pragma unroll
        for (int a = 0; a <= D; ++a) load_vertex<D>(qv, v[a], x[a]);
        bool deg = false;
        double vol = element_volume<D, CORE>(x, deg);
        if (deg) atomicMin(bad, (unsigned long long)k);
        vols[k] = vol;
    }
}

// ---------------------------------------------------------------------------
// symbolic phase

template <int D>
__global__ void k_inc_count(const typename IdxT<D>::type *__restrict__ me, int64_t nme, int64_t nb0, int64_t nb1,
                            unsigned long long *__restrict__ cnt)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nme; e += (int64_t)gridDim.x * blockDim.x) {
        int v[D + 1];
        load_element<D>(me, e, v);
#pragma unroll
        for (int a = 0; a <= D; ++a)
            if (v[a] >= nb0 && v[a] < nb1) atomicAdd(cnt + (v[a] - nb0), 1ull);
    }
}

template <int D>
__global__ void k_inc_fill(const typename IdxT<D>::type *__restrict__ me, int64_t nme, int64_t nb0, int64_t nb1,
                           const int64_t *__restrict__ inc_ptr, unsigned long long *__restrict__ cursor,
                           uint2 *__restrict__ inc)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nme; e += (int64_t)gridDim.x * blockDim.x) {
        int v[D + 1];
        load_element<D>(me, e, v);
#pragma unroll
        for (int a = 0; a <= D; ++a)
            if (v[a] >= nb0 && v[a] < nb1) {
                int64_t nl = v[a] - nb0;
                int64_t pos = inc_ptr[nl] + (int64_t)atomicAdd(cursor + nl, 1ull);
                inc[pos] = make_uint2((unsigned)e | ((unsigned)a << 30), 0u);
            }
    }
}

// ascending element order per node (the reference's triplet order is
// element-major, so each entry's contributions are summed in element order)
__global__ void k_inc_sort(const int64_t *__restrict__ inc_ptr, int64_t nnodes, uint2 *__restrict__ inc)
{
    int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl >= nnodes) return;
    int64_t t0 = inc_ptr[nl], t1 = inc_ptr[nl + 1];
    for (int64_t t = t0 + 1; t < t1; ++t) {
        uint2 x = inc[t];
        unsigned key = x.x & 0x3fffffffu;
        int64_t u = t - 1;
        while (u >= t0 && (inc[u].x & 0x3fffffffu) > key) { inc[u + 1] = inc[u]; --u; }
        inc[u + 1] = x;
    }
}

// sorted unique neighbour nodes of node nl (write == nullptr: count only)
template <int D>
__global__ void k_node_cols(const typename IdxT<D>::type *__restrict__ me, const int64_t *__restrict__ inc_ptr,
                            const uint2 *__restrict__ inc, int64_t nnodes, int64_t *__restrict__ ncol,
                            const int64_t *__restrict__ colptr, int32_t *__restrict__ cols,
                            unsigned long long *cap_flag)
{
    int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl >= nnodes) return;
    int buf[MAXC];
    int n = 0;
    bool over = false;
    for (int64_t t = inc_ptr[nl]; t < inc_ptr[nl + 1] && !over; ++t) {
        int v[D + 1];
        load_element<D>(me, inc[t].x & 0x3fffffffu, v);
        for (int a = 0; a <= D; ++a) {
            int x = v[a];
            int lo = 0, hi = n;
            while (lo < hi) { int mid = (lo + hi) >> 1; if (buf[mid] < x) lo = mid + 1; else hi = mid; }
            if (lo < n && buf[lo] == x) continue;
            if (n == MAXC) { over = true; break; }
            for (int u = n; u > lo; --u) buf[u] = buf[u - 1];
            buf[lo] = x;
            ++n;
        }
    }
    if (over) { atomicOr(cap_flag, 1ull); n = 0; }
    if (cols == nullptr) {
        ncol[nl] = n;
    } else {
        int64_t base = colptr[nl];
        for (int u = 0; u < n; ++u) cols[base + u] = buf[u];
    }
}

template <int D>
__global__ void k_inc_ranks(const typename IdxT<D>::type *__restrict__ me, const int64_t *__restrict__ inc_ptr,
                            uint2 *__restrict__ inc, int64_t nnodes, const int64_t *__restrict__ colptr,
                            const int32_t *__restrict__ cols)
{
    int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl >= nnodes) return;
    const int64_t c0 = colptr[nl];
    const int n = (int)(colptr[nl + 1] - c0);
    for (int64_t t = inc_ptr[nl]; t < inc_ptr[nl + 1]; ++t) {
        uint2 rec = inc[t];
        int v[D + 1];
        load_element<D>(me, rec.x & 0x3fffffffu, v);
        unsigned ranks = 0;
        for (int a = 0; a <= D; ++a) {
            int lo = 0, hi = n;
            while (lo < hi) { int mid = (lo + hi) >> 1; if (cols[c0 + mid] < v[a]) lo = mid + 1; else hi = mid; }
            ranks |= (unsigned)lo << (8 * a);
        }
        rec.y = ranks;
        inc[t] = rec;
    }
}

// dof-level CSR of the block: row m*nl+l has columns m*cols[k]+n
__global__ void k_dof_csr(const int64_t *__restrict__ colptr, const int32_t *__restrict__ cols, int64_t nnodes,
                          int m, int64_t *__restrict__ indptr, int32_t *__restrict__ indices)
{
    int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl > nnodes) return;
    const int64_t c0 = colptr[nl];
    if (nl == nnodes) { indptr[(int64_t)m * nnodes] = (int64_t)m * m * c0; return; }
    const int deg = (int)(colptr[nl + 1] - c0);
    for (int l = 0; l < m; ++l) {
        int64_t p = (int64_t)m * m * c0 + (int64_t)l * m * deg;
        indptr[(int64_t)m * nl + l] = p;
        for (int k = 0; k < deg; ++k)
            for (int n = 0; n < m; ++n) indices[p + (int64_t)k * m + n] = m * cols[c0 + k] + n;
    }
}

// ---------------------------------------------------------------------------
// numeric phase

struct NumArgs {
    const void *qv;
    const void *me;
    const double *vols;
    int64_t nnodes;
    int64_t node_begin;
    const int64_t *inc_ptr;
    const uint2 *inc;
    const int64_t *colptr;
    const int64_t *indptr;
    int acc_stride;  // smem accumulator rows per output (m*m*max_deg)
    double *vals[2];
    int64_t *counters;
    // coefficients
    const double *w; double w_const;
    const double *lamb; double lamb_const;
    const double *mu; double mu_const;
    const double *A; const double *b; const double *c; const double *a0;
    double A_const[9]; double a0_const;
    double mass_coef_diag, mass_coef_off;  // 2/((d+1)(d+2)(d+3)), 1/(...) as Python computes them
};

template <int OPS>
__host__ __device__ constexpr int n_outputs()
{
    return ((OPS & OP_MASS) ? 1 : 0) + ((OPS & OP_STIFF) ? 1 : 0) + ((OPS & OP_ELASTIC) ? 1 : 0) +
           ((OPS & OP_GENERAL) ? 1 : 0);
}

template <int D>
__device__ __forceinline__ double nodal(const double *p, double cst, int v)
{
    return p ? __ldg(p + v) : cst;
}

// Fold element e's row(s) for local vertex alpha into the accumulators.
template <int D, int M, int OPS, int CORE>
__device__ __forceinline__ void fold_incidence(const NumArgs &a, uint2 rec, double *acc, int tid, int nthr,
                                               bool &degenerate)
{
    constexpr int NOUT = n_outputs<OPS>();
    const int64_t e = rec.x & 0x3fffffffu;
    const int alpha = rec.x >> 30;
    const unsigned ranks = rec.y;
    int v[D + 1];
    load_element<D>((const typename IdxT<D>::type *)a.me, e, v);
    const double vol = __ldg(a.vols + e);
    double x[D + 1][D];
    double G[D + 1][D];
    if constexpr ((OPS & (OP_STIFF | OP_ELASTIC | OP_GENERAL)) != 0) {
#pragma unroll
        for (int g = 0; g <= D; ++g) load_vertex<D>((const typename VecT<D>::type *)a.qv, v[g], x[g]);
        degenerate |= element_gradients<D, CORE>(x, G);
    }
    double ga[D];
    if constexpr ((OPS & (OP_STIFF | OP_ELASTIC | OP_GENERAL)) != 0) select_row<D>(G, alpha, ga);

    int o = 0;
    if constexpr ((OPS & OP_MASS) != 0) {
        double W[D + 1];
#pragma unroll
        for (int g = 0; g <= D; ++g) W[g] = nodal<D>(a.w, a.w_const, v[g]);
        double wsum = W[0];
#pragma unroll
        for (int g = 1; g <= D; ++g) wsum = SA_ADD(wsum, W[g]);
        const double wa = select_val<D>(W, alpha);
        const double cd = SA_MUL(a.mass_coef_diag, vol), co = SA_MUL(a.mass_coef_off, vol);
        const double wsa = SA_ADD(wsum, wa);
#pragma unroll
        for (int b = 0; b <= D; ++b) {
            double val = SA_MUL(b == alpha ? cd : co, SA_ADD(wsa, W[b]));
            int r = (ranks >> (8 * b)) & 0xff;
            acc[(o * a.acc_stride + r) * nthr + tid] += val;
        }
        ++o;
    }
    if constexpr ((OPS & OP_STIFF) != 0) {
#pragma unroll
        for (int b = 0; b <= D; ++b) {
            double val = stiff_entry<D>(ga, G[b], vol);
            int r = (ranks >> (8 * b)) & 0xff;
            acc[(o * a.acc_stride + r) * nthr + tid] += val;
        }
        ++o;
    }
    if constexpr ((OPS & OP_ELASTIC) != 0) {
        // lambs = (sum_g lamb_g) * (vols / (d+1))   kernels.py:354-356
        const double scale = __ddiv_rn(vol, (double)(D + 1));
        double ls = nodal<D>(a.lamb, a.lamb_const, v[0]), ms = nodal<D>(a.mu, a.mu_const, v[0]);
#pragma unroll
        for (int g = 1; g <= D; ++g) {
            ls = SA_ADD(ls, nodal<D>(a.lamb, a.lamb_const, v[g]));
            ms = SA_ADD(ms, nodal<D>(a.mu, a.mu_const, v[g]));
        }
        const double lambs = SA_MUL(ls, scale), mus = SA_MUL(ms, scale);
        const int deg_stride = a.acc_stride / M;  // = M * max_deg
#pragma unroll
        for (int b = 0; b <= D; ++b) {
            const int r = (ranks >> (8 * b)) & 0xff;
#pragma unroll
            for (int l = 0; l < M; ++l)
#pragma unroll
                for (int n = 0; n < M; ++n) {
                    double val = elastic_entry<D>(ga, G[b], l, n, lambs, mus);
                    acc[(o * a.acc_stride + l * deg_stride + r * M + n) * nthr + tid] += val;
                }
        }
        ++o;
    }
    if constexpr ((OPS & OP_GENERAL) != 0) {
        double As[D][D], bs[D], cs[D], a0s;
        double bb[D + 1][D], cc[D], a0v[D + 1];
#pragma unroll
        for (int g = 0; g <= D; ++g) {
            const int vg = v[g];
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    double t = a.A ? __ldg(a.A + (int64_t)vg * D * D + i * D + j) : a.A_const[i * D + j];
                    As[i][j] = g == 0 ? t : SA_ADD(As[i][j], t);
                }
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double tb = a.b ? __ldg(a.b + (int64_t)vg * D + i) : 0.0;
                double tc = a.c ? __ldg(a.c + (int64_t)vg * D + i) : 0.0;
                bb[g][i] = tb;
                bs[i] = g == 0 ? tb : SA_ADD(bs[i], tb);
                cs[i] = g == 0 ? tc : SA_ADD(cs[i], tc);
                if (g == alpha) cc[i] = tc;
            }
            a0v[g] = a.a0 ? __ldg(a.a0 + vg) : a.a0_const;
            a0s = g == 0 ? a0v[0] : SA_ADD(a0s, a0v[g]);
        }
        const double s1 = __ddiv_rn(vol, (double)(D + 1));
        const double s2 = __ddiv_rn(vol, (double)((D + 1) * (D + 2)));
        const double cd = SA_MUL(a.mass_coef_diag, vol), co = SA_MUL(a.mass_coef_off, vol);
        const double a0a = select_val<D>(a0v, alpha);
#pragma unroll
        for (int b = 0; b <= D; ++b) {
            double AG[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double t = SA_MUL(As[i][0], G[b][0]);
#pragma unroll
                for (int j = 1; j < D; ++j) t = SA_ADD(t, SA_MUL(As[i][j], G[b][j]));
                AG[i] = t;
            }
            double diff = SA_MUL(ga[0], AG[0]);
            double conv = SA_MUL(SA_ADD(bs[0], bb[b][0]), ga[0]);
            double tran = SA_MUL(SA_ADD(cs[0], cc[0]), G[b][0]);
#pragma unroll
            for (int i = 1; i < D; ++i) {
                diff = SA_ADD(diff, SA_MUL(ga[i], AG[i]));
                conv = SA_ADD(conv, SA_MUL(SA_ADD(bs[i], bb[b][i]), ga[i]));
                tran = SA_ADD(tran, SA_MUL(SA_ADD(cs[i], cc[i]), G[b][i]));
            }
            double rea = SA_MUL(b == alpha ? cd : co, SA_ADD(SA_ADD(a0s, a0a), a0v[b]));
            double val = SA_ADD(SA_ADD(SA_SUB(SA_MUL(diff, s1), SA_MUL(conv, s2)), SA_MUL(tran, s2)), rea);
            int r = (ranks >> (8 * b)) & 0xff;
            acc[(o * a.acc_stride + r) * nthr + tid] += val;
        }
        ++o;
    }
}

template <int D, int M, int OPS, int CORE>
__global__ void __launch_bounds__(128) k_numeric_rowgather(NumArgs a)
{
    constexpr int NOUT = n_outputs<OPS>();
    extern __shared__ double smem_acc[];
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int64_t nl = blockIdx.x * (int64_t)blockDim.x + tid;
    int nz[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) nz[o] = 0;
    if (nl < a.nnodes) {
        const int64_t c0 = a.colptr[nl];
        const int deg = (int)(a.colptr[nl + 1] - c0);
        const int deg_stride = M * deg;
        for (int o = 0; o < NOUT; ++o)
            for (int l = 0; l < M; ++l)
                for (int k = 0; k < deg_stride; ++k)
                    smem_acc[(o * a.acc_stride + l * (a.acc_stride / M) + k) * nthr + tid] = 0.0;
        const int64_t t1 = a.inc_ptr[nl + 1];
        int64_t emin = INT64_MAX;
        for (int64_t t = a.inc_ptr[nl]; t < t1; ++t) {
            uint2 rec = __ldg(a.inc + t);
            bool dg = false;
            fold_incidence<D, M, OPS, CORE>(a, rec, smem_acc, tid, nthr, dg);
            if (dg) emin = min(emin, (int64_t)(rec.x & 0x3fffffffu));
        }
        if (emin != INT64_MAX) {
            atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)emin);
        }
        for (int o = 0; o < NOUT; ++o) {
            double *out = a.vals[o];
            for (int l = 0; l < M; ++l) {
                const int64_t p = a.indptr[M * nl + l];
                for (int k = 0; k < deg_stride; ++k) {
                    double val = smem_acc[(o * a.acc_stride + l * (a.acc_stride / M) + k) * nthr + tid];
                    out[p + k] = val;
                    nz[o] += (val == 0.0);
                }
            }
        }
    }
    // deterministic integer reduction of the exact-zero counts
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
        int v = nz[o];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
        if ((tid & 31) == 0 && v) atomicAdd((unsigned long long *)(a.counters + o), (unsigned long long)v);
    }
}

// compaction (K5): drop exact-zero entries (sparse.py:108-111)
__global__ void k_row_nonzeros(const int64_t *__restrict__ indptr, const double *__restrict__ vals, int64_t nrows,
                               int64_t *__restrict__ cnt)
{
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    int64_t c = 0;
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p) c += (vals[p] != 0.0);
    cnt[r] = c;
}

__global__ void k_compact(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                          const double *__restrict__ vals, int64_t nrows, const int64_t *__restrict__ new_ptr,
                          int32_t *__restrict__ out_idx, double *__restrict__ out_val)
{
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    int64_t w = new_ptr[r];
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p) {
        double v = vals[p];
        if (v != 0.0) { out_idx[w] = indices[p]; out_val[w] = v; ++w; }
    }
}

// ---------------------------------------------------------------------------
// dispatch helpers

template <int D>
int mesh_kernels(sa_mesh *M, const double *q, const int64_t *me, const double *vols, cudaStream_t st)
{
    typedef typename VecT<D>::type V;
    typedef typename IdxT<D>::type I;
    unsigned long long *bad = (unsigned long long *)M->scratch;
    SA_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
    const int B = 256;
    unsigned gq = std::min<int64_t>(grid_for(M->nq, B), 148 * 32);
    unsigned ge = std::min<int64_t>(grid_for(M->nme, B), 148 * 32);
    if (M->nq) SA_LAUNCH(k_pack_q<D>, gq, B, 0, st, q, M->nq, (V *)M->qv);
    if (M->nme) SA_LAUNCH(k_pack_me<D>, ge, B, 0, st, me, M->nq, M->nme, (I *)M->me, bad);
    unsigned long long hbad = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    if (hbad != ~0ull) {
        err_state().bad = (int64_t)hbad;
        return set_error(SA_ERR_INDEX_RANGE, "connectivity entry me[%lld, %lld] out of range [0, %lld)",
                         (long long)(hbad / M->nme), (long long)(hbad % M->nme), (long long)M->nq);
    }
    if (vols) {
        SA_CUDA_TRY(cudaMemcpyAsync(M->vols, vols, M->nme * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else if (M->nme) {
        SA_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
        if (M->core == CORE_SKYLAKEX)
            SA_LAUNCH((k_volumes<D, CORE_SKYLAKEX>), ge, B, 0, st, (const V *)M->qv, (const I *)M->me, M->nme, M->vols, bad);
        else
            SA_LAUNCH((k_volumes<D, CORE_HASWELL>), ge, B, 0, st, (const V *)M->qv, (const I *)M->me, M->nme, M->vols, bad);
        SA_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        if (hbad != ~0ull) {
            err_state().bad = (int64_t)hbad;
            return set_error(SA_ERR_DEGENERATE, "simplex %lld is degenerate (zero volume)", (long long)hbad);
        }
    }
    return SA_OK;
}

template <int D>
int symbolic_kernels(sa_plan *P, cudaStream_t st)
{
    typedef typename IdxT<D>::type I;
    const sa_mesh *M = P->mesh;
    const int B = 256;
    const int64_t nn = P->nnodes;
    unsigned ge = std::min<int64_t>(grid_for(M->nme, B), 148 * 32);
    int64_t *cnt = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&cnt, (nn + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMemsetAsync(cnt, 0, (nn + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->inc_ptr, (nn + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->colptr, (nn + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->scan_tmp, (scan_tmp_elems(std::max<int64_t>(nn, P->nrows) + 1) + 1) * sizeof(int64_t), st));
    if (M->nme)
        SA_LAUNCH(k_inc_count<D>, ge, B, 0, st, (const I *)M->me, M->nme, P->node_begin, P->node_end,
                  (unsigned long long *)cnt);
    SA_TRY(exclusive_scan_i64(cnt, P->inc_ptr, nn, P->scan_tmp, st));
    SA_CUDA_TRY(cudaMemcpyAsync(&P->n_inc, P->inc_ptr + nn, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->inc, std::max<int64_t>(P->n_inc, 1) * sizeof(uint2), st));
    SA_CUDA_TRY(cudaMemsetAsync(cnt, 0, (nn + 1) * sizeof(int64_t), st));
    if (M->nme)
        SA_LAUNCH(k_inc_fill<D>, ge, B, 0, st, (const I *)M->me, M->nme, P->node_begin, P->node_end, P->inc_ptr,
                  (unsigned long long *)cnt, P->inc);
    if (nn) {
        SA_LAUNCH(k_inc_sort, grid_for(nn, 128), 128, 0, st, P->inc_ptr, nn, P->inc);
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 5, 0, sizeof(int64_t), st));
        SA_LAUNCH(k_node_cols<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, cnt,
                  (const int64_t *)nullptr, (int32_t *)nullptr, (unsigned long long *)(P->counters + 5));
    }
    SA_TRY(exclusive_scan_i64(cnt, P->colptr, nn, P->scan_tmp, st));
    int64_t cap = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&P->n_colnodes, P->colptr + nn, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaMemcpyAsync(&cap, P->counters + 5, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    if (cap) return set_error(SA_ERR_CAPACITY, "a node has more than %d distinct neighbours", MAXC);
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->cols, std::max<int64_t>(P->n_colnodes, 1) * sizeof(int32_t), st));
    if (nn) {
        SA_LAUNCH(k_node_cols<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, cnt,
                  (const int64_t *)P->colptr, P->cols, (unsigned long long *)(P->counters + 5));
        SA_LAUNCH(k_inc_ranks<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, P->colptr,
                  P->cols);
    }
    // max node degree (host side from the node-level colptr)
    std::vector<int64_t> hcp(nn + 1);
    SA_CUDA_TRY(cudaMemcpyAsync(hcp.data(), P->colptr, (nn + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    int64_t md = 0;
    for (int64_t i = 0; i < nn; ++i) md = std::max(md, hcp[i + 1] - hcp[i]);
    P->max_deg = md;
    const int m = P->m;
    P->nnz = (int64_t)m * m * P->n_colnodes;
    if (P->nnz >= ((int64_t)1 << 31) || (int64_t)m * M->nq >= ((int64_t)1 << 31))
        return set_error(SA_ERR_CAPACITY, "block has %lld structural entries; int32 column indices overflow",
                         (long long)P->nnz);
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->indptr, (P->nrows + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->indices, std::max<int64_t>(P->nnz, 1) * sizeof(int32_t), st));
    SA_LAUNCH(k_dof_csr, grid_for(nn + 1, 128), 128, 0, st, P->colptr, P->cols, nn, m, P->indptr, P->indices);
    SA_CUDA_TRY(cudaFreeAsync(cnt, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    return SA_OK;
}

template <int D, int M, int OPS, int CORE>
int launch_numeric(const NumArgs &a, int64_t nnodes, cudaStream_t st)
{
    constexpr int NOUT = n_outputs<OPS>();
    int block = 128;
    size_t smem = (size_t)NOUT * a.acc_stride * block * sizeof(double);
    while (smem > 200 * 1024 && block > 32) { block /= 2; smem /= 2; }
    if (smem > 200 * 1024)
        return set_error(SA_ERR_CAPACITY, "row accumulators need %zu B of shared memory per 32 threads", smem);
    auto kern = k_numeric_rowgather<D, M, OPS, CORE>;
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (nnodes) SA_LAUNCH(kern, grid_for(nnodes, block), block, smem, st, a);
    return SA_OK;
}

template <int D, int M, int OPS>
int launch_numeric_core(const NumArgs &a, int64_t nnodes, int core, cudaStream_t st)
{
    if (core == CORE_SKYLAKEX) return launch_numeric<D, M, OPS, CORE_SKYLAKEX>(a, nnodes, st);
    return launch_numeric<D, M, OPS, CORE_HASWELL>(a, nnodes, st);
}

template <int D>
int dispatch_numeric(const NumArgs &a, int ops, int m, int64_t nnodes, int core, cudaStream_t st)
{
    switch (ops) {
        case OP_MASS: return launch_numeric_core<D, 1, OP_MASS>(a, nnodes, core, st);
        case OP_STIFF: return launch_numeric_core<D, 1, OP_STIFF>(a, nnodes, core, st);
        case OP_MASS | OP_STIFF: return launch_numeric_core<D, 1, OP_MASS | OP_STIFF>(a, nnodes, core, st);
        case OP_GENERAL: return launch_numeric_core<D, 1, OP_GENERAL>(a, nnodes, core, st);
        case OP_ELASTIC:
            if constexpr (D >= 2) {
                if (m == D) return launch_numeric_core<D, D, OP_ELASTIC>(a, nnodes, core, st);
            }
            return set_error(SA_ERR_ARG, "elastic operator needs d in {2,3} and m == d");
        default: return set_error(SA_ERR_ARG, "unsupported operator combination %d", ops);
    }
}

}  // namespace

// ===========================================================================
// C ABI

extern "C" {

const char *sa_last_error(void) { return err_state().msg.c_str(); }
int64_t sa_bad_index(void) { return err_state().bad; }
int64_t sa_launch_count(int reset)
{
    int64_t v = err_state().launches;
    if (reset) err_state().launches = 0;
    return v;
}

int sa_mesh_create(int d, int64_t nq, int64_t nme, const double *q_dev, const int64_t *me_dev,
                   const double *vols_dev, int core, int device, void *stream, sa_mesh **out)
{
    err_state().msg.clear();
    err_state().bad = -1;
    if (!out) return set_error(SA_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (d < 1 || d > 3) return set_error(SA_ERR_ARG, "dimension must be 1, 2 or 3, got %d", d);
    if (core != CORE_SKYLAKEX && core != CORE_HASWELL) return set_error(SA_ERR_ARG, "unknown core %d", core);
    if (nq < 0 || nme < 0) return set_error(SA_ERR_ARG, "negative sizes");
    if (nq >= ((int64_t)1 << 31) || nme >= ((int64_t)1 << 30))
        return set_error(SA_ERR_CAPACITY, "mesh with nq=%lld nme=%lld exceeds the int32 index range",
                         (long long)nq, (long long)nme);
    SA_TRY(set_device(device));
    cudaStream_t st = (cudaStream_t)stream;
    sa_mesh *M = new sa_mesh();
    M->d = d; M->nq = nq; M->nme = nme; M->core = core; M->device = device;
    size_t vsz = d == 1 ? 8 : (d == 2 ? 16 : 32);
    size_t isz = d == 1 ? 8 : 16;
    int rc = SA_OK;
    auto fail = [&](int r) { sa_mesh_destroy(M); return r; };
    if (cudaMalloc(&M->qv, std::max<int64_t>(nq, 1) * vsz) != cudaSuccess ||
        cudaMalloc(&M->me, std::max<int64_t>(nme, 1) * isz) != cudaSuccess ||
        cudaMalloc((void **)&M->vols, std::max<int64_t>(nme, 1) * sizeof(double)) != cudaSuccess ||
        cudaMalloc((void **)&M->scratch, 8 * sizeof(int64_t)) != cudaSuccess)
        return fail(set_error(SA_ERR_NOMEM, "device allocation for the mesh failed"));
    if (d == 1) rc = mesh_kernels<1>(M, q_dev, me_dev, vols_dev, st);
    else if (d == 2) rc = mesh_kernels<2>(M, q_dev, me_dev, vols_dev, st);
    else rc = mesh_kernels<3>(M, q_dev, me_dev, vols_dev, st);
    if (rc != SA_OK) return fail(rc);
    *out = M;
    return SA_OK;
}

int sa_mesh_vols(const sa_mesh *M, double *vols_dev_out, void *stream)
{
    if (!M) return set_error(SA_ERR_ARG, "mesh is NULL");
    SA_CUDA_TRY(cudaMemcpyAsync(vols_dev_out, M->vols, M->nme * sizeof(double), cudaMemcpyDeviceToDevice,
                                (cudaStream_t)stream));
    return SA_OK;
}

int sa_mesh_destroy(sa_mesh *M)
{
    if (!M) return SA_OK;
    cudaFree(M->qv);
    cudaFree(M->me);
    cudaFree(M->vols);
    cudaFree(M->scratch);
    delete M;
    return SA_OK;
}

int sa_plan_destroy(sa_plan *P)
{
    if (!P) return SA_OK;
    cudaDeviceSynchronize();
    cudaFree(P->inc_ptr); cudaFree(P->inc); cudaFree(P->colptr); cudaFree(P->cols);
    cudaFree(P->indptr); cudaFree(P->indices); cudaFree(P->counters); cudaFree(P->scan_tmp);
    delete P;
    return SA_OK;
}

int sa_plan_create(const sa_mesh *M, int m, int64_t row_begin, int64_t row_end, void *stream, sa_plan **out)
{
    err_state().msg.clear();
    err_state().bad = -1;
    if (!M || !out) return set_error(SA_ERR_ARG, "mesh/out is NULL");
    *out = nullptr;
    if (m < 1 || m > 3) return set_error(SA_ERR_ARG, "m must be 1..3, got %d", m);
    const int64_t ndof = (int64_t)m * M->nq;
    if (row_begin < 0 || row_end > ndof || row_begin > row_end || row_begin % m || row_end % m)
        return set_error(SA_ERR_ARG, "row block [%lld, %lld) invalid for %lld dofs with m=%d",
                         (long long)row_begin, (long long)row_end, (long long)ndof, m);
    SA_TRY(set_device(M->device));
    cudaStream_t st = (cudaStream_t)stream;
    sa_plan *P = new sa_plan();
    P->mesh = M; P->m = m; P->row_begin = row_begin; P->row_end = row_end; P->nrows = row_end - row_begin;
    P->node_begin = row_begin / m; P->node_end = row_end / m; P->nnodes = P->node_end - P->node_begin;
    if (cudaMalloc((void **)&P->counters, 8 * sizeof(int64_t)) != cudaSuccess) {
        delete P;
        return set_error(SA_ERR_NOMEM, "device allocation failed");
    }
    int rc;
    if (M->d == 1) rc = symbolic_kernels<1>(P, st);
    else if (M->d == 2) rc = symbolic_kernels<2>(P, st);
    else rc = symbolic_kernels<3>(P, st);
    if (rc != SA_OK) {
        std::string msg = err_state().msg;
        cudaStreamSynchronize(st);
        sa_plan_destroy(P);
        err_state().msg = msg;
        return rc;
    }
    *out = P;
    return SA_OK;
}

int sa_plan_info(const sa_plan *P, int64_t *nrows, int64_t *nnz, int64_t *max_row_nodes)
{
    if (!P) return set_error(SA_ERR_ARG, "plan is NULL");
    if (nrows) *nrows = P->nrows;
    if (nnz) *nnz = P->nnz;
    if (max_row_nodes) *max_row_nodes = P->max_deg;
    return SA_OK;
}

int sa_plan_pattern(const sa_plan *P, int64_t *indptr_dev, int32_t *indices_dev, void *stream)
{
    if (!P) return set_error(SA_ERR_ARG, "plan is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    if (indptr_dev)
        SA_CUDA_TRY(cudaMemcpyAsync(indptr_dev, P->indptr, (P->nrows + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    if (indices_dev && P->nnz)
        SA_CUDA_TRY(cudaMemcpyAsync(indices_dev, P->indices, P->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    return SA_OK;
}

int sa_numeric(sa_plan *P, int ops, const sa_coeffs *cf, double *const *vals_dev, int64_t *n_zero_out, void *stream)
{
    if (!P || !vals_dev) return set_error(SA_ERR_ARG, "plan/vals is NULL");
    const sa_mesh *M = P->mesh;
    const int d = M->d;
    if ((ops & SA_OP_ELASTIC) && P->m != d) return set_error(SA_ERR_ARG, "elastic operator needs a plan with m = d");
    if (!(ops & SA_OP_ELASTIC) && P->m != 1) return set_error(SA_ERR_ARG, "scalar operators need a plan with m = 1");
    SA_TRY(set_device(M->device));
    cudaStream_t st = (cudaStream_t)stream;
    NumArgs a;
    memset(&a, 0, sizeof a);
    a.qv = M->qv; a.me = M->me; a.vols = M->vols;
    a.nnodes = P->nnodes; a.node_begin = P->node_begin;
    a.inc_ptr = P->inc_ptr; a.inc = P->inc; a.colptr = P->colptr; a.indptr = P->indptr;
    a.acc_stride = (int)(P->m * P->m * std::max<int64_t>(P->max_deg, 1));
    int nout = 0;
    for (int bit = 1; bit <= 8; bit <<= 1)
        if (ops & bit) { a.vals[nout] = vals_dev[nout]; ++nout; }
    a.counters = P->counters;
    sa_coeffs z;
    memset(&z, 0, sizeof z);
    if (!cf) { cf = &z; z.w_const = 1.0; z.lamb_const = 1.0; z.mu_const = 1.0; }
    a.w = cf->w; a.w_const = cf->w_const;
    a.lamb = cf->lamb; a.lamb_const = cf->lamb_const;
    a.mu = cf->mu; a.mu_const = cf->mu_const;
    a.A = cf->A; a.b = cf->b; a.c = cf->c; a.a0 = cf->a0;
    memcpy(a.A_const, cf->A_const, sizeof a.A_const);
    a.a0_const = cf->a0_const;
    const double den = (double)((d + 1) * (d + 2) * (d + 3));
    a.mass_coef_diag = 2.0 / den;
    a.mass_coef_off = 1.0 / den;
    SA_CUDA_TRY(cudaMemsetAsync(P->counters, 0, 4 * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMemsetAsync(P->counters + 4, 0x7f, sizeof(int64_t), st));
    int rc;
    if (d == 1) rc = dispatch_numeric<1>(a, ops, P->m, P->nnodes, M->core, st);
    else if (d == 2) rc = dispatch_numeric<2>(a, ops, P->m, P->nnodes, M->core, st);
    else rc = dispatch_numeric<3>(a, ops, P->m, P->nnodes, M->core, st);
    if (rc != SA_OK) return rc;
    if (n_zero_out) {
        int64_t h[5];
        SA_CUDA_TRY(cudaMemcpyAsync(h, P->counters, 5 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        for (int o = 0; o < nout; ++o) n_zero_out[o] = h[o];
        if (h[4] != 0x7f7f7f7f7f7f7f7fLL) {
            err_state().bad = h[4];
            return set_error(SA_ERR_DEGENERATE, "simplex %lld is degenerate (zero volume)", (long long)h[4]);
        }
    }
    return SA_OK;
}

int sa_compact(const sa_plan *P, const double *vals_dev, int64_t *indptr_out, int32_t *indices_out, double *vals_out,
               void *stream)
{
    if (!P) return set_error(SA_ERR_ARG, "plan is NULL");
    SA_TRY(set_device(P->mesh->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nr = P->nrows;
    int64_t *cnt = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&cnt, (nr + 1) * sizeof(int64_t), st));
    if (nr) SA_LAUNCH(k_row_nonzeros, grid_for(nr, 256), 256, 0, st, P->indptr, vals_dev, nr, cnt);
    SA_TRY(exclusive_scan_i64(cnt, indptr_out, nr, P->scan_tmp, st));
    if (nr) SA_LAUNCH(k_compact, grid_for(nr, 256), 256, 0, st, P->indptr, P->indices, vals_dev, nr, indptr_out,
                      indices_out, vals_out);
    SA_CUDA_TRY(cudaFreeAsync(cnt, st));
    return SA_OK;
}

}  // extern "C"
