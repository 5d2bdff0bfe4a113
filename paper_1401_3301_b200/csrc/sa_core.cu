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
#include <climits>
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
    bool coords = false;         // q packed and vols set (sa_mesh_create with q, or sa_mesh_set_coords)
    bool vols_ready = false;     // vols set (the 3D symbolic phase copies them into its records)
};

// Warp-interleaved incidence record (row-gather kernel): everything an
// incidence needs besides the vertex coordinates / nodal coefficients, in one
// 32-byte sector.  Records of the 32 rows of a warp are interleaved
// (record k of lane j at wseg[w] + 32 k + j), so each step of the warp reads
// one contiguous 1 KB run instead of three dependent gathers (record,
// connectivity, volume).
struct __align__(32) IncRec {
    uint32_t ea;      // e | alpha << 30
    uint32_t ranks;   // 4 x 8-bit column ranks of the element's vertices in the row
    int32_t v[4];     // the element's vertices (unused slots 0)
    double vol;       // mesh.vols[e]
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
    IncRec *winc = nullptr;       // warp-interleaved records (padded to each warp's max degree)
    int64_t *wseg = nullptr;      // (nwarps+1) record offset of each warp of 32 node rows
    int64_t n_winc = 0;
    // two-pass numeric ("element rows"): incidence slot of every (element, alpha)
    // of the block's element range, and the per-incidence local-row buffer
    uint4 *epos = nullptr;         // (e_hi - e_lo): slot t of (e, alpha) in inc, or ~0u
    int64_t e_lo = 0, e_hi = 0;
    double *kbuf = nullptr;        // (n_slots * stride) local rows in warp-interleaved slot order
    int64_t kbuf_elems = 0;
    unsigned *tp_rank = nullptr;   // (n_slots) column ranks per slot (warp-interleaved like winc)
    int64_t tp_nslots = 0;
    // element batches (two-pass element pass, 3D general operator): per batch
    // of EB_SIZE consecutive elements its sorted unique vertices (EB_CAP max;
    // count -1 = too many, direct gathers) and 8-bit local vertex ids per element
    int32_t *eb_verts = nullptr, *eb_count = nullptr;
    uint32_t *eb_loc = nullptr;
    int eb_maxn = 0;
    bool eb_allfit = false;        // every batch staged (no direct-gather fallback compiled in)
    // fast general operator: rows whose zero guard tripped (recomputed in
    // reference order by k_guard_fixup)
    uint32_t *gd_flag_rows = nullptr;
    int *gd_nflag = nullptr;
    // heavy rows (degree above the light cap): assembled by k_heavy_rows
    int64_t light_deg = 0, n_heavy = 0;
    uint32_t *heavy_rows = nullptr;
};

// numeric-phase arguments (shared by the per-dimension translation units)
struct NumArgs {
    const void *qv;
    const void *me;
    const double *vols;
    int64_t nnodes;
    int64_t node_begin;
    const int64_t *inc_ptr;
    const uint2 *inc;
    const IncRec *winc;   // warp-interleaved records (row-gather), or NULL
    const int64_t *wseg;
    const int64_t *colptr;
    const int64_t *indptr;
    const int32_t *cols;  // node-level sorted neighbour nodes (row-gather coordinate cache)
    int acc_stride;  // smem accumulator rows per output (m*m*light_deg)
    double *vals[2];
    int64_t *counters;
    // coefficients
    const double *w; double w_const;
    const double *lamb; double lamb_const;
    const double *mu; double mu_const;
    const double *A; const double *b; const double *c; const double *a0;
    double A_const[9]; double a0_const;
    const double *gen_packed;  // (nq, 16) AoS [A(9) b(3) c(3) a0] or NULL
    const double *lambs_e, *mus_e;   // elastic: per-element scaled Lame sums (reference ElasticKernel) or NULL
    // two-pass numeric: element pass writes local rows to kbuf (stride kstride
    // doubles per incidence), the ordered fold pass reads them
    double *kbuf; int kstride;
    const uint4 *epos; int64_t e_lo, ne;
    const unsigned *tp_rank;   // slot of incidence k of row nl: wseg[nl >> 5] + 32 k + (nl & 31)
    const int32_t *eb_verts, *eb_count;
    const uint32_t *eb_loc;
    int eb_maxn;
    int eb_allfit;
    int64_t eb_b0, eb_b1;      // element-pass batch range of this launch
    double mass_coef_diag, mass_coef_off;  // 2/((d+1)(d+2)(d+3)), 1/(...) as Python computes them
    double mass_wc;  // constant weight: (wsum + w) + w, the same for every (alpha, beta)
    int exact;       // general operator: reference-order (bitwise) element values
    int *nflag;          // fast general operator: guarded-row count + list
    uint32_t *flag_rows;
    int light_deg;       // rows with more columns are heavy (k_heavy_rows), skipped by the row kernels
    const uint32_t *heavy_rows;
    int64_t n_heavy;
};

namespace {

constexpr int MAXC = 255;  // 8-bit ranks: at most 255 distinct neighbour nodes per node
// fast general operator: |entry| <= SA_GUARD_TAU * (sum of |contributions| of
// its row) sends the row to the reference-order recomputation
constexpr double SA_GUARD_TAU = 1e-9;

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

// (rows [0, rows32) of me may arrive as int32 -- narrowed and range-checked on
// the host while uploading, sa_host_narrow_upload -- the others as int64)
template <int D>
__global__ void k_pack_me(const int64_t *__restrict__ me, const int32_t *__restrict__ me32, int rows32, int64_t nq,
                          int64_t nme, typename IdxT<D>::type *__restrict__ out, unsigned long long *bad)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nme; k += (int64_t)gridDim.x * blockDim.x) {
        int v[4] = {0, 0, 0, 0};
#pragma unroll
        for (int a = 0; a <= D; ++a) {
            int64_t x = a < rows32 ? (int64_t)me32[a * nme + k] : me[(a - rows32) * nme + k];
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
                            unsigned long long *nheavy, uint32_t *heavy)
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
    if (over) {   // more than MAXC neighbours: k_heavy_cols builds this node's list
        if (cols == nullptr) heavy[atomicAdd(nheavy, 1ull)] = (uint32_t)nl;
        return;
    }
    if (cols == nullptr) {
        ncol[nl] = n;
    } else {
        int64_t base = colptr[nl];
        for (int u = 0; u < n; ++u) cols[base + u] = buf[u];
    }
}


// Nodes with more than MAXC distinct neighbours (k_node_cols' heavy list):
// one CTA per node gathers the vertices of its incidences into shared
// memory, bitonic-sorts them and keeps the unique ones (count, then fill).
// Their incidence ranks are not used (heavy rows are assembled by
// k_heavy_rows, which looks columns up in the sorted list).
constexpr int HEAVY_CAP = 16384;   // vertex references (4 per 3D incidence) per heavy node
template <int D>
__global__ void __launch_bounds__(1024) k_heavy_cols(const typename IdxT<D>::type *__restrict__ me,
                                                     const int64_t *__restrict__ inc_ptr, const uint2 *__restrict__ inc,
                                                     const uint32_t *__restrict__ heavy, int64_t *__restrict__ ncol,
                                                     const int64_t *__restrict__ colptr, int32_t *__restrict__ cols,
                                                     unsigned long long *too_big)
{
    extern __shared__ int hk[];
    __shared__ int s_part[32], s_n;
    const uint32_t nl = heavy[blockIdx.x];
    const int64_t t0 = inc_ptr[nl];
    const int ni = (int)(inc_ptr[nl + 1] - t0);
    const int nk = ni * (D + 1);
    if (nk > HEAVY_CAP) {
        if (threadIdx.x == 0) atomicOr(too_big, 1ull);
        return;
    }
    int P = 1;
    while (P < nk) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        int x = INT_MAX;
        if (i < nk) {
            int v[D + 1];
            load_element<D>(me, inc[t0 + i / (D + 1)].x & 0x3fffffffu, v);
            x = v[i % (D + 1)];
        }
        hk[i] = x;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int h = k >> 1; h > 0; h >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int p = i ^ h;
                if (p > i) {
                    const int a = hk[i], b = hk[p];
                    if ((a > b) == ((i & k) == 0)) { hk[i] = b; hk[p] = a; }
                }
            }
            __syncthreads();
        }
    // unique: heads among each thread's contiguous chunk, block scan of counts
    const int per = (P + blockDim.x - 1) / blockDim.x;
    const int c0 = threadIdx.x * per, c1 = min(c0 + per, nk);
    int cnt = 0;
    for (int i = c0; i < c1; ++i) cnt += (i == 0 || hk[i] != hk[i - 1]);
    int incl = cnt;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int sh = 1; sh < 32; sh <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, sh);
        if (lane >= sh) incl += y;
    }
    if (lane == 31) s_part[w] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { const int t = s_part[i]; s_part[i] = run; run += t; }
        s_n = run;
    }
    __syncthreads();
    if (cols == nullptr) {
        if (threadIdx.x == 0) ncol[nl] = s_n;
        return;
    }
    int pos = s_part[w] + incl - cnt;
    const int64_t base = colptr[nl];
    for (int i = c0; i < c1; ++i)
        if (i == 0 || hk[i] != hk[i - 1]) cols[base + pos++] = hk[i];
}

// rows above the light-row degree cap (heavy rows), and the largest light degree
__global__ void k_heavy_rows_list(const int64_t *__restrict__ colptr, int64_t nnodes, int64_t cap,
                                  uint32_t *__restrict__ list, unsigned long long *__restrict__ cnt_max)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnodes; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t deg = colptr[i + 1] - colptr[i];
        if (deg > cap) list[atomicAdd(cnt_max, 1ull)] = (uint32_t)i;
        else atomicMax(cnt_max + 1, (unsigned long long)deg);
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

// Fused node pass of the symbolic phase (fast path, every node with at most
// NS_CAPI incidences and NS_CAPC distinct neighbours): one thread per node
// row, its incidences and its sorted neighbour list in private shared-memory
// columns ([k][thread]: conflict-free).  FILL = false: sort the incidences in
// ascending element order (written back) and count the neighbours;
// FILL = true: (incidences already sorted) write the neighbours and the
// 8-bit column ranks of every incidence.  Replaces k_inc_sort + 2 x
// k_node_cols + k_inc_ranks (global-memory insertion sort, local-memory
// neighbour buffers).
constexpr int NS_THREADS = 64;
constexpr int NS_CAPI = 48;
constexpr int NS_CAPC = 64;

template <int D, bool FILL>
__global__ void __launch_bounds__(NS_THREADS) k_node_symbolic(const typename IdxT<D>::type *__restrict__ me,
                                                              const int64_t *__restrict__ inc_ptr,
                                                              uint2 *__restrict__ inc, int64_t nnodes,
                                                              int64_t *__restrict__ ncol,
                                                              const int64_t *__restrict__ colptr,
                                                              int32_t *__restrict__ cols,
                                                              unsigned long long *overflow)
{
    __shared__ unsigned s_inc[NS_CAPI][NS_THREADS];
    __shared__ int s_col[NS_CAPC][NS_THREADS];
    const int tid = threadIdx.x;
    const int64_t nl = blockIdx.x * (int64_t)NS_THREADS + tid;
    if (nl >= nnodes) return;
    const int64_t t0 = inc_ptr[nl];
    const int n = (int)(inc_ptr[nl + 1] - t0);
    if (n > NS_CAPI) { atomicOr(overflow, 1ull); return; }
    if (!FILL) {
        for (int k = 0; k < n; ++k) {
            const unsigned x = inc[t0 + k].x;
            const unsigned key = x & 0x3fffffffu;
            int u = k - 1;
            while (u >= 0 && (s_inc[u][tid] & 0x3fffffffu) > key) { s_inc[u + 1][tid] = s_inc[u][tid]; --u; }
            s_inc[u + 1][tid] = x;
        }
    } else {
        for (int k = 0; k < n; ++k) s_inc[k][tid] = inc[t0 + k].x;
    }
    int nc = 0;
    for (int k = 0; k < n; ++k) {
        int v[D + 1];
        load_element<D>(me, s_inc[k][tid] & 0x3fffffffu, v);
#pragma unroll
        for (int a = 0; a <= D; ++a) {
            const int x = v[a];
            int lo = 0, hi = nc;
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_col[mid][tid] < x) lo = mid + 1; else hi = mid; }
            if (lo < nc && s_col[lo][tid] == x) continue;
            if (nc == NS_CAPC) { atomicOr(overflow, 1ull); return; }
            for (int u = nc; u > lo; --u) s_col[u][tid] = s_col[u - 1][tid];
            s_col[lo][tid] = x;
            ++nc;
        }
    }
    if (!FILL) {
        for (int k = 0; k < n; ++k) inc[t0 + k] = make_uint2(s_inc[k][tid], 0u);
        ncol[nl] = nc;
        return;
    }
    const int64_t c0 = colptr[nl];
    for (int u = 0; u < nc; ++u) cols[c0 + u] = s_col[u][tid];
    for (int k = 0; k < n; ++k) {
        const unsigned x = s_inc[k][tid];
        int v[D + 1];
        load_element<D>(me, x & 0x3fffffffu, v);
        unsigned ranks = 0;
#pragma unroll
        for (int a = 0; a <= D; ++a) {
            int lo = 0, hi = nc;
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_col[mid][tid] < v[a]) lo = mid + 1; else hi = mid; }
            ranks |= (unsigned)lo << (8 * a);
        }
        inc[t0 + k] = make_uint2(x, ranks);
    }
}

// records per warp of 32 node rows: 32 x the warp's largest incidence count
__global__ void k_warp_span(const int64_t *__restrict__ inc_ptr, int64_t nnodes, int64_t *__restrict__ span)
{
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r0 = w * 32;
    if (r0 >= nnodes) return;
    const int64_t r1 = min(r0 + 32, nnodes);
    int64_t md = 0;
    for (int64_t r = r0; r < r1; ++r) md = max(md, inc_ptr[r + 1] - inc_ptr[r]);
    span[w] = 32 * md;
}

template <int D>
__global__ void k_winc_fill(const typename IdxT<D>::type *__restrict__ me, const double *__restrict__ vols,
                            const int64_t *__restrict__ inc_ptr, const uint2 *__restrict__ inc, int64_t nnodes,
                            const int64_t *__restrict__ wseg, IncRec *__restrict__ winc)
{
    const int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl >= nnodes) return;
    IncRec *out = winc + wseg[nl >> 5] + (nl & 31);
    const int64_t t0 = inc_ptr[nl], n = inc_ptr[nl + 1] - t0;
    for (int64_t k = 0; k < n; ++k) {
        const uint2 rec = inc[t0 + k];
        const int64_t e = rec.x & 0x3fffffffu;
        int v[D + 1];
        load_element<D>(me, e, v);
        IncRec r;
        r.ea = rec.x;
        r.ranks = rec.y;
#pragma unroll
        for (int a = 0; a < 4; ++a) r.v[a] = a <= D ? v[a < D + 1 ? a : 0] : 0;
        r.vol = vols[e];
        out[32 * k] = r;
    }
}

// max_i (p[i+1] - p[i]) over a prefix array
__global__ void k_max_diff(const int64_t *__restrict__ p, int64_t n, unsigned long long *out)
{
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (unsigned long long)(p[i + 1] - p[i]));
    for (int s = 16; s > 0; s >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, s));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
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

// Per-element state shared by the rows a tile needs from that element.
template <int D>
struct ElemGeo {
    int v[D + 1];
    double vol;
    double G[D + 1][D];
    double W[D + 1], wsum;                      // mass
    double lambs, mus;                          // elastic
    double As[D][D], bs[D], cs[D], a0s;         // general
    double bv[D + 1][D], cv[D + 1][D], a0v[D + 1];
};

// Raw per-element inputs, loaded in two stages (connectivity + volume, then
// vertices + nodal coefficients) so a lane can keep two elements' loads in
// flight before it computes either.
template <int D>
struct ElemRaw {
    int v[D + 1];
    double vol;
    double x[D + 1][D];
    double W[D + 1], lam[D + 1], mu[D + 1];
    double elam, emu;   // elastic, per-element input (lambs_e/mus_e), used when pre_lm
    int pre_lm;
    // general: coefficient sums accumulated while loading (in vertex order,
    // as the reference-order restatement sums them) + the per-vertex terms
    double As[D][D], bs[D], cs[D], a0s;
    double bv[D + 1][D], cv[D + 1][D], a0v[D + 1];
};

// elastic with the reference's per-element lambs/mus (kernels.py:354-356)
template <int D, int OPS>
__device__ __forceinline__ void element_load_lm(const NumArgs &a, int64_t e, ElemRaw<D> &r)
{
    if constexpr ((OPS & OP_ELASTIC) != 0) {
        r.pre_lm = a.lambs_e != nullptr;
        if (r.pre_lm) {
            r.elam = __ldg(a.lambs_e + e);
            r.emu = __ldg(a.mus_e + e);
        }
    }
}

template <int D, int OPS>
__device__ __forceinline__ void element_load1(const NumArgs &a, int64_t e, ElemRaw<D> &r)
{
    load_element<D>((const typename IdxT<D>::type *)a.me, e, r.v);
    r.vol = __ldg(a.vols + e);
    element_load_lm<D, OPS>(a, e, r);
}

// nodal coefficients of the element's vertices (r.v loaded)
template <int D, int OPS>
__device__ __forceinline__ void element_load_coeffs(const NumArgs &a, ElemRaw<D> &r)
{
#pragma unroll
    for (int k = 0; k <= D; ++k) {
        const int vk = r.v[k];
        if constexpr ((OPS & OP_MASS) != 0) r.W[k] = a.w ? __ldg(a.w + vk) : 0.0;
        if constexpr ((OPS & OP_ELASTIC) != 0) {
            r.lam[k] = nodal<D>(a.lamb, a.lamb_const, vk);
            r.mu[k] = nodal<D>(a.mu, a.mu_const, vk);
        }
        if constexpr ((OPS & OP_GENERAL) != 0) {
            if (a.gen_packed) {
                // one 128-byte line per node: [A 3x3 | b | c | a0]
                const double *pp = a.gen_packed + (int64_t)vk * 16;
                double w[16];
#pragma unroll
                for (int h = 0; h < 4; ++h) ldg256(pp + 4 * h, w[4 * h], w[4 * h + 1], w[4 * h + 2], w[4 * h + 3]);
#pragma unroll
                for (int i = 0; i < D; ++i) {
#pragma unroll
                    for (int j = 0; j < D; ++j) r.As[i][j] = k == 0 ? w[i * 3 + j] : SA_ADD(r.As[i][j], w[i * 3 + j]);
                    r.bv[k][i] = w[9 + i];
                    r.cv[k][i] = w[12 + i];
                    r.bs[i] = k == 0 ? w[9 + i] : SA_ADD(r.bs[i], w[9 + i]);
                    r.cs[i] = k == 0 ? w[12 + i] : SA_ADD(r.cs[i], w[12 + i]);
                }
                r.a0v[k] = w[15];
                r.a0s = k == 0 ? w[15] : SA_ADD(r.a0s, w[15]);
            } else {
#pragma unroll
                for (int i = 0; i < D; ++i) {
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        const double t = a.A ? __ldg(a.A + (int64_t)vk * D * D + i * D + j) : a.A_const[i * D + j];
                        r.As[i][j] = k == 0 ? t : SA_ADD(r.As[i][j], t);
                    }
                    const double tb = a.b ? __ldg(a.b + (int64_t)vk * D + i) : 0.0;
                    const double tc = a.c ? __ldg(a.c + (int64_t)vk * D + i) : 0.0;
                    r.bv[k][i] = tb;
                    r.cv[k][i] = tc;
                    r.bs[i] = k == 0 ? tb : SA_ADD(r.bs[i], tb);
                    r.cs[i] = k == 0 ? tc : SA_ADD(r.cs[i], tc);
                }
                const double t0 = a.a0 ? __ldg(a.a0 + vk) : a.a0_const;
                r.a0v[k] = t0;
                r.a0s = k == 0 ? t0 : SA_ADD(r.a0s, t0);
            }
        }
    }
}

template <int D, int OPS>
__device__ __forceinline__ void element_load2(const NumArgs &a, ElemRaw<D> &r)
{
    if constexpr ((OPS & (OP_STIFF | OP_ELASTIC | OP_GENERAL)) != 0) {
#pragma unroll
        for (int k = 0; k <= D; ++k) load_vertex<D>((const typename VecT<D>::type *)a.qv, r.v[k], r.x[k]);
    }
    element_load_coeffs<D, OPS>(a, r);
}

// K1: bit-exact gradients and per-element coefficient sums from raw inputs.
template <int D, int OPS, int CORE>
__device__ __forceinline__ bool element_compute(const ElemRaw<D> &r, ElemGeo<D> &g)
{
    g.vol = r.vol;
    bool degenerate = false;
    if constexpr ((OPS & (OP_STIFF | OP_ELASTIC | OP_GENERAL)) != 0) degenerate = element_gradients<D, CORE>(r.x, g.G);
    if constexpr ((OPS & OP_MASS) != 0) {
#pragma unroll
        for (int k = 0; k <= D; ++k) g.W[k] = r.W[k];
        g.wsum = r.W[0];
#pragma unroll
        for (int k = 1; k <= D; ++k) g.wsum = SA_ADD(g.wsum, r.W[k]);
    }
    if constexpr ((OPS & OP_ELASTIC) != 0) {
        if (r.pre_lm) {
            g.lambs = r.elam;
            g.mus = r.emu;
        } else {
            // lambs = (sum_k lamb_k) * (vols / (d+1))   kernels.py:354-356
            const double scale = __ddiv_rn(r.vol, (double)(D + 1));
            double ls = r.lam[0], ms = r.mu[0];
#pragma unroll
            for (int k = 1; k <= D; ++k) { ls = SA_ADD(ls, r.lam[k]); ms = SA_ADD(ms, r.mu[k]); }
            g.lambs = SA_MUL(ls, scale);
            g.mus = SA_MUL(ms, scale);
        }
    }
    if constexpr ((OPS & OP_GENERAL) != 0) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
#pragma unroll
            for (int j = 0; j < D; ++j) g.As[i][j] = r.As[i][j];
            g.bs[i] = r.bs[i];
            g.cs[i] = r.cs[i];
        }
        g.a0s = r.a0s;
#pragma unroll
        for (int k = 0; k <= D; ++k) {
#pragma unroll
            for (int i = 0; i < D; ++i) { g.bv[k][i] = r.bv[k][i]; g.cv[k][i] = r.cv[k][i]; }
            g.a0v[k] = r.a0v[k];
        }
    }
    return degenerate;
}

// vol / (d+1): for d = 1, 3 a power-of-two divisor, so the product with its
// exact reciprocal is the same correctly rounded value as the division
template <int D>
__device__ __forceinline__ double general_s1(double vol)
{
    if constexpr (D == 1) return SA_MUL(vol, 0.5);
    else if constexpr (D == 3) return SA_MUL(vol, 0.25);
    else return __ddiv_rn(vol, (double)(D + 1));
}

// General operator, all (d+1)^2 local entries of one element with the
// subexpressions every row shares computed once (A^s G_beta, b^s + b_beta,
// c^s + c_alpha, a0^s + a0_alpha, the volume scalings).  Each entry's
// operations and their order are element_krow's: bitwise the same values.
template <int D>
__device__ __forceinline__ void general_all_rows(const NumArgs &a, const ElemGeo<D> &g, double (&K)[D + 1][D + 1])
{
    const double s1 = general_s1<D>(g.vol);
    const double s2 = __ddiv_rn(g.vol, (double)((D + 1) * (D + 2)));
    const double cd = SA_MUL(a.mass_coef_diag, g.vol), co = SA_MUL(a.mass_coef_off, g.vol);
    double AG[D + 1][D], bb[D + 1][D], cc[D + 1][D], a0a[D + 1];
#pragma unroll
    for (int b = 0; b <= D; ++b) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double t = SA_MUL(g.As[i][0], g.G[b][0]);
#pragma unroll
            for (int j = 1; j < D; ++j) t = SA_ADD(t, SA_MUL(g.As[i][j], g.G[b][j]));
            AG[b][i] = t;
            bb[b][i] = SA_ADD(g.bs[i], g.bv[b][i]);
            cc[b][i] = SA_ADD(g.cs[i], g.cv[b][i]);
        }
        a0a[b] = SA_ADD(g.a0s, g.a0v[b]);
    }
#pragma unroll
    for (int al = 0; al <= D; ++al) {
        const double(&ga)[D] = g.G[al];
#pragma unroll
        for (int b = 0; b <= D; ++b) {
            double diff = SA_MUL(ga[0], AG[b][0]);
            double conv = SA_MUL(bb[b][0], ga[0]);
            double tran = SA_MUL(cc[al][0], g.G[b][0]);
#pragma unroll
            for (int i = 1; i < D; ++i) {
                diff = SA_ADD(diff, SA_MUL(ga[i], AG[b][i]));
                conv = SA_ADD(conv, SA_MUL(bb[b][i], ga[i]));
                tran = SA_ADD(tran, SA_MUL(cc[al][i], g.G[b][i]));
            }
            const double rea = SA_MUL(b == al ? cd : co, SA_ADD(a0a[al], g.a0v[b]));
            K[al][b] = SA_ADD(SA_ADD(SA_SUB(SA_MUL(diff, s1), SA_MUL(conv, s2)), SA_MUL(tran, s2)), rea);
        }
    }
}

// K2: local row ALPHA of every requested operator, stored to dst with layout
// dst[((b * NOUT + o) * M + l) * M + n] (entry (dof row (l, ALPHA), dof col (n, b))).
template <int D, int M, int OPS, int ALPHA>
__device__ __forceinline__ void element_krow(const NumArgs &a, const ElemGeo<D> &g, double *dst)
{
    constexpr int NOUT = n_outputs<OPS>();
    int o = 0;
    if constexpr ((OPS & OP_MASS) != 0) {
        // kernels.py:76-78: (coef * vols) * ((wsum + W[alpha]) + W[beta])
        const double cd = SA_MUL(a.mass_coef_diag, g.vol), co = SA_MUL(a.mass_coef_off, g.vol);
        if (a.w) {
            const double wsa = SA_ADD(g.wsum, g.W[ALPHA]);
#pragma unroll
            for (int b = 0; b <= D; ++b) dst[(b * NOUT + o) * M * M] = SA_MUL(b == ALPHA ? cd : co, SA_ADD(wsa, g.W[b]));
        } else {
            // constant weight: (wsum + W[alpha]) + W[beta] is one constant
            const double vd = SA_MUL(cd, a.mass_wc), vo = SA_MUL(co, a.mass_wc);
#pragma unroll
            for (int b = 0; b <= D; ++b) dst[(b * NOUT + o) * M * M] = b == ALPHA ? vd : vo;
        }
        ++o;
    }
    if constexpr ((OPS & OP_STIFF) != 0) {
#pragma unroll
        for (int b = 0; b <= D; ++b) dst[(b * NOUT + o) * M * M] = stiff_entry<D>(g.G[ALPHA], g.G[b], g.vol);
        ++o;
    }
    if constexpr ((OPS & OP_ELASTIC) != 0) {
#pragma unroll
        for (int b = 0; b <= D; ++b)
#pragma unroll
            for (int l = 0; l < M; ++l)
#pragma unroll
                for (int n = 0; n < M; ++n)
                    dst[((b * NOUT + o) * M + l) * M + n] = elastic_entry<D>(g.G[ALPHA], g.G[b], l, n, g.lambs, g.mus);
        ++o;
    }
    if constexpr ((OPS & OP_GENERAL) != 0) {
        const double s1 = general_s1<D>(g.vol);
        const double s2 = __ddiv_rn(g.vol, (double)((D + 1) * (D + 2)));
        const double cd = SA_MUL(a.mass_coef_diag, g.vol), co = SA_MUL(a.mass_coef_off, g.vol);
        const double(&ga)[D] = g.G[ALPHA];
#pragma unroll
        for (int b = 0; b <= D; ++b) {
            double AG[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double t = SA_MUL(g.As[i][0], g.G[b][0]);
#pragma unroll
                for (int j = 1; j < D; ++j) t = SA_ADD(t, SA_MUL(g.As[i][j], g.G[b][j]));
                AG[i] = t;
            }
            double diff = SA_MUL(ga[0], AG[0]);
            double conv = SA_MUL(SA_ADD(g.bs[0], g.bv[b][0]), ga[0]);
            double tran = SA_MUL(SA_ADD(g.cs[0], g.cv[ALPHA][0]), g.G[b][0]);
#pragma unroll
            for (int i = 1; i < D; ++i) {
                diff = SA_ADD(diff, SA_MUL(ga[i], AG[i]));
                conv = SA_ADD(conv, SA_MUL(SA_ADD(g.bs[i], g.bv[b][i]), ga[i]));
                tran = SA_ADD(tran, SA_MUL(SA_ADD(g.cs[i], g.cv[ALPHA][i]), g.G[b][i]));
            }
            const double rea = SA_MUL(b == ALPHA ? cd : co, SA_ADD(SA_ADD(g.a0s, g.a0v[ALPHA]), g.a0v[b]));
            dst[(b * NOUT + o) * M * M] =
                SA_ADD(SA_ADD(SA_SUB(SA_MUL(diff, s1), SA_MUL(conv, s2)), SA_MUL(tran, s2)), rea);
        }
        ++o;
    }
}

// Local row alpha of constant-weight mass and/or stiffness with alpha chosen
// by selects instead of a branch per alpha: one copy of the arithmetic
// (G_alpha selected, then element_krow's operations in element_krow's order:
// the same values bit for bit).  Lean row-gather instances use it.
template <int D, int OPS>
__device__ __forceinline__ void element_krow_sel(const NumArgs &a, const ElemGeo<D> &g, int alpha, double *dst)
{
    constexpr int NOUT = n_outputs<OPS>();
    int o = 0;
    if constexpr ((OPS & OP_MASS) != 0) {
        const double cd = SA_MUL(a.mass_coef_diag, g.vol), co = SA_MUL(a.mass_coef_off, g.vol);
        const double vd = SA_MUL(cd, a.mass_wc), vo = SA_MUL(co, a.mass_wc);
#pragma unroll
        for (int b = 0; b <= D; ++b) dst[b * NOUT + o] = b == alpha ? vd : vo;
        ++o;
    }
    if constexpr ((OPS & OP_STIFF) != 0) {
        double ga[D];
        select_row<D>(g.G, alpha, ga);
#pragma unroll
        for (int b = 0; b <= D; ++b) dst[b * NOUT + o] = stiff_entry<D>(ga, g.G[b], g.vol);
        ++o;
    }
    if constexpr ((OPS & OP_ELASTIC) != 0) {   // OPS == OP_ELASTIC, M == D
        double ga[D];
        select_row<D>(g.G, alpha, ga);
#pragma unroll
        for (int b = 0; b <= D; ++b)
#pragma unroll
            for (int l = 0; l < D; ++l)
#pragma unroll
                for (int n = 0; n < D; ++n)
                    dst[(b * D + l) * D + n] = elastic_entry<D>(ga, g.G[b], l, n, g.lambs, g.mus);
    }
}

// runtime local row alpha -> compile-time element_krow<alpha>
template <int D, int M, int OPS, int A = 0>
__device__ __forceinline__ void krow_runtime(const NumArgs &a, const ElemGeo<D> &g, int alpha, double *vals)
{
    if (alpha == A) element_krow<D, M, OPS, A>(a, g, vals);
    else if constexpr (A < D) krow_runtime<D, M, OPS, A + 1>(a, g, alpha, vals);
}

// v1 / fallback numeric kernel: one thread per node row, private smem
// accumulators indexed by the 8-bit column ranks stored with each incidence.
// Used when a node has more than 31 incidences or the block kernel's shared
// memory does not fit.
template <int D, int M, int OPS, int CORE, int ILP, int MINB, bool PRE = false, bool LEAN = false, bool GUARD = false>
__global__ void __launch_bounds__(128, MINB) k_numeric_rowgather(NumArgs a_in)
{
    // LEAN: a constant mass weight, known at compile time (the local copy is
    // scalar-replaced; w == nullptr folds the weight loads away)
    NumArgs a = a_in;
    if constexpr (LEAN) a.w = nullptr;
    constexpr int NOUT = n_outputs<OPS>();
    extern __shared__ double smem_acc[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t nl = blockIdx.x * (int64_t)blockDim.x + tid;
    // Accumulators: per warp and output a plane of 32 lane rows of S doubles;
    // lane j's dof row l, column k at wacc[o*32*S + j*S + l*M*deg + k].  When
    // the warp's rows all have degree d0, S = M*M*d0 and the plane IS the
    // warp's CSR run (row-major, consecutive rows), so the store phase is a
    // straight coalesced copy; otherwise S is padded to the warp's largest
    // row (odd, so lane strides hit distinct banks) and rows store their own
    // segments.
    const unsigned full = 0xffffffffu;
    const bool in_range = nl < a.nnodes;
    const int64_t c0 = in_range ? a.colptr[nl] : 0;
    const int deg_row = in_range ? (int)(a.colptr[nl + 1] - c0) : -1;
    const bool active = in_range && deg_row <= a.light_deg;   // heavy rows: k_heavy_rows
    const int deg = active ? deg_row : -1;
    // the row's CSR base, loaded with the degree (independent loads: one
    // round trip) rather than after the incidence loop
    const int64_t row_base = active ? a.indptr[M * nl] : 0;
    const int64_t inc0 = active ? a.inc_ptr[nl] : 0, inc1 = active ? a.inc_ptr[nl + 1] : 0;
    const int d0 = __shfl_sync(full, deg, 0);
    const bool uniform = __all_sync(full, deg == d0) && d0 > 0;
    int dmax = deg;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) dmax = max(dmax, __shfl_xor_sync(full, dmax, sh));
    const int S = uniform ? M * M * d0 : ((M * M * max(dmax, 0)) | 1);
    double *wacc = smem_acc + (size_t)(tid >> 5) * NOUT * 32 * (a.acc_stride | 1) + lane * S;
    int nz[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) nz[o] = 0;
    double rbound = 0.0;   // GUARD: sum over the row's contributions of |K[alpha][beta]|
    if (active) {
        const int deg_stride = M * deg;
        for (int o = 0; o < NOUT; ++o)
            for (int k = 0; k < M * deg_stride; ++k) wacc[o * 32 * S + k] = 0.0;
        const int64_t t1 = inc1;
        int64_t emin = INT64_MAX;
        constexpr int MM = M * M;
        constexpr int VPR = (D + 1) * NOUT * MM;
        // fold one local row set into the row accumulators (ranks: 8-bit
        // column rank of each element vertex within this row)
        auto accum = [&](const double(&vals)[VPR], unsigned ranks) {
            if constexpr (GUARD) {   // fast values: the zero guard's magnitude, sum of |contributions|
#pragma unroll
                for (int i = 0; i < VPR; ++i) rbound += fabs(vals[i]);
            }
#pragma unroll
            for (int b = 0; b <= D; ++b) {
                const int r = (ranks >> (8 * b)) & 0xff;
#pragma unroll
                for (int o = 0; o < NOUT; ++o)
#pragma unroll
                    for (int l = 0; l < M; ++l)
#pragma unroll
                        for (int n = 0; n < M; ++n)
                            wacc[o * 32 * S + l * deg_stride + r * M + n] += vals[(b * NOUT + o) * MM + l * M + n];
            }
        };
        auto fold = [&](const ElemRaw<D> &x, uint2 rec) {
            ElemGeo<D> g;
            const int64_t e = rec.x & 0x3fffffffu;
            if (element_compute<D, OPS, CORE>(x, g)) emin = min(emin, e);
            double vals[(D + 1) * NOUT * MM];
            if constexpr (LEAN && ((M == 1 && (OPS & ~(OP_MASS | OP_STIFF)) == 0) || OPS == OP_ELASTIC))
                element_krow_sel<D, OPS>(a, g, rec.x >> 30, vals);
            else
                krow_runtime<D, M, OPS>(a, g, rec.x >> 30, vals);
            accum(vals, rec.y);
        };
        const int64_t t0 = inc0;
        // (lean instances: warp-interleaved records exactly in 3D)
        const bool use_w = LEAN ? D == 3 : a.winc != nullptr;
        const IncRec *wrec = use_w ? a.winc + a.wseg[nl >> 5] + (nl & 31) : nullptr;
        // stage 1 of incidence t: its record, connectivity and volume
        auto load1 = [&](int64_t t, uint2 &rec, ElemRaw<D> &x) {
            if (use_w) {
                unsigned long long u0, u1, u2, u3;
                asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                    : "=l"(u0), "=l"(u1), "=l"(u2), "=l"(u3)
                    : "l"(wrec + 32 * (t - t0)));
                rec = make_uint2((unsigned)u0, (unsigned)(u0 >> 32));
                x.v[0] = (int)(unsigned)u1;
                if constexpr (D >= 1) x.v[1] = (int)(unsigned)(u1 >> 32);
                if constexpr (D >= 2) x.v[2] = (int)(unsigned)u2;
                if constexpr (D >= 3) x.v[3] = (int)(unsigned)(u2 >> 32);
                x.vol = __longlong_as_double((long long)u3);
                element_load_lm<D, OPS>(a, rec.x & 0x3fffffffu, x);
            } else {
                rec = __ldg(a.inc + t);
                element_load1<D, OPS>(a, rec.x & 0x3fffffffu, x);
            }
        };
        int64_t t = t0;
        if constexpr (PRE) {
            // two-pass fold: the element pass left this incidence's local
            // row(s) in its slot (warp-interleaved: incidence k of lane j of
            // the warp at wseg + 32 k + j, so each warp load is one contiguous
            // run); ranks and rows are independent loads -- no gather chain,
            // U incidences in flight
            const int64_t sb = a.wseg[nl >> 5] + lane;
            auto loadk = [&](int64_t slot, double(&v)[VPR]) {
                const double *src = a.kbuf + slot * a.kstride;
                if constexpr (VPR % 4 == 0) {
#pragma unroll
                    for (int i = 0; i < VPR; i += 4) ldg256_cs(src + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
                } else if constexpr (VPR % 2 == 0) {
#pragma unroll
                    for (int i = 0; i < VPR; i += 2) {
                        const double2 w = __ldg((const double2 *)(src + i));
                        v[i] = w.x;
                        v[i + 1] = w.y;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < VPR; ++i) v[i] = __ldg(src + i);
                }
            };
            constexpr int U = ILP < 1 ? 1 : ILP;
            for (; t + U <= t1; t += U) {
                unsigned rk[U];
                double v[U][VPR];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t slot = sb + 32 * (t + u - t0);
                    rk[u] = __ldcs(a.tp_rank + slot);
                    loadk(slot, v[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) accum(v[u], rk[u]);
            }
            for (; t < t1; ++t) {
                double v[VPR];
                const int64_t slot = sb + 32 * (t - t0);
                const unsigned rk = __ldcs(a.tp_rank + slot);
                loadk(slot, v);
                accum(v, rk);
            }
        } else if constexpr (ILP == 3) {
            // software pipeline: while incidence t is folded, the vertex /
            // coefficient gathers of t+1 and the record of t+2 are in flight
            // (index clamped to the row's last incidence: the tail re-reads it)
            if (t < t1) {
                const int64_t last = t1 - 1;
                uint2 rc, rn;
                ElemRaw<D> xc, xn;
                load1(t, rc, xc);
                load1(min(t + 1, last), rn, xn);
                element_load2<D, OPS>(a, xc);
                for (; t < t1; ++t) {
                    uint2 rnn;
                    ElemRaw<D> xnn;
                    load1(min(t + 2, last), rnn, xnn);
                    element_load2<D, OPS>(a, xn);
                    fold(xc, rc);
                    xc = xn;
                    rc = rn;
                    xn = xnn;
                    rn = rnn;
                }
            }
        }
        for (; !PRE && ILP == 2 && t + 1 < t1; t += 2) {
            uint2 r1, r2;
            ElemRaw<D> x1, x2;
            load1(t, r1, x1);
            load1(t + 1, r2, x2);
            element_load2<D, OPS>(a, x1);
            element_load2<D, OPS>(a, x2);
            fold(x1, r1);
            fold(x2, r2);
        }
        for (; !PRE && t < t1; ++t) {
            uint2 r1;
            ElemRaw<D> x1;
            load1(t, r1, x1);
            element_load2<D, OPS>(a, x1);
            fold(x1, r1);
        }
        if (emin != INT64_MAX) atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)emin);
    }
    // Stores (see the accumulator layout above)
    __syncwarp();
    if constexpr (GUARD) {
        // an entry this small relative to its row's contributions may be an
        // exact zero of the reference-order sum: the row is recomputed in
        // reference order (k_guard_fixup) and its zeros counted there
        if (active) {
            bool flag = false;
            const double thr = SA_GUARD_TAU * rbound;
            for (int k = 0; k < M * M * deg; ++k) flag |= fabs(wacc[k]) <= thr;
            if (flag) a.flag_rows[atomicAdd(a.nflag, 1)] = (uint32_t)nl;
        }
    }
    if (uniform) {
        const int64_t base = __shfl_sync(full, row_base, 0);
        const double *plane = wacc - lane * S;
        for (int i = lane; i < 32 * S; i += 32) {
#pragma unroll
            for (int o = 0; o < NOUT; ++o) {
                const double val = plane[o * 32 * S + i];
                a.vals[o][base + i] = val;
                if constexpr (!GUARD) nz[o] += (val == 0.0);
            }
        }
    } else if (active) {
        for (int o = 0; o < NOUT; ++o) {
            double *out = a.vals[o];
            for (int l = 0; l < M; ++l) {
                const int64_t p = a.indptr[M * nl + l];
                for (int k = 0; k < M * deg; ++k) {
                    const double val = wacc[o * 32 * S + l * M * deg + k];
                    out[p + k] = val;
                    if constexpr (!GUARD) nz[o] += (val == 0.0);
                }
            }
        }
    }
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
        int v = nz[o];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
        if ((tid & 31) == 0 && v) atomicAdd((unsigned long long *)(a.counters + o), (unsigned long long)v);
    }
}

// ---------------------------------------------------------------------------
// Two-pass numeric ("element rows"): pass 1 computes every element of the
// block ONCE (geometry + all its local rows the block owns) and writes each
// local row to the slot of its incidence; pass 2 is the row-gather fold
// (k_numeric_rowgather<PRE = true>) streaming those rows in ascending element
// order.  Same per-element arithmetic, same fold order: bitwise the one-pass
// result.  Pays 2 x (local row bytes) of HBM traffic per incidence to save
// (d+1)-fold recomputation and the per-incidence gathers of vertex
// coordinates and nodal coefficients (the general operator's 4 x 128 B).

// 256-bit store (sm_100)
__device__ __forceinline__ void st256(double *p, double a, double b, double c, double d)
{
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
// streaming variants (evict-first): data touched once -- the two-pass local
// rows, slot maps -- should not push the staged vertex records out of L2
__device__ __forceinline__ void st256_cs(double *p, double a, double b, double c, double d)
{
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

template <int VPR>
__device__ __forceinline__ void store_row(double *dst, const double (&vals)[VPR])
{
    if constexpr (VPR % 4 == 0) {
#pragma unroll
        for (int i = 0; i < VPR; i += 4) st256_cs(dst + i, vals[i], vals[i + 1], vals[i + 2], vals[i + 3]);
    } else if constexpr (VPR % 2 == 0) {
#pragma unroll
        for (int i = 0; i < VPR; i += 2) *(double2 *)(dst + i) = make_double2(vals[i], vals[i + 1]);
    } else {
#pragma unroll
        for (int i = 0; i < VPR; ++i) dst[i] = vals[i];
    }
}

template <int D, int M, int OPS, int A = 0>
__device__ __forceinline__ void element_rows_store(const NumArgs &a, const ElemGeo<D> &g, const unsigned (&pos)[4])
{
    constexpr int VPR = (D + 1) * n_outputs<OPS>() * M * M;
    if constexpr (OPS == OP_GENERAL && A == 0) {
        double K[D + 1][D + 1];
        general_all_rows<D>(a, g, K);
#pragma unroll
        for (int al = 0; al <= D; ++al)
            if (pos[al] != 0xffffffffu) store_row<D + 1>(a.kbuf + (int64_t)pos[al] * a.kstride, K[al]);
        return;
    }
    if (pos[A] != 0xffffffffu) {
        double vals[VPR];
        element_krow<D, M, OPS, A>(a, g, vals);
        double *dst = a.kbuf + (int64_t)pos[A] * a.kstride;
        if constexpr (VPR % 4 == 0) {
#pragma unroll
            for (int i = 0; i < VPR; i += 4) st256(dst + i, vals[i], vals[i + 1], vals[i + 2], vals[i + 3]);
        } else if constexpr (VPR % 2 == 0) {
#pragma unroll
            for (int i = 0; i < VPR; i += 2) *(double2 *)(dst + i) = make_double2(vals[i], vals[i + 1]);
        } else {
#pragma unroll
            for (int i = 0; i < VPR; ++i) dst[i] = vals[i];
        }
    }
    if constexpr (A < D) element_rows_store<D, M, OPS, A + 1>(a, g, pos);
}

template <int D, int M, int OPS, int CORE, int MINB>
__global__ void __launch_bounds__(128, MINB) k_element_rows(NumArgs a)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.ne) return;
    const int64_t e = a.e_lo + i;
    // slot map, connectivity and volume are independent: one round trip
    const uint4 p = __ldg(a.epos + i);
    ElemRaw<D> x;
    element_load1<D, OPS>(a, e, x);
    const unsigned pos[4] = {p.x, p.y, p.z, p.w};
    bool any = false;
#pragma unroll
    for (int k = 0; k <= D; ++k) any |= pos[k] != 0xffffffffu;
    if (!any) return;   // element does not touch the block
    element_load2<D, OPS>(a, x);
    ElemGeo<D> g;
    if (element_compute<D, OPS, CORE>(x, g)) atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)e);
    element_rows_store<D, M, OPS>(a, g, pos);
}

// ---------------------------------------------------------------------------
// Batched element pass: a block takes EB_SIZE consecutive elements, stages
// the batch's distinct vertices (coordinates + packed nodal coefficients,
// EB_REC doubles each) ONCE in shared memory with cp.async, then every
// thread computes its element from the stage.  A vertex is shared by ~24
// tetrahedra, so a batch of 128 consecutive elements of a Kuhn mesh needs
// ~90 records instead of 512 register gathers; the compute phase holds no
// load destinations, so more warps fit and the fp64 pipe stays fed.
constexpr int EB_SIZE = 256;   // elements per batch (C5: ~150 distinct vertices staged per batch)
constexpr int EB_CAP = 255;    // distinct vertices per batch (8-bit local ids)
// staged doubles per vertex: q (4, padded) + [A(9) b(3) c(3) a0] + 2 pad: a
// 176-byte stride = 11 x 16 B (odd), so the 128-bit shared loads of lanes
// reading different vertices spread over the banks (the 160-byte stride put
// every 4th vertex on the same bank group: L1 at 81 % of peak in C5)
constexpr int EB_REC = 22;

// one staged vertex record as 10 x 128-bit shared loads: c[0..3] = q (padded), w[0..15]
__device__ __forceinline__ void stage_record(const double *__restrict__ rec, double (&c)[4], double (&w)[16])
{
    const double2 *r2 = reinterpret_cast<const double2 *>(rec);
    double2 t = r2[0];
    c[0] = t.x; c[1] = t.y;
    t = r2[1];
    c[2] = t.x; c[3] = t.y;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        t = r2[2 + h];
        w[2 * h] = t.x;
        w[2 * h + 1] = t.y;
    }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// symbolic (once per plan): sorted unique vertices of every batch, local ids
template <int D>
__global__ void __launch_bounds__(EB_SIZE) k_eb_build(const typename IdxT<D>::type *__restrict__ me, int64_t e_lo,
                                                      int64_t ne, int32_t *__restrict__ verts,
                                                      int32_t *__restrict__ count, uint32_t *__restrict__ loc,
                                                      unsigned long long *maxn)
{
    constexpr int NK = 4 * EB_SIZE;
    __shared__ int keys[NK];
    __shared__ int part[EB_SIZE / 32];
    __shared__ int nuniq;
    const int t = threadIdx.x;
    const int64_t b = blockIdx.x, i = b * EB_SIZE + t;
    int v[D + 1];
    if (i < ne) load_element<D>(me, e_lo + i, v);
#pragma unroll
    for (int k = 0; k < 4; ++k) keys[k * EB_SIZE + t] = (i < ne && k <= D) ? v[k < D + 1 ? k : 0] : INT_MAX;
    __syncthreads();
    // bitonic sort, NK/2 compare pairs per stage
    for (int kk = 2; kk <= NK; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int pi = t; pi < NK / 2; pi += EB_SIZE) {
                const int lo = 2 * j * (pi / j) + (pi % j), hi = lo + j;
                const bool up = (lo & kk) == 0;
                const int x = keys[lo], y = keys[hi];
                if ((x > y) == up) { keys[lo] = y; keys[hi] = x; }
            }
            __syncthreads();
        }
    // unique: heads among this thread's 4 consecutive keys, block scan
    int h[4], cnt = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int j = 4 * t + k;
        h[k] = keys[j] != INT_MAX && (j == 0 || keys[j] != keys[j - 1]);
        cnt += h[k];
    }
    int incl = cnt;
#pragma unroll
    for (int sh = 1; sh < 32; sh <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, sh);
        if ((t & 31) >= sh) incl += y;
    }
    if ((t & 31) == 31) part[t >> 5] = incl;
    __syncthreads();
    int off = incl - cnt;
    for (int w = 0; w < (t >> 5); ++w) off += part[w];
    if (t == EB_SIZE - 1) nuniq = off + cnt;
    int u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { u[k] = off; off += h[k]; }
    int kv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) kv[k] = keys[4 * t + k];
    __syncthreads();
    const int n = nuniq;
    // compact the unique keys to the front of keys[] and to the batch list
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (h[k]) {
            keys[u[k]] = kv[k];
            if (n <= EB_CAP) verts[b * EB_CAP + u[k]] = kv[k];
        }
    __syncthreads();
    if (t == 0) {
        count[b] = n <= EB_CAP ? n : -1;
        atomicMax(maxn, (unsigned long long)n);   // > EB_CAP: some batch takes the direct path
    }
    if (i < ne && n <= EB_CAP) {
        unsigned l = 0;
#pragma unroll
        for (int k = 0; k <= D; ++k) {
            int lo = 0, hi = n;
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (keys[mid] < v[k]) lo = mid + 1; else hi = mid; }
            l |= (unsigned)lo << (8 * k);
        }
        loc[i] = l;
    }
}

// ElemRaw from the staged vertex records (same summation order as
// element_load_coeffs: vertex 0..d, packed general coefficients)
template <int D, int OPS>
__device__ __forceinline__ void element_from_stage(const double *__restrict__ vrec, unsigned lc, ElemRaw<D> &r)
{
#pragma unroll
    for (int k = 0; k <= D; ++k) {
        double cq[4], w[16];
        stage_record(vrec + ((lc >> (8 * k)) & 0xff) * EB_REC, cq, w);
#pragma unroll
        for (int c = 0; c < D; ++c) r.x[k][c] = cq[c];
#pragma unroll
        for (int ii = 0; ii < D; ++ii) {
#pragma unroll
            for (int j = 0; j < D; ++j) r.As[ii][j] = k == 0 ? w[ii * 3 + j] : SA_ADD(r.As[ii][j], w[ii * 3 + j]);
            r.bv[k][ii] = w[9 + ii];
            r.cv[k][ii] = w[12 + ii];
            r.bs[ii] = k == 0 ? w[9 + ii] : SA_ADD(r.bs[ii], w[9 + ii]);
            r.cs[ii] = k == 0 ? w[12 + ii] : SA_ADD(r.cs[ii], w[12 + ii]);
        }
        r.a0v[k] = w[15];
        r.a0s = k == 0 ? w[15] : SA_ADD(r.a0s, w[15]);
    }
}


// General operator, fast mode, from the staged vertex records (EB_REC
// doubles: q padded to 4 | [A 3x3 | b | c | a0]): gradients bitwise
// (element_gradients -- the same degeneracy test as exact mode), the local
// matrix regrouped for fused multiply-adds:
//   Q_b = s1 As G_b - s2 (bs + b_b),  R_a = s2 (cs + c_a),
//   K[a][b] = G_a . Q_b + G_b . R_a + (a == b ? cd : co) ((a0s + a0_a) + a0_b)
// ~210 fp64 instructions for the 16 entries instead of ~370 in reference
// order.  Rows go to their incidence slots (pos) as in element_rows_store.
template <int D, int CORE>
__device__ __forceinline__ bool stage_general_fast(const NumArgs &a, const double *__restrict__ vrec, unsigned lc,
                                                   double vol, const unsigned (&pos)[4])
{
    const double2 *rk[D + 1];   // records as 16-byte words (EB_REC even, 16 B aligned)
#pragma unroll
    for (int k = 0; k <= D; ++k) rk[k] = reinterpret_cast<const double2 *>(vrec + ((lc >> (8 * k)) & 0xff) * EB_REC);
    double G[D + 1][D];
    bool deg;
    {
        double x[D + 1][D];
#pragma unroll
        for (int k = 0; k <= D; ++k) {
            const double2 t0 = rk[k][0], t1 = rk[k][1];
            const double c4[4] = {t0.x, t0.y, t1.x, t1.y};
#pragma unroll
            for (int c = 0; c < D; ++c) x[k][c] = c4[c];
        }
        deg = element_gradients<D, CORE>(x, G);
    }
    const double s1 = vol * (1.0 / (D + 1));
    const double s2 = vol * (1.0 / ((D + 1) * (D + 2)));
    const double cd = a.mass_coef_diag * vol, co = a.mass_coef_off * vol;
    double As[D][D], bs[D], cs[D], a0s;
#pragma unroll
    for (int k = 0; k <= D; ++k) {
        double w[16];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            const double2 t = rk[k][2 + h];
            w[2 * h] = t.x;
            w[2 * h + 1] = t.y;
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
#pragma unroll
            for (int j = 0; j < D; ++j) As[i][j] = k == 0 ? w[i * 3 + j] : As[i][j] + w[i * 3 + j];
            bs[i] = k == 0 ? w[9 + i] : bs[i] + w[9 + i];
            cs[i] = k == 0 ? w[12 + i] : cs[i] + w[12 + i];
        }
        a0s = k == 0 ? w[15] : a0s + w[15];
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) As[i][j] *= s1;
        bs[i] *= -s2;
        cs[i] *= s2;
    }
    double Rv[D + 1][D], ea[D + 1], a0v[D + 1];
#pragma unroll
    for (int k = 0; k <= D; ++k) {
        const double2 t6 = rk[k][8], t7 = rk[k][9];   // w[12..15] = c (3) | a0
        const double cw[3] = {t6.x, t6.y, t7.x};
#pragma unroll
        for (int i = 0; i < D; ++i) Rv[k][i] = __fma_rn(s2, cw[i], cs[i]);
        a0v[k] = t7.y;
        ea[k] = a0s + t7.y;
    }
    double K[D + 1][D + 1];
#pragma unroll
    for (int b = 0; b <= D; ++b) {
        const double2 t4 = rk[b][6], t5 = rk[b][7];   // w[8..11]: w[9..11] = b
        const double bw[3] = {t4.y, t5.x, t5.y};
        double Q[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double t = __fma_rn(-s2, bw[i], bs[i]);
#pragma unroll
            for (int j = 0; j < D; ++j) t = __fma_rn(As[i][j], G[b][j], t);
            Q[i] = t;
        }
#pragma unroll
        for (int al = 0; al <= D; ++al) {
            double t = (al == b ? cd : co) * (ea[al] + a0v[b]);
#pragma unroll
            for (int i = 0; i < D; ++i) t = __fma_rn(G[al][i], Q[i], t);
#pragma unroll
            for (int i = 0; i < D; ++i) t = __fma_rn(G[b][i], Rv[al][i], t);
            K[al][b] = t;
        }
    }
#pragma unroll
    for (int al = 0; al <= D; ++al)
        if (pos[al] != 0xffffffffu) store_row<D + 1>(a.kbuf + (int64_t)pos[al] * a.kstride, K[al]);
    return deg;
}

// Pipelined batched element pass (every batch staged): persistent blocks
// walk batches b, b + G, b + 2G, ... with a three-stage cp.async pipeline --
// the vertex list of batch k+2 and the vertex records of batch k+1 are in
// flight while batch k is computed -- so the staging latency hides behind
// the fp64 work instead of alternating with it.  Same per-element values.
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int D, int M, int OPS, int CORE, int MINB, bool FAST = false>
__global__ void __launch_bounds__(EB_SIZE, MINB) k_element_rows_pipe(NumArgs a)
{
    extern __shared__ double dyn[];
    double *recs = dyn;                                                 // [2][maxn][EB_REC]
    int *svs = (int *)(dyn + 2 * (size_t)a.eb_maxn * EB_REC);           // [3][EB_CAP + 1] (+ count)
    const int t = threadIdx.x;
    const int64_t nb = a.eb_b1;   // batches [eb_b0, eb_b1) of this launch
    const int64_t G = gridDim.x;
    const int RS = a.eb_maxn * EB_REC;
    auto issue_list = [&](int64_t bb, int stage) {   // vertex list + count of batch bb
        if (bb >= nb) return;
        int *sv = svs + stage * (EB_CAP + 1);
        const int32_t *vl = a.eb_verts + bb * EB_CAP;
        for (int s = t; s < EB_CAP; s += EB_SIZE) cp_async4(sv + s, vl + s);
        if (t == 0) cp_async4(sv + EB_CAP, a.eb_count + bb);
    };
    auto issue_recs = [&](int64_t bb, int lstage, int rstage) {   // vertex records of batch bb
        if (bb >= nb) return;
        const int *sv = svs + lstage * (EB_CAP + 1);
        double *rec = recs + (size_t)rstage * RS;
        const int n = sv[EB_CAP];
        for (int c = t; c < n * 10; c += EB_SIZE) {
            const int s = c / 10, h = c - 10 * s;
            const int64_t vv = sv[s];
            const double *src = h < 2 ? (const double *)a.qv + vv * 4 + 2 * h : a.gen_packed + vv * 16 + 2 * (h - 2);
            cp_async16(rec + s * EB_REC + 2 * h, src);
        }
    };
    const int64_t b0 = a.eb_b0 + blockIdx.x;
    if (b0 >= nb) return;
    // prologue: lists of batches 0 and 1, then records of batch 0
    issue_list(b0, 0);
    cp_async_commit();
    issue_list(b0 + G, 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    issue_recs(b0, 0, 0);
    cp_async_commit();
    // this thread's element data of the current batch (registers, one ahead)
    auto own = [&](int64_t bb, uint4 &p, unsigned &lc, double &vol) {
        const int64_t i = bb * EB_SIZE + t;
        p = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
        lc = 0;
        vol = 0.0;
        if (bb < nb && i < a.ne) {
            p = __ldcs(a.epos + i);
            lc = __ldcs(a.eb_loc + i);
            vol = __ldcs(a.vols + a.e_lo + i);
        }
    };
    uint4 p;
    unsigned lc;
    double vol;
    own(b0, p, lc, vol);
    for (int64_t k = 0;; ++k) {
        const int64_t b = b0 + k * G;
        if (b >= nb) break;
        issue_list(b + 2 * G, (int)((k + 2) % 3));
        cp_async_commit();
        cp_async_wait<1>();   // records of batch k and the list of batch k+1 have landed
        __syncthreads();
        issue_recs(b + G, (int)((k + 1) % 3), (int)((k + 1) & 1));
        cp_async_commit();
        uint4 pn;
        unsigned lcn;
        double voln;
        own(b + G, pn, lcn, voln);
        const int64_t i = b * EB_SIZE + t;
        const unsigned pos[4] = {p.x, p.y, p.z, p.w};
        bool any = false;
#pragma unroll
        for (int kk = 0; kk <= D; ++kk) any |= pos[kk] != 0xffffffffu;
        if (i < a.ne && any) {
            if constexpr (FAST && OPS == OP_GENERAL) {
                if (stage_general_fast<D, CORE>(a, recs + (size_t)(k & 1) * RS, lc, vol, pos))
                    atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)(a.e_lo + i));
            } else {
                ElemRaw<D> x;
                x.vol = vol;
                element_from_stage<D, OPS>(recs + (size_t)(k & 1) * RS, lc, x);
                ElemGeo<D> g;
                if (element_compute<D, OPS, CORE>(x, g))
                    atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)(a.e_lo + i));
                element_rows_store<D, M, OPS>(a, g, pos);
            }
        }
        p = pn;
        lc = lcn;
        vol = voln;
        __syncthreads();   // stage k & 1 is rewritten by the records of batch k+2
    }
    cp_async_wait<0>();
}

// element range of the block's incidences: out[0] = min e, out[1] = max e
__global__ void k_inc_erange(const uint2 *__restrict__ inc, int64_t n, unsigned long long *out)
{
    unsigned lo = 0xffffffffu, hi = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const unsigned e = inc[t].x & 0x3fffffffu;
        lo = min(lo, e);
        hi = max(hi, e);
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, sh));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, sh));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out, (unsigned long long)lo);
        atomicMax(out + 1, (unsigned long long)hi);
    }
}

// slots of node row nl's incidences (warp-interleaved, as winc): slot map of
// (e, alpha) and the column ranks per slot
__global__ void k_tp_slots(const int64_t *__restrict__ inc_ptr, const uint2 *__restrict__ inc, int64_t nnodes,
                           const int64_t *__restrict__ wseg, unsigned e_lo, unsigned *__restrict__ epos,
                           unsigned *__restrict__ rank)
{
    const int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl >= nnodes) return;
    const int64_t base = wseg[nl >> 5] + (nl & 31);
    const int64_t t0 = inc_ptr[nl], n = inc_ptr[nl + 1] - t0;
    for (int64_t k = 0; k < n; ++k) {
        const uint2 rec = inc[t0 + k];
        const int64_t slot = base + 32 * k;
        epos[(int64_t)((rec.x & 0x3fffffffu) - e_lo) * 4 + (rec.x >> 30)] = (unsigned)slot;
        rank[slot] = rec.y;
    }
}

// compaction (K5): drop exact-zero entries (sparse.py:108-111).  Exact zeros
// are rare, so the passes are streaming: every entry is read coalesced once to
// find the zeros (each one looks its row up by binary search and bumps the
// row's counter), and once more by a warp-per-32-rows stream compaction whose
// output offset is the scanned zero count -- no per-row strided walks.
__global__ void k_zero_rows(const int64_t *__restrict__ indptr, const double *__restrict__ vals, int64_t nnz,
                            int64_t nrows, unsigned long long *__restrict__ zcnt)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
        if (vals[p] != 0.0) continue;
        int64_t lo = 0, hi = nrows;   // last row r with indptr[r] <= p
        while (hi - lo > 1) { const int64_t mid = (lo + hi) >> 1; if (indptr[mid] <= p) lo = mid; else hi = mid; }
        atomicAdd(zcnt + lo, 1ull);
    }
}

__global__ void k_new_ptr(const int64_t *__restrict__ indptr, const int64_t *__restrict__ zpre, int64_t nrows,
                          int64_t *__restrict__ out)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r <= nrows) out[r] = indptr[r] - zpre[r];
}

__global__ void k_compact(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                          const double *__restrict__ vals, int64_t nrows, const int64_t *__restrict__ new_ptr,
                          int32_t *__restrict__ out_idx, double *__restrict__ out_val)
{
    const int lane = threadIdx.x & 31;
    const int64_t r0 = 32 * ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (r0 >= nrows) return;
    const int64_t e0 = indptr[r0], e1 = indptr[min(r0 + 32, nrows)];
    int64_t w = new_ptr[r0];
    for (int64_t p = e0 + lane; p - lane < e1; p += 32) {
        const bool in = p < e1;
        const double v = in ? vals[p] : 0.0;
        const int32_t c = in ? indices[p] : 0;
        const bool keep = in && v != 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int64_t q = w + __popc(m & ((1u << lane) - 1));
            out_idx[q] = c;
            out_val[q] = v;
        }
        w += __popc(m);
    }
}

// general-operator coefficient records from their column-compacted upload:
// column j of the 16-double record is column map[j] of the nv uploaded ones,
// or the constant cst[j] when map[j] < 0 (columns that are constant over the
// nodes, or equal to another column -- a symmetric A -- do not cross PCIe)
struct UnpackCols {
    int map[16];
    double cst[16];
};
__global__ void k_unpack_columns(const double *__restrict__ src, int nv, UnpackCols u, int64_t nq, double *__restrict__ dst)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq * 16; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t node = i >> 4;
        const int j = (int)(i & 15);
        const int m = u.map[j];
        dst[i] = m >= 0 ? src[node * nv + m] : u.cst[j];
    }
}

// canonical CSR from a structural one (shared by sa_compact / sa_pk_compact)
inline int compact_csr(const int64_t *indptr, const int32_t *indices, const double *vals, int64_t nr, int64_t nnz,
                       int64_t *scan_tmp, int64_t *indptr_out, int32_t *indices_out, double *vals_out, cudaStream_t st)
{
    int64_t *cnt = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&cnt, (nr + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMemsetAsync(cnt, 0, (nr + 1) * sizeof(int64_t), st));
    if (nr && nnz)
        SA_LAUNCH(k_zero_rows, std::min<int64_t>(grid_for(nnz, 256), 148 * 16), 256, 0, st, indptr, vals, nnz, nr,
                  (unsigned long long *)cnt);
    SA_TRY(exclusive_scan_i64(cnt, cnt, nr, scan_tmp, st));
    SA_LAUNCH(k_new_ptr, grid_for(nr + 1, 256), 256, 0, st, indptr, cnt, nr, indptr_out);
    if (nr) SA_LAUNCH(k_compact, grid_for(nr, 256), 256, 0, st, indptr, indices, vals, nr, indptr_out, indices_out,
                      vals_out);
    SA_CUDA_TRY(cudaFreeAsync(cnt, st));
    return SA_OK;
}

// ---------------------------------------------------------------------------
// dispatch helpers

template <int D>
int mesh_coords(sa_mesh *M, const double *q, const double *vols, cudaStream_t st);

template <int D>
int mesh_kernels(sa_mesh *M, const double *q, const int64_t *me, const int32_t *me32, int rows32, const double *vols,
                 cudaStream_t st)
{
    typedef typename VecT<D>::type V;
    typedef typename IdxT<D>::type I;
    unsigned long long *bad = (unsigned long long *)M->scratch;
    SA_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
    const int B = 256;
    unsigned gq = std::min<int64_t>(grid_for(M->nq, B), 148 * 32);
    unsigned ge = std::min<int64_t>(grid_for(M->nme, B), 148 * 32);
    if (M->nq && q) SA_LAUNCH(k_pack_q<D>, gq, B, 0, st, q, M->nq, (V *)M->qv);
    if (M->nme) SA_LAUNCH(k_pack_me<D>, ge, B, 0, st, me, me32, rows32, M->nq, M->nme, (I *)M->me, bad);
    unsigned long long hbad = 0;
    SA_TRY(readback(&hbad, bad, sizeof hbad, st));
    SA_TRY(sync_stream(st));
    if (hbad != ~0ull) {
        err_state().bad = (int64_t)hbad;
        return set_error(SA_ERR_INDEX_RANGE, "connectivity entry me[%lld, %lld] out of range [0, %lld)",
                         (long long)(hbad / M->nme), (long long)(hbad % M->nme), (long long)M->nq);
    }
    if (!q) {   // coordinates later (sa_mesh_set_coords); given volumes now
        if (vols) {
            SA_CUDA_TRY(cudaMemcpyAsync(M->vols, vols, M->nme * sizeof(double), cudaMemcpyDeviceToDevice, st));
            M->vols_ready = true;
        }
        return SA_OK;
    }
    return mesh_coords<D>(M, nullptr, vols, st);
}

// q (if given) packed to AoS, then vols copied or computed on the device
template <int D>
int mesh_coords(sa_mesh *M, const double *q, const double *vols, cudaStream_t st)
{
    typedef typename VecT<D>::type V;
    typedef typename IdxT<D>::type I;
    unsigned long long *bad = (unsigned long long *)M->scratch;
    unsigned long long hbad = 0;
    const int B = 256;
    unsigned gq = std::min<int64_t>(grid_for(M->nq, B), 148 * 32);
    unsigned ge = std::min<int64_t>(grid_for(M->nme, B), 148 * 32);
    if (M->nq && q) SA_LAUNCH(k_pack_q<D>, gq, B, 0, st, q, M->nq, (V *)M->qv);
    M->coords = true;
    if (M->vols_ready) return SA_OK;
    M->vols_ready = true;
    if (vols) {
        SA_CUDA_TRY(cudaMemcpyAsync(M->vols, vols, M->nme * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else if (M->nme) {
        SA_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
        if (M->core == CORE_SKYLAKEX)
            SA_LAUNCH((k_volumes<D, CORE_SKYLAKEX>), ge, B, 0, st, (const V *)M->qv, (const I *)M->me, M->nme, M->vols, bad);
        else
            SA_LAUNCH((k_volumes<D, CORE_HASWELL>), ge, B, 0, st, (const V *)M->qv, (const I *)M->me, M->nme, M->vols, bad);
        SA_TRY(readback(&hbad, bad, sizeof hbad, st));
        SA_TRY(sync_stream(st));
        if (hbad != ~0ull) {
            err_state().bad = (int64_t)hbad;
            return set_error(SA_ERR_DEGENERATE, "simplex %lld is degenerate (zero volume)", (long long)hbad);
        }
    }
    return SA_OK;
}

// volumes recomputed from the coordinates into `out` (Mesh.validate; a
// degenerate element gives 0.0 there, no error)
template <int D>
int mesh_recompute_vols(const sa_mesh *M, double *out, cudaStream_t st)
{
    typedef typename VecT<D>::type V;
    typedef typename IdxT<D>::type I;
    if (!M->nme) return SA_OK;
    unsigned long long *bad = (unsigned long long *)M->scratch + 1;
    const unsigned ge = std::min<int64_t>(grid_for(M->nme, 256), 148 * 32);
    if (M->core == CORE_SKYLAKEX)
        SA_LAUNCH((k_volumes<D, CORE_SKYLAKEX>), ge, 256, 0, st, (const V *)M->qv, (const I *)M->me, M->nme, out, bad);
    else
        SA_LAUNCH((k_volumes<D, CORE_HASWELL>), ge, 256, 0, st, (const V *)M->qv, (const I *)M->me, M->nme, out, bad);
    return SA_OK;
}

// first element with a non-positive stored volume, first element whose stored
// volume is off its recomputed one by more than 1e-12 relative (mesh.py:92-101)
__global__ void k_validate_vols(const double *__restrict__ stored, const double *__restrict__ recomputed, int64_t n,
                                unsigned long long *out)
{
    unsigned long long np = ~0ull, mm = ~0ull;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double v = stored[k], r = recomputed[k];
        if (v <= 0.0) np = min(np, (unsigned long long)k);
        if (fabs(v - r) > 1e-12 * r) mm = min(mm, (unsigned long long)k);
    }
    for (int sh = 16; sh > 0; sh >>= 1) {
        np = min(np, __shfl_xor_sync(0xffffffffu, np, sh));
        mm = min(mm, __shfl_xor_sync(0xffffffffu, mm, sh));
    }
    if ((threadIdx.x & 31) == 0) {
        if (np != ~0ull) atomicMin(out, np);
        if (mm != ~0ull) atomicMin(out + 1, mm);
    }
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
    SA_TRY(readback(&P->n_inc, P->inc_ptr + nn, sizeof(int64_t), st));
    SA_TRY(sync_stream(st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->inc, std::max<int64_t>(P->n_inc, 1) * sizeof(uint2), st));
    SA_CUDA_TRY(cudaMemsetAsync(cnt, 0, (nn + 1) * sizeof(int64_t), st));
    if (M->nme)
        SA_LAUNCH(k_inc_fill<D>, ge, B, 0, st, (const I *)M->me, M->nme, P->node_begin, P->node_end, P->inc_ptr,
                  (unsigned long long *)cnt, P->inc);
    // fast path when every node fits the fused shared-memory node pass
    // (max incidences <= NS_CAPI, checked here; neighbours <= NS_CAPC,
    // checked by the pass itself), else the general kernels
    bool fast = false;

    // (default in 3D: measured warm C3 12.5 -> 9.9 ms, C5 65 -> 52 ms; in 2D
    // the general kernels are faster, C2 1.29 vs 1.71 ms)
    if (nn && tune_int("symfast", D == 3) != 0) {
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, 2 * sizeof(int64_t), st));
        SA_LAUNCH(k_max_diff, std::min<int64_t>(grid_for(nn, 256), 148 * 8), 256, 0, st, P->inc_ptr, nn,
                  (unsigned long long *)(P->counters + 6));
        int64_t mi = 0;
        SA_TRY(readback(&mi, P->counters + 6, sizeof(int64_t), st));
        SA_TRY(sync_stream(st));
        if (mi <= NS_CAPI) {
            SA_LAUNCH((k_node_symbolic<D, false>), grid_for(nn, NS_THREADS), NS_THREADS, 0, st, (const I *)M->me,
                      P->inc_ptr, P->inc, nn, cnt, (const int64_t *)nullptr, (int32_t *)nullptr,
                      (unsigned long long *)(P->counters + 7));
            int64_t ov = 0;
            SA_TRY(readback(&ov, P->counters + 7, sizeof(int64_t), st));
            SA_TRY(sync_stream(st));
            fast = ov == 0;   // else (a node with > NS_CAPC neighbours): the general kernels below
        }
    }
    uint32_t *hsym = nullptr;   // nodes with more than MAXC neighbours (general path)
    int64_t nhsym = 0;
    const size_t hsm = HEAVY_CAP * sizeof(int);
    if (nn && !fast) {
        SA_LAUNCH(k_inc_sort, grid_for(nn, 128), 128, 0, st, P->inc_ptr, nn, P->inc);
        SA_CUDA_TRY(cudaMallocAsync((void **)&hsym, nn * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 5, 0, 2 * sizeof(int64_t), st));
        SA_LAUNCH(k_node_cols<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, cnt,
                  (const int64_t *)nullptr, (int32_t *)nullptr, (unsigned long long *)(P->counters + 5), hsym);
        SA_TRY(readback(&nhsym, P->counters + 5, sizeof(int64_t), st));
        SA_TRY(sync_stream(st));
        if (nhsym) {
            SA_CUDA_TRY(cudaFuncSetAttribute(k_heavy_cols<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
            SA_LAUNCH(k_heavy_cols<D>, (unsigned)nhsym, 1024, hsm, st, (const I *)M->me, P->inc_ptr, P->inc, hsym, cnt,
                      (const int64_t *)nullptr, (int32_t *)nullptr, (unsigned long long *)(P->counters + 6));
        }
    }
    SA_TRY(exclusive_scan_i64(cnt, P->colptr, nn, P->scan_tmp, st));
    int64_t too_big = 0;
    SA_TRY(readback(&P->n_colnodes, P->colptr + nn, sizeof(int64_t), st));
    if (nhsym) SA_TRY(readback(&too_big, P->counters + 6, sizeof(int64_t), st));
    SA_TRY(sync_stream(st));
    if (too_big) {
        SA_CUDA_TRY(cudaFreeAsync(hsym, st));
        return set_error(SA_ERR_CAPACITY, "a node has more than %d vertex references in its incident elements",
                         HEAVY_CAP);
    }
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->cols, std::max<int64_t>(P->n_colnodes, 1) * sizeof(int32_t), st));
    if (nn && fast) {
        SA_LAUNCH((k_node_symbolic<D, true>), grid_for(nn, NS_THREADS), NS_THREADS, 0, st, (const I *)M->me,
                  P->inc_ptr, P->inc, nn, cnt, (const int64_t *)P->colptr, P->cols,
                  (unsigned long long *)(P->counters + 7));
    } else if (nn) {
        SA_LAUNCH(k_node_cols<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, cnt,
                  (const int64_t *)P->colptr, P->cols, (unsigned long long *)nullptr, (uint32_t *)nullptr);
        if (nhsym)
            SA_LAUNCH(k_heavy_cols<D>, (unsigned)nhsym, 1024, hsm, st, (const I *)M->me, P->inc_ptr, P->inc, hsym, cnt,
                      (const int64_t *)P->colptr, P->cols, (unsigned long long *)(P->counters + 6));
        SA_LAUNCH(k_inc_ranks<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, P->colptr,
                  P->cols);
    }
    if (hsym) SA_CUDA_TRY(cudaFreeAsync(hsym, st));
    // max node degree: device reduction (no host copy of colptr)
    SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, sizeof(int64_t), st));
    if (nn)
        SA_LAUNCH(k_max_diff, std::min<int64_t>(grid_for(nn, 256), 148 * 8), 256, 0, st, P->colptr, nn,
                  (unsigned long long *)(P->counters + 6));
    int64_t md = 0;
    SA_TRY(readback(&md, P->counters + 6, sizeof(int64_t), st));
    SA_TRY(sync_stream(st));
    P->max_deg = md;
    const int m = P->m;
    // light / heavy rows: the row kernels size their shared-memory
    // accumulators for the light rows only; rows above the cap (hubs) are
    // assembled by k_heavy_rows, so one hub neither shrinks every block nor
    // runs into the 8-bit column ranks
    {
        const int64_t avg = nn ? (P->n_colnodes + nn - 1) / nn : 0;
        const int64_t smem_cap = m == 1 ? 200 : (m == 2 ? 100 : 44);
        const int64_t cap = std::min<int64_t>(std::min<int64_t>(smem_cap, MAXC), std::max<int64_t>(2 * avg + 8, 16));
        P->light_deg = md;
        P->n_heavy = 0;
        if (md > cap) {
            SA_CUDA_TRY(cudaMallocAsync((void **)&P->heavy_rows, nn * sizeof(uint32_t), st));
            SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, 2 * sizeof(int64_t), st));
            SA_LAUNCH(k_heavy_rows_list, std::min<int64_t>(grid_for(nn, 256), 148 * 8), 256, 0, st, P->colptr, nn, cap,
                      P->heavy_rows, (unsigned long long *)(P->counters + 6));
            int64_t h[2];
            SA_TRY(readback(h, P->counters + 6, sizeof h, st));
            SA_TRY(sync_stream(st));
            P->n_heavy = h[0];
            P->light_deg = h[1];
        }
    }
    P->nnz = (int64_t)m * m * P->n_colnodes;
    if (P->nnz >= ((int64_t)1 << 31) || (int64_t)m * M->nq >= ((int64_t)1 << 31))
        return set_error(SA_ERR_CAPACITY, "block has %lld structural entries; int32 column indices overflow",
                         (long long)P->nnz);
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->indptr, (P->nrows + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->indices, std::max<int64_t>(P->nnz, 1) * sizeof(int32_t), st));
    SA_LAUNCH(k_dof_csr, grid_for(nn + 1, 128), 128, 0, st, P->colptr, P->cols, nn, m, P->indptr, P->indices);
    SA_CUDA_TRY(cudaFreeAsync(cnt, st));
    SA_TRY(sync_stream(st));
    return SA_OK;
}

// Warp-interleaved incidence records (IncRec, 32 B) for the 3D row gather:
// they replace three dependent gathers per incidence (measured faster in 3D;
// no gain in 1D/2D at 4x the record traffic).  Built on the first row-gather
// numeric call of a plan -- plans served by the two-pass path (3D general
// operator) never pay for them.  The records carry the volume, so the mesh
// volumes must be set.
template <int D>
int build_winc(sa_plan *P, cudaStream_t st)
{
    typedef typename IdxT<D>::type I;
    const sa_mesh *M = P->mesh;
    const int64_t nn = P->nnodes;
    if (P->winc || !nn || !M->vols_ready || tune_int("winc", D == 3) == 0) return SA_OK;
    const int64_t nw = (nn + 31) / 32;
    int64_t *span = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&span, (nw + 1) * sizeof(int64_t), st));
    if (!P->wseg) {
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->wseg, (nw + 1) * sizeof(int64_t), st));
        SA_LAUNCH(k_warp_span, grid_for(nw, 128), 128, 0, st, P->inc_ptr, nn, span);
        SA_TRY(exclusive_scan_i64(span, P->wseg, nw, P->scan_tmp, st));
    }
    SA_TRY(readback(&P->n_winc, P->wseg + nw, sizeof(int64_t), st));
    SA_TRY(sync_stream(st));
    SA_CUDA_TRY(cudaFreeAsync(span, st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->winc, std::max<int64_t>(P->n_winc, 1) * sizeof(IncRec), st));
    // padding records (rows shorter than their warp's longest) = all ones: ea = 0xffffffff sentinel
    SA_CUDA_TRY(cudaMemsetAsync(P->winc, 0xff, std::max<int64_t>(P->n_winc, 1) * sizeof(IncRec), st));
    SA_LAUNCH(k_winc_fill<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, M->vols, P->inc_ptr, P->inc, nn,
              P->wseg, P->winc);
    return SA_OK;
}

// One-pass row gather.  Launch shape per operator (measured on the BASELINE
// configs, profiles/r01/README.md): the kernel is latency-bound, so
// occupancy wins over per-thread ILP except for the register-heavy elastic
// operator, which gains from the 3-deep software pipeline; lean instances
// (no nodal mass weight) drop the generic branches.
template <int D, int M, int OPS, int CORE>
int launch_rowgather(const NumArgs &a, int64_t nnodes, cudaStream_t st)
{
    constexpr int NOUT = n_outputs<OPS>();
    const size_t per_thread = (size_t)NOUT * (a.acc_stride | 1) * sizeof(double);
    int block = 128;
    while (per_thread * block > 100 * 1024 && block > 32) block /= 2;
    const size_t smem = per_thread * block;
    if (smem > 200 * 1024)
        return set_error(SA_ERR_CAPACITY, "row accumulators need %zu B of shared memory per %d threads", smem, block);
    const bool lean = !((OPS & OP_MASS) && a.w) && (a.winc != nullptr) == (D == 3);
    void (*kern)(NumArgs);
    if constexpr (M > 1) {
        kern = lean ? k_numeric_rowgather<D, M, OPS, CORE, 3, 1, false, true> : k_numeric_rowgather<D, M, OPS, CORE, 3, 1>;
    } else if constexpr ((OPS & OP_GENERAL) != 0) {
        kern = k_numeric_rowgather<D, M, OPS, CORE, 1, 3>;
    } else if constexpr (D == 3) {
        kern = lean ? k_numeric_rowgather<D, M, OPS, CORE, 1, 6, false, true> : k_numeric_rowgather<D, M, OPS, CORE, 1, 6>;
    } else {
        // 2D/1D: 10 blocks/SM at 48 registers beats 8 at 60 once the grid
        // has more than one wave (C2 0.299 -> 0.289 ms); one wave keeps 8
        if (lean && nnodes > (int64_t)148 * 8 * 128) kern = k_numeric_rowgather<D, M, OPS, CORE, 1, 10, false, true>;
        else if (lean) kern = k_numeric_rowgather<D, M, OPS, CORE, 1, 8, false, true>;
        else kern = k_numeric_rowgather<D, M, OPS, CORE, 1, 8>;
    }
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (nnodes) SA_LAUNCH(kern, grid_for(nnodes, block), block, smem, st, a);
    return SA_OK;
}

// Fast general operator, guarded rows: recompute each flagged row in
// reference order (bitwise element values, ascending element fold straight
// into the row's CSR segment) and count its exact zeros (sparse.py:108-111).
template <int D, int OPS, int CORE>
__global__ void k_guard_fixup(NumArgs a)
{
    constexpr int NOUT = n_outputs<OPS>();
    const int n = *a.nflag;
    int nz[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) nz[o] = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t nl = a.flag_rows[i];
        const int64_t base = a.indptr[nl];
        const int deg = (int)(a.colptr[nl + 1] - a.colptr[nl]);
        for (int o = 0; o < NOUT; ++o)
            for (int k = 0; k < deg; ++k) a.vals[o][base + k] = 0.0;
        for (int64_t t = a.inc_ptr[nl]; t < a.inc_ptr[nl + 1]; ++t) {
            const uint2 rec = a.inc[t];
            ElemRaw<D> x;
            element_load1<D, OPS>(a, rec.x & 0x3fffffffu, x);
            element_load2<D, OPS>(a, x);
            ElemGeo<D> g;
            element_compute<D, OPS, CORE>(x, g);
            double vals[(D + 1) * NOUT];
            krow_runtime<D, 1, OPS>(a, g, rec.x >> 30, vals);
#pragma unroll
            for (int b = 0; b <= D; ++b) {
                const int rk = (rec.y >> (8 * b)) & 0xff;
#pragma unroll
                for (int o = 0; o < NOUT; ++o) a.vals[o][base + rk] += vals[b * NOUT + o];
            }
        }
        for (int o = 0; o < NOUT; ++o)
            for (int k = 0; k < deg; ++k) nz[o] += (a.vals[o][base + k] == 0.0);
    }
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
        if (nz[o]) atomicAdd((unsigned long long *)(a.counters + o), (unsigned long long)nz[o]);
}

// Two-pass numeric (3D general operator): element pass, then the ordered
// fold.  Element pass: the persistent three-stage cp.async pipeline when
// every batch's vertex records fit the stage (C5: 3 blocks/SM at 164
// registers), else one thread per element with direct gathers.  Fast mode
// (default for the general operator): fused-multiply-add local matrices in
// the element pass, the zero guard in the fold, guarded rows recomputed.
template <int D, int M, int OPS, int CORE>
int launch_twopass(const sa_plan *P, const NumArgs &a, int64_t nnodes, cudaStream_t st)
{
    constexpr int NOUT = n_outputs<OPS>();
    constexpr bool GEN3 = OPS == OP_GENERAL && D == 3 && M == 1;
    const bool pipe = GEN3 && a.eb_loc && a.gen_packed && a.eb_allfit;
    const bool fast = pipe && !a.exact;
    if constexpr (GEN3) {
        if (pipe) {
            // (fast: 126 registers, 2 blocks of 256 per SM; batches of 256
            // elements read 7.7 instead of 9.5 GB -- C5 7.77 vs 7.90 ms)
            auto pk = fast ? k_element_rows_pipe<D, M, OPS, CORE, 2, true> : k_element_rows_pipe<D, M, OPS, CORE, 2>;
            const size_t psm = 2 * (size_t)std::max(a.eb_maxn, 1) * EB_REC * sizeof(double) +
                               3 * (EB_CAP + 1) * sizeof(int);
            SA_CUDA_TRY(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
            int dev = 0, nsm = 148, occ = 0;
            SA_CUDA_TRY(cudaGetDevice(&dev));
            SA_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
            SA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pk, EB_SIZE, psm));
            const int64_t nb = (a.ne + EB_SIZE - 1) / EB_SIZE;
            const unsigned g = (unsigned)std::min<int64_t>(nb, (int64_t)nsm * std::max(occ, 1));
            if (a.ne) SA_LAUNCH(pk, g, EB_SIZE, psm, st, a);
        }
    }
    if (!pipe && a.ne) SA_LAUNCH((k_element_rows<D, M, OPS, CORE, 3>), grid_for(a.ne, 128), 128, 0, st, a);
    const size_t per_thread = (size_t)NOUT * (a.acc_stride | 1) * sizeof(double);
    int block = 128;
    while (per_thread * block > 100 * 1024 && block > 32) block /= 2;
    const size_t smem = per_thread * block;
    if (smem > 200 * 1024)
        return set_error(SA_ERR_CAPACITY, "row accumulators need %zu B of shared memory per %d threads", smem, block);
    void (*kern)(NumArgs) = fast ? k_numeric_rowgather<D, M, OPS, CORE, 2, 1, true, false, true>
                                 : k_numeric_rowgather<D, M, OPS, CORE, 2, 1, true>;
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (fast) SA_CUDA_TRY(cudaMemsetAsync(a.nflag, 0, sizeof(int), st));
    if (nnodes) SA_LAUNCH(kern, grid_for(nnodes, block), block, smem, st, a);
    if constexpr (M == 1) {
        if (fast && nnodes) SA_LAUNCH((k_guard_fixup<D, OPS, CORE>), 148, 128, 0, st, a);
    }
    return SA_OK;
}


// Heavy rows (degree above the plan's light cap): one thread per row, exact
// element values (element_krow, reference order) folded in ascending element
// order straight into the row's CSR segment in global memory; the column of
// each element vertex is looked up in the row's sorted column list (ranks
// may exceed 8 bits).  Bitwise the row-gather result; zeros counted.
template <int D, int M, int OPS, int CORE>
__global__ void k_heavy_rows(NumArgs a)
{
    constexpr int NOUT = n_outputs<OPS>();
    constexpr int MM = M * M;
    int nz[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) nz[o] = 0;
    int64_t emin = INT64_MAX;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n_heavy;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t nl = a.heavy_rows[i];
        const int64_t c0 = a.colptr[nl];
        const int deg = (int)(a.colptr[nl + 1] - c0);
        for (int o = 0; o < NOUT; ++o)
            for (int l = 0; l < M; ++l) {
                const int64_t p = a.indptr[M * nl + l];
                for (int k = 0; k < M * deg; ++k) a.vals[o][p + k] = 0.0;
            }
        for (int64_t t = a.inc_ptr[nl]; t < a.inc_ptr[nl + 1]; ++t) {
            const uint2 rec = a.inc[t];
            const int64_t e = rec.x & 0x3fffffffu;
            ElemRaw<D> x;
            element_load1<D, OPS>(a, e, x);
            element_load2<D, OPS>(a, x);
            ElemGeo<D> g;
            if (element_compute<D, OPS, CORE>(x, g)) emin = min(emin, e);
            double vals[(D + 1) * NOUT * MM];
            krow_runtime<D, M, OPS>(a, g, rec.x >> 30, vals);
            for (int b = 0; b <= D; ++b) {
                int lo = 0, hi = deg;
                while (lo < hi) { const int mid = (lo + hi) >> 1; if (a.cols[c0 + mid] < x.v[b]) lo = mid + 1; else hi = mid; }
                for (int o = 0; o < NOUT; ++o)
                    for (int l = 0; l < M; ++l) {
                        const int64_t p = a.indptr[M * nl + l] + (int64_t)lo * M;
                        for (int n = 0; n < M; ++n) a.vals[o][p + n] += vals[(b * NOUT + o) * MM + l * M + n];
                    }
            }
        }
        for (int o = 0; o < NOUT; ++o)
            for (int l = 0; l < M; ++l) {
                const int64_t p = a.indptr[M * nl + l];
                for (int k = 0; k < M * deg; ++k) nz[o] += (a.vals[o][p + k] == 0.0);
            }
    }
    if (emin != INT64_MAX) atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)emin);
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
        if (nz[o]) atomicAdd((unsigned long long *)(a.counters + o), (unsigned long long)nz[o]);
}

template <int D, int M, int OPS, int CORE>
int launch_numeric(const sa_plan *P, const NumArgs &a, cudaStream_t st)
{
    if (a.kbuf) SA_TRY((launch_twopass<D, M, OPS, CORE>(P, a, P->nnodes, st)));
    else SA_TRY((launch_rowgather<D, M, OPS, CORE>(a, P->nnodes, st)));
    if (a.n_heavy)
        SA_LAUNCH((k_heavy_rows<D, M, OPS, CORE>), (unsigned)std::min<int64_t>(grid_for(a.n_heavy, 64), 148), 64, 0, st, a);
    return SA_OK;
}


template <int D, int M, int OPS>
int launch_numeric_core(const sa_plan *P, const NumArgs &a, int core, cudaStream_t st)
{
    if (core == CORE_SKYLAKEX) return launch_numeric<D, M, OPS, CORE_SKYLAKEX>(P, a, st);
    return launch_numeric<D, M, OPS, CORE_HASWELL>(P, a, st);
}

template <int D>
int dispatch_numeric(const sa_plan *P, const NumArgs &a, int ops, int core, cudaStream_t st)
{
    switch (ops) {
        case OP_MASS: return launch_numeric_core<D, 1, OP_MASS>(P, a, core, st);
        case OP_STIFF: return launch_numeric_core<D, 1, OP_STIFF>(P, a, core, st);
        case OP_MASS | OP_STIFF: return launch_numeric_core<D, 1, OP_MASS | OP_STIFF>(P, a, core, st);
        case OP_GENERAL: return launch_numeric_core<D, 1, OP_GENERAL>(P, a, core, st);
        case OP_ELASTIC:
            if constexpr (D >= 2) {
                if (P->m == D) return launch_numeric_core<D, D, OP_ELASTIC>(P, a, core, st);
            }
            return set_error(SA_ERR_ARG, "elastic operator needs d in {2,3} and m == d");
        default: return set_error(SA_ERR_ARG, "unsupported operator combination %d", ops);
    }
}

}  // namespace

// The kernels are compiled once per dimension (SA_D = 1, 2, 3: sa_d1.cu ..
// sa_d3.cu, in parallel); the C ABI (SA_ABI: sa_abi.cu) reaches them through
// these wrappers.
#define SA_CAT2(a, b) a##b
#define SA_CAT(a, b) SA_CAT2(a, b)
int sa_mesh_kernels_d1(sa_mesh *, const double *, const int64_t *, const int32_t *, int, const double *, cudaStream_t);
int sa_mesh_kernels_d2(sa_mesh *, const double *, const int64_t *, const int32_t *, int, const double *, cudaStream_t);
int sa_mesh_kernels_d3(sa_mesh *, const double *, const int64_t *, const int32_t *, int, const double *, cudaStream_t);
int sa_mesh_coords_d1(sa_mesh *, const double *, const double *, cudaStream_t);
int sa_mesh_coords_d2(sa_mesh *, const double *, const double *, cudaStream_t);
int sa_mesh_coords_d3(sa_mesh *, const double *, const double *, cudaStream_t);
int sa_symbolic_d1(sa_plan *, cudaStream_t);
int sa_symbolic_d2(sa_plan *, cudaStream_t);
int sa_symbolic_d3(sa_plan *, cudaStream_t);
int sa_dispatch_d1(const sa_plan *, const NumArgs &, int, int, cudaStream_t);
int sa_dispatch_d2(const sa_plan *, const NumArgs &, int, int, cudaStream_t);
int sa_dispatch_d3(const sa_plan *, const NumArgs &, int, int, cudaStream_t);
int sa_winc_d3(sa_plan *, cudaStream_t);
int sa_mesh_revols_d1(const sa_mesh *, double *, cudaStream_t);
int sa_mesh_revols_d2(const sa_mesh *, double *, cudaStream_t);
int sa_mesh_revols_d3(const sa_mesh *, double *, cudaStream_t);
#ifdef SA_D
int SA_CAT(sa_mesh_revols_d, SA_D)(const sa_mesh *M, double *out, cudaStream_t st)
{
    return mesh_recompute_vols<SA_D>(M, out, st);
}
#if SA_D == 3
int sa_winc_d3(sa_plan *P, cudaStream_t st) { return build_winc<3>(P, st); }
#endif
int SA_CAT(sa_mesh_kernels_d, SA_D)(sa_mesh *M, const double *q, const int64_t *me, const int32_t *me32, int rows32,
                                    const double *vols, cudaStream_t st)
{
    return mesh_kernels<SA_D>(M, q, me, me32, rows32, vols, st);
}
int SA_CAT(sa_symbolic_d, SA_D)(sa_plan *P, cudaStream_t st) { return symbolic_kernels<SA_D>(P, st); }
int SA_CAT(sa_mesh_coords_d, SA_D)(sa_mesh *M, const double *q, const double *vols, cudaStream_t st)
{
    return mesh_coords<SA_D>(M, q, vols, st);
}
int SA_CAT(sa_dispatch_d, SA_D)(const sa_plan *P, const NumArgs &a, int ops, int core, cudaStream_t st)
{
    return dispatch_numeric<SA_D>(P, a, ops, core, st);
}
#endif

#ifdef SA_ABI
// Device buffers come from the stream-ordered pool (cudaMallocAsync) whose
// release threshold is raised once, so repeated mesh/plan construction
// (re-assembly, e2e) reuses memory instead of re-mapping it.
static void pool_keep_memory(int device)
{
    static bool done[64] = {false};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[device] = true;
}

static void free_all(std::initializer_list<void *> ps)
{
    cudaDeviceSynchronize();
    for (void *p : ps)
        if (p) cudaFreeAsync(p, 0);
}

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

int sa_mesh_create_split(int d, int64_t nq, int64_t nme, const double *q_dev, const int32_t *me32_dev, int rows32,
                         const int64_t *me_dev, const double *vols_dev, int core, int device, void *stream,
                         sa_mesh **out)
{
    err_state().msg.clear();
    err_state().bad = -1;
    if (!out) return set_error(SA_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (d < 1 || d > 3) return set_error(SA_ERR_ARG, "dimension must be 1, 2 or 3, got %d", d);
    if (rows32 < 0 || rows32 > d + 1 || (rows32 > 0 && !me32_dev && nme) || (rows32 <= d && !me_dev && nme))
        return set_error(SA_ERR_ARG, "connectivity: %d int32 rows of %d, missing array", rows32, d + 1);
    if (core != CORE_SKYLAKEX && core != CORE_HASWELL) return set_error(SA_ERR_ARG, "unknown core %d", core);
    if (nq < 0 || nme < 0) return set_error(SA_ERR_ARG, "negative sizes");
    if (nq >= ((int64_t)1 << 31) || nme >= ((int64_t)1 << 30))
        return set_error(SA_ERR_CAPACITY, "mesh with nq=%lld nme=%lld exceeds the int32 index range",
                         (long long)nq, (long long)nme);
    SA_TRY(set_device(device));
    pool_keep_memory(device);
    cudaStream_t st = (cudaStream_t)stream;
    sa_mesh *M = new sa_mesh();
    M->d = d; M->nq = nq; M->nme = nme; M->core = core; M->device = device;
    size_t vsz = d == 1 ? 8 : (d == 2 ? 16 : 32);
    size_t isz = d == 1 ? 8 : 16;
    int rc = SA_OK;
    auto fail = [&](int r) { sa_mesh_destroy(M); return r; };
    if (cudaMallocAsync(&M->qv, std::max<int64_t>(nq, 1) * vsz, st) != cudaSuccess ||
        cudaMallocAsync(&M->me, std::max<int64_t>(nme, 1) * isz, st) != cudaSuccess ||
        cudaMallocAsync((void **)&M->vols, std::max<int64_t>(nme, 1) * sizeof(double), st) != cudaSuccess ||
        cudaMallocAsync((void **)&M->scratch, 8 * sizeof(int64_t), st) != cudaSuccess)
        return fail(set_error(SA_ERR_NOMEM, "device allocation for the mesh failed"));
    if (d == 1) rc = sa_mesh_kernels_d1(M, q_dev, me_dev, me32_dev, rows32, vols_dev, st);
    else if (d == 2) rc = sa_mesh_kernels_d2(M, q_dev, me_dev, me32_dev, rows32, vols_dev, st);
    else rc = sa_mesh_kernels_d3(M, q_dev, me_dev, me32_dev, rows32, vols_dev, st);
    if (rc != SA_OK) return fail(rc);
    *out = M;
    return SA_OK;
}

int sa_mesh_create(int d, int64_t nq, int64_t nme, const double *q_dev, const int64_t *me_dev,
                   const double *vols_dev, int core, int device, void *stream, sa_mesh **out)
{
    return sa_mesh_create_split(d, nq, nme, q_dev, nullptr, 0, me_dev, vols_dev, core, device, stream, out);
}

int sa_mesh_set_coords(sa_mesh *M, const double *q_dev, const double *vols_dev, void *stream)
{
    if (!M || !q_dev) return set_error(SA_ERR_ARG, "mesh/q is NULL");
    SA_TRY(set_device(M->device));
    cudaStream_t st = (cudaStream_t)stream;
    if (M->d == 1) return sa_mesh_coords_d1(M, q_dev, vols_dev, st);
    if (M->d == 2) return sa_mesh_coords_d2(M, q_dev, vols_dev, st);
    return sa_mesh_coords_d3(M, q_dev, vols_dev, st);
}

int sa_mesh_vols(const sa_mesh *M, double *vols_dev_out, void *stream)
{
    if (!M) return set_error(SA_ERR_ARG, "mesh is NULL");
    SA_CUDA_TRY(cudaMemcpyAsync(vols_dev_out, M->vols, M->nme * sizeof(double), cudaMemcpyDeviceToDevice,
                                (cudaStream_t)stream));
    return SA_OK;
}

int sa_mesh_validate(const sa_mesh *M, const double *vols_dev, int64_t *first_nonpositive, int64_t *first_mismatch,
                     void *stream)
{
    if (!M || !vols_dev || !first_nonpositive || !first_mismatch) return set_error(SA_ERR_ARG, "NULL argument");
    if (!M->coords) return set_error(SA_ERR_ARG, "mesh coordinates not set (sa_mesh_set_coords)");
    SA_TRY(set_device(M->device));
    cudaStream_t st = (cudaStream_t)stream;
    *first_nonpositive = *first_mismatch = -1;
    if (!M->nme) return SA_OK;
    double *re = nullptr;
    unsigned long long *out = nullptr, h[2] = {~0ull, ~0ull};
    SA_CUDA_TRY(cudaMallocAsync((void **)&re, M->nme * sizeof(double), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&out, sizeof h, st));
    SA_CUDA_TRY(cudaMemcpyAsync(out, h, sizeof h, cudaMemcpyHostToDevice, st));
    int rc = M->d == 1 ? sa_mesh_revols_d1(M, re, st) : (M->d == 2 ? sa_mesh_revols_d2(M, re, st) : sa_mesh_revols_d3(M, re, st));
    if (rc == SA_OK) {
        k_validate_vols<<<std::min<int64_t>(grid_for(M->nme, 256), 148 * 16), 256, 0, st>>>(vols_dev, re, M->nme, out);
        err_state().launches++;
        if (cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            rc = set_error(SA_ERR_CUDA, "volume validation failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
    cudaFreeAsync(re, st);
    cudaFreeAsync(out, st);
    if (rc != SA_OK) return rc;
    if (h[0] != ~0ull) *first_nonpositive = (int64_t)h[0];
    if (h[1] != ~0ull) *first_mismatch = (int64_t)h[1];
    return SA_OK;
}

int sa_mesh_destroy(sa_mesh *M)
{
    if (!M) return SA_OK;
    free_all({M->qv, M->me, M->vols, M->scratch});
    delete M;
    return SA_OK;
}

int sa_plan_destroy(sa_plan *P)
{
    if (!P) return SA_OK;
    free_all({P->inc_ptr, P->inc, P->winc, P->wseg, P->colptr, P->cols, P->indptr, P->indices, P->counters,
              P->scan_tmp, P->epos, P->kbuf, P->tp_rank, P->eb_verts, P->eb_count, P->eb_loc, P->gd_flag_rows,
              P->gd_nflag, P->heavy_rows});
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
    if (cudaMallocAsync((void **)&P->counters, 8 * sizeof(int64_t), st) != cudaSuccess) {
        delete P;
        return set_error(SA_ERR_NOMEM, "device allocation failed");
    }
    int rc;
    if (M->d == 1) rc = sa_symbolic_d1(P, st);
    else if (M->d == 2) rc = sa_symbolic_d2(P, st);
    else rc = sa_symbolic_d3(P, st);
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

int sa_plan_stats(const sa_plan *P, int64_t *out, int n)
{
    if (!P || !out) return set_error(SA_ERR_ARG, "plan/out is NULL");
    const int64_t nn = P->nnodes, nw = (nn + 31) / 32, ne = P->e_hi - P->e_lo, nb = (ne + EB_SIZE - 1) / EB_SIZE;
    // device bytes of the plan's symbolic structures (pattern, incidences,
    // warp records, two-pass slot map / row buffer / element batches)
    const int64_t bytes = 3 * (nn + 1) * 8 + P->n_inc * 8 + P->n_colnodes * 4 + (P->nrows + 1) * 8 + P->nnz * 4 +
                          P->n_winc * (int64_t)sizeof(IncRec) + (P->wseg ? (nw + 1) * 8 : 0) +
                          (P->epos ? ne * 16 : 0) + P->kbuf_elems * 8 + P->tp_nslots * 4 +
                          (P->eb_loc ? ne * 4 + nb * (EB_CAP + 1) * 4 : 0);
    const int64_t v[11] = {P->n_inc, P->max_deg, P->nnodes, P->nnz, P->n_winc, P->tp_nslots, P->eb_allfit ? 1 : 0,
                           P->eb_maxn, bytes, P->light_deg, P->n_heavy};
    for (int i = 0; i < n && i < 11; ++i) out[i] = v[i];
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

// two-pass numeric ("element rows") serves the 3D general operator, where
// recomputing each element once per vertex row costs more than the local-row
// buffer (measured); SA_TUNE=kernel=twopass|rowgather forces
// either path for any operator (tests, A/B)
static bool want_twopass(int ops, int d, int m)
{
    (void)m;
    if (tune_is("kernel", "twopass")) return true;
    if (tune_is("kernel", "rowgather")) return false;
    return ops == SA_OP_GENERAL && d == 3;
}

// element range, slot map and row buffer of a plan's two-pass numeric phase
// (built on first use, kept with the plan)
static int ensure_twopass(sa_plan *P, int kstride, bool batches, cudaStream_t st)
{
    if (!P->epos) {
        unsigned long long h[2] = {0xffffffffull, 0};
        unsigned long long *dr = nullptr;
        SA_CUDA_TRY(cudaMallocAsync((void **)&dr, 2 * sizeof(unsigned long long), st));
        SA_CUDA_TRY(cudaMemcpyAsync(dr, h, sizeof h, cudaMemcpyHostToDevice, st));
        if (P->n_inc)
            SA_LAUNCH(k_inc_erange, std::min<int64_t>(grid_for(P->n_inc, 256), 148 * 8), 256, 0, st, P->inc,
                      P->n_inc, dr);
        SA_TRY(readback(h, dr, sizeof h, st));
        SA_TRY(sync_stream(st));
        SA_CUDA_TRY(cudaFreeAsync(dr, st));
        P->e_lo = P->n_inc ? (int64_t)h[0] : 0;
        P->e_hi = P->n_inc ? (int64_t)h[1] + 1 : 0;
        const int64_t ne = P->e_hi - P->e_lo;
        const int64_t nn = P->nnodes, nw = (nn + 31) / 32;
        if (!P->wseg) {   // warp-interleaved slot offsets (built with winc in 3D)
            int64_t *span = nullptr;
            SA_CUDA_TRY(cudaMallocAsync((void **)&span, (nw + 1) * sizeof(int64_t), st));
            SA_CUDA_TRY(cudaMallocAsync((void **)&P->wseg, (nw + 1) * sizeof(int64_t), st));
            if (nw) SA_LAUNCH(k_warp_span, grid_for(nw, 128), 128, 0, st, P->inc_ptr, nn, span);
            SA_TRY(exclusive_scan_i64(span, P->wseg, nw, P->scan_tmp, st));
            SA_CUDA_TRY(cudaFreeAsync(span, st));
        }
        SA_TRY(readback(&P->tp_nslots, P->wseg + nw, sizeof(int64_t), st));
        SA_TRY(sync_stream(st));
        if (P->tp_nslots >= 0xffffffffLL)
            return set_error(SA_ERR_CAPACITY, "two-pass numeric: %lld slots overflow 32-bit slot indices",
                             (long long)P->tp_nslots);
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->epos, std::max<int64_t>(ne, 1) * sizeof(uint4), st));
        SA_CUDA_TRY(cudaMemsetAsync(P->epos, 0xff, std::max<int64_t>(ne, 1) * sizeof(uint4), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->tp_rank, std::max<int64_t>(P->tp_nslots, 1) * sizeof(unsigned), st));
        if (nn)
            SA_LAUNCH(k_tp_slots, grid_for(nn, 128), 128, 0, st, P->inc_ptr, P->inc, nn, P->wseg, (unsigned)P->e_lo,
                      (unsigned *)P->epos, P->tp_rank);
    }
    if (batches && !P->eb_loc && P->mesh->d == 3) {
        const int64_t ne = P->e_hi - P->e_lo, nb = (ne + EB_SIZE - 1) / EB_SIZE;
        unsigned long long *mx = nullptr;
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->eb_verts, std::max<int64_t>(nb * EB_CAP, 1) * sizeof(int32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->eb_count, std::max<int64_t>(nb, 1) * sizeof(int32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->eb_loc, std::max<int64_t>(ne, 1) * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&mx, sizeof(unsigned long long), st));
        SA_CUDA_TRY(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st));
        if (nb)
            SA_LAUNCH(k_eb_build<3>, (unsigned)nb, EB_SIZE, 0, st, (const int4 *)P->mesh->me, P->e_lo, ne, P->eb_verts,
                      P->eb_count, P->eb_loc, mx);
        unsigned long long h = 0;
        SA_TRY(readback(&h, mx, sizeof h, st));
        SA_TRY(sync_stream(st));
        SA_CUDA_TRY(cudaFreeAsync(mx, st));
        P->eb_maxn = (int)std::min<unsigned long long>(h, EB_CAP);
        P->eb_allfit = h <= EB_CAP;
    }
    if (!P->gd_nflag) {   // fast general operator: guarded-row list
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->gd_flag_rows, std::max<int64_t>(P->nnodes, 1) * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->gd_nflag, sizeof(int), st));
    }
    const int64_t kelems = (int64_t)kstride * P->tp_nslots;
    if (P->kbuf_elems < kelems) {
        if (P->kbuf) SA_CUDA_TRY(cudaFreeAsync(P->kbuf, st));
        P->kbuf = nullptr;
        P->kbuf_elems = 0;
        if (cudaMallocAsync((void **)&P->kbuf, std::max<int64_t>(kelems, 1) * sizeof(double), st) != cudaSuccess)
            return set_error(SA_ERR_NOMEM, "two-pass row buffer (%lld doubles) does not fit", (long long)kelems);
        P->kbuf_elems = kelems;
    }
    return SA_OK;
}

static bool want_batches(int ops, int d) { return ops == SA_OP_GENERAL && d == 3; }

static int plan_nout(int ops)
{
    int n = 0;
    for (int bit = 1; bit <= 8; bit <<= 1) n += (ops & bit) ? 1 : 0;
    return n;
}

int sa_plan_prepare(sa_plan *P, int ops, void *stream)
{
    if (!P) return set_error(SA_ERR_ARG, "plan is NULL");
    const int d = P->mesh->d;
    SA_TRY(set_device(P->mesh->device));
    ops &= 15;
    if (d == 3 && !(want_twopass(ops, d, P->m) && P->n_inc < 0xffffffffLL))
        SA_TRY(sa_winc_d3(P, (cudaStream_t)stream));
    if (want_twopass(ops, d, P->m) && P->n_inc < 0xffffffffLL) {
        const int ks = (d + 1) * plan_nout(ops) * P->m * P->m;
        SA_TRY(ensure_twopass(P, ks, want_batches(ops, d), (cudaStream_t)stream));
    }
    return SA_OK;
}

int sa_numeric(sa_plan *P, int ops, const sa_coeffs *cf, double *const *vals_dev, int64_t *n_zero_out, void *stream)
{
    if (!P || !vals_dev) return set_error(SA_ERR_ARG, "plan/vals is NULL");
    const sa_mesh *M = P->mesh;
    if (!M->coords) return set_error(SA_ERR_ARG, "mesh coordinates not set (sa_mesh_set_coords)");
    const int d = M->d;
    if ((ops & SA_OP_ELASTIC) && P->m != d) return set_error(SA_ERR_ARG, "elastic operator needs a plan with m = d");
    if (!(ops & SA_OP_ELASTIC) && P->m != 1) return set_error(SA_ERR_ARG, "scalar operators need a plan with m = 1");
    SA_TRY(set_device(M->device));
    cudaStream_t st = (cudaStream_t)stream;
    NumArgs a;
    memset(&a, 0, sizeof a);
    a.exact = (ops & SA_OP_EXACT) ? 1 : 0;
    ops &= 15;
    if (d == 3 && !(want_twopass(ops, d, P->m) && P->n_inc < 0xffffffffLL)) SA_TRY(sa_winc_d3(P, st));

    a.qv = M->qv; a.me = M->me; a.vols = M->vols;
    a.nnodes = P->nnodes; a.node_begin = P->node_begin;
    a.inc_ptr = P->inc_ptr; a.inc = P->inc; a.winc = P->winc; a.wseg = P->wseg; a.colptr = P->colptr; a.indptr = P->indptr; a.cols = P->cols;
    a.acc_stride = (int)(P->m * P->m * std::max<int64_t>(P->light_deg, 1));
    a.light_deg = (int)P->light_deg;
    a.heavy_rows = P->heavy_rows;
    a.n_heavy = P->n_heavy;
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
    a.A = cf->A; a.b = cf->b; a.c = cf->c; a.a0 = cf->a0; a.gen_packed = cf->gen_packed;
    a.lambs_e = cf->lambs_e; a.mus_e = cf->mus_e;
    if ((a.lambs_e == nullptr) != (a.mus_e == nullptr))
        return set_error(SA_ERR_ARG, "per-element lambs_e and mus_e must be given together");
    memcpy(a.A_const, cf->A_const, sizeof a.A_const);
    a.a0_const = cf->a0_const;
    const double den = (double)((d + 1) * (d + 2) * (d + 3));
    a.mass_coef_diag = 2.0 / den;
    a.mass_coef_off = 1.0 / den;
    {
        // ((W0 + W1) + ... + Wd) + W[alpha]) + W[beta] with every W = w_const
        double ws = a.w_const;
        for (int k = 1; k <= d; ++k) ws = ws + a.w_const;
        a.mass_wc = (ws + a.w_const) + a.w_const;
    }
    if (want_twopass(ops, d, P->m) && P->n_inc < 0xffffffffLL) {
        const int vpr = (d + 1) * nout * P->m * P->m;
        const int ks = vpr;   // row alignment follows from the row size (see loadk)
        const bool batches = want_batches(ops, d);
        SA_TRY(ensure_twopass(P, ks, batches, st));
        if (batches) {
            a.eb_verts = P->eb_verts;
            a.eb_count = P->eb_count;
            a.eb_loc = P->eb_loc;
            a.eb_maxn = P->eb_maxn;
            a.eb_allfit = P->eb_allfit ? 1 : 0;
            a.eb_b0 = 0;
            a.eb_b1 = (P->e_hi - P->e_lo + EB_SIZE - 1) / EB_SIZE;
        }
        a.kbuf = P->kbuf;
        a.kstride = ks;
        a.epos = P->epos;
        a.e_lo = P->e_lo;
        a.ne = P->e_hi - P->e_lo;
        a.tp_rank = P->tp_rank;
        a.wseg = P->wseg;
        a.nflag = P->gd_nflag;
        a.flag_rows = P->gd_flag_rows;
    }
    SA_CUDA_TRY(cudaMemsetAsync(P->counters, 0, 4 * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMemsetAsync(P->counters + 4, 0x7f, sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMemsetAsync(P->counters + 7, 0, sizeof(int64_t), st));
    int rc;
    if (d == 1) rc = sa_dispatch_d1(P, a, ops, M->core, st);
    else if (d == 2) rc = sa_dispatch_d2(P, a, ops, M->core, st);
    else rc = sa_dispatch_d3(P, a, ops, M->core, st);
    if (rc != SA_OK) return rc;
    if (n_zero_out) {
        int64_t h[8];
        SA_TRY(readback(h, P->counters, 8 * sizeof(int64_t), st));
        SA_TRY(sync_stream(st));
        if (h[7]) return set_error(SA_ERR_CUDA, "chunk kernel: a carry wait timed out (internal error)");
        for (int o = 0; o < nout; ++o) n_zero_out[o] = h[o];
        if (h[4] != 0x7f7f7f7f7f7f7f7fLL) {
            err_state().bad = h[4];
            return set_error(SA_ERR_DEGENERATE, "simplex %lld is degenerate (zero volume)", (long long)h[4]);
        }
    }
    return SA_OK;
}

int sa_unpack_columns(const double *src_dev, int nv, const int32_t *colmap16_host, const double *consts16_host, int64_t nq,
                      double *dst_dev, void *stream)
{
    if (!dst_dev || !colmap16_host || !consts16_host || nv < 0 || nv > 16 || (nv > 0 && !src_dev))
        return set_error(SA_ERR_ARG, "sa_unpack_columns: bad argument");
    UnpackCols u;
    for (int j = 0; j < 16; ++j) {
        if (colmap16_host[j] >= nv) return set_error(SA_ERR_ARG, "sa_unpack_columns: column map entry out of range");
        u.map[j] = colmap16_host[j];
        u.cst[j] = consts16_host[j];
    }
    if (nq > 0)
        SA_LAUNCH(k_unpack_columns, std::min<int64_t>(grid_for(nq * 16, 256), 148 * 32), 256, 0, (cudaStream_t)stream,
                  src_dev, nv, u, nq, dst_dev);
    return SA_OK;
}

int sa_compact(const sa_plan *P, const double *vals_dev, int64_t *indptr_out, int32_t *indices_out, double *vals_out,
               void *stream)
{
    if (!P) return set_error(SA_ERR_ARG, "plan is NULL");
    SA_TRY(set_device(P->mesh->device));
    cudaStream_t st = (cudaStream_t)stream;
    return compact_csr(P->indptr, P->indices, vals_dev, P->nrows, P->nnz, P->scan_tmp, indptr_out, indices_out, vals_out,
                       st);
}

}  // extern "C"

#include "sa_pk.cuh"
#endif  // SA_ABI
