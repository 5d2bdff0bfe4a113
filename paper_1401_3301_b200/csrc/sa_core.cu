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
#include <unordered_map>
#include <vector>

#include "sa_common.cuh"
#include "sa_geometry.cuh"
#include "sa_radix.cuh"

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
    // block numeric kernel: compact incidences + fold program
    uint32_t *inc_e = nullptr;    // (n_inc) e | alpha<<30
    uint16_t *fold = nullptr;     // ((d+1) n_inc) per slot: u | beta<<6 | last<<8
    bool fold_ok = false;         // every node has <= 64 incidences
    // fold templates (tile kernel)
    bool tm_ok = false;
    int64_t n_templates = 0, tm_nwords = 0;
    int tile_rows = 0;
    uint32_t *tile_e0 = nullptr, *tile_tm = nullptr, *tm_off = nullptr, *tm = nullptr;
    // per tile size R = 2^c (c = 0..5): max incidences / node-level entries in one tile of R rows
    int64_t tile_max_inc[6] = {0, 0, 0, 0, 0, 0};
    int64_t tile_max_ent[6] = {0, 0, 0, 0, 0, 0};
    // chunk kernel
    bool ck_ok = false;
    unsigned ck_emin = 0, ck_emax = 0;
    int ck_C = 0;
    int64_t ck_nchunks = 0, ck_ntemplates = 0, ck_nwords = 0;
    uint32_t *ck_tm = nullptr, *ck_pb = nullptr, *ck_tm_off = nullptr, *ck_tmw = nullptr;
    unsigned *ck_flags = nullptr;  // nrec record flags + 1 ticket
    uint32_t *ck_rs = nullptr;     // first record index per chunk
    int64_t ck_nrec = 0;
    int64_t ck_maxw = 0;           // largest chunk template (words)
    unsigned ck_epoch = 0;         // bumped per launch
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
    // overlap of the element pass (compute) with the fold (DRAM): element
    // batch chunks and the warp-aligned row segments whose elements they hold
    std::vector<int64_t> ov_bcut, ov_wcut;   // (K+1) batch cuts, (K+1) warp cuts
    cudaStream_t ov_stream = nullptr;
    std::vector<cudaEvent_t> ov_events;
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
    int dbg;              // diagnostics (SA_DBG): 1 = loads only, 2 = loads + element math, no folds, 3 = stores only
    int acc_stride;  // smem accumulator rows per output (m*m*max_deg)
    double *vals[2];
    int64_t *counters;
    // coefficients
    const double *w; double w_const;
    const double *lamb; double lamb_const;
    const double *mu; double mu_const;
    const double *A; const double *b; const double *c; const double *a0;
    double A_const[9]; double a0_const;
    const double *gen_packed;  // (nq, 16) AoS [A(9) b(3) c(3) a0] or NULL
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
    int64_t row0, row1;        // fold (PRE) row range of this launch (row0 % 32 == 0)
    double mass_coef_diag, mass_coef_off;  // 2/((d+1)(d+2)(d+3)), 1/(...) as Python computes them
    double mass_wc;  // constant weight: (wsum + w) + w, the same for every (alpha, beta)
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

// Fold program of node row nl: for each column k (ascending), the
// contributing (incidence u, local vertex beta) pairs in ascending element
// order, as u | beta << 6; the last pair of each column has bit 8 set.
template <int D>
__global__ void k_fold_lists(const int64_t *__restrict__ inc_ptr, const uint2 *__restrict__ inc, int64_t nnodes,
                             const int64_t *__restrict__ colptr, uint32_t *__restrict__ inc_e,
                             uint16_t *__restrict__ fold, unsigned long long *too_many)
{
    int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl >= nnodes) return;
    const int64_t t0 = inc_ptr[nl];
    const int ni = (int)(inc_ptr[nl + 1] - t0);
    for (int u = 0; u < ni; ++u) inc_e[t0 + u] = inc[t0 + u].x;
    if (ni > 64) { atomicOr(too_many, 1ull); return; }
    const int deg = (int)(colptr[nl + 1] - colptr[nl]);
    uint16_t *out = fold + (int64_t)(D + 1) * t0;
    int w = 0;
    for (int k = 0; k < deg; ++k) {
        int last = -1;
        for (int u = 0; u < ni; ++u) {
            const unsigned r = inc[t0 + u].y;
            for (int b = 0; b <= D; ++b)
                if ((int)((r >> (8 * b)) & 0xff) == k) { out[w] = (uint16_t)(u | (b << 6)); last = w; ++w; }
        }
        if (last >= 0) out[last] |= 256;
    }
}

// ---- tile templates -------------------------------------------------------
// A tile is R consecutive node rows, processed by one warp.  Its template
// (relative to the tile's smallest element id e_base) holds
//   w[0] = n_elem | nrows << 8 | nslots << 16,  w[1] = NE node-level entries
//   w[2 .. 2+ne)            de[j]: the tile's distinct elements, ascending
//   w[2+ne .. 2+2ne)        per element: 4 x 8-bit slot id of local row
//                           alpha = 0..3 (0xff: vertex not in the tile)
//   w[2+2ne .. 2+2ne+2NI)   per slot (= incidence, row-major, ascending
//                           element per row): 4 x 16-bit fold positions,
//                           one per local column beta
//   w[PB .. PB+nrows)       per row: deg | entb << 16
//   w[OB .. OB+(NE+2)/2)    NE+1 uint16 entry offsets into the fold array
//   w[LB .. LB+17)          33 uint16: lane l sums entries [ls[l], ls[l+1]),
//                           split so every lane gets ~1/32 of the contributions
// The fold array of a tile is entry-major: entry k's contributions occupy
// [off[k], off[k+1]) in ascending element order.  Element lanes scatter their
// local rows straight into it; row lanes then sum contiguous runs.
// Tiles with equal templates share one copy: all interior tiles of a
// structured mesh collapse to a few dozen.
__device__ __forceinline__ uint64_t fnv_step(uint64_t h, uint32_t x)
{
#pragma unroll
    for (int i = 0; i < 4; ++i) { h ^= (x >> (8 * i)) & 0xff; h *= 1099511628211ull; }
    return h;
}

constexpr int TILE_MAX_ELEM = 255;

__host__ __device__ inline int64_t tile_stride_bound(int64_t NI, int64_t NE, int64_t R)
{
    return 2 + 2 * (NI < TILE_MAX_ELEM ? NI : TILE_MAX_ELEM) + 2 * NI + R + (NE + 2) / 2 + 17 + 4;
}

template <int D>
__global__ void k_tile_build(const int64_t *__restrict__ inc_ptr, const uint32_t *__restrict__ inc_e,
                             const uint16_t *__restrict__ fold, const int64_t *__restrict__ colptr, int64_t nnodes,
                             int R, int64_t ntiles, int stride, uint32_t *__restrict__ scratch,
                             uint32_t *__restrict__ words_out, uint64_t *__restrict__ sig,
                             uint32_t *__restrict__ tile_e0, unsigned long long *fail)
{
    const int64_t T = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (T >= ntiles) return;
    const int64_t r0 = T * R;
    const int nr = (int)min((int64_t)R, nnodes - r0);
    uint32_t *w = scratch + T * (int64_t)stride;
    const int64_t t0 = inc_ptr[r0];
    const int NI = (int)(inc_ptr[r0 + nr] - t0);
    const int64_t c0 = colptr[r0];
    const int NE = (int)(colptr[r0 + nr] - c0);
    uint32_t el[TILE_MAX_ELEM];
    int ne = 0;
    bool bad = NI > 254 || (D + 1) * NI > 65535 || NE > 65534;
    for (int i = 0; i < NI && !bad; ++i) {
        const uint32_t e = inc_e[t0 + i] & 0x3fffffffu;
        int lo = 0, hi = ne;
        while (lo < hi) { int mid = (lo + hi) >> 1; if (el[mid] < e) lo = mid + 1; else hi = mid; }
        if (lo < ne && el[lo] == e) continue;
        if (ne == TILE_MAX_ELEM) { bad = true; break; }
        for (int k = ne; k > lo; --k) el[k] = el[k - 1];
        el[lo] = e;
        ++ne;
    }
    if (bad) { atomicOr(fail, 1ull); words_out[T] = 0; return; }
    const uint32_t eb = ne ? el[0] : 0u;
    tile_e0[T] = eb;
    w[0] = (uint32_t)ne | ((uint32_t)nr << 8) | ((uint32_t)NI << 16);
    w[1] = (uint32_t)NE;
    for (int j = 0; j < ne; ++j) { w[2 + j] = el[j] - eb; w[2 + ne + j] = 0xffffffffu; }
    for (int i = 0; i < NI; ++i) {
        const uint32_t r = inc_e[t0 + i];
        const uint32_t e = r & 0x3fffffffu, alpha = r >> 30;
        int lo = 0, hi = ne;
        while (lo < hi) { int mid = (lo + hi) >> 1; if (el[mid] < e) lo = mid + 1; else hi = mid; }
        uint32_t &sw = w[2 + ne + lo];
        sw = (sw & ~(0xffu << (8 * alpha))) | ((uint32_t)i << (8 * alpha));
    }
    const uint32_t SB = 2 + 2 * ne, PB = SB + 2 * NI, OB = PB + nr, LB = OB + ((NE + 2) >> 1);
    const uint32_t end = LB + 17;
    for (uint32_t x = SB; x < end; ++x) w[x] = 0;
    for (int row = 0; row < nr; ++row) {
        const int64_t ip = inc_ptr[r0 + row];
        const int ni = (int)(inc_ptr[r0 + row + 1] - ip);
        const int deg = (int)(colptr[r0 + row + 1] - colptr[r0 + row]);
        const int incb = (int)(ip - t0);
        const int entb = (int)(colptr[r0 + row] - c0);
        w[PB + row] = (uint32_t)deg | ((uint32_t)entb << 16);
        int k = 0;
        for (int s = 0; s < (D + 1) * ni; ++s) {
            const uint16_t f = fold[(D + 1) * ip + s];
            const uint32_t slot = incb + (f & 63), beta = (f >> 6) & 3;
            const uint32_t pos = (uint32_t)((D + 1) * incb + s);
            w[SB + 2 * slot + (beta >> 1)] |= pos << (16 * (beta & 1));
            if (f & 256) {
                ++k;
                const uint32_t kg = entb + k;
                w[OB + (kg >> 1)] |= (pos + 1) << (16 * (kg & 1));
            }
        }
    }
    // lane starts: lane l takes the entries whose runs start in [l*NC/32, (l+1)*NC/32)
    {
        const uint32_t NC = (uint32_t)((D + 1) * NI);
        int k = 0;
        for (int l = 0; l <= 32; ++l) {
            const uint32_t target = (uint32_t)(((uint64_t)NC * l) / 32);
            while (k < NE && ((w[OB + (k >> 1)] >> (16 * (k & 1))) & 0xffff) < target) ++k;
            const uint32_t v = l == 32 ? (uint32_t)NE : (uint32_t)k;
            w[LB + (l >> 1)] |= v << (16 * (l & 1));
        }
    }
    words_out[T] = end;
    uint64_t h = 1469598103934665603ull;
    for (uint32_t x = 0; x < end; ++x) h = fnv_step(h, w[x]);
    sig[T] = h;
}

__global__ void k_tile_pack(const int64_t *__restrict__ rep, int64_t ntm, const uint32_t *__restrict__ scratch,
                            int stride, const uint32_t *__restrict__ words, const uint32_t *__restrict__ tm_off,
                            uint32_t *__restrict__ tm)
{
    // one warp per template
    const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= ntm) return;
    const uint32_t *src = scratch + rep[t] * (int64_t)stride;
    uint32_t *dst = tm + tm_off[t];
    const uint32_t n = words[rep[t]];
    for (uint32_t i = lane; i < n; i += 32) dst[i] = src[i];
}

__global__ void k_tile_verify(const uint32_t *__restrict__ scratch, int stride, const uint32_t *__restrict__ words,
                              int64_t ntiles, const uint32_t *__restrict__ tile_tm,
                              const uint32_t *__restrict__ tm_off, const uint32_t *__restrict__ tm,
                              unsigned long long *bad)
{
    const int64_t T = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (T >= ntiles) return;
    const uint32_t *a = scratch + T * (int64_t)stride;
    const uint32_t *b = tm + tm_off[tile_tm[T]];
    const uint32_t n = words[T];
    bool ok = true;
    for (uint32_t i = lane; i < n; i += 32) ok &= (a[i] == b[i]);
    if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicOr(bad, 1ull);
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
    // general: coefficient sums accumulated while loading (in vertex order,
    // as the reference-order restatement sums them) + the per-vertex terms
    double As[D][D], bs[D], cs[D], a0s;
    double bv[D + 1][D], cv[D + 1][D], a0v[D + 1];
};

template <int D, int OPS>
__device__ __forceinline__ void element_load1(const NumArgs &a, int64_t e, ElemRaw<D> &r)
{
    load_element<D>((const typename IdxT<D>::type *)a.me, e, r.v);
    r.vol = __ldg(a.vols + e);
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
        // lambs = (sum_k lamb_k) * (vols / (d+1))   kernels.py:354-356
        const double scale = __ddiv_rn(r.vol, (double)(D + 1));
        double ls = r.lam[0], ms = r.mu[0];
#pragma unroll
        for (int k = 1; k <= D; ++k) { ls = SA_ADD(ls, r.lam[k]); ms = SA_ADD(ms, r.mu[k]); }
        g.lambs = SA_MUL(ls, scale);
        g.mus = SA_MUL(ms, scale);
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
template <int D, int M, int OPS, int CORE, int ILP, int MINB, bool PRE = false, bool LEAN = false>
__global__ void __launch_bounds__(128, MINB) k_numeric_rowgather(NumArgs a_in)
{
    // LEAN: no diagnostics and a constant mass weight, known at compile time
    // (the local copy is scalar-replaced; w == nullptr and dbg == 0 fold the
    // weight loads and the diagnostic branches away)
    NumArgs a = a_in;
    if constexpr (LEAN) {
        a.w = nullptr;
        a.dbg = 0;
    }
    constexpr int NOUT = n_outputs<OPS>();
    extern __shared__ double smem_acc[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t nl = (PRE ? a.row0 : 0) + blockIdx.x * (int64_t)blockDim.x + tid;
    // Accumulators: per warp and output a plane of 32 lane rows of S doubles;
    // lane j's dof row l, column k at wacc[o*32*S + j*S + l*M*deg + k].  When
    // the warp's rows all have degree d0, S = M*M*d0 and the plane IS the
    // warp's CSR run (row-major, consecutive rows), so the store phase is a
    // straight coalesced copy; otherwise S is padded to the warp's largest
    // row (odd, so lane strides hit distinct banks) and rows store their own
    // segments.
    const unsigned full = 0xffffffffu;
    const bool active = nl < (PRE ? a.row1 : a.nnodes);
    const int64_t c0 = active ? a.colptr[nl] : 0;
    const int deg = active ? (int)(a.colptr[nl + 1] - c0) : -1;
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
    if (active) {
        const int deg_stride = M * deg;
        for (int o = 0; o < NOUT; ++o)
            for (int k = 0; k < M * deg_stride; ++k) wacc[o * 32 * S + k] = 0.0;
        const int64_t t1 = a.dbg >= 3 ? inc0 : inc1;   // 3: stores only, 4: neither
        int64_t emin = INT64_MAX;
        constexpr int MM = M * M;
        double dsum = 0.0;
        constexpr int VPR = (D + 1) * NOUT * MM;
        // fold one local row set into the row accumulators (ranks: 8-bit
        // column rank of each element vertex within this row)
        auto accum = [&](const double(&vals)[VPR], unsigned ranks) {
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
            if (a.dbg == 1) {   // diagnostics: memory traffic only
#pragma unroll
                for (int b = 0; b <= D; ++b)
#pragma unroll
                    for (int c = 0; c < D; ++c) dsum += x.x[b][c];
                dsum += x.vol + (double)x.v[0] + (double)rec.y;
                return;
            }
            ElemGeo<D> g;
            const int64_t e = rec.x & 0x3fffffffu;
            if (element_compute<D, OPS, CORE>(x, g)) emin = min(emin, e);
            double vals[(D + 1) * NOUT * MM];
            if constexpr (LEAN && ((M == 1 && (OPS & ~(OP_MASS | OP_STIFF)) == 0) || OPS == OP_ELASTIC))
                element_krow_sel<D, OPS>(a, g, rec.x >> 30, vals);
            else
                krow_runtime<D, M, OPS>(a, g, rec.x >> 30, vals);
            if (a.dbg == 2) {   // diagnostics: no folds
#pragma unroll
                for (int i = 0; i < (D + 1) * NOUT * MM; ++i) dsum += vals[i];
                return;
            }
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
                    for (int i = 0; i < VPR; i += 4) ldg256(src + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
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
                    rk[u] = __ldg(a.tp_rank + slot);
                    loadk(slot, v[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) accum(v[u], rk[u]);
            }
            for (; t < t1; ++t) {
                double v[VPR];
                const int64_t slot = sb + 32 * (t - t0);
                const unsigned rk = __ldg(a.tp_rank + slot);
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
        if (a.dbg) wacc[0] = dsum;
    }
    // Stores (see the accumulator layout above)
    __syncwarp();
    if (a.dbg == 4) {   // diagnostics: metadata + zero-init only, no stores
    } else if (uniform) {
        const int64_t base = __shfl_sync(full, row_base, 0);
        const double *plane = wacc - lane * S;
        for (int i = lane; i < 32 * S; i += 32) {
#pragma unroll
            for (int o = 0; o < NOUT; ++o) {
                const double val = plane[o * 32 * S + i];
                a.vals[o][base + i] = val;
                nz[o] += (val == 0.0);
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
                    nz[o] += (val == 0.0);
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

template <int VPR>
__device__ __forceinline__ void store_row(double *dst, const double (&vals)[VPR])
{
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
constexpr int EB_SIZE = 128;   // elements per batch
constexpr int EB_CAP = 255;    // distinct vertices per batch (8-bit local ids)
constexpr int EB_REC = 20;     // staged doubles per vertex: q (4, padded) + [A(9) b(3) c(3) a0]

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
        const double *rec = vrec + ((lc >> (8 * k)) & 0xff) * EB_REC;
#pragma unroll
        for (int c = 0; c < D; ++c) r.x[k][c] = rec[c];
        const double *w = rec + 4;
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

template <int D, int M, int OPS, int CORE, int MINB, bool ALLFIT = false>
__global__ void __launch_bounds__(EB_SIZE, MINB) k_element_rows_batched(NumArgs a)
{
    extern __shared__ double vrec[];
    const int t = threadIdx.x;
    const int64_t b = blockIdx.x, i = b * EB_SIZE + t;
    const bool in = i < a.ne;
    const int64_t e = a.e_lo + i;
    // ALLFIT: every batch is staged (the direct-gather fallback is not compiled)
    const int n = ALLFIT ? max(__ldg(a.eb_count + b), 0) : __ldg(a.eb_count + b);
    uint4 p = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    unsigned lc = 0;
    ElemRaw<D> x;
    if (in) {
        p = __ldg(a.epos + i);
        x.vol = __ldg(a.vols + e);
        if (n >= 0) lc = __ldg(a.eb_loc + i);
        else load_element<D>((const typename IdxT<D>::type *)a.me, e, x.v);
    }
    if (n >= 0) {   // uniform per block
        // the batch's vertex list first (one coalesced load), then every
        // cp.async of the stage issues without a dependent load
        __shared__ int sv[EB_CAP + 1];
        const int32_t *vl = a.eb_verts + b * EB_CAP;
        for (int s = t; s < n; s += EB_SIZE) sv[s] = __ldg(vl + s);
        __syncthreads();
        for (int c = t; c < n * 10; c += EB_SIZE) {
            const int s = c / 10, h = c - 10 * s;
            const int64_t vv = sv[s];
            const double *src = h < 2 ? (const double *)a.qv + vv * 4 + 2 * h : a.gen_packed + vv * 16 + 2 * (h - 2);
            cp_async16(vrec + s * EB_REC + 2 * h, src);
        }
        cp_async_wait_all();
        __syncthreads();
    }
    if (!in) return;
    const unsigned pos[4] = {p.x, p.y, p.z, p.w};
    bool any = false;
#pragma unroll
    for (int k = 0; k <= D; ++k) any |= pos[k] != 0xffffffffu;
    if (!any) return;
    if (n >= 0) element_from_stage<D, OPS>(vrec, lc, x);
    else element_load2<D, OPS>(a, x);
    ElemGeo<D> g;
    if (element_compute<D, OPS, CORE>(x, g)) atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)e);
    element_rows_store<D, M, OPS>(a, g, pos);
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

template <int D, int M, int OPS, int CORE, int MINB>
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
            p = __ldg(a.epos + i);
            lc = __ldg(a.eb_loc + i);
            vol = __ldg(a.vols + a.e_lo + i);
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
            ElemRaw<D> x;
            x.vol = vol;
            element_from_stage<D, OPS>(recs + (size_t)(k & 1) * RS, lc, x);
            ElemGeo<D> g;
            if (element_compute<D, OPS, CORE>(x, g))
                atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)(a.e_lo + i));
            element_rows_store<D, M, OPS>(a, g, pos);
        }
        p = pn;
        lc = lcn;
        vol = voln;
        __syncthreads();   // stage k & 1 is rewritten by the records of batch k+2
    }
    cp_async_wait<0>();
}

// largest element of each warp's 32 rows (incidences are sorted per row)
__global__ void k_warp_emax(const int64_t *__restrict__ inc_ptr, const uint2 *__restrict__ inc, int64_t nnodes,
                            unsigned *__restrict__ out)
{
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r0 = w * 32;
    if (r0 >= nnodes) return;
    const int64_t r1 = min(r0 + 32, nnodes);
    unsigned m = 0;
    for (int64_t r = r0; r < r1; ++r)
        if (inc_ptr[r + 1] > inc_ptr[r]) m = max(m, inc[inc_ptr[r + 1] - 1].x & 0x3fffffffu);
    out[w] = m;
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

// element lane: local row A of the element -> scatter into the fold array
template <int D, int M, int OPS, int A = 0>
__device__ __forceinline__ void element_rows_scatter(const NumArgs &a, const ElemGeo<D> &g, unsigned sw,
                                                     const uint32_t *__restrict__ tm, unsigned sb, double *F, int FS)
{
    constexpr int NOUT = n_outputs<OPS>();
    constexpr int MM = M * M;
    const unsigned slot = (sw >> (8 * A)) & 0xff;
    if (slot != 0xff) {
        double vals[(D + 1) * NOUT * MM];
        element_krow<D, M, OPS, A>(a, g, vals);
        const unsigned p01 = __ldg(tm + sb + 2 * slot), p23 = __ldg(tm + sb + 2 * slot + 1);
#pragma unroll
        for (int b = 0; b <= D; ++b) {
            const unsigned pos = ((b < 2 ? p01 : p23) >> (16 * (b & 1))) & 0xffff;
#pragma unroll
            for (int o = 0; o < NOUT; ++o)
#pragma unroll
                for (int i = 0; i < MM; ++i) F[(o * FS + pos) * MM + i] = vals[(b * NOUT + o) * MM + i];
        }
    }
    if constexpr (A < D) element_rows_scatter<D, M, OPS, A + 1>(a, g, sw, tm, sb, F, FS);
}

// Tile numeric kernel (K1 + K2 + K4), the production path.
//
// One warp owns one tile (R = 32/L consecutive node rows, L lanes per row);
// warps never synchronise with each other, so the SM overlaps one warp's
// loads with another's arithmetic.
//   phase 1  lanes over the tile's distinct elements: loads for two elements
//            in flight, geometry once per element, then each local row the
//            tile needs, scattered into the tile's entry-major fold array in
//            warp-private shared memory;
//   phase 2  each row's L lanes sum their entries' contiguous runs in
//            registers (ascending element order) into an output segment;
//   phase 3  the tile's rows are consecutive, so their CSR segment is one
//            contiguous range: coalesced stores.
// Every entry is the left-to-right sum of its contributions in ascending
// element index: bitwise the reference's optv2 value.
struct TileArgs {
    const uint32_t *tile_e0;   // (ntiles) smallest element of each tile
    const uint32_t *tile_tm;   // (ntiles) template id
    const uint32_t *tm_off;    // (ntemplates) word offset of each template
    const uint32_t *tm;        // template words
    int max_inc;               // max incidences (slots) in one tile
    int max_ent;               // max node-level entries in one tile
};

// Kernel choice: the row-gather kernel is the default (fastest measured on
// every BASELINE config so far); SA_KERNEL=tile selects the tile kernel, whose
// templates are then built in the symbolic phase.
inline bool want_tile_kernel()
{
    const char *k = getenv("SA_KERNEL");
    return k && strcmp(k, "tile") == 0;
}
// SA_KERNEL=chunk selects the element-chunk kernel (its symbolic data is then
// built); the row-gather kernel is the default (fastest measured, profiles/)
inline bool want_chunk_kernel()
{
    const char *k = getenv("SA_KERNEL");
    return k && strcmp(k, "chunk") == 0;
}

// lanes per row (R = 32/L rows per warp tile): default per (d, m), override
// with SA_TILE_LANES at plan creation (tuning).
inline int default_lanes(int d, int m)
{
    return d == 1 ? 1 : (m == 1 ? (d == 2 ? 2 : 4) : (d == 2 ? 4 : 16));
}
inline int tile_lanes(int d, int m)
{
    const char *v = getenv("SA_TILE_LANES");
    int L = v ? atoi(v) : default_lanes(d, m);
    if (L != 1 && L != 2 && L != 4 && L != 8 && L != 16) L = default_lanes(d, m);
    return L;
}

template <int D, int M, int OPS, int CORE, int L>
__global__ void __launch_bounds__(128) k_numeric_tiles(NumArgs a, TileArgs t)
{
    constexpr int NOUT = n_outputs<OPS>();
    constexpr int MM = M * M;
    constexpr int R = 32 / L;
    constexpr int WARPS = 4;
    extern __shared__ __align__(16) double smem_d[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t T = (int64_t)blockIdx.x * WARPS + wid;
    const int64_t r0 = T * R;
    if (r0 >= a.nnodes) return;
    const int FS = (D + 1) * t.max_inc;          // fold positions per output
    const int OS = M > 1 ? MM * t.max_ent : 0;   // output staging (vector case only)
    double *F = smem_d + (size_t)wid * NOUT * ((size_t)FS * MM + OS);
    double *outs = F + (size_t)NOUT * FS * MM;

    const unsigned to = __ldg(t.tm_off + __ldg(t.tile_tm + T));
    const unsigned eb = __ldg(t.tile_e0 + T);
    const unsigned hdr = __ldg(t.tm + to);
    const int ne = hdr & 0xff, nr = (hdr >> 8) & 0xff, NI = hdr >> 16;
    const int NE = __ldg(t.tm + to + 1);
    const unsigned SB = to + 2 + 2 * ne, PB = SB + 2 * NI, OB = PB + nr;

    // phase 1: each distinct element once, two per lane in flight
    int64_t emin = INT64_MAX;
    for (int j = lane; j < ne; j += 64) {
        const bool two = j + 32 < ne;
        const int64_t e1 = (int64_t)eb + __ldg(t.tm + to + 2 + j);
        const unsigned sw1 = __ldg(t.tm + to + 2 + ne + j);
        const int64_t e2 = two ? (int64_t)eb + __ldg(t.tm + to + 2 + j + 32) : e1;
        const unsigned sw2 = two ? __ldg(t.tm + to + 2 + ne + j + 32) : 0xffffffffu;
        ElemRaw<D> x1, x2;
        element_load1<D, OPS>(a, e1, x1);
        element_load1<D, OPS>(a, e2, x2);
        element_load2<D, OPS>(a, x1);
        element_load2<D, OPS>(a, x2);
        ElemGeo<D> g;
        if (element_compute<D, OPS, CORE>(x1, g)) emin = min(emin, e1);
        element_rows_scatter<D, M, OPS>(a, g, sw1, t.tm, SB, F, FS);
        if (two) {
            if (element_compute<D, OPS, CORE>(x2, g)) emin = min(emin, e2);
            element_rows_scatter<D, M, OPS>(a, g, sw2, t.tm, SB, F, FS);
        }
    }
    if (emin != INT64_MAX) atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)emin);
    __syncwarp();

    int nz[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) nz[o] = 0;
    const int64_t base = a.indptr[(int64_t)M * r0];
    if constexpr (M == 1) {
        // phase 2 (scalar): the tile's entries are in CSR order and their runs
        // are contiguous in the fold array; lane l sums the entries whose runs
        // start in its 1/32 of the contributions (balanced, no carries: each
        // run is summed left to right by one lane) and stores each result to
        // its CSR position.
        const unsigned LB = OB + ((NE + 2) >> 1);
        const int kb = (__ldg(t.tm + LB + (lane >> 1)) >> (16 * (lane & 1))) & 0xffff;
        const int ke = (__ldg(t.tm + LB + ((lane + 1) >> 1)) >> (16 * ((lane + 1) & 1))) & 0xffff;
        if (kb < ke) {
            auto off = [&](int k) { return (int)((__ldg(t.tm + OB + (k >> 1)) >> (16 * (k & 1))) & 0xffff); };
            int k = kb;
            int s = off(kb), next = off(kb + 1);
            const int se = off(ke);
            double acc[NOUT];
#pragma unroll
            for (int o = 0; o < NOUT; ++o) acc[o] = 0.0;
            for (; s < se; ++s) {
#pragma unroll
                for (int o = 0; o < NOUT; ++o) acc[o] = SA_ADD(acc[o], F[o * FS + s]);
                if (s + 1 == next) {
#pragma unroll
                    for (int o = 0; o < NOUT; ++o) {
                        a.vals[o][base + k] = acc[o];
                        nz[o] += (acc[o] == 0.0);
                        acc[o] = 0.0;
                    }
                    ++k;
                    if (k < ke) next = off(k + 1);
                }
            }
        }
    } else {
        // phase 2 (vector): each row's L lanes sum their entries' runs
        const int row = lane / L, jl = lane % L;
        if (row < nr) {
            const unsigned rw = __ldg(t.tm + PB + row);
            const int deg = rw & 0xffff, entb = rw >> 16;
            for (int k = jl; k < deg; k += L) {
                const int kg = entb + k;
                const unsigned s0 = (__ldg(t.tm + OB + (kg >> 1)) >> (16 * (kg & 1))) & 0xffff;
                const unsigned s1 = (__ldg(t.tm + OB + ((kg + 1) >> 1)) >> (16 * ((kg + 1) & 1))) & 0xffff;
#pragma unroll
                for (int o = 0; o < NOUT; ++o) {
                    double acc[MM];
#pragma unroll
                    for (int i = 0; i < MM; ++i) acc[i] = 0.0;
                    const double *src = F + (size_t)o * FS * MM;
                    for (unsigned s = s0; s < s1; ++s)
#pragma unroll
                        for (int i = 0; i < MM; ++i) acc[i] = SA_ADD(acc[i], src[s * MM + i]);
                    double *orow = outs + o * OS + MM * entb;
#pragma unroll
                    for (int l = 0; l < M; ++l)
#pragma unroll
                        for (int n = 0; n < M; ++n) orow[l * M * deg + k * M + n] = acc[l * M + n];
                }
            }
        }
        __syncwarp();
        // phase 3: the tile's CSR segment is contiguous -> coalesced stores
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
            double *dst = a.vals[o] + base;
            const double *src = outs + o * OS;
            for (int i = lane; i < MM * NE; i += 32) {
                const double v = src[i];
                dst[i] = v;
                nz[o] += (v == 0.0);
            }
        }
    }
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
        int v = nz[o];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
        if (lane == 0 && v) atomicAdd((unsigned long long *)(a.counters + o), (unsigned long long)v);
    }
}

#include "sa_chunk.cuh"

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
int mesh_coords(sa_mesh *M, const double *q, const double *vols, cudaStream_t st);

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
    if (M->nq && q) SA_LAUNCH(k_pack_q<D>, gq, B, 0, st, q, M->nq, (V *)M->qv);
    if (M->nme) SA_LAUNCH(k_pack_me<D>, ge, B, 0, st, me, M->nq, M->nme, (I *)M->me, bad);
    unsigned long long hbad = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
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
        SA_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        if (hbad != ~0ull) {
            err_state().bad = (int64_t)hbad;
            return set_error(SA_ERR_DEGENERATE, "simplex %lld is degenerate (zero volume)", (long long)hbad);
        }
    }
    return SA_OK;
}

// Host side of the tile-template dedupe: build every tile in scratch, dedupe
// by 64-bit signature, pack one copy per template, then verify every tile
// word for word against its template (a hash collision disables templates).
template <int D>
int build_tile_templates(sa_plan *P, int R, cudaStream_t st)
{
    const int64_t nn = P->nnodes;
    const int64_t ntiles = (nn + R - 1) / R;
    int c = 0;
    while ((1 << c) < R) ++c;
    const int64_t NI = P->tile_max_inc[c], NE = P->tile_max_ent[c];
    if (NI > 254) return SA_OK;  // tiles too wide for 8-bit slots: row-gather kernel
    const int64_t stride64 = tile_stride_bound(NI, NE, R);
    const int stride = (int)stride64;
    uint32_t *scratch = nullptr, *words = nullptr;
    uint64_t *sig = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&scratch, ntiles * stride64 * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&words, ntiles * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&sig, ntiles * sizeof(uint64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->tile_e0, ntiles * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->tile_tm, ntiles * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, sizeof(int64_t), st));
    SA_LAUNCH(k_tile_build<D>, grid_for(ntiles, 64), 64, 0, st, P->inc_ptr, P->inc_e, P->fold, P->colptr, nn, R,
              ntiles, stride, scratch, words, sig, P->tile_e0, (unsigned long long *)(P->counters + 6));
    std::vector<uint64_t> hs(ntiles);
    std::vector<uint32_t> hw(ntiles);
    int64_t fail = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(hs.data(), sig, ntiles * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaMemcpyAsync(hw.data(), words, ntiles * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaMemcpyAsync(&fail, P->counters + 6, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    int rc = SA_OK;
    if (!fail) {
        std::unordered_map<uint64_t, uint32_t> ids;
        std::vector<uint32_t> ttm(ntiles), off;
        std::vector<int64_t> rep;
        uint64_t total = 0;
        for (int64_t i = 0; i < ntiles; ++i) {
            auto it = ids.find(hs[i]);
            if (it == ids.end()) {
                const uint32_t id = (uint32_t)rep.size();
                ids.emplace(hs[i], id);
                rep.push_back(i);
                off.push_back((uint32_t)total);
                total += hw[i];
                ttm[i] = id;
            } else {
                ttm[i] = it->second;
            }
        }
        if (total < ((uint64_t)1 << 32)) {
            P->n_templates = (int64_t)rep.size();
            P->tm_nwords = (int64_t)total;
            P->tile_rows = R;
            int64_t *drep = nullptr;
            SA_CUDA_TRY(cudaMallocAsync((void **)&drep, rep.size() * sizeof(int64_t), st));
            SA_CUDA_TRY(cudaMallocAsync((void **)&P->tm_off, off.size() * sizeof(uint32_t), st));
            SA_CUDA_TRY(cudaMallocAsync((void **)&P->tm, std::max<uint64_t>(total, 1) * sizeof(uint32_t), st));
            SA_CUDA_TRY(cudaMemcpyAsync(drep, rep.data(), rep.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
            SA_CUDA_TRY(cudaMemcpyAsync(P->tm_off, off.data(), off.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            SA_CUDA_TRY(cudaMemcpyAsync(P->tile_tm, ttm.data(), ntiles * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            SA_LAUNCH(k_tile_pack, grid_for((int64_t)rep.size() * 32, 128), 128, 0, st, drep, (int64_t)rep.size(),
                      scratch, stride, words, P->tm_off, P->tm);
            SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, sizeof(int64_t), st));
            SA_LAUNCH(k_tile_verify, grid_for(ntiles * 32, 128), 128, 0, st, scratch, stride, words, ntiles,
                      P->tile_tm, P->tm_off, P->tm, (unsigned long long *)(P->counters + 6));
            int64_t bad = 0;
            SA_CUDA_TRY(cudaMemcpyAsync(&bad, P->counters + 6, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            SA_CUDA_TRY(cudaStreamSynchronize(st));
            SA_CUDA_TRY(cudaFreeAsync(drep, st));
            P->tm_ok = (bad == 0);
        }
    }
    SA_CUDA_TRY(cudaFreeAsync(scratch, st));
    SA_CUDA_TRY(cudaFreeAsync(words, st));
    SA_CUDA_TRY(cudaFreeAsync(sig, st));
    return rc;
}

// Host side of the chunk kernel's symbolic data (see sa_chunk.cuh).
template <int D>
int build_chunks(sa_plan *P, cudaStream_t st)
{
    const int64_t nn = P->nnodes;
    if (!nn || !P->n_inc) return SA_OK;
    unsigned *mm = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&mm, 2 * sizeof(unsigned), st));
    const unsigned init[2] = {0xffffffffu, 0u};
    SA_CUDA_TRY(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st));
    SA_LAUNCH(k_inc_minmax<D>, std::min<int64_t>(grid_for(P->n_inc, 256), 148 * 8), 256, 0, st, P->inc_e, P->n_inc, mm);
    unsigned hmm[2];
    SA_CUDA_TRY(cudaMemcpyAsync(hmm, mm, sizeof hmm, cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    SA_CUDA_TRY(cudaFreeAsync(mm, st));
    const int C = chunk_elems(D, P->m);
    const int64_t nchunks = ((int64_t)hmm[1] - hmm[0]) / C + 1;
    P->ck_emin = hmm[0];
    P->ck_emax = hmm[1];
    P->ck_C = C;
    P->ck_nchunks = nchunks;

    // records: count, scan, fill
    int64_t *rcount = nullptr, *rstart = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&rcount, (nn + 1) * sizeof(int64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&rstart, (nn + 1) * sizeof(int64_t), st));
    SA_LAUNCH(k_chunk_records<D>, grid_for(nn, 128), 128, 0, st, P->inc_ptr, P->inc_e, P->fold, P->colptr, P->indptr,
              nn, P->m, hmm[0], C, rcount, (const int64_t *)nullptr, (uint64_t *)nullptr, (uint32_t *)nullptr,
              (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint16_t *)nullptr);
    SA_TRY(exclusive_scan_i64(rcount, rstart, nn, P->scan_tmp, st));
    int64_t nrec = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&nrec, rstart + nn, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    if (nrec >= ((int64_t)1 << 32)) {
        SA_CUDA_TRY(cudaFreeAsync(rcount, st));
        SA_CUDA_TRY(cudaFreeAsync(rstart, st));
        return SA_OK;
    }
    uint64_t *k0 = nullptr, *k1 = nullptr;
    uint32_t *v0 = nullptr, *v1 = nullptr, *rp = nullptr, *rmeta = nullptr, *rprev = nullptr, *rcoff = nullptr;
    uint16_t *contrib = nullptr;
    const int64_t nr1 = std::max<int64_t>(nrec, 1);
    SA_CUDA_TRY(cudaMallocAsync((void **)&k0, nr1 * sizeof(uint64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&k1, nr1 * sizeof(uint64_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&v0, nr1 * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&v1, nr1 * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&rp, nr1 * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&rmeta, nr1 * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&rprev, nr1 * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&rcoff, nr1 * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&contrib, (D + 1) * P->n_inc * sizeof(uint16_t), st));
    SA_LAUNCH(k_chunk_records<D>, grid_for(nn, 128), 128, 0, st, P->inc_ptr, P->inc_e, P->fold, P->colptr, P->indptr,
              nn, P->m, hmm[0], C, (int64_t *)nullptr, (const int64_t *)rstart, k0, v0, rp, rmeta, rprev, rcoff,
              contrib);
    int kbits = 0;
    while (((int64_t)1 << kbits) < nchunks) ++kbits;
    int which = 0;
    SA_TRY(radix::sort_pairs(k0, v0, k1, v1, nrec, std::max(8, (kbits + 7) & ~7), st, &which));
    const uint64_t *skey = which ? k1 : k0;
    const uint32_t *order = which ? v1 : v0;
    int64_t *cstart = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&cstart, (nchunks + 1) * sizeof(int64_t), st));
    SA_LAUNCH(k_chunk_bounds, grid_for(nrec, 256), 256, 0, st, skey, nrec, nchunks, cstart);
    std::vector<int64_t> hcs(nchunks + 1);
    SA_CUDA_TRY(cudaMemcpyAsync(hcs.data(), cstart, (nchunks + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    int64_t maxrec = 0;
    for (int64_t k = 0; k < nchunks; ++k) maxrec = std::max(maxrec, hcs[k + 1] - hcs[k]);
    const int64_t stride = 2 + 5 * maxrec + (int64_t)C * (D + 1) * (D + 1) / 2 + 8;
    uint32_t *inv = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&inv, nr1 * sizeof(uint32_t), st));
    SA_LAUNCH(k_inverse, grid_for(nrec, 256), 256, 0, st, order, nrec, inv);
    uint32_t *fpos = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&fpos, nr1 * sizeof(uint32_t), st));
    SA_LAUNCH(k_chunk_order, grid_for(nchunks, 128), 128, 0, st, (const int64_t *)cstart, nchunks, order, rmeta, fpos);

    // templates, built and deduplicated in batches of chunks (bounded scratch)
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->ck_tm, nchunks * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->ck_pb, nchunks * sizeof(uint32_t), st));
    const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(nchunks, ((int64_t)1 << 29) / (stride * 4)));
    uint32_t *scratch = nullptr, *words = nullptr;
    uint64_t *sig = nullptr;
    SA_CUDA_TRY(cudaMallocAsync((void **)&scratch, batch * stride * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&words, batch * sizeof(uint32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&sig, batch * sizeof(uint64_t), st));
    std::unordered_map<uint64_t, uint32_t> ids;
    std::vector<uint32_t> tm_off_h;
    std::vector<uint32_t> tm_h;        // packed template words (host copy)
    std::vector<uint32_t> ctm(nchunks);
    std::vector<uint64_t> hs(batch);
    std::vector<uint32_t> hw(batch);
    bool ok = true;
    for (int64_t b0 = 0; b0 < nchunks && ok; b0 += batch) {
        const int64_t nb = std::min(batch, nchunks - b0);
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, sizeof(int64_t), st));
        SA_LAUNCH(k_chunk_build, grid_for(nb, 64), 64, 0, st, (const int64_t *)cstart, b0, nb, order, inv, skey, rp,
                  rmeta, rcoff, contrib, (const uint32_t *)fpos, stride, scratch, words, sig, P->ck_pb + b0,
                  (unsigned long long *)(P->counters + 6));
        int64_t fail = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(hs.data(), sig, nb * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaMemcpyAsync(hw.data(), words, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaMemcpyAsync(&fail, P->counters + 6, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        if (fail) { ok = false; break; }
        // new templates of this batch: copy their words back (small for structured meshes)
        std::vector<int64_t> fresh;
        for (int64_t i = 0; i < nb; ++i) {
            auto it = ids.find(hs[i]);
            if (it == ids.end()) {
                const uint32_t id = (uint32_t)tm_off_h.size();
                ids.emplace(hs[i], id);
                tm_off_h.push_back((uint32_t)tm_h.size());
                const size_t at = tm_h.size();
                tm_h.resize(at + hw[i]);
                SA_CUDA_TRY(cudaMemcpyAsync(tm_h.data() + at, scratch + i * stride, hw[i] * sizeof(uint32_t),
                                            cudaMemcpyDeviceToHost, st));
                ctm[b0 + i] = id;
            } else {
                ctm[b0 + i] = it->second;
            }
        }
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        // exact verification of this batch against the templates so far
        if (tm_h.size() >= ((size_t)1 << 31)) { ok = false; break; }
        uint32_t *dtm = nullptr, *doff = nullptr, *dctm = nullptr;
        SA_CUDA_TRY(cudaMallocAsync((void **)&dtm, std::max<size_t>(tm_h.size(), 1) * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&doff, tm_off_h.size() * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&dctm, nb * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMemcpyAsync(dtm, tm_h.data(), tm_h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        SA_CUDA_TRY(cudaMemcpyAsync(doff, tm_off_h.data(), tm_off_h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        SA_CUDA_TRY(cudaMemcpyAsync(dctm, ctm.data() + b0, nb * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, sizeof(int64_t), st));
        SA_LAUNCH(k_tile_verify, grid_for(nb * 32, 128), 128, 0, st, scratch, (int)stride, words, nb, dctm, doff, dtm,
                  (unsigned long long *)(P->counters + 6));
        int64_t bad = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&bad, P->counters + 6, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        SA_CUDA_TRY(cudaFreeAsync(dtm, st));
        SA_CUDA_TRY(cudaFreeAsync(doff, st));
        SA_CUDA_TRY(cudaFreeAsync(dctm, st));
        if (bad) ok = false;
    }
    if (ok) {
        for (size_t t = 0; t < tm_off_h.size(); ++t) {
            const size_t end = t + 1 < tm_off_h.size() ? tm_off_h[t + 1] : tm_h.size();
            P->ck_maxw = std::max<int64_t>(P->ck_maxw, (int64_t)(end - tm_off_h[t]));
        }
        tm_off_h.push_back((uint32_t)tm_h.size());   // sentinel: template t spans [off[t], off[t+1])
        P->ck_ntemplates = (int64_t)tm_off_h.size() - 1;
        P->ck_nwords = (int64_t)tm_h.size();
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->ck_tm_off, std::max<size_t>(tm_off_h.size(), 1) * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->ck_tmw, std::max<size_t>(tm_h.size(), 1) * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->ck_flags, (nrec + 1) * sizeof(unsigned), st));
        SA_CUDA_TRY(cudaMemsetAsync(P->ck_flags, 0, (nrec + 1) * sizeof(unsigned), st));
        std::vector<uint32_t> rs(nchunks);
        for (int64_t k = 0; k < nchunks; ++k) rs[k] = (uint32_t)hcs[k];
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->ck_rs, nchunks * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMemcpyAsync(P->ck_rs, rs.data(), nchunks * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        P->ck_nrec = nrec;
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        SA_CUDA_TRY(cudaMemcpyAsync(P->ck_tm_off, tm_off_h.data(), tm_off_h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        SA_CUDA_TRY(cudaMemcpyAsync(P->ck_tmw, tm_h.data(), tm_h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        SA_CUDA_TRY(cudaMemcpyAsync(P->ck_tm, ctm.data(), nchunks * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    }
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    for (void *p : {(void *)rcount, (void *)rstart, (void *)k0, (void *)k1, (void *)v0, (void *)v1, (void *)rp,
                    (void *)rmeta, (void *)rprev, (void *)rcoff, (void *)contrib, (void *)cstart, (void *)scratch,
                    (void *)words, (void *)sig, (void *)inv, (void *)fpos})
        SA_CUDA_TRY(cudaFreeAsync(p, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    P->ck_ok = ok;
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
    // fast path when every node fits the fused shared-memory node pass
    // (max incidences <= NS_CAPI, checked here; neighbours <= NS_CAPC,
    // checked by the pass itself), else the general kernels
    bool fast = false;
    const char *ns_s = getenv("SA_SYMFAST");
    // (default in 3D: measured warm C3 12.5 -> 9.9 ms, C5 65 -> 52 ms; in 2D
    // the general kernels are faster, C2 1.29 vs 1.71 ms)
    if (nn && (ns_s ? atoi(ns_s) != 0 : D == 3)) {
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, 2 * sizeof(int64_t), st));
        SA_LAUNCH(k_max_diff, std::min<int64_t>(grid_for(nn, 256), 148 * 8), 256, 0, st, P->inc_ptr, nn,
                  (unsigned long long *)(P->counters + 6));
        int64_t mi = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&mi, P->counters + 6, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        if (mi <= NS_CAPI) {
            SA_LAUNCH((k_node_symbolic<D, false>), grid_for(nn, NS_THREADS), NS_THREADS, 0, st, (const I *)M->me,
                      P->inc_ptr, P->inc, nn, cnt, (const int64_t *)nullptr, (int32_t *)nullptr,
                      (unsigned long long *)(P->counters + 7));
            int64_t ov = 0;
            SA_CUDA_TRY(cudaMemcpyAsync(&ov, P->counters + 7, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            SA_CUDA_TRY(cudaStreamSynchronize(st));
            fast = ov == 0;   // else (a node with > NS_CAPC neighbours): the general kernels below
        }
    }
    if (nn && !fast) {
        SA_LAUNCH(k_inc_sort, grid_for(nn, 128), 128, 0, st, P->inc_ptr, nn, P->inc);
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 5, 0, sizeof(int64_t), st));
        SA_LAUNCH(k_node_cols<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, cnt,
                  (const int64_t *)nullptr, (int32_t *)nullptr, (unsigned long long *)(P->counters + 5));
    }
    SA_TRY(exclusive_scan_i64(cnt, P->colptr, nn, P->scan_tmp, st));
    int64_t cap = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&P->n_colnodes, P->colptr + nn, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (!fast) SA_CUDA_TRY(cudaMemcpyAsync(&cap, P->counters + 5, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    if (cap) return set_error(SA_ERR_CAPACITY, "a node has more than %d distinct neighbours", MAXC);
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->cols, std::max<int64_t>(P->n_colnodes, 1) * sizeof(int32_t), st));
    if (nn && fast) {
        SA_LAUNCH((k_node_symbolic<D, true>), grid_for(nn, NS_THREADS), NS_THREADS, 0, st, (const I *)M->me,
                  P->inc_ptr, P->inc, nn, cnt, (const int64_t *)P->colptr, P->cols,
                  (unsigned long long *)(P->counters + 7));
    } else if (nn) {
        SA_LAUNCH(k_node_cols<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, cnt,
                  (const int64_t *)P->colptr, P->cols, (unsigned long long *)(P->counters + 5));
        SA_LAUNCH(k_inc_ranks<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, P->inc_ptr, P->inc, nn, P->colptr,
                  P->cols);
    }
    // max node degree: device reduction (no host copy of colptr)
    SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, sizeof(int64_t), st));
    if (nn)
        SA_LAUNCH(k_max_diff, std::min<int64_t>(grid_for(nn, 256), 148 * 8), 256, 0, st, P->colptr, nn,
                  (unsigned long long *)(P->counters + 6));
    int64_t md = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&md, P->counters + 6, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    P->max_deg = md;
    // warp-interleaved records for the row-gather kernel: on by default in 3D
    // (they replace three dependent gathers per incidence; measured faster),
    // off in 1D/2D (same speed there, 4x the record traffic); SA_WINC=0|1
    const char *wi_s = getenv("SA_WINC");
    // (the records carry the volume: without it yet -- a mesh created
    // without coordinates or volumes -- the plan uses the 8-byte records)
    const bool want_winc = (wi_s ? atoi(wi_s) != 0 : D == 3) && M->vols_ready;
    if (nn && want_winc) {
        const int64_t nw = (nn + 31) / 32;
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->wseg, (nw + 1) * sizeof(int64_t), st));
        SA_LAUNCH(k_warp_span, grid_for(nw, 128), 128, 0, st, P->inc_ptr, nn, cnt);
        SA_TRY(exclusive_scan_i64(cnt, P->wseg, nw, P->scan_tmp, st));
        SA_CUDA_TRY(cudaMemcpyAsync(&P->n_winc, P->wseg + nw, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->winc, std::max<int64_t>(P->n_winc, 1) * sizeof(IncRec), st));
        // padding records (rows shorter than their warp's longest) = all ones: ea = 0xffffffff sentinel
        SA_CUDA_TRY(cudaMemsetAsync(P->winc, 0xff, std::max<int64_t>(P->n_winc, 1) * sizeof(IncRec), st));
        SA_LAUNCH(k_winc_fill<D>, grid_for(nn, 128), 128, 0, st, (const I *)M->me, M->vols, P->inc_ptr, P->inc, nn,
                  P->wseg, P->winc);
    }
    // fold programs + templates: only for the tile / chunk kernels
    if (want_tile_kernel() || want_chunk_kernel()) {
        std::vector<int64_t> hcp(nn + 1), hip(nn + 1);
        SA_CUDA_TRY(cudaMemcpyAsync(hcp.data(), P->colptr, (nn + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaMemcpyAsync(hip.data(), P->inc_ptr, (nn + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->inc_e, std::max<int64_t>(P->n_inc, 1) * sizeof(uint32_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->fold, std::max<int64_t>((D + 1) * P->n_inc, 1) * sizeof(uint16_t), st));
        SA_CUDA_TRY(cudaMemsetAsync(P->counters + 6, 0, sizeof(int64_t), st));
        if (nn)
            SA_LAUNCH(k_fold_lists<D>, grid_for(nn, 128), 128, 0, st, P->inc_ptr, P->inc, nn, P->colptr, P->inc_e,
                      P->fold, (unsigned long long *)(P->counters + 6));
        int64_t too_many = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&too_many, P->counters + 6, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        P->fold_ok = (too_many == 0);
        for (int c = 0; c < 6; ++c) {
            const int64_t R = (int64_t)1 << c;
            int64_t mi = 0, mz = 0;
            for (int64_t r0 = 0; r0 < nn; r0 += R) {
                mi = std::max(mi, hip[std::min(nn, r0 + R)] - hip[r0]);
                mz = std::max(mz, hcp[std::min(nn, r0 + R)] - hcp[r0]);
            }
            P->tile_max_inc[c] = mi;
            P->tile_max_ent[c] = mz;
        }
        if (P->fold_ok && md <= 255 && nn && want_tile_kernel()) {
            SA_TRY(build_tile_templates<D>(P, 32 / tile_lanes(D, P->m), st));
        }
    }
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
    if (P->fold_ok && want_chunk_kernel()) SA_TRY(build_chunks<D>(P, st));
    return SA_OK;
}

// Kernel selection: the tile kernel whenever the plan has verified fold
// templates; SA_KERNEL=rowgather forces the v1 kernel (tests, comparison).
template <int D, int M, int OPS, int CORE>
int launch_rowgather(const NumArgs &a, int64_t nnodes, cudaStream_t st)
{
    constexpr int NOUT = n_outputs<OPS>();
    // SA_ILP (1|2|3): incidences in flight per thread (3 = software
    // pipeline); SA_MINB (0|3|6|8): minimum resident 128-thread blocks per SM
    // the single-incidence kernel is register-capped for (0 = no cap)
    const char *ilp_s = getenv("SA_ILP"), *mb_s = getenv("SA_MINB");
    // defaults measured on the BASELINE configs (profiles/r01): the kernel is
    // latency-bound, so occupancy wins over per-thread ILP except for the
    // register-heavy elastic operator, which gains from the pipeline
    const int ilp = ilp_s ? atoi(ilp_s) : (M > 1 ? 3 : 1);
    int minb = mb_s ? atoi(mb_s) : (M > 1 ? 0 : (OPS & OP_GENERAL) ? 3 : (D <= 2 ? 8 : 6));
    // (2D, more than one wave of 8 blocks/SM: 10 blocks/SM at 48 registers
    // beats 8 at 60 despite an 8-byte spill -- C2 0.299 -> 0.289 ms; a
    // single wave (C1) keeps 8)

    const size_t per_thread = (size_t)NOUT * (a.acc_stride | 1) * sizeof(double);
    int block = 128;
    while (per_thread * block > 100 * 1024 && block > 32) block /= 2;
    const size_t smem = per_thread * block;
    if (smem > 200 * 1024)
        return set_error(SA_ERR_CAPACITY, "row accumulators need %zu B of shared memory per %d threads", smem, block);
    void (*kern)(NumArgs);
    // lean instances (SA_LEAN=0 disables) when no diagnostics run and any mass
    // weight is constant
    const char *ln_s = getenv("SA_LEAN");
    const bool lean = (ln_s ? atoi(ln_s) != 0 : true) && a.dbg == 0 && !((OPS & OP_MASS) && a.w) &&
                      (a.winc != nullptr) == (D == 3);
    if (!mb_s && lean && D <= 2 && M == 1 && !(OPS & OP_GENERAL) && nnodes > (int64_t)148 * 8 * 128) minb = 10;
    if (ilp == 2) kern = k_numeric_rowgather<D, M, OPS, CORE, 2, 1>;
    else if (ilp == 3) kern = lean ? k_numeric_rowgather<D, M, OPS, CORE, 3, 1, false, true>
                                   : k_numeric_rowgather<D, M, OPS, CORE, 3, 1>;
    else if (minb == 8) kern = lean ? k_numeric_rowgather<D, M, OPS, CORE, 1, 8, false, true>
                                    : k_numeric_rowgather<D, M, OPS, CORE, 1, 8>;
    else if (minb == 6) kern = lean ? k_numeric_rowgather<D, M, OPS, CORE, 1, 6, false, true>
                                    : k_numeric_rowgather<D, M, OPS, CORE, 1, 6>;
    else if (minb == 7 && lean && M == 1) kern = k_numeric_rowgather<D, M, OPS, CORE, 1, 7, false, true>;
    else if (minb == 10 && lean && M == 1) kern = k_numeric_rowgather<D, M, OPS, CORE, 1, 10, false, true>;
    else if (minb == 12 && lean && M == 1) kern = k_numeric_rowgather<D, M, OPS, CORE, 1, 12, false, true>;
    else if (minb == 3) kern = lean ? k_numeric_rowgather<D, M, OPS, CORE, 1, 3, false, true>
                                    : k_numeric_rowgather<D, M, OPS, CORE, 1, 3>;
    else kern = lean ? k_numeric_rowgather<D, M, OPS, CORE, 1, 1, false, true>
                     : k_numeric_rowgather<D, M, OPS, CORE, 1, 1>;
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (nnodes) SA_LAUNCH(kern, grid_for(nnodes, block), block, smem, st, a);
    return SA_OK;
}

// returns SA_OK after launching, 1000 when the kernel's staging does not fit
#define SA_TRY_OR_FALL(...)                  \
    do {                                     \
        int _r = (__VA_ARGS__);              \
        if (_r == SA_OK) return SA_OK;       \
        if (_r != 1000) return _r;           \
    } while (0)

template <int D, int M, int OPS, int CORE, int L>
int launch_tiles(const sa_plan *P, const NumArgs &a, cudaStream_t st)
{
    constexpr int NOUT = n_outputs<OPS>();
    constexpr int VPI = NOUT * M * M * (D + 1);
    constexpr int R = 32 / L;
    constexpr int LOG2R = R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : R == 16 ? 4 : 5;
    TileArgs t;
    t.tile_e0 = P->tile_e0;
    t.tile_tm = P->tile_tm;
    t.tm_off = P->tm_off;
    t.tm = P->tm;
    t.max_inc = (int)P->tile_max_inc[LOG2R];
    t.max_ent = (int)P->tile_max_ent[LOG2R];
    const size_t warp_bytes =
        (size_t)NOUT * ((size_t)(D + 1) * t.max_inc * M * M + (M > 1 ? (size_t)M * M * t.max_ent : 0)) * 8;
    const size_t smem = 4 * warp_bytes;
    if (smem > 200 * 1024) return 1000;
    (void)VPI;
    auto kern = k_numeric_tiles<D, M, OPS, CORE, L>;
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (P->nnodes) SA_LAUNCH(kern, grid_for(P->nnodes, 4 * R), 128, smem, st, a, t);
    return SA_OK;
}

template <int D, int M, int OPS, int CORE>
int launch_chunks(const sa_plan *P, const NumArgs &a, cudaStream_t st)
{
    constexpr int NOUT = n_outputs<OPS>();
    constexpr int VPE = NOUT * M * M * (D + 1) * (D + 1);
    const size_t smem = (size_t)P->ck_C * VPE * sizeof(double) + (size_t)P->ck_maxw * sizeof(uint32_t);
    if (smem > 200 * 1024) return 1000;
    auto kern = k_numeric_chunks<D, M, OPS, CORE>;
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, nsm = 148, occ = 1;
    SA_CUDA_TRY(cudaGetDevice(&dev));
    SA_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int threads = std::max(64, std::min(256, P->ck_C));
    SA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    ChunkArgs c;
    c.chunk_tm = P->ck_tm;
    c.chunk_pb = P->ck_pb;
    c.tm_off = P->ck_tm_off;
    c.tm = P->ck_tmw;
    c.chunk_rs = P->ck_rs;
    c.rflags = P->ck_flags;
    c.ticket = P->ck_flags + P->ck_nrec;
    c.epoch = ++const_cast<sa_plan *>(P)->ck_epoch;
    c.nowait = getenv("SA_CHUNK_NOWAIT") != nullptr;
    c.max_words = (int)P->ck_maxw;
    c.nchunks = P->ck_nchunks;
    c.emin = P->ck_emin;
    c.emax = P->ck_emax;
    c.C = P->ck_C;
    SA_CUDA_TRY(cudaMemsetAsync(c.ticket, 0, sizeof(unsigned), st));
    const int64_t grid = std::min<int64_t>(P->ck_nchunks, (int64_t)nsm * std::max(occ, 1));
    if (grid > 0) SA_LAUNCH(kern, (unsigned)grid, threads, smem, st, a, c);
    return SA_OK;
}

// the fold of the overlapped two-pass (ILP 2, 128 threads)
template <int D, int M, int OPS, int CORE>
auto fold_kernel() -> void (*)(NumArgs)
{
    return k_numeric_rowgather<D, M, OPS, CORE, 2, 1, true>;
}
template <int OPS>
size_t fold_smem(const NumArgs &a)
{
    return (size_t)n_outputs<OPS>() * (a.acc_stride | 1) * sizeof(double) * 128;
}

template <int D, int M, int OPS, int CORE>
int launch_twopass(const sa_plan *P, const NumArgs &a, int64_t nnodes, cudaStream_t st)
{
    constexpr int NOUT = n_outputs<OPS>();
    // SA_EMINB (0|3|4): minimum resident 128-thread blocks per SM of the
    // element pass (register cap)
    const char *emb_s = getenv("SA_EMINB");
    // (measured on C5: no cap 210 registers 11.8 ms, 3 blocks 8.6 ms, 4 blocks 9.0 ms)
    const int eminb = emb_s ? atoi(emb_s) : 3;
    bool batched = false;
    if constexpr (OPS == OP_GENERAL && D == 3) {
        if (a.eb_loc && a.gen_packed) {
            // batched element pass (vertex records deduplicated per batch in smem)
            batched = true;
            const size_t smem = (size_t)std::max(a.eb_maxn, 1) * EB_REC * sizeof(double);
            // SA_EMINB for the batched pass: 3 | 4 (default) | 5 blocks per SM
            const int bm = emb_s ? atoi(emb_s) : 4;
            const char *pp_s = getenv("SA_EPIPE");
            const bool pipe = a.eb_allfit && (pp_s ? atoi(pp_s) != 0 : true);
            if (pipe) {
                // persistent, three-stage cp.async pipeline
                // (C5: 3 blocks/SM at 164 registers 6.73 ms, 4 at 128 + spill 6.79,
                // unpipelined batched 7.18)
                const int pm = pp_s && atoi(pp_s) > 1 ? atoi(pp_s) : 3;
                auto pk = pm == 3 ? k_element_rows_pipe<D, M, OPS, CORE, 3> : k_element_rows_pipe<D, M, OPS, CORE, 4>;
                const size_t psm = 2 * (size_t)std::max(a.eb_maxn, 1) * EB_REC * sizeof(double) +
                                   3 * (EB_CAP + 1) * sizeof(int);
                SA_CUDA_TRY(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
                int dev = 0, nsm = 148, occ = 0;
                SA_CUDA_TRY(cudaGetDevice(&dev));
                SA_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
                SA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pk, EB_SIZE, psm));
                const int64_t nb = (a.ne + EB_SIZE - 1) / EB_SIZE;
                const int K = (int)P->ov_bcut.size() - 1;
                if (K >= 1 && P->ov_stream) {
                    // element chunk k on st, then the fold of the rows whose
                    // elements are all in chunks <= k on the second stream:
                    // fold k (DRAM-bound) overlaps element chunk k+1 (fp64)
                    auto fk = fold_kernel<D, M, OPS, CORE>();
                    const size_t fsm = fold_smem<OPS>(a);
                    SA_CUDA_TRY(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
                    for (int k = 0; k < K; ++k) {
                        NumArgs ak = a;
                        ak.eb_b0 = P->ov_bcut[k];
                        ak.eb_b1 = P->ov_bcut[k + 1];
                        const unsigned g = (unsigned)std::min<int64_t>(std::max<int64_t>(ak.eb_b1 - ak.eb_b0, 1),
                                                                       (int64_t)nsm * std::max(occ, 1));
                        if (ak.eb_b1 > ak.eb_b0) SA_LAUNCH(pk, g, EB_SIZE, psm, st, ak);
                        SA_CUDA_TRY(cudaEventRecord(P->ov_events[k], st));
                        SA_CUDA_TRY(cudaStreamWaitEvent(P->ov_stream, P->ov_events[k], 0));
                        ak.row0 = 32 * P->ov_wcut[k];
                        ak.row1 = std::min<int64_t>(nnodes, 32 * P->ov_wcut[k + 1]);
                        if (ak.row1 > ak.row0)
                            SA_LAUNCH(fk, grid_for(ak.row1 - ak.row0, 128), 128, fsm, P->ov_stream, ak);
                    }
                    SA_CUDA_TRY(cudaEventRecord(P->ov_events[K], P->ov_stream));
                    SA_CUDA_TRY(cudaStreamWaitEvent(st, P->ov_events[K], 0));
                    return SA_OK;
                }
                const unsigned g = (unsigned)std::min<int64_t>(nb, (int64_t)nsm * std::max(occ, 1));
                if (a.ne) SA_LAUNCH(pk, g, EB_SIZE, psm, st, a);
            } else {
                auto kern = bm == 3 ? k_element_rows_batched<D, M, OPS, CORE, 3>
                            : bm == 5 ? k_element_rows_batched<D, M, OPS, CORE, 5>
                            : a.eb_allfit ? k_element_rows_batched<D, M, OPS, CORE, 4, true>
                                          : k_element_rows_batched<D, M, OPS, CORE, 4>;
                SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                if (a.ne) SA_LAUNCH(kern, grid_for(a.ne, EB_SIZE), EB_SIZE, smem, st, a);
            }
        }
    }
    if (batched) {
    } else if (a.ne) {
        if (eminb == 4) SA_LAUNCH((k_element_rows<D, M, OPS, CORE, 4>), grid_for(a.ne, 128), 128, 0, st, a);
        else if (eminb == 3) SA_LAUNCH((k_element_rows<D, M, OPS, CORE, 3>), grid_for(a.ne, 128), 128, 0, st, a);
        else SA_LAUNCH((k_element_rows<D, M, OPS, CORE, 1>), grid_for(a.ne, 128), 128, 0, st, a);
    }
    const char *ilp_s = getenv("SA_ILP");
    const int ilp = ilp_s ? atoi(ilp_s) : 2;
    const size_t per_thread = (size_t)NOUT * (a.acc_stride | 1) * sizeof(double);
    int block = 128;
    while (per_thread * block > 100 * 1024 && block > 32) block /= 2;
    const size_t smem = per_thread * block;
    if (smem > 200 * 1024)
        return set_error(SA_ERR_CAPACITY, "row accumulators need %zu B of shared memory per %d threads", smem, block);
    void (*kern)(NumArgs);
    if (ilp >= 4) kern = k_numeric_rowgather<D, M, OPS, CORE, 4, 1, true>;
    else if (ilp == 2 || ilp == 3) kern = k_numeric_rowgather<D, M, OPS, CORE, 2, 1, true>;
    else kern = k_numeric_rowgather<D, M, OPS, CORE, 1, 1, true>;
    SA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (nnodes) SA_LAUNCH(kern, grid_for(nnodes, block), block, smem, st, a);
    return SA_OK;
}

template <int D, int M, int OPS, int CORE>
int launch_numeric(const sa_plan *P, const NumArgs &a, cudaStream_t st)
{
    if (a.kbuf) return launch_twopass<D, M, OPS, CORE>(P, a, P->nnodes, st);
    if (P->ck_ok && want_chunk_kernel()) SA_TRY_OR_FALL(launch_chunks<D, M, OPS, CORE>(P, a, st));

    const int64_t nnodes = P->nnodes;
    const bool use_tile = P->tm_ok && want_tile_kernel();
    if (use_tile) {
        switch (32 / P->tile_rows) {
            case 1: SA_TRY_OR_FALL(launch_tiles<D, M, OPS, CORE, 1>(P, a, st)); break;
            case 2: SA_TRY_OR_FALL(launch_tiles<D, M, OPS, CORE, 2>(P, a, st)); break;
            case 4: SA_TRY_OR_FALL(launch_tiles<D, M, OPS, CORE, 4>(P, a, st)); break;
            case 8: SA_TRY_OR_FALL(launch_tiles<D, M, OPS, CORE, 8>(P, a, st)); break;
            case 16: SA_TRY_OR_FALL(launch_tiles<D, M, OPS, CORE, 16>(P, a, st)); break;
            default: break;
        }
    }
    return launch_rowgather<D, M, OPS, CORE>(a, nnodes, st);
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
int sa_mesh_kernels_d1(sa_mesh *, const double *, const int64_t *, const double *, cudaStream_t);
int sa_mesh_kernels_d2(sa_mesh *, const double *, const int64_t *, const double *, cudaStream_t);
int sa_mesh_kernels_d3(sa_mesh *, const double *, const int64_t *, const double *, cudaStream_t);
int sa_mesh_coords_d1(sa_mesh *, const double *, const double *, cudaStream_t);
int sa_mesh_coords_d2(sa_mesh *, const double *, const double *, cudaStream_t);
int sa_mesh_coords_d3(sa_mesh *, const double *, const double *, cudaStream_t);
int sa_symbolic_d1(sa_plan *, cudaStream_t);
int sa_symbolic_d2(sa_plan *, cudaStream_t);
int sa_symbolic_d3(sa_plan *, cudaStream_t);
int sa_dispatch_d1(const sa_plan *, const NumArgs &, int, int, cudaStream_t);
int sa_dispatch_d2(const sa_plan *, const NumArgs &, int, int, cudaStream_t);
int sa_dispatch_d3(const sa_plan *, const NumArgs &, int, int, cudaStream_t);
#ifdef SA_D
int SA_CAT(sa_mesh_kernels_d, SA_D)(sa_mesh *M, const double *q, const int64_t *me, const double *vols, cudaStream_t st)
{
    return mesh_kernels<SA_D>(M, q, me, vols, st);
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
    if (d == 1) rc = sa_mesh_kernels_d1(M, q_dev, me_dev, vols_dev, st);
    else if (d == 2) rc = sa_mesh_kernels_d2(M, q_dev, me_dev, vols_dev, st);
    else rc = sa_mesh_kernels_d3(M, q_dev, me_dev, vols_dev, st);
    if (rc != SA_OK) return fail(rc);
    *out = M;
    return SA_OK;
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
    if (P->ov_stream) {
        cudaStreamSynchronize(P->ov_stream);
        cudaStreamDestroy(P->ov_stream);
    }
    for (auto ev : P->ov_events) cudaEventDestroy(ev);
    free_all({P->inc_ptr, P->inc, P->winc, P->wseg, P->colptr, P->cols, P->indptr, P->indices, P->counters, P->scan_tmp, P->inc_e,
              P->fold, P->tile_e0, P->tile_tm, P->tm_off, P->tm, P->ck_tm, P->ck_pb, P->ck_tm_off, P->ck_tmw,
              P->ck_flags, P->ck_rs, P->epos, P->kbuf, P->tp_rank, P->eb_verts,
              P->eb_count, P->eb_loc});
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
    const int64_t v[12] = {P->n_templates, P->tm_ok ? 1 : 0, P->fold_ok ? 1 : 0, P->n_inc,
                           P->tm_nwords, P->max_deg, P->nnodes, P->nnz,
                           P->ck_ok ? 1 : 0, P->ck_nchunks, P->ck_ntemplates, P->ck_nwords};
    for (int i = 0; i < n && i < 12; ++i) out[i] = v[i];
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

// two-pass numeric ("element rows"): SA_KERNEL=twopass|rowgather forces it
// on/off; by default it serves the operators where it measured faster
static bool want_twopass(int ops, int d, int m)
{
    const char *k = getenv("SA_KERNEL");
    if (k && *k) return strcmp(k, "twopass") == 0;
    (void)m;
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
        SA_CUDA_TRY(cudaMemcpyAsync(h, dr, sizeof h, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
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
        SA_CUDA_TRY(cudaMemcpyAsync(&P->tp_nslots, P->wseg + nw, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
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
        SA_CUDA_TRY(cudaMemcpyAsync(&h, mx, sizeof h, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        SA_CUDA_TRY(cudaFreeAsync(mx, st));
        P->eb_maxn = (int)std::min<unsigned long long>(h, EB_CAP);
        P->eb_allfit = h <= EB_CAP;
        // overlap chunks (opt-in SA_OVERLAP = K): batch cuts, and per chunk
        // the warps whose rows' largest element lies before the chunk's end.
        // Off by default: measured C5 9.03 ms without, 9.07 / 9.12 / 9.22 ms
        // with K = 2 / 4 / 8 -- the element pass holds the whole register
        // file (3 x 128 threads x 164), so fold blocks cannot co-reside
        const char *ov_s = getenv("SA_OVERLAP");
        const int K = ov_s ? atoi(ov_s) : 0;
        const int64_t nn = P->nnodes, nw = (nn + 31) / 32;
        if (K >= 2 && P->eb_allfit && nb >= 4 * K && nw > 0) {
            unsigned *wm = nullptr;
            SA_CUDA_TRY(cudaMallocAsync((void **)&wm, nw * sizeof(unsigned), st));
            SA_LAUNCH(k_warp_emax, grid_for(nw, 128), 128, 0, st, P->inc_ptr, P->inc, nn, wm);
            std::vector<unsigned> hw(nw);
            SA_CUDA_TRY(cudaMemcpyAsync(hw.data(), wm, nw * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
            SA_CUDA_TRY(cudaStreamSynchronize(st));
            SA_CUDA_TRY(cudaFreeAsync(wm, st));
            P->ov_bcut.assign(K + 1, 0);
            P->ov_wcut.assign(K + 1, 0);
            for (int k = 0; k <= K; ++k) P->ov_bcut[k] = nb * k / K;
            unsigned pm = 0;
            int64_t w = 0;
            for (int k = 0; k < K; ++k) {
                const int64_t e_end = P->e_lo + std::min<int64_t>(P->ov_bcut[k + 1] * EB_SIZE, ne);
                while (w < nw && (int64_t)std::max(pm, hw[w]) < e_end) pm = std::max(pm, hw[w++]);
                P->ov_wcut[k + 1] = k + 1 == K ? nw : w;
            }
            SA_CUDA_TRY(cudaStreamCreateWithFlags(&P->ov_stream, cudaStreamNonBlocking));
            P->ov_events.resize(K + 1);
            for (auto &ev : P->ov_events) SA_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
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

static bool want_batches(int ops, int d)
{
    const char *eb_s = getenv("SA_EBATCH");
    return ops == SA_OP_GENERAL && d == 3 && (eb_s ? atoi(eb_s) != 0 : true);
}

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
    a.qv = M->qv; a.me = M->me; a.vols = M->vols;
    a.nnodes = P->nnodes; a.node_begin = P->node_begin;
    a.inc_ptr = P->inc_ptr; a.inc = P->inc; a.winc = P->winc; a.wseg = P->wseg; a.colptr = P->colptr; a.indptr = P->indptr; a.cols = P->cols;
    a.dbg = getenv("SA_DBG") ? atoi(getenv("SA_DBG")) : 0;
    a.row0 = 0;
    a.row1 = P->nnodes;
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
    a.A = cf->A; a.b = cf->b; a.c = cf->c; a.a0 = cf->a0; a.gen_packed = cf->gen_packed;
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
        SA_CUDA_TRY(cudaMemcpyAsync(h, P->counters, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        if (h[7]) return set_error(SA_ERR_CUDA, "chunk kernel: a carry wait timed out (internal error)");
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

#include "sa_pk.cuh"
#endif  // SA_ABI
