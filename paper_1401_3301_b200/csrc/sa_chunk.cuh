// sa_chunk.cuh -- element-chunk numeric kernel ("carry" kernel), included by
// sa_core.cu inside its anonymous namespace.
//
// Every element is computed exactly once, by the CTA that owns its chunk of
// C consecutive element ids (coalesced connectivity/volume loads, vertex
// gathers local in the mesh).  Each CSR entry's contributions are summed
// left to right in ascending element index, exactly as the reference's
// optv2 does (sparse.py:97-106): a chunk continues the partial sums left in
// the output array by the previous chunk that touched the entry ("carry"),
// after waiting for that record's flag (per record, so waits chain only
// along one entry's few chunks); chunks are taken in ascending order through
// a ticket counter (decoupled look-back style), so every wait is on an older
// chunk and cannot deadlock.  Flags hold the launch epoch: no reset pass.
//
// Symbolic data (built once per plan):
//   records  one per (entry, chunk) pair with contributions: dof position of
//            the entry's (l=0, n=0) value, first/last flags, dof row stride,
//            chunk delta to the entry's previous record, its contributions
//            (local element | alpha << 8 | beta << 10, ascending element);
//   grouped by chunk with the stable radix sort, serialised into chunk
//   templates (deduplicated by signature, verified word for word):
//     w[0] = nrec, w[1] = 0
//     w[2 .. 2+nrec)           word offset of each record
//     record: [rel dof position] [nc | first<<8 | last<<9 | stride<<16]
//             [pred: chunk delta << 16 | record index in that chunk] (if !first)
//             [contribs, 2 per word]
//   per chunk: template id, dof position base, first record index.
#pragma once

constexpr int CHUNK_MAX_PRED = 255;

inline int chunk_elems(int d, int m)
{
    const char *v = getenv("SA_CHUNK");
    if (v && atoi(v) > 0 && atoi(v) <= 256) return atoi(v);
    if (m > 1) return d == 2 ? 128 : 32;
    return d == 2 ? 256 : 128;
}

template <int D>
__global__ void k_inc_minmax(const uint32_t *__restrict__ inc_e, int64_t n, unsigned *__restrict__ mm)
{
    unsigned lo = 0xffffffffu, hi = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned e = inc_e[i] & 0x3fffffffu;
        lo = min(lo, e);
        hi = max(hi, e);
    }
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
}

// records per node row (pass 1 counts, pass 2 writes); contributions of row
// slot s live at (d+1)*inc_ptr[row] + s (one per fold slot)
template <int D>
__global__ void k_chunk_records(const int64_t *__restrict__ inc_ptr, const uint32_t *__restrict__ inc_e,
                                const uint16_t *__restrict__ fold, const int64_t *__restrict__ colptr,
                                const int64_t *__restrict__ indptr, int64_t nnodes, int m, unsigned emin, int C,
                                int64_t *__restrict__ rcount, const int64_t *__restrict__ rstart,
                                uint64_t *__restrict__ key, uint32_t *__restrict__ val, uint32_t *__restrict__ rp,
                                uint32_t *__restrict__ rmeta, uint32_t *__restrict__ rprev,
                                uint32_t *__restrict__ rcoff, uint16_t *__restrict__ contrib)
{
    const int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl >= nnodes) return;
    const int64_t t0 = inc_ptr[nl];
    const int deg = (int)(colptr[nl + 1] - colptr[nl]);
    const uint16_t *f = fold + (int64_t)(D + 1) * t0;
    const int64_t dof0 = indptr[(int64_t)m * nl];
    const uint32_t stride = (uint32_t)(m * deg);
    int64_t w = rcount ? 0 : rstart[nl];
    int s = 0;
    for (int k = 0; k < deg; ++k) {
        int prev_chunk = -1;
        int64_t cur = -1;          // record being filled
        int cur_chunk = -1;
        while (true) {
            const uint16_t x = f[s];
            const uint32_t r = inc_e[t0 + (x & 63)];
            const unsigned e = r & 0x3fffffffu;
            const int ch = (int)((e - emin) / (unsigned)C);
            if (ch != cur_chunk) {
                // close the previous record of this entry, open a new one
                if (cur >= 0 && !rcount) rmeta[cur] &= ~(1u << 9);
                prev_chunk = cur_chunk;
                cur_chunk = ch;
                if (!rcount) {
                    cur = w;
                    key[w] = (uint64_t)ch;
                    val[w] = (uint32_t)w;
                    rp[w] = (uint32_t)(dof0 + (int64_t)k * m);
                    rmeta[w] = (prev_chunk < 0 ? (1u << 8) : 0u) | (1u << 9) | (stride << 16);
                    rprev[w] = prev_chunk < 0 ? 0u : (uint32_t)(ch - prev_chunk);
                    rcoff[w] = (uint32_t)((int64_t)(D + 1) * t0 + s);
                } else {
                    cur = w;
                }
                ++w;
            }
            if (!rcount) {
                const unsigned local = e - emin - (unsigned)ch * (unsigned)C;
                const unsigned alpha = r >> 30, beta = (x >> 6) & 3;
                contrib[(int64_t)(D + 1) * t0 + s] = (uint16_t)(local | (alpha << 8) | (beta << 10));
                rmeta[cur] += 1;     // nc
            }
            const bool last = x & 256;
            ++s;
            if (last) break;
        }
    }
    if (rcount) rcount[nl] = w;
}

// chunk boundaries in the sorted record order
__global__ void k_chunk_bounds(const uint64_t *__restrict__ skey, int64_t n, int64_t nchunks,
                               int64_t *__restrict__ cstart)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t c = (int64_t)skey[i];
    const int64_t prev = i ? (int64_t)skey[i - 1] : -1;
    for (int64_t x = prev + 1; x <= c; ++x) cstart[x] = i;
    if (i == n - 1)
        for (int64_t x = c + 1; x <= nchunks; ++x) cstart[x] = n;
}

// inverse permutation of the sort: generation index -> sorted position
__global__ void k_inverse(const uint32_t *__restrict__ order, int64_t n, uint32_t *__restrict__ inv)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) inv[order[i]] = (uint32_t)i;
}

// in-chunk record order: records that feed a later chunk (not last) first, so
// the successor's waits resolve at the start of this chunk's phase C instead
// of its end (which would chain chunk after chunk into a wavefront)
__global__ void k_chunk_order(const int64_t *__restrict__ cstart, int64_t nchunks, const uint32_t *__restrict__ order,
                              const uint32_t *__restrict__ rmeta, uint32_t *__restrict__ fpos)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nchunks) return;
    uint32_t j = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (int64_t i = cstart[k]; i < cstart[k + 1]; ++i) {
            const bool last = rmeta[order[i]] & (1u << 9);
            if (last == (pass == 1)) fpos[i] = j++;
        }
}

__global__ void k_chunk_build(const int64_t *__restrict__ cstart, int64_t k0, int64_t nchunks,
                              const uint32_t *__restrict__ order, const uint32_t *__restrict__ inv,
                              const uint64_t *__restrict__ skey, const uint32_t *__restrict__ rp,
                              const uint32_t *__restrict__ rmeta, const uint32_t *__restrict__ rcoff,
                              const uint16_t *__restrict__ contrib, const uint32_t *__restrict__ fpos,
                              int64_t stride, uint32_t *__restrict__ scratch,
                              uint32_t *__restrict__ words_out, uint64_t *__restrict__ sig,
                              uint32_t *__restrict__ chunk_pb, unsigned long long *fail)
{
    const int64_t kl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (kl >= nchunks) return;
    const int64_t k = k0 + kl;
    const int64_t r0 = cstart[k], r1 = cstart[k + 1];
    const int nrec = (int)(r1 - r0);
    uint32_t *w = scratch + kl * stride;
    if (nrec >= (1 << 16)) { atomicOr(fail, 1ull); words_out[kl] = 0; chunk_pb[kl] = 0; return; }
    const uint32_t pb = nrec ? rp[order[r0]] : 0u;
    chunk_pb[kl] = pb;
    w[0] = (uint32_t)nrec;
    w[1] = 0;
    uint32_t pos = 2 + nrec;
    bool bad = false;
    for (int64_t i = r0; i < r1; ++i) {
        const uint32_t g = order[i];
        const uint32_t meta = rmeta[g];
        const int nc = meta & 0xff;
        const uint32_t j = fpos[i];
        w[2 + j] = pos;
        w[pos] = rp[g] - pb;
        w[pos + 1] = meta;
        pos += 2;
        if (!(meta & (1u << 8))) {
            // predecessor = the previous record of the same entry (generation g-1)
            const uint32_t ip = inv[g - 1];
            const int64_t kp = (int64_t)skey[ip];
            const int64_t d = k - kp, jp = fpos[ip];
            if (d <= 0 || d >= (1 << 16) || jp >= (1 << 16)) bad = true;
            w[pos++] = (uint32_t)(d << 16) | (uint32_t)jp;
        }
        for (int c = 0; c < nc; c += 2) {
            const uint32_t lo = contrib[rcoff[g] + c];
            const uint32_t hi = c + 1 < nc ? contrib[rcoff[g] + c + 1] : 0u;
            w[pos + (c >> 1)] = lo | (hi << 16);
        }
        pos += (nc + 1) >> 1;
    }
    if (bad) { atomicOr(fail, 1ull); words_out[kl] = 0; return; }
    words_out[kl] = pos;
    uint64_t h = 1469598103934665603ull;
    for (uint32_t x = 0; x < pos; ++x) h = fnv_step(h, w[x]);
    sig[kl] = h;
}

// ---------------------------------------------------------------------------
// numeric kernel

struct ChunkArgs {
    const uint32_t *chunk_tm;    // (nchunks) template id
    const uint32_t *chunk_pb;    // (nchunks) dof position base
    const uint32_t *tm_off;      // template word offsets
    const uint32_t *tm;          // template words
    const uint32_t *chunk_rs;    // (nchunks) first record index of each chunk
    unsigned *rflags;            // (nrec) per-record carry flags (launch epoch)
    unsigned *ticket;            // ticket counter (zeroed per launch)
    unsigned epoch;              // this launch's flag value
    int nowait;                  // diagnostics only (SA_CHUNK_NOWAIT): skip carry waits, results invalid
    int max_words;               // largest template (shared-memory copy per chunk)
    int64_t nchunks;
    unsigned emin;               // first element of chunk 0
    unsigned emax;               // last element touching the plan
    int C;                       // elements per chunk
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// element lane: every local row of the element into the staging area
template <int D, int M, int OPS, int A = 0>
__device__ __forceinline__ void element_all_rows(const NumArgs &a, const ElemGeo<D> &g, double *dst)
{
    constexpr int VPR = n_outputs<OPS>() * M * M * (D + 1);   // values per local row
    element_krow<D, M, OPS, A>(a, g, dst + A * VPR);
    if constexpr (A < D) element_all_rows<D, M, OPS, A + 1>(a, g, dst);
}

template <int D, int M, int OPS, int CORE>
__global__ void __launch_bounds__(256) k_numeric_chunks(NumArgs a, ChunkArgs c)
{
    constexpr int NOUT = n_outputs<OPS>();
    constexpr int MM = M * M;
    constexpr int VPR = NOUT * MM * (D + 1);    // staged values per local row
    constexpr int VPE = VPR * (D + 1);          // per element
    extern __shared__ __align__(16) double staged[];
    uint32_t *tms = reinterpret_cast<uint32_t *>(staged + (size_t)c.C * VPE);   // template copy
    __shared__ int64_t s_k;
    int nz[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) nz[o] = 0;
    int64_t emin_deg = INT64_MAX;
    while (true) {
        if (threadIdx.x == 0) s_k = (int64_t)atomicAdd(c.ticket, 1u);
        __syncthreads();
        const int64_t k = s_k;
        if (k >= c.nchunks) break;
        const int64_t e0 = (int64_t)c.emin + k * c.C;
        const int ne = (int)min((int64_t)c.C, (int64_t)c.emax + 1 - e0);

        // phase A: every element of the chunk once, two per thread in flight
        for (int j = threadIdx.x; j < ne; j += 2 * blockDim.x) {
            const int j2 = j + blockDim.x;
            const bool two = j2 < ne;
            ElemRaw<D> x1, x2;
            element_load1<D, OPS>(a, e0 + j, x1);
            element_load1<D, OPS>(a, two ? e0 + j2 : e0 + j, x2);
            element_load2<D, OPS>(a, x1);
            element_load2<D, OPS>(a, x2);
            ElemGeo<D> g;
            if (element_compute<D, OPS, CORE>(x1, g)) emin_deg = min(emin_deg, e0 + j);
            element_all_rows<D, M, OPS>(a, g, staged + (size_t)j * VPE);
            if (two) {
                if (element_compute<D, OPS, CORE>(x2, g)) emin_deg = min(emin_deg, e0 + j2);
                element_all_rows<D, M, OPS>(a, g, staged + (size_t)j2 * VPE);
            }
        }
        // the chunk's template -> shared memory (coalesced; records are then
        // read with LDS instead of scattered global loads)
        const unsigned to = __ldg(c.tm_off + __ldg(c.chunk_tm + k));
        const int nw = (int)(__ldg(c.tm_off + __ldg(c.chunk_tm + k) + 1) - to);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) tms[i] = __ldg(c.tm + to + i);
        const int64_t pb = __ldg(c.chunk_pb + k);
        const unsigned rs = __ldg(c.chunk_rs + k);
        __syncthreads();   // staged rows and template complete
        const int nrec = tms[0] & 0xffffff;

        // phase C: continue each touched entry's left-to-right sum
        for (int r = threadIdx.x; r < nrec; r += blockDim.x) {
            unsigned ro = tms[2 + r];
            const int64_t p = pb + (int64_t)tms[ro];
            const unsigned meta = tms[ro + 1];
            ro += 2;
            const int nc = meta & 0xff;
            const bool first = meta & (1u << 8), last = meta & (1u << 9);
            const int stride = meta >> 16;
            double acc[NOUT][MM];
            if (first) {
#pragma unroll
                for (int o = 0; o < NOUT; ++o)
#pragma unroll
                    for (int x = 0; x < MM; ++x) acc[o][x] = 0.0;
            } else {
                const unsigned pw = tms[ro++];
                const int64_t kp = k - (int64_t)(pw >> 16);
                const unsigned *fl = c.rflags + __ldg(c.chunk_rs + kp) + (pw & 0xffff);
                // bounded spin on the predecessor record's flag
                unsigned spins = 0;
                while (!c.nowait && ld_acquire(fl) != c.epoch) {
                    if (++spins > (1u << 22) || *(volatile int64_t *)(a.counters + 7)) {
                        atomicOr((unsigned long long *)(a.counters + 7), 1ull);
                        break;
                    }
                    __nanosleep(32);
                }
#pragma unroll
                for (int o = 0; o < NOUT; ++o)
#pragma unroll
                    for (int l = 0; l < M; ++l)
#pragma unroll
                        for (int n = 0; n < M; ++n) acc[o][l * M + n] = __ldcg(a.vals[o] + p + (int64_t)l * stride + n);
            }
            for (int i = 0; i < nc; ++i) {
                const unsigned cw = (tms[ro + (i >> 1)] >> (16 * (i & 1))) & 0xffff;
                const double *src = staged + (size_t)(cw & 0xff) * VPE + ((cw >> 8) & 3) * VPR +
                                    ((cw >> 10) & 3) * (NOUT * MM);
#pragma unroll
                for (int o = 0; o < NOUT; ++o)
#pragma unroll
                    for (int x = 0; x < MM; ++x) acc[o][x] = SA_ADD(acc[o][x], src[o * MM + x]);
            }
#pragma unroll
            for (int o = 0; o < NOUT; ++o)
#pragma unroll
                for (int l = 0; l < M; ++l)
#pragma unroll
                    for (int n = 0; n < M; ++n) {
                        const double v = acc[o][l * M + n];
                        __stcg(a.vals[o] + p + (int64_t)l * stride + n, v);
                        if (last) nz[o] += (v == 0.0);
                    }
            if (!last) st_release(c.rflags + rs + r, c.epoch);
        }
        __syncthreads();   // staging area reused by the next chunk
    }
    if (emin_deg != INT64_MAX) atomicMin((unsigned long long *)(a.counters + 4), (unsigned long long)emin_deg);
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
        int v = nz[o];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd((unsigned long long *)(a.counters + o), (unsigned long long)v);
    }
}
