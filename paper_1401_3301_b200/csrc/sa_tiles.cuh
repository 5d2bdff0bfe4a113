// sa_tiles.cuh -- plan-time construction of the tiled two-pass schedule
// (3D general operator; included by sa_core.cu in the C-ABI translation unit).
//
// The two-pass numeric phase writes one 32-byte local row per incidence and
// reads it back in the fold: 2 x 12.9 GB of DRAM traffic on C5 against 5.8 GB
// of algorithmic bytes.  Here the rows of the block are grouped into spatial
// TILES whose local rows fit the L2 (126 MB on B200).  Per tile the element
// pass computes every element touching the tile's rows (elements on a tile
// face are computed once per tile they touch: a halo of ~10 % for bricks of
// ~35^3 nodes) and stores the local rows of the tile's own rows into a ring
// buffer that every tile reuses; the tile's fold reads them back while they
// are still in L2.  Neither the values nor the fold order change, so the
// result is bitwise that of the untiled two-pass (and of the row gather).
//
// A tile is a run of WARPS (32 consecutive node rows, the unit the fold's
// warp-interleaved slots and coalesced CSR stores are built on) in brick
// order: warps are keyed by the brick of a uniform grid that holds their
// centroid, stably sorted by key (1-bit split passes on the existing scan),
// and runs of whole bricks are packed greedily up to the slot budget (a brick
// above the budget is split).  Meshes whose numbering has no locality give
// tiles with large halos; the caller keeps the untiled path when the
// recomputation factor exceeds 1.6.
#pragma once

namespace {


__device__ __forceinline__ unsigned long long ordered_bits(double x)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
inline double from_ordered_bits(unsigned long long u)
{
    const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    double x;
    memcpy(&x, &b, sizeof x);
    return x;
}

// bounding box of the block's nodes: out[0..2] = min, out[3..5] = max (ordered bits)
__global__ void k_tile_bbox(const double4 *__restrict__ qv, int64_t node_begin, int64_t nn, unsigned long long *out)
{
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
        const double4 c = qv[node_begin + i];
        const unsigned long long k[3] = {ordered_bits(c.x), ordered_bits(c.y), ordered_bits(c.z)};
#pragma unroll
        for (int j = 0; j < 3; ++j) { lo[j] = min(lo[j], k[j]); hi[j] = max(hi[j], k[j]); }
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        for (int s = 16; s > 0; s >>= 1) {
            lo[j] = min(lo[j], __shfl_xor_sync(0xffffffffu, lo[j], s));
            hi[j] = max(hi[j], __shfl_xor_sync(0xffffffffu, hi[j], s));
        }
        if ((threadIdx.x & 31) == 0) { atomicMin(out + j, lo[j]); atomicMax(out + 3 + j, hi[j]); }
    }
}

// brick key of each warp (centroid of its node rows), identity permutation
__global__ void k_tile_keys(const double4 *__restrict__ qv, int64_t node_begin, int64_t nn, int64_t nw, double lx,
                            double ly, double lz, double ihx, double ihy, double ihz, int nbx, int nby, int nbz,
                            uint32_t *__restrict__ key, uint32_t *__restrict__ idx)
{
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w >= nw) return;
    const int64_t r0 = 32 * w, r1 = min(r0 + 32, nn);
    double sx = 0, sy = 0, sz = 0;
    for (int64_t r = r0; r < r1; ++r) {
        const double4 c = qv[node_begin + r];
        sx += c.x; sy += c.y; sz += c.z;
    }
    const double inv = 1.0 / (double)(r1 - r0);
    const int bx = min(max((int)((sx * inv - lx) * ihx), 0), nbx - 1);
    const int by = min(max((int)((sy * inv - ly) * ihy), 0), nby - 1);
    const int bz = min(max((int)((sz * inv - lz) * ihz), 0), nbz - 1);
    key[w] = (uint32_t)((bx * nby + by) * nbz + bz);
    idx[w] = (uint32_t)w;
}

// stable split on one key bit: zeros first
__global__ void k_split_flag(const uint32_t *__restrict__ key, int64_t n, int bit, int64_t *__restrict__ flag)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = ((key[i] >> bit) & 1u) ? 0 : 1;
}
__global__ void k_split_scatter(const uint32_t *__restrict__ key, const uint32_t *__restrict__ idx, int64_t n, int bit,
                                const int64_t *__restrict__ pos0, uint32_t *__restrict__ key_out,
                                uint32_t *__restrict__ idx_out)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = key[i];
    const int64_t z = pos0[i];
    const int64_t dst = ((k >> bit) & 1u) ? pos0[n] + (i - z) : z;
    key_out[dst] = k;
    idx_out[dst] = idx[i];
}

// span of the warp at each sorted position
__global__ void k_tile_gather_span(const int64_t *__restrict__ span, const uint32_t *__restrict__ order, int64_t nw,
                                   int64_t *__restrict__ out)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < nw) out[p] = span[order[p]];
}

// per warp (natural index): its tile and its virtual slot offset
__global__ void k_tile_warp_maps(const uint32_t *__restrict__ order, const int64_t *__restrict__ vseg, int64_t nw,
                                 const int64_t *__restrict__ tile_w0, int nt, int32_t *__restrict__ wtile,
                                 int64_t *__restrict__ wvseg)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= nw) return;
    int lo = 0, hi = nt;   // last t with tile_w0[t] <= p
    while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (tile_w0[mid] <= p) lo = mid; else hi = mid; }
    const uint32_t w = order[p];
    wtile[w] = lo;
    wvseg[w] = vseg[p];
}

// tile-relative slot of every (element, alpha) of the block, column ranks in
// virtual slot order (the tiled counterpart of k_tp_slots)
__global__ void k_tile_slots(const int64_t *__restrict__ inc_ptr, const uint2 *__restrict__ inc, int64_t nnodes,
                             const int32_t *__restrict__ wtile, const int64_t *__restrict__ wvseg,
                             const int64_t *__restrict__ tbase, unsigned e_lo, unsigned *__restrict__ epos,
                             unsigned *__restrict__ rank)
{
    const int64_t nl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (nl >= nnodes) return;
    const int64_t w = nl >> 5;
    const int64_t vbase = wvseg[w] + (nl & 31);
    const int64_t rel = vbase - tbase[wtile[w]];
    const int64_t t0 = inc_ptr[nl], n = inc_ptr[nl + 1] - t0;
    for (int64_t k = 0; k < n; ++k) {
        const uint2 rec = inc[t0 + k];
        epos[(int64_t)((rec.x & 0x3fffffffu) - e_lo) * 4 + (rec.x >> 30)] = (unsigned)(rel + 32 * k);
        rank[vbase + 32 * k] = rec.y;
    }
}

// An element is listed once per tile it touches, by its first vertex (lowest
// alpha) whose row lies in that tile.  Virtual row vr = 32 p + lane.
__device__ __forceinline__ bool tile_owner(const int4 v, int alpha, int t, int64_t nb0, int64_t nb1,
                                           const int32_t *__restrict__ wtile)
{
    const int vv[4] = {v.x, v.y, v.z, v.w};
    for (int b = 0; b < alpha; ++b)
        if (vv[b] >= nb0 && vv[b] < nb1 && wtile[(vv[b] - nb0) >> 5] == t) return false;
    return true;
}

__global__ void k_tile_count(const int4 *__restrict__ me, const int64_t *__restrict__ inc_ptr,
                             const uint2 *__restrict__ inc, int64_t nnodes, int64_t nb0, const uint32_t *__restrict__ order,
                             int64_t nw, const int32_t *__restrict__ wtile, int64_t *__restrict__ cnt)
{
    const int64_t vr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (vr >= 32 * nw) return;
    const int64_t w = order[vr >> 5], nl = 32 * w + (vr & 31);
    int64_t c = 0;
    if (nl < nnodes) {
        const int t = wtile[w];
        for (int64_t k = inc_ptr[nl]; k < inc_ptr[nl + 1]; ++k) {
            const unsigned x = inc[k].x;
            c += tile_owner(__ldg(me + (x & 0x3fffffffu)), (int)(x >> 30), t, nb0, nb0 + nnodes, wtile);
        }
    }
    cnt[vr] = c;
}

__global__ void k_tile_pick(const int64_t *__restrict__ vpre, const int64_t *__restrict__ tile_w0, int nt,
                            int64_t *__restrict__ out)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t <= nt) out[t] = vpre[32 * tile_w0[t]];
}

__global__ void k_tile_fill(const int4 *__restrict__ me, const int64_t *__restrict__ inc_ptr,
                            const uint2 *__restrict__ inc, int64_t nnodes, int64_t nb0, const uint32_t *__restrict__ order,
                            int64_t nw, const int32_t *__restrict__ wtile, const int64_t *__restrict__ vpre,
                            const int64_t *__restrict__ tshift, unsigned e_lo, const unsigned *__restrict__ epos,
                            int32_t *__restrict__ tv_elem, uint4 *__restrict__ tv_pos)
{
    const int64_t vr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (vr >= 32 * nw) return;
    const int64_t w = order[vr >> 5], nl = 32 * w + (vr & 31);
    if (nl >= nnodes) return;
    const int t = wtile[w];
    const int64_t nb1 = nb0 + nnodes;
    int64_t i = vpre[vr] + tshift[t];
    for (int64_t k = inc_ptr[nl]; k < inc_ptr[nl + 1]; ++k) {
        const unsigned x = inc[k].x;
        const unsigned e = x & 0x3fffffffu;
        const int4 v = __ldg(me + e);
        if (!tile_owner(v, (int)(x >> 30), t, nb0, nb1, wtile)) continue;
        const int vv[4] = {v.x, v.y, v.z, v.w};
        unsigned p[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const bool in = vv[b] >= nb0 && vv[b] < nb1 && wtile[(vv[b] - nb0) >> 5] == t;
            p[b] = in ? epos[(int64_t)(e - e_lo) * 4 + b] : 0xffffffffu;
        }
        tv_elem[i] = (int32_t)e;
        tv_pos[i] = make_uint4(p[0], p[1], p[2], p[3]);
        ++i;
    }
}

struct TmpBufs {   // stream-ordered temporaries, freed on every exit path
    cudaStream_t st;
    std::vector<void *> ps;
    explicit TmpBufs(cudaStream_t s) : st(s) {}
    template <typename T>
    cudaError_t get(T **p, int64_t n)
    {
        cudaError_t e = cudaMallocAsync((void **)p, (size_t)std::max<int64_t>(n, 1) * sizeof(T), st);
        if (e == cudaSuccess) ps.push_back(*p);
        return e;
    }
    ~TmpBufs()
    {
        for (void *p : ps)
            if (p) cudaFreeAsync(p, st);
    }
};

// Build the tiled schedule of plan P (3D, coordinates set, e_lo / e_hi and
// the natural-order warp spans `span` known).  On success P->tiled is set
// and P->tp_rank (virtual slot order), tv_elem / tv_pos, the element batches
// over the virtual list and the ring buffer size (tile_max_slots) are in
// place; P->tiled stays false (nothing kept) when tiling does not pay.
int build_tiles(sa_plan *P, const int64_t *span, int64_t slot_budget, cudaStream_t st)
{
    const sa_mesh *M = P->mesh;
    const int64_t nn = P->nnodes, nw = (nn + 31) / 32;
    const int64_t ne = P->e_hi - P->e_lo;
    if (!nn || !ne || !M->coords || M->d != 3) return SA_OK;
    P->tile_tried = true;
    const double4 *qv = (const double4 *)M->qv;
    const int4 *me = (const int4 *)M->me;
    TmpBufs tmp(st);
    const int B = 256;

    // --- brick grid from the bounding box and the slot budget
    unsigned long long *dbox = nullptr, hbox[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
    SA_CUDA_TRY(tmp.get(&dbox, 6));
    SA_CUDA_TRY(cudaMemcpyAsync(dbox, hbox, sizeof hbox, cudaMemcpyHostToDevice, st));
    SA_LAUNCH(k_tile_bbox, std::min<int64_t>(grid_for(nn, B), 148 * 8), B, 0, st, qv, P->node_begin, nn, dbox);
    int64_t total_slots = 0;
    int64_t *vseg_nat = nullptr;   // natural-order scan only to get the total
    SA_CUDA_TRY(tmp.get(&vseg_nat, nw + 1));
    SA_TRY(exclusive_scan_i64(span, vseg_nat, nw, P->scan_tmp, st));
    SA_CUDA_TRY(cudaMemcpyAsync(&total_slots, vseg_nat + nw, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaMemcpyAsync(hbox, dbox, sizeof hbox, cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    if (total_slots <= slot_budget || total_slots >= 0xffffffffLL * 32) return SA_OK;   // one tile: nothing to gain
    double lo[3], ext[3];
    for (int j = 0; j < 3; ++j) {
        lo[j] = from_ordered_bits(hbox[j]);
        ext[j] = from_ordered_bits(hbox[3 + j]) - lo[j];
        if (!(ext[j] > 0)) ext[j] = 0;
    }
    // bricks of ~0.8 budgets, cubic in the box's metric
    const double nbricks = std::max(1.0, (double)total_slots / (0.8 * (double)slot_budget));
    double vol = 1.0;
    int ndim = 0;
    for (int j = 0; j < 3; ++j)
        if (ext[j] > 0) { vol *= ext[j]; ++ndim; }
    if (!ndim) return SA_OK;
    const double h = std::pow(vol / nbricks, 1.0 / ndim);
    int nb[3];
    double ih[3];
    for (int j = 0; j < 3; ++j) {
        nb[j] = ext[j] > 0 ? (int)std::min(1024.0, std::max(1.0, std::ceil(ext[j] / h - 1e-9))) : 1;
        ih[j] = ext[j] > 0 ? nb[j] / ext[j] : 0.0;
    }
    const int64_t nkeys = (int64_t)nb[0] * nb[1] * nb[2];
    int nbits = 0;
    while (((int64_t)1 << nbits) < nkeys) ++nbits;

    // --- warps sorted by brick key (stable)
    uint32_t *key[2] = {nullptr, nullptr}, *idx[2] = {nullptr, nullptr};
    int64_t *flag = nullptr;
    SA_CUDA_TRY(tmp.get(&key[0], nw));
    SA_CUDA_TRY(tmp.get(&key[1], nw));
    SA_CUDA_TRY(tmp.get(&idx[1], nw));
    SA_CUDA_TRY(tmp.get(&flag, nw + 1));
    SA_CUDA_TRY(cudaMallocAsync((void **)&idx[0], nw * sizeof(uint32_t), st));   // becomes P->tw_order (either buffer)
    tmp.ps.push_back(idx[0]);
    SA_LAUNCH(k_tile_keys, grid_for(nw, B), B, 0, st, qv, P->node_begin, nn, nw, lo[0], lo[1], lo[2], ih[0], ih[1], ih[2],
              nb[0], nb[1], nb[2], key[0], idx[0]);
    int cur = 0;
    for (int bit = 0; bit < nbits; ++bit) {
        SA_LAUNCH(k_split_flag, grid_for(nw, B), B, 0, st, key[cur], nw, bit, flag);
        SA_TRY(exclusive_scan_i64(flag, flag, nw, P->scan_tmp, st));
        SA_LAUNCH(k_split_scatter, grid_for(nw, B), B, 0, st, key[cur], idx[cur], nw, bit, flag, key[cur ^ 1],
                  idx[cur ^ 1]);
        cur ^= 1;
    }
    uint32_t *order = idx[cur];

    // --- tiles: whole bricks packed up to the budget, oversized bricks split
    int64_t *sspan = nullptr, *vseg = nullptr;
    SA_CUDA_TRY(tmp.get(&sspan, nw + 1));
    SA_CUDA_TRY(cudaMallocAsync((void **)&vseg, (nw + 1) * sizeof(int64_t), st));
    tmp.ps.push_back(vseg);
    SA_LAUNCH(k_tile_gather_span, grid_for(nw, B), B, 0, st, span, order, nw, sspan);
    std::vector<uint32_t> hkey(nw);
    std::vector<int64_t> hspan(nw);
    SA_CUDA_TRY(cudaMemcpyAsync(hkey.data(), key[cur], nw * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaMemcpyAsync(hspan.data(), sspan, nw * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_TRY(exclusive_scan_i64(sspan, vseg, nw, P->scan_tmp, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<int64_t> w0;   // tile starts (sorted positions)
    {
        int64_t cur_slots = 0;
        w0.push_back(0);
        int64_t p = 0;
        while (p < nw) {
            int64_t q = p, bs = 0;   // brick run [p, q), its slots
            while (q < nw && hkey[q] == hkey[p]) bs += hspan[q++];
            if (bs > slot_budget) {
                if (cur_slots > 0) { w0.push_back(p); cur_slots = 0; }
                for (int64_t r = p; r < q; ++r) {
                    if (cur_slots > 0 && cur_slots + hspan[r] > slot_budget) { w0.push_back(r); cur_slots = 0; }
                    cur_slots += hspan[r];
                }
            } else {
                if (cur_slots > 0 && cur_slots + bs > slot_budget) { w0.push_back(p); cur_slots = 0; }
                cur_slots += bs;
            }
            p = q;
        }
        w0.push_back(nw);
    }
    const int nt = (int)w0.size() - 1;
    if (nt < 2) return SA_OK;
    int64_t max_slots = 0;
    {
        std::vector<int64_t> pre(nw + 1, 0);
        for (int64_t p = 0; p < nw; ++p) pre[p + 1] = pre[p] + hspan[p];
        for (int t = 0; t < nt; ++t) max_slots = std::max(max_slots, pre[w0[t + 1]] - pre[w0[t]]);
        if (max_slots >= 0xffffffffLL) return SA_OK;
    }

    // --- per-warp maps, virtual element counts per tile
    int64_t *d_w0 = nullptr, *tbase = nullptr, *wvseg = nullptr, *cnt = nullptr, *tpre = nullptr, *tshift = nullptr;
    int32_t *wtile = nullptr;
    SA_CUDA_TRY(tmp.get(&d_w0, nt + 1));
    SA_CUDA_TRY(tmp.get(&tbase, nt + 1));
    SA_CUDA_TRY(tmp.get(&wvseg, nw));
    SA_CUDA_TRY(tmp.get(&wtile, nw));
    SA_CUDA_TRY(tmp.get(&cnt, 32 * nw + 1));
    SA_CUDA_TRY(tmp.get(&tpre, nt + 1));
    SA_CUDA_TRY(tmp.get(&tshift, nt + 1));
    SA_CUDA_TRY(cudaMemcpyAsync(d_w0, w0.data(), (nt + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    SA_LAUNCH(k_tile_warp_maps, grid_for(nw, B), B, 0, st, order, vseg, nw, d_w0, nt, wtile, wvseg);
    SA_LAUNCH(k_tile_count, grid_for(32 * nw, B), B, 0, st, me, P->inc_ptr, P->inc, nn, P->node_begin, order, nw, wtile,
              cnt);
    // (the scan scratch of the plan is sized for nn + 1 entries; 32 nw + 1 <= nn + 32)
    int64_t *scan_tmp = nullptr;
    SA_CUDA_TRY(tmp.get(&scan_tmp, scan_tmp_elems(32 * nw + 1) + 1));
    SA_TRY(exclusive_scan_i64(cnt, cnt, 32 * nw, scan_tmp, st));
    SA_LAUNCH(k_tile_pick, grid_for(nt + 1, B), B, 0, st, cnt, d_w0, nt, tpre);
    std::vector<int64_t> hpre(nt + 1), v0(nt + 1), hshift(nt + 1, 0), hbase(nt + 1);
    SA_CUDA_TRY(cudaMemcpyAsync(hpre.data(), tpre, (nt + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    v0[0] = 0;
    for (int t = 0; t < nt; ++t) {
        const int64_t c = hpre[t + 1] - hpre[t];
        hshift[t] = v0[t] - hpre[t];
        v0[t + 1] = v0[t] + (c + EB_SIZE - 1) / EB_SIZE * EB_SIZE;
    }
    const int64_t nv = v0[nt];
    // halos too large (SA_TUNE tile_maxf, percent: tests force tiny tiles)
    if ((double)hpre[nt] > 0.01 * tune_int("tile_maxf", 160) * (double)ne || nv >= 0x7fffffffLL) return SA_OK;
    {
        std::vector<int64_t> pre(nw + 1, 0);
        for (int64_t p = 0; p < nw; ++p) pre[p + 1] = pre[p] + hspan[p];
        for (int t = 0; t <= nt; ++t) hbase[t] = pre[w0[t]];
    }
    SA_CUDA_TRY(cudaMemcpyAsync(tshift, hshift.data(), (nt + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    SA_CUDA_TRY(cudaMemcpyAsync(tbase, hbase.data(), (nt + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));

    // --- slots, virtual element lists, element batches
    unsigned *epos_t = nullptr;
    SA_CUDA_TRY(tmp.get(&epos_t, 4 * ne));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->tp_rank, std::max<int64_t>(total_slots, 1) * sizeof(unsigned), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->tv_elem, std::max<int64_t>(nv, 1) * sizeof(int32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->tv_pos, std::max<int64_t>(nv, 1) * sizeof(uint4), st));
    SA_CUDA_TRY(cudaMemsetAsync(P->tv_elem, 0xff, std::max<int64_t>(nv, 1) * sizeof(int32_t), st));
    SA_CUDA_TRY(cudaMemsetAsync(P->tv_pos, 0xff, std::max<int64_t>(nv, 1) * sizeof(uint4), st));
    SA_LAUNCH(k_tile_slots, grid_for(nn, 128), 128, 0, st, P->inc_ptr, P->inc, nn, wtile, wvseg, tbase, (unsigned)P->e_lo,
              epos_t, P->tp_rank);
    SA_LAUNCH(k_tile_fill, grid_for(32 * nw, B), B, 0, st, me, P->inc_ptr, P->inc, nn, P->node_begin, order, nw, wtile, cnt,
              tshift, (unsigned)P->e_lo, epos_t, P->tv_elem, P->tv_pos);
    const int64_t nbat = nv / EB_SIZE;
    unsigned long long *mx = nullptr;
    SA_CUDA_TRY(tmp.get(&mx, 1));
    SA_CUDA_TRY(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->eb_verts, std::max<int64_t>(nbat * EB_CAP, 1) * sizeof(int32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->eb_count, std::max<int64_t>(nbat, 1) * sizeof(int32_t), st));
    SA_CUDA_TRY(cudaMallocAsync((void **)&P->eb_loc, std::max<int64_t>(nv, 1) * sizeof(uint32_t), st));
    if (nbat)
        SA_LAUNCH(k_eb_build<3>, (unsigned)nbat, EB_SIZE, 0, st, me, (int64_t)0, nv, P->eb_verts, P->eb_count, P->eb_loc,
                  mx, (const int32_t *)P->tv_elem);
    unsigned long long hmx = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&hmx, mx, sizeof hmx, cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    if (hmx > (unsigned long long)EB_CAP) {
        // a batch with too many distinct vertices: the untiled path (with its
        // direct-gather fallback) serves this plan
        for (void *p : {(void *)P->tp_rank, (void *)P->tv_elem, (void *)P->tv_pos, (void *)P->eb_verts,
                        (void *)P->eb_count, (void *)P->eb_loc})
            cudaFreeAsync(p, st);
        P->tp_rank = nullptr; P->tv_elem = nullptr; P->tv_pos = nullptr;
        P->eb_verts = nullptr; P->eb_count = nullptr; P->eb_loc = nullptr;
        return SA_OK;
    }
    P->eb_maxn = (int)hmx;
    P->eb_allfit = true;
    {   // per-tile prefix arrays of the fused kernel: batches, sorted warps, fold chunks
        std::vector<int64_t> hd(3 * (nt + 1));
        for (int t = 0; t <= nt; ++t) {
            hd[t] = v0[t] / EB_SIZE;
            hd[(nt + 1) + t] = w0[t];
        }
        hd[2 * (nt + 1)] = 0;
        for (int t = 0; t < nt; ++t)
            hd[2 * (nt + 1) + t + 1] = hd[2 * (nt + 1) + t] + (w0[t + 1] - w0[t] + TILE_FCH - 1) / TILE_FCH;
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->tile_dev, hd.size() * sizeof(int64_t), st));
        SA_CUDA_TRY(cudaMallocAsync((void **)&P->tile_sync, 2 * (size_t)nt * sizeof(unsigned), st));
        SA_CUDA_TRY(cudaMemcpyAsync(P->tile_dev, hd.data(), hd.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
    }
    // keep: order, vseg (taken out of the temporaries)
    for (void *&p : tmp.ps)
        if (p == (void *)order || p == (void *)vseg) p = nullptr;
    P->tw_order = order;
    P->tw_vseg = vseg;
    P->tile_w0 = w0;
    P->tile_v0 = v0;
    P->nt = nt;
    P->nv = nv;
    P->tile_max_slots = max_slots;
    P->tp_nslots = total_slots;
    P->tiled = true;
    return SA_OK;
}

}  // namespace
