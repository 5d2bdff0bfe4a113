// sa_meshgen.cu -- the benchmark meshes generated on the device, bitwise the
// host generator's arrays (the host build of C3/C5 takes
// tens of seconds, more than the assembly).
//
//   * Kuhn triangulation of [0,1]^d (mesh.py:104-140): q = grid / float(n),
//     grid points in row-major order (first coordinate slowest); d! simplices
//     per cell, one per axis permutation in itertools.permutations order, the
//     simplices of a cell adjacent; vertex j+1 = vertex j + stride[perm[j]].
//   * Seeded interior jitter: numpy's
//     default_rng(seed).uniform(lo, hi, size=(d, n_interior)) added to the
//     interior nodes.  numpy's PCG64 (128-bit LCG, XSL-RR output; the
//     generator state after SeedSequence seeding is passed in) is restated
//     with LCG jump-ahead, so each thread starts at its own draw; a draw is
//     lo + (hi - lo) * ((x >> 11) * 2^-53), added as q + v.
#include <cuda_runtime.h>
#include <cstdint>

#include "sa_common.cuh"

using namespace sa;

namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult()
{
    return ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
}

__device__ __forceinline__ uint64_t pcg_output(u128 s)
{
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned r = (unsigned)(s >> 122);
    return (x >> r) | (x << ((64u - r) & 63u));
}

// state after `delta` LCG steps (O(log delta) 128-bit products)
__device__ u128 pcg_advance(u128 state, uint64_t delta, u128 inc)
{
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

__global__ void k_kuhn_q(int d, int64_t n, int64_t nq, double *__restrict__ q)
{
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= nq) return;
    int64_t r = v;
    for (int a = d - 1; a >= 0; --a) {
        q[a * nq + v] = __ddiv_rn((double)(r % (n + 1)), (double)n);
        r /= n + 1;
    }
}

constexpr int JIT_CHUNK = 64;   // consecutive draws per thread

__global__ void k_kuhn_jitter(int d, int64_t n, int64_t nq, int64_t nint, int64_t ndraw, double lo, double range,
                              uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, double *__restrict__ q)
{
    const int64_t k0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * JIT_CHUNK;
    if (k0 >= ndraw) return;
    const u128 inc = ((u128)i_hi << 64) | i_lo;
    u128 s = pcg_advance(((u128)s_hi << 64) | s_lo, (uint64_t)k0, inc);
    const int64_t k1 = min(k0 + JIT_CHUNK, ndraw);
    for (int64_t k = k0; k < k1; ++k) {
        s = s * pcg_mult() + inc;   // numpy steps, then outputs the new state
        const double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
        const double val = __dadd_rn(lo, __dmul_rn(range, u));
        const int a = (int)(k / nint);
        int64_t j = k - a * nint, node = 0, w = 1;
        for (int b = d - 1; b >= 0; --b) {   // interior index -> node (row-major)
            node += (1 + j % (n - 1)) * w;
            j /= n - 1;
            w *= n + 1;
        }
        q[a * nq + node] = __dadd_rn(q[a * nq + node], val);
    }
}

__constant__ int c_perm[6][3];

__global__ void k_kuhn_me(int d, int dfact, int64_t n, int64_t nme, int64_t *__restrict__ me)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= nme) return;
    const int64_t cell = e / dfact;
    const int p = (int)(e - cell * dfact);
    int64_t stride[3], base = 0, r = cell, s = 1;
    for (int a = d - 1; a >= 0; --a) {
        stride[a] = s;
        base += (r % n) * s;
        r /= n;
        s *= n + 1;
    }
    int64_t v = base;
    me[e] = v;
    for (int j = 0; j < d; ++j) {
        v += stride[c_perm[p][j]];
        me[(int64_t)(j + 1) * nme + e] = v;
    }
}

// A node window [v0, v0 + nv) with its jitter (each interior node's d
// draws by jump-ahead: draw k = axis * n_interior + interior index) and an
// element window [e0, e0 + ne) with node ids relative to v0: a rank's slab
// without the global mesh.
__global__ void k_kuhn_q_range(int d, int64_t n, int64_t v0, int64_t nv, int64_t nint, int jitter, double lo,
                               double range, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                               double *__restrict__ q)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nv) return;
    const int64_t v = v0 + t;
    int64_t idx[3], r = v;
    bool interior = true;
    for (int a = d - 1; a >= 0; --a) {
        idx[a] = r % (n + 1);
        r /= n + 1;
        interior &= idx[a] >= 1 && idx[a] <= n - 1;
    }
    int64_t j = 0;
    for (int a = 0; a < d; ++a) j = j * (n - 1) + (idx[a] - 1);
    const u128 s0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)i_hi << 64) | i_lo;
    for (int a = 0; a < d; ++a) {
        double x = __ddiv_rn((double)idx[a], (double)n);
        if (jitter && interior) {
            const u128 s = pcg_advance(s0, (uint64_t)(a * nint + j) + 1, inc);
            const double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
            x = __dadd_rn(x, __dadd_rn(lo, __dmul_rn(range, u)));
        }
        q[a * nv + t] = x;
    }
}

__global__ void k_kuhn_me_range(int d, int dfact, int64_t n, int64_t e0, int64_t ne, int64_t v0,
                                int64_t *__restrict__ me)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= ne) return;
    const int64_t e = e0 + t;
    const int64_t cell = e / dfact;
    const int p = (int)(e - cell * dfact);
    int64_t stride[3], base = 0, r = cell, s = 1;
    for (int a = d - 1; a >= 0; --a) {
        stride[a] = s;
        base += (r % n) * s;
        r /= n;
        s *= n + 1;
    }
    int64_t v = base;
    me[t] = v - v0;
    for (int j = 0; j < d; ++j) {
        v += stride[c_perm[p][j]];
        me[(int64_t)(j + 1) * ne + t] = v - v0;
    }
}

}  // namespace

static void kuhn_perms(int d, int (&perm)[6][3])
{
    int cur[3] = {0, 1, 2}, k = 0, dfact = 1;
    for (int a = 2; a <= d; ++a) dfact *= a;
    do {
        for (int j = 0; j < d; ++j) perm[k][j] = cur[j];
        ++k;
        int i = d - 2;
        while (i >= 0 && cur[i] > cur[i + 1]) --i;
        if (i < 0) break;
        int j = d - 1;
        while (cur[j] < cur[i]) --j;
        int t = cur[i]; cur[i] = cur[j]; cur[j] = t;
        for (int a = i + 1, b = d - 1; a < b; ++a, --b) { t = cur[a]; cur[a] = cur[b]; cur[b] = t; }
    } while (k < dfact);
}

extern "C" int sa_kuhn_slab(int d, int64_t n, int jitter, double lo, double range, uint64_t state_hi,
                            uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t v0, int64_t v1, int64_t e0,
                            int64_t e1, double *q_dev, int64_t *me_dev, void *stream)
{
    if (d < 1 || d > 3) return set_error(SA_ERR_ARG, "dimension must be 1, 2 or 3, got %d", d);
    if (n < 1) return set_error(SA_ERR_ARG, "subdivision count must be >= 1, got %lld", (long long)n);
    cudaStream_t st = (cudaStream_t)stream;
    int64_t nq = 1, ncell = 1, nint = 1;
    int dfact = 1;
    for (int a = 0; a < d; ++a) { nq *= n + 1; ncell *= n; nint *= n - 1; dfact *= a + 1; }
    if (v0 < 0 || v1 > nq || v0 > v1 || e0 < 0 || e1 > ncell * dfact || e0 > e1)
        return set_error(SA_ERR_ARG, "slab window out of range");
    int perm[6][3] = {{0}};
    kuhn_perms(d, perm);
    SA_CUDA_TRY(cudaMemcpyToSymbolAsync(c_perm, perm, sizeof perm, 0, cudaMemcpyHostToDevice, st));
    if (q_dev && v1 > v0)
        SA_LAUNCH(k_kuhn_q_range, grid_for(v1 - v0, 128), 128, 0, st, d, n, v0, v1 - v0, nint, jitter && n >= 2, lo,
                  range, state_hi, state_lo, inc_hi, inc_lo, q_dev);
    if (me_dev && e1 > e0)
        SA_LAUNCH(k_kuhn_me_range, grid_for(e1 - e0, 256), 256, 0, st, d, dfact, n, e0, e1 - e0, v0, me_dev);
    return SA_OK;
}

extern "C" int sa_kuhn_mesh(int d, int64_t n, int jitter, double lo, double range, uint64_t state_hi,
                            uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, double *q_dev, int64_t *me_dev,
                            void *stream)
{
    if (d < 1 || d > 3) return set_error(SA_ERR_ARG, "dimension must be 1, 2 or 3, got %d", d);
    if (n < 1) return set_error(SA_ERR_ARG, "subdivision count must be >= 1, got %lld", (long long)n);
    cudaStream_t st = (cudaStream_t)stream;
    int64_t nq = 1, ncell = 1, nint = 1;
    int dfact = 1;
    for (int a = 0; a < d; ++a) { nq *= n + 1; ncell *= n; nint *= n - 1; dfact *= a + 1; }
    const int64_t nme = ncell * dfact;
    // itertools.permutations(range(d)) order (lexicographic)
    int perm[6][3] = {{0}};
    {
        int cur[3] = {0, 1, 2}, k = 0;
        do {
            for (int j = 0; j < d; ++j) perm[k][j] = cur[j];
            ++k;
            // next lexicographic permutation of cur[0..d)
            int i = d - 2;
            while (i >= 0 && cur[i] > cur[i + 1]) --i;
            if (i < 0) break;
            int j = d - 1;
            while (cur[j] < cur[i]) --j;
            int t = cur[i]; cur[i] = cur[j]; cur[j] = t;
            for (int a = i + 1, b = d - 1; a < b; ++a, --b) { t = cur[a]; cur[a] = cur[b]; cur[b] = t; }
        } while (k < dfact);
    }
    SA_CUDA_TRY(cudaMemcpyToSymbolAsync(c_perm, perm, sizeof perm, 0, cudaMemcpyHostToDevice, st));
    if (q_dev && nq) SA_LAUNCH(k_kuhn_q, grid_for(nq, 256), 256, 0, st, d, n, nq, q_dev);
    if (q_dev && jitter && n >= 2) {
        const int64_t ndraw = (int64_t)d * nint;
        SA_LAUNCH(k_kuhn_jitter, grid_for((ndraw + JIT_CHUNK - 1) / JIT_CHUNK, 128), 128, 0, st, d, n, nq, nint,
                  ndraw, lo, range, state_hi, state_lo, inc_hi, inc_lo, q_dev);
    }
    if (me_dev && nme) SA_LAUNCH(k_kuhn_me, grid_for(nme, 256), 256, 0, st, d, dfact, n, nme, me_dev);
    return SA_OK;
}
