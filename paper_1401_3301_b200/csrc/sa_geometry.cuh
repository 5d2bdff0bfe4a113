// sa_geometry.cuh -- per-simplex geometry (K1) and local element rows (K2).
//
// Bit-exact restatement on sm_100a of:
//   compute_gradients   kernels.py:49-65   -> numpy.linalg.solve(B^T, [-1|I])
//                                             = OpenBLAS dgesv; operation order of
//                                             the SkylakeX / Haswell kernels
//
//   mass_kernel         kernels.py:68-78   (coef*vols) * ((wsum + W[a]) + W[b])
//   stiffness_kernel    kernels.py:81-88   ((G_b0*G_a0 + G_b1*G_a1) + ...) * vols
//   elastic_kernel      kernels.py:155-172 lambs*dot_mat_vec_g(Q) + mus*dot_mat_vec_g(S)
//   general operator
// Every multiply/add/fma is an explicit round-to-nearest intrinsic so that
// nvcc never contracts or reassociates them: the values are bitwise those of
// the reference, which is what makes the value-dependent CSR pattern exact.
#pragma once
#include <cstdint>

#define SA_MUL(a, b) __dmul_rn((a), (b))
#define SA_ADD(a, b) __dadd_rn((a), (b))
#define SA_SUB(a, b) __dsub_rn((a), (b))
#define SA_FMA(a, b, c) __fma_rn((a), (b), (c))
#define SA_RCP(a) __drcp_rn(a)

namespace sa {

enum { CORE_SKYLAKEX = 0, CORE_HASWELL = 1 };
enum { OP_MASS = 1, OP_STIFF = 2, OP_ELASTIC = 4, OP_GENERAL = 8 };

template <int D> struct VecT;
template <> struct VecT<1> { typedef double type; };
template <> struct VecT<2> { typedef double2 type; };
template <> struct VecT<3> { typedef double4 type; };
template <int D> struct IdxT;
template <> struct IdxT<1> { typedef int2 type; };
template <> struct IdxT<2> { typedef int4 type; };
template <> struct IdxT<3> { typedef int4 type; };

// One 32-byte read-only load (sm_100: LDG.E.ENL2.256): a whole sector per
// lane in a single request, half the L1 requests of two 16-byte loads.
__device__ __forceinline__ void ldg256(const void *p, double &a, double &b, double &c, double &d)
{
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// streaming (evict-first) 32-byte load: data read exactly once
__device__ __forceinline__ void ldg256_cs(const void *p, double &a, double &b, double &c, double &d)
{
    asm("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

template <int D>
__device__ __forceinline__ void load_vertex(const typename VecT<D>::type *__restrict__ qv, int v, double (&x)[D])
{
    if constexpr (D == 1) { x[0] = __ldg(qv + v); }
    else if constexpr (D == 2) { double2 t = __ldg(qv + v); x[0] = t.x; x[1] = t.y; }
    else {
        double pad;
        ldg256(qv + v, x[0], x[1], x[2], pad);
    }
}

template <int D>
__device__ __forceinline__ void load_element(const typename IdxT<D>::type *__restrict__ me, int64_t e, int (&v)[D + 1])
{
    typename IdxT<D>::type t = __ldg(me + e);
    v[0] = t.x; v[1] = t.y;
    if constexpr (D >= 2) v[2] = t.z;
    if constexpr (D >= 3) v[3] = t.w;
}

// s = fma(a, b, s) (SkylakeX dot kernels) or s + a*b (Haswell)
template <int CORE>
__device__ __forceinline__ double acc_step(double s, double a, double b)
{
    if constexpr (CORE == CORE_SKYLAKEX) return SA_FMA(a, b, s);
    else return SA_ADD(s, SA_MUL(a, b));
}

// Left-looking LU with partial pivoting (OpenBLAS getf2 structure).
// a: d x d row-major, in place.  perm[i] = source row of row i.
// rcp[j] = 1.0 / u_jj.  Returns true if some pivot is exactly zero.
template <int D, int CORE>
__device__ __forceinline__ bool lu_factor(double (&a)[D][D], int (&perm)[D], double (&rcp)[D])
{
#pragma unroll
    for (int i = 0; i < D; ++i) perm[i] = i;
    bool sing = false;
#pragma unroll
    for (int j = 0; j < D; ++j) {
#pragma unroll
        for (int i = 1; i < j; ++i) {
            double s = SA_MUL(a[i][0], a[0][j]);
#pragma unroll
            for (int k = 1; k < i; ++k) s = acc_step<CORE>(s, a[i][k], a[k][j]);
            a[i][j] = SA_SUB(a[i][j], s);
        }
        if (j > 0) {
#pragma unroll
            for (int i = j; i < D; ++i) {
                double s = SA_MUL(a[i][0], a[0][j]);
#pragma unroll
                for (int k = 1; k < j; ++k) s = acc_step<CORE>(s, a[i][k], a[k][j]);
                a[i][j] = SA_SUB(a[i][j], s);
            }
        }
        int p = j;
        double best = fabs(a[j][j]);
#pragma unroll
        for (int i = j + 1; i < D; ++i) {
            double v = fabs(a[i][j]);
            if (v > best) { best = v; p = i; }
        }
#pragma unroll
        for (int i = j + 1; i < D; ++i) {
            if (p == i) {
#pragma unroll
                for (int c = 0; c < D; ++c) { double t = a[j][c]; a[j][c] = a[i][c]; a[i][c] = t; }
                int t = perm[j]; perm[j] = perm[i]; perm[i] = t;
            }
        }
        sing |= (a[j][j] == 0.0);
        rcp[j] = SA_RCP(a[j][j]);
#pragma unroll
        for (int i = j + 1; i < D; ++i) a[i][j] = SA_MUL(a[i][j], rcp[j]);
    }
    return sing;
}

// getrs for the rhs [-1 | I_d]; G[alpha][nu] = X[nu][alpha] (kernels.py:64-65).
template <int D, int CORE>
__device__ __forceinline__ void solve_ref_gradients(const double (&a)[D][D], const int (&perm)[D],
                                                    const double (&rcp)[D], double (&G)[D + 1][D])
{
#pragma unroll
    for (int col = 0; col <= D; ++col) {
        double b[D];
#pragma unroll
        for (int i = 0; i < D; ++i) b[i] = (col == 0) ? -1.0 : (perm[i] == col - 1 ? 1.0 : 0.0);
        if constexpr (D == 1) {
            b[0] = SA_MUL(b[0], rcp[0]);
        } else if constexpr (D == 2) {
            const double l10 = a[1][0], u01 = a[0][1];
            if constexpr (CORE == CORE_SKYLAKEX) b[1] = SA_FMA(-l10, b[0], b[1]);
            else b[1] = SA_SUB(b[1], SA_MUL(l10, b[0]));
            b[1] = SA_MUL(b[1], rcp[1]);
            if constexpr (CORE == CORE_SKYLAKEX) b[0] = SA_FMA(-u01, b[1], b[0]);
            else b[0] = SA_SUB(b[0], SA_MUL(u01, b[1]));
            b[0] = SA_MUL(b[0], rcp[0]);
        } else {
            const double l10 = a[1][0], l20 = a[2][0], l21 = a[2][1];
            const double u01 = a[0][1], u02 = a[0][2], u12 = a[1][2];
            if constexpr (CORE == CORE_SKYLAKEX) b[1] = SA_FMA(-l10, b[0], b[1]);
            else b[1] = SA_SUB(b[1], SA_MUL(l10, b[0]));
            double acc = SA_MUL(l20, b[0]);
            acc = SA_FMA(l21, b[1], acc);
            b[2] = SA_SUB(b[2], acc);
            b[2] = SA_MUL(b[2], rcp[2]);
            b[0] = SA_SUB(b[0], SA_MUL(u02, b[2]));
            b[1] = SA_SUB(b[1], SA_MUL(u12, b[2]));
            b[1] = SA_MUL(b[1], rcp[1]);
            if constexpr (CORE == CORE_SKYLAKEX) b[0] = SA_FMA(-b[1], u01, b[0]);
            else b[0] = SA_SUB(b[0], SA_MUL(u01, b[1]));
            b[0] = SA_MUL(b[0], rcp[0]);
        }
#pragma unroll
        for (int nu = 0; nu < D; ++nu) G[col][nu] = b[nu];
    }
}

// Edge rows A[r][c] = x[r+1][c] - x[0][c]  (kernels.py:57, one subtraction).
template <int D>
__device__ __forceinline__ void edge_rows(const double (&x)[D + 1][D], double (&A)[D][D])
{
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) A[r][c] = SA_SUB(x[r + 1][c], x[0][c]);
}

// Full gradient computation; returns true if degenerate.
template <int D, int CORE>
__device__ __forceinline__ bool element_gradients(const double (&x)[D + 1][D], double (&G)[D + 1][D])
{
    double a[D][D];
    int perm[D];
    double rcp[D];
    edge_rows<D>(x, a);
    bool sing = lu_factor<D, CORE>(a, perm, rcp);
    solve_ref_gradients<D, CORE>(a, perm, rcp, G);
    return sing;
}

// numpy det of B = A^T (mesh.py:38-43): LU of B, sign * exp(sum log|u_jj|).
// CUDA's log/exp stand in for glibc's (<= 1 ulp apart), so device volumes
// are within a few ulp of Mesh.vols, not bitwise.  Returns |det| / d!.
template <int D, int CORE>
__device__ __forceinline__ double element_volume(const double (&x)[D + 1][D], bool &degenerate)
{
    double A[D][D], B[D][D];
    edge_rows<D>(x, A);
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) B[i][j] = A[j][i];
    int perm[D];
    double rcp[D];
    bool sing = lu_factor<D, CORE>(B, perm, rcp);
    degenerate = sing;
    if (sing) return 0.0;
    int sign = 1;
    // permutation parity by counting inversions
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i + 1; j < D; ++j)
            if (perm[i] > perm[j]) sign = -sign;
    double logdet = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double u = B[i][i];
        if (u < 0) { sign = -sign; u = -u; }
        logdet = SA_ADD(logdet, log(u));
    }
    double det = exp(logdet);
    if (det == 0.0) degenerate = true;
    const double fact = D == 1 ? 1.0 : (D == 2 ? 2.0 : 6.0);
    return __ddiv_rn(det, fact);
}

// select G[alpha] for runtime alpha without dynamic register indexing
template <int D>
__device__ __forceinline__ void select_row(const double (&G)[D + 1][D], int alpha, double (&g)[D])
{
#pragma unroll
    for (int nu = 0; nu < D; ++nu) g[nu] = G[0][nu];
#pragma unroll
    for (int a = 1; a <= D; ++a)
        if (alpha == a)
#pragma unroll
            for (int nu = 0; nu < D; ++nu) g[nu] = G[a][nu];
}

template <int D>
__device__ __forceinline__ double select_val(const double (&w)[D + 1], int alpha)
{
    double r = w[0];
#pragma unroll
    for (int a = 1; a <= D; ++a)
        if (alpha == a) r = w[a];
    return r;
}

// Stiffness entry (alpha, beta): ((G_b0*G_a0 + G_b1*G_a1) + G_b2*G_a2) * vol
template <int D>
__device__ __forceinline__ double stiff_entry(const double (&ga)[D], const double (&gb)[D], double vol)
{
    double acc = SA_MUL(gb[0], ga[0]);
#pragma unroll
    for (int i = 1; i < D; ++i) acc = SA_ADD(acc, SA_MUL(gb[i], ga[i]));
    return SA_MUL(acc, vol);
}

// dot_mat_vec_g(Q[n][l]) = G_a[l]*G_b[n];  dot_mat_vec_g(S[n][l]) as in
// kernels.py:141-152 with the d=2,3 tables of build_elastic_tables (:114-138):
//   Q[n][l][j][i] = [j==n][i==l]
//   S[n][l][j][i] = n==l ? [i==j]*(i==l ? 2 : 1) : [j==l][i==n]
template <int D>
__device__ __forceinline__ double elastic_entry(const double (&ga)[D], const double (&gb)[D], int l, int n,
                                                double lambs, double mus)
{
    double xq = SA_MUL(ga[l], gb[n]);
    double xs;
    if (n != l) {
        xs = SA_MUL(ga[n], gb[l]);
    } else {
        xs = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double p = SA_MUL(ga[i], gb[i]);
            if (i == l) p = SA_MUL(2.0, p);
            xs = (i == 0) ? p : SA_ADD(xs, p);
        }
    }
    return SA_ADD(SA_MUL(lambs, xq), SA_MUL(mus, xs));
}

}  // namespace sa
