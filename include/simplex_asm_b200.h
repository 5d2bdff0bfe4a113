/*
 * simplex_asm_b200.h -- C ABI of the B200-native P1 assembly path.
 *
 * This is the drop-in boundary for the reference's assembly drivers
 * (reference = /root/reference/pkg/src/simplex_asm).  The reference is pure
 * Python; its "FFI" for this path is the Python driver protocol
 *     driver(mesh: Mesh, kernel) -> SparseMatrix        assembly.py:295-308
 * The Python package paper_1401_3301_b200 binds these symbols with ctypes
 * (INTEGRATION.md shows the binding) and re-exposes that protocol.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Pointers named *_dev are CUDA device
 *     pointers on `device`; `stream` is a cudaStream_t (NULL = legacy default).
 *   - Every entry point returns an sa_status; 0 = success.  On failure
 *     sa_last_error() gives a thread-local message and sa_bad_index() the
 *     element / position the reference would name in its exception.
 *   - Results are bitwise deterministic run to run.
 */
#ifndef SIMPLEX_ASM_B200_H
#define SIMPLEX_ASM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sa_status {
    SA_OK = 0,
    SA_ERR_DEGENERATE = 1,   /* -> DegenerateSimplexError(element)   errors.py:12-17, kernels.py:60-62 */
    SA_ERR_INDEX_RANGE = 2,  /* -> IndexRangeError                   errors.py:20-21, mesh.py:83-87 */
    SA_ERR_CAPACITY = 3,     /* -> CapacityError                     errors.py:8-9 */
    SA_ERR_ARG = 4,          /* -> ValueError                        */
    SA_ERR_CUDA = 5,         /* -> RuntimeError (CUDA error text)    */
    SA_ERR_NOMEM = 6         /* -> MemoryError                       */
} sa_status;

/* Operators (bit mask: MASS|STIFF may be fused into one numeric pass). */
enum {
    SA_OP_MASS = 1,      /* MassKernel       kernels.py:281-303 (mass_kernel :68-78)      */
    SA_OP_STIFF = 2,     /* StiffnessKernel  kernels.py:306-329 (stiffness_kernel :81-88) */
    SA_OP_ELASTIC = 4,   /* ElasticKernel    kernels.py:332-387 (elastic_kernel :155-172) */
    SA_OP_GENERAL = 8,   /* -div(A grad u)+div(b u)+c.grad u+a0 u */
    /* modifier: the general operator's element values in the reference's
     * operation order (bitwise the oracle).  Without it the general operator's
     * local matrices use fused multiply-adds: values within a few ulp of the
     * contributions, the exact-zero pattern still the reference's (guarded
     * rows are recomputed in reference order).  Mass, stiffness and elastic
     * are always bitwise. */
    SA_OP_EXACT = 16
};

/* OpenBLAS kernel family whose dgesv/dgetrf bits the gradients reproduce
 * (kernels.py:64 -> numpy -> OpenBLAS). */
enum { SA_CORE_SKYLAKEX = 0, SA_CORE_HASWELL = 1 };

typedef struct sa_mesh sa_mesh;   /* device-resident mesh (Mesh, mesh.py:46-101) */
typedef struct sa_plan sa_plan;   /* symbolic phase for one dof-row block        */

/* ---- mesh ------------------------------------------------------------- */

/* Upload-side mesh construction, replacing Mesh.from_arrays (mesh.py:54-58)
 * + compute_volumes (mesh.py:29-43).
 *   q_dev    (d, nq) f64 row-major, the reference layout of Mesh.q
 *   me_dev   (d+1, nme) int64 row-major (Mesh.me); checked against [0, nq)
 *            -> SA_ERR_INDEX_RANGE, sa_bad_index() = a*nme + k of the first
 *            bad entry in row-major order (mesh.py:83-87 names me[a, k]).
 *   vols_dev (nme,) f64 Mesh.vols, or NULL: volumes are then computed on the
 *            device from the numpy-det factorisation (mesh.py:38-43); zero
 *            volume -> SA_ERR_DEGENERATE with the first element.
 * The mesh keeps private device copies (q as padded AoS, me as int32). */
int sa_mesh_create(int d, int64_t nq, int64_t nme, const double *q_dev, const int64_t *me_dev,
                   const double *vols_dev, int core, int device, void *stream, sa_mesh **out);
/* Connectivity with its first rows32 rows as int32 ((rows32, nme), narrowed
 * on the host while uploading: sa_host_narrow_upload) and the remaining
 * d+1-rows32 rows as int64; otherwise sa_mesh_create. */
int sa_mesh_create_split(int d, int64_t nq, int64_t nme, const double *q_dev, const int32_t *me32_dev, int rows32,
                         const int64_t *me_dev, const double *vols_dev, int core, int device, void *stream,
                         sa_mesh **out);
/* Host side of the upload: n int64 entries of me (HOST memory) are narrowed
 * to int32 by nthreads host threads into `staging` (pinned host memory, n
 * entries), range-checked against [0, nq) in the same pass (first_bad = flat
 * index a * nme + k of the first bad entry, or -1: the reference's
 * IndexRangeError, mesh.py:83-87), and copied to dst_dev (device, n entries)
 * chunk by chunk on `stream` while later chunks are still being narrowed. */
int sa_host_narrow_upload(const int64_t *src_host, int64_t n, int64_t nq, int32_t *staging_pinned, int32_t *dst_dev,
                          int nthreads, int device, void *stream, int64_t *first_bad);
/* dst[i] = (int64) src[i] + offset on the same host thread pool: the int32
 * column indices that crossed PCIe, widened to the reference's int64
 * (sparse.py:53-55); offset shifts a slab's columns to global dofs. */
int sa_host_widen_i32(const int32_t *src_host, int64_t n, int64_t offset, int64_t *dst_host, int nthreads);
/* q_dev may be NULL in sa_mesh_create: the connectivity is packed and the
 * symbolic phase (which needs only me) can run while the coordinates are
 * still uploading; sa_mesh_set_coords then packs q and copies / computes
 * vols (as sa_mesh_create would).  sa_numeric fails until they are set. */
int sa_mesh_set_coords(sa_mesh *mesh, const double *q_dev, const double *vols_dev, void *stream);
int sa_mesh_vols(const sa_mesh *mesh, double *vols_dev_out, void *stream);
/* Mesh.validate's volume checks (reference mesh.py:92-101) on the device:
 * volumes are recomputed from the coordinates (numpy-det factorisation) and
 * compared with the stored ones (vols_dev, nme).  Outputs the first element
 * with a non-positive stored volume and the first whose stored volume is off
 * its recomputed one by more than 1e-12 relative (-1 = none).  The index
 * range check is sa_mesh_create's (SA_ERR_INDEX_RANGE). */
int sa_mesh_validate(const sa_mesh *mesh, const double *vols_dev, int64_t *first_nonpositive,
                     int64_t *first_mismatch, void *stream);
int sa_mesh_destroy(sa_mesh *mesh);

/* ---- symbolic phase (once per mesh and row block) ---------------------- */

/* Pattern of dof rows [row_begin, row_end) of an m-unknowns-per-node system
 * (m = 1 scalar, m = d elastic; interleaved dofs r = m*i + l, assembly.py:181-183).
 * row_begin/row_end must be multiples of m.  Replaces the structural part of
 * _canonicalize (sparse.py:91-115): node->element incidences in ascending
 * element order, sorted unique columns per row, indptr.  The structural
 * pattern is the optv2 pattern before exact-zero sums are dropped. */
int sa_plan_create(const sa_mesh *mesh, int m, int64_t row_begin, int64_t row_end, void *stream,
                   sa_plan **out);
/* nrows = row_end - row_begin; nnz = structural entries of the block. */
int sa_plan_info(const sa_plan *plan, int64_t *nrows, int64_t *nnz_structural,
                 int64_t *max_row_nodes);
/* Structural CSR of the block (indptr relative, int64 (nrows+1); indices
 * global column dofs int32 (nnz)), into caller-allocated device buffers. */
int sa_plan_pattern(const sa_plan *plan, int64_t *indptr_dev, int32_t *indices_dev, void *stream);
/* Diagnostics: out[0..n) = {incidences, max row nodes, nodes, nnz, warp
 * interleaved records, two-pass slots, every element batch staged (0/1),
 * largest batch vertex count, device bytes of the plan's structures,
 * largest light-row degree, heavy rows (assembled by the hub kernel)}. */
int sa_plan_stats(const sa_plan *plan, int64_t *out, int n);
int sa_plan_destroy(sa_plan *plan);

/* General-operator coefficient records (nq, 16) = [A 3x3 | b | c | a0] from a
 * column-compacted upload (nq, nv): record column j is uploaded column
 * colmap16[j], or the constant consts16[j] when colmap16[j] < 0.  Columns that
 * are constant over the nodes or repeat another column (a symmetric A) stay
 * on the host.  colmap16 / consts16 are HOST arrays of 16 entries. */
int sa_unpack_columns(const double *src_dev, int nv, const int32_t *colmap16_host, const double *consts16_host,
                      int64_t nq, double *dst_dev, void *stream);

/* ---- numeric phase (repeated for new coefficients) --------------------- */

/* Nodal coefficients (device pointers, nq entries unless stated) or
 * constants when the pointer is NULL -- the values _nodal_values produces
 * (kernels.py:268-278). */
typedef struct sa_coeffs {
    const double *w;     double w_const;      /* mass weight               */
    const double *lamb;  double lamb_const;   /* Lame lambda (elastic)     */
    const double *mu;    double mu_const;     /* Lame mu (elastic)         */
    const double *A;     /* general: (nq, d, d) row-major; NULL = A_const  */
    const double *b;     /* general: (nq, d); NULL = 0                     */
    const double *c;     /* general: (nq, d); NULL = 0                     */
    const double *a0;    /* general: (nq,);  NULL = a0_const               */
    double A_const[9];
    double a0_const;
    /* general, preferred: nodal AoS, 16 doubles per node
     * [A (3x3 row-major, zero-padded for d < 3) | b (3) | c (3) | a0], one
     * 128-byte line per node; overrides A/b/c/a0 when non-NULL */
    const double *gen_packed;
    /* elastic, optional: per-element Lame sums already scaled, exactly the
     * reference ElasticKernel's arrays lambs = (sum_g lamb_g) * vols/(d+1)
     * and mus (kernels.py:354-356), (nme,) each; override lamb/mu */
    const double *lambs_e;
    const double *mus_e;
} sa_coeffs;

/* Assemble the values of every structural entry of the block into
 * vals_dev[k] (k-th op in ascending SA_OP bit order, each nnz_structural
 * doubles, so MASS|STIFF writes mass at vals_dev[0] and stiffness at
 * vals_dev[1]).  Each entry is the left-to-right sum of its element
 * contributions in ascending element order -- bitwise the optv2 value
 * (assembly.py:92-111, sparse.py:97-106).  n_zero_out[k] = number of
 * structural entries whose sum is exactly +-0.0 (sparse.py:108-111 drops
 * them; see sa_compact).  q is read from the mesh; vols too.
 * Degenerate element (zero pivot) -> SA_ERR_DEGENERATE, sa_bad_index() = the
 * smallest such element (kernels.py:59-62). */
int sa_numeric(sa_plan *plan, int ops, const sa_coeffs *coeffs, double *const *vals_dev,
               int64_t *n_zero_out, void *stream);

/* Optional: build the per-plan structures the numeric kernel selected for
 * `ops` needs (the two-pass slot map, local-row buffer and element batches
 * of the 3D general operator) now instead of on the first sa_numeric call,
 * so that they are accounted to the symbolic phase.  No reference
 * counterpart (the reference re-sorts on every assembly). */
int sa_plan_prepare(sa_plan *plan, int ops, void *stream);

/* Drop exact-zero entries (sparse.py:108-111) from one op's values:
 * writes the canonical block CSR (indptr_out relative int64, indices_out
 * int32, vals_out f64, sized from sa_numeric's n_zero). */
int sa_compact(const sa_plan *plan, const double *vals_dev, int64_t *indptr_out_dev,
               int32_t *indices_out_dev, double *vals_out_dev, void *stream);

/* ---- diagnostics ------------------------------------------------------- */
const char *sa_last_error(void);
int64_t sa_bad_index(void);
/* Number of sa_* kernel launches issued by this thread since the last reset
 * (bench.py's gpu_launches). */
int64_t sa_launch_count(int reset);

/* ---- Pk mass matrix (order-k node lattices; csrc/sa_pk.cuh) ------------ */

/* Replaces assemble_mass_pk (assembly.py:265-292): every local entry is
 * (d! C[a][b]) * |K| with an element-independent table C.  me_dev is the
 * lattice connectivity (ndfe, nme) int64 (PkMesh.me, mesh.py:167-192);
 * ndfe <= 84, <= 255 distinct neighbours per node.  The symbolic plan holds
 * the structural pattern (CSR over nq x nq); sa_pk_mass folds every entry in
 * ascending element order (cs_dev = d! * C, row-major [a][b], computed as
 * the reference computes dfact * C[a, b]); sa_pk_compact drops exact-zero
 * sums (sparse.py:108-111). */
typedef struct sa_pk_plan sa_pk_plan;
int sa_pk_plan_create(int ndfe, int64_t nq, int64_t nme, const int64_t *me_dev, int device, void *stream,
                      sa_pk_plan **out);
int sa_pk_plan_info(const sa_pk_plan *plan, int64_t *nnz, int64_t *max_row_nodes);
int sa_pk_plan_pattern(const sa_pk_plan *plan, int64_t *indptr_dev, int32_t *indices_dev, void *stream);
int sa_pk_mass(sa_pk_plan *plan, const double *cs_dev, const double *vols_dev, double *vals_dev,
               int64_t *n_zero_out, void *stream);
int sa_pk_compact(const sa_pk_plan *plan, const double *vals_dev, int64_t *indptr_out, int32_t *indices_out,
                  double *vals_out, void *stream);
int sa_pk_plan_destroy(sa_pk_plan *plan);

/* ---- benchmark meshes on the device (sa_meshgen.cu) ------------------- */

/* Kuhn triangulation of [0,1]^d, n cells per axis, written to caller-owned
 * device buffers q_dev (d, (n+1)^d) f64 and me_dev (d+1, d! n^d) int64 --
 * bitwise the arrays of generate_hypercube_mesh (mesh.py:104-140).  With
 * jitter != 0 the interior nodes move by numpy's
 * default_rng(seed).uniform(lo, lo + range, size=(d, (n-1)^d)) (SURVEY.md
 * 8(d)); (state, inc) = np.random.PCG64(seed).state after seeding.
 * Either buffer may be NULL. */
int sa_kuhn_mesh(int d, int64_t n, int jitter, double lo, double range, uint64_t state_hi, uint64_t state_lo,
                 uint64_t inc_hi, uint64_t inc_lo, double *q_dev, int64_t *me_dev, void *stream);
/* The window of that mesh a rank needs: nodes [v0, v1) -> q_dev (d, v1-v0)
 * (jitter by PCG64 jump-ahead to each node's draws) and elements [e0, e1) ->
 * me_dev (d+1, e1-e0) with node ids relative to v0; bitwise the
 * corresponding slices of sa_kuhn_mesh's arrays. */
int sa_kuhn_slab(int d, int64_t n, int jitter, double lo, double range, uint64_t state_hi, uint64_t state_lo,
                 uint64_t inc_hi, uint64_t inc_lo, int64_t v0, int64_t v1, int64_t e0, int64_t e1, double *q_dev,
                 int64_t *me_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif
