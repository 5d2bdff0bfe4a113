"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden fixtures and the CPU oracle.  Bar: bit-exact CSR pattern and -- since
every entry is folded in ascending element order with bit-exact element
values -- bit-exact values too (north_star's tolerance, 1e-12 of the row max,
is asserted as well so a failure says which bar broke).  The general
operator's default (fast) mode forms local matrices with fused multiply-adds:
there the bar is north_star's -- pattern bit-exact, values within 1e-12 of
each row's max -- and exact=True must be bitwise."""

import hashlib
import os

import numpy as np
import pytest

import paper_1401_3301_b200 as P
from conftest import device_kernel_for, golden_cases, load_golden, oracle_op_for

pytestmark = pytest.mark.gpu

VAL_RTOL = 1e-12  # north_star: fp64 values within 1e-12 relative to each row's max magnitude


def assert_csr_equal(got, rp, ci, va, bitwise=True):
    assert np.array_equal(got.row_ptr, rp), "row_ptr differs"
    assert np.array_equal(got.col_idx, ci), "col_idx differs"
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    rowmax = np.zeros(len(rp) - 1)
    np.maximum.at(rowmax, rows, np.abs(va))
    err = np.abs(got.vals - va)
    assert np.all(err <= VAL_RTOL * rowmax[rows]), f"max rel err {np.max(err / np.maximum(rowmax[rows], 1e-300))}"
    if bitwise:
        assert np.array_equal(got.vals, va), f"{np.count_nonzero(got.vals != va)} values not bitwise"


def golden_mesh(g):
    return P.Mesh(g["q"], g["me"], g["vols"])


@pytest.mark.parametrize("name", golden_cases())
def test_golden_bitwise(cuda_ok, name):
    g = load_golden(name)
    mesh = golden_mesh(g)
    k = device_kernel_for(name, g, mesh)
    got = P.assemble_vector_b200(mesh, k) if k.m > 1 else P.assemble_b200(mesh, k)
    assert got.shape == tuple(g["shape"])
    assert_csr_equal(got, g["row_ptr"], g["col_idx"], g["vals"])


def _jittered(d, n, seed):
    from oracle import oracle as O

    q, me = P.hypercube_arrays(d, n)
    q = P.jitter_interior(q, n, 0.2 if d == 2 else 0.15, seed)
    return P.Mesh(q, me, O.volumes(q, me))


def _oracle(mesh, kind, nthreads=16, **kw):
    from oracle import oracle as O

    op = O.OracleOp(kind, mesh.q.shape[0], mesh.vols, **kw)
    return O.assemble(mesh.q, mesh.me, op, nthreads=nthreads)


def tune(monkeypatch, **kw):
    """SA_TUNE: the library's single developer switch (kernel=..., symfast=...)."""
    monkeypatch.setenv("SA_TUNE", ",".join(f"{k}={v}" for k, v in kw.items()))


@pytest.mark.parametrize("symfast", ["1", "0"])
@pytest.mark.parametrize("d,n", [(2, 200), (3, 40)])
def test_fused_mass_stiffness_vs_oracle(cuda_ok, d, n, symfast, monkeypatch):
    # symfast: the fused shared-memory symbolic node pass (default) and the
    # general symbolic kernels give the same plan
    tune(monkeypatch, symfast=symfast)
    # C1 is d=2, n=200 (configs[0]); fused numeric pass, two outputs
    mesh = _jittered(d, n, 14013301)
    mass, stiff = P.assemble_many_b200(mesh, [P.MassKernel(mesh), P.StiffnessKernel(mesh)])
    assert_csr_equal(mass, *_oracle(mesh, "mass", w=np.ones(mesh.q.shape[1])))
    assert_csr_equal(stiff, *_oracle(mesh, "stiffness"))


def test_elastic_vs_oracle(cuda_ok):
    mesh = _jittered(3, 16, 14013304)
    lam = 1.0 + mesh.q[0]
    mu = 0.5 + mesh.q[2] ** 2
    got = P.assemble_vector_b200(mesh, P.ElasticKernel(mesh, lam, mu))
    assert_csr_equal(got, *_oracle(mesh, "elastic", lamb=lam, mu=mu))


def _c5_fields(nq, seed, d=3):
    rng = np.random.default_rng(seed)
    R = rng.standard_normal((nq, d, d))
    A = np.eye(d)[None] + 0.5 * np.einsum("nij,nkj->nik", R, R) / 3.0
    return dict(A=A, b=rng.standard_normal((nq, d)), c=rng.standard_normal((nq, d)), a0=rng.uniform(0, 1, nq))


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("kernel", ["rowgather", "twopass"])
def test_general_vs_oracle(cuda_ok, kernel, exact, monkeypatch):
    # exact: bitwise; fast (default, two-pass FMA element math): pattern exact,
    # values within 1e-12 of the row max
    tune(monkeypatch, kernel=kernel)
    mesh = _jittered(3, 20, 14013305)
    f = _c5_fields(mesh.q.shape[1], 14013305)
    got = P.assemble_b200(mesh, P.GeneralKernel(mesh, exact=exact, **f))
    assert_csr_equal(got, *_oracle(mesh, "general", **f), bitwise=exact or kernel == "rowgather")


@pytest.mark.parametrize("d,n", [(3, 8), (3, 12)])
def test_general_fast_guard_keeps_exact_zero_pattern(cuda_ok, d, n):
    # unjittered Kuhn cube, A = I and no lower-order terms: the stiffness
    # structure with its exact cancellations (3D N=8 keeps 4,617 of 9,097
    # entries).  Fast local matrices would leave ~1e-17 residues; the guard
    # sends those rows to the reference-order recomputation, so the pattern
    # and the zero count are the oracle's
    from paper_1401_3301_b200.device import DeviceMesh

    q, me = P.hypercube_arrays(d, n)
    from oracle import oracle as O

    mesh = P.Mesh(q, me, O.volumes(q, me))
    nq = q.shape[1]
    k = P.GeneralKernel(mesh, A=np.eye(d))
    got = P.assemble_b200(mesh, k)
    z = dict(A=np.broadcast_to(np.eye(d), (nq, d, d)), b=np.zeros((nq, d)), c=np.zeros((nq, d)), a0=np.zeros(nq))
    rp, ci, va = _oracle(mesh, "general", **z)
    assert_csr_equal(got, rp, ci, va, bitwise=False)
    plan = DeviceMesh(mesh.q, mesh.me, mesh.vols).plan(1)
    _, zeros = plan.numeric([k])
    assert zeros[0] == plan.nnz - len(va) > 0


@pytest.mark.parametrize("exact", [True, False])
def test_general_reduces_to_stiffness_and_mass(cuda_ok, exact):
    mesh = _jittered(3, 10, 3)
    st = P.assemble_b200(mesh, P.StiffnessKernel(mesh))
    g = P.assemble_b200(mesh, P.GeneralKernel(mesh, A=np.eye(3), exact=exact))
    assert_csr_equal(g, st.row_ptr, st.col_idx, st.vals, bitwise=exact)  # d=3: (4a)(v/4) == a*v exactly
    w = 1.0 + mesh.q[1]
    m = P.assemble_b200(mesh, P.MassKernel(mesh, w))
    g2 = P.assemble_b200(mesh, P.GeneralKernel(mesh, a0=w, exact=exact))
    assert_csr_equal(g2, m.row_ptr, m.col_idx, m.vals, bitwise=exact)


@pytest.mark.parametrize("kernel", ["rowgather", "twopass"])
def test_row_blocks_stitch_bitwise(cuda_ok, kernel, monkeypatch):
    from paper_1401_3301_b200 import parallel
    from paper_1401_3301_b200.device import DeviceMesh

    tune(monkeypatch, kernel=kernel)
    mesh = _jittered(3, 18, 9)
    full = P.assemble_b200(mesh, P.StiffnessKernel(mesh))
    dm = DeviceMesh(mesh.q, mesh.me, mesh.vols)
    blocks = []
    for rb, re_ in parallel.row_blocks(mesh.q.shape[1], 1, 3):
        (csr,) = dm.plan(1, rb, re_).assemble([P.StiffnessKernel(mesh)])
        blocks.append((rb, re_, csr.indptr.cpu().numpy(), csr.indices.cpu().numpy(), csr.vals.cpu().numpy()))
    rp, ci, va = parallel.stitch(blocks, mesh.q.shape[1], mesh.q.shape[1])
    assert_csr_equal(full, rp, ci, va)


def test_deterministic_run_to_run(cuda_ok):
    from paper_1401_3301_b200.device import DeviceMesh

    mesh = _jittered(2, 300, 1)
    dm = DeviceMesh(mesh.q, mesh.me, mesh.vols)
    plan = dm.plan(1)
    ks = [P.MassKernel(mesh), P.StiffnessKernel(mesh)]
    h = set()
    for _ in range(3):
        vals, _z = plan.numeric(ks)
        h.add(tuple(hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest() for v in vals))
    assert len(h) == 1


@pytest.mark.parametrize("kernel", ["rowgather", "twopass"])
def test_degenerate_element_named(cuda_ok, kernel, monkeypatch):
    tune(monkeypatch, kernel=kernel)
    q = np.array([[0.0, 1.0, 2.0, 0.0], [0.0, 1.0, 2.0, 1.0]])
    me = np.array([[0, 0], [3, 1], [1, 2]])
    mesh = P.Mesh(q, me, np.array([0.5, 0.0]))
    with pytest.raises(P.DegenerateSimplexError) as ei:
        P.assemble_b200(mesh, P.StiffnessKernel(mesh))
    assert ei.value.element == 1
    with pytest.raises(P.DegenerateSimplexError) as ei:
        P.Mesh.from_arrays(q, me)
    assert ei.value.element == 1


def test_index_range_error(cuda_ok):
    q, me = P.hypercube_arrays(2, 2)
    me = me.copy()
    me[2, 5] = q.shape[1]
    mesh = P.Mesh(q, me, np.full(me.shape[1], 0.125))
    with pytest.raises(P.IndexRangeError, match=r"me\[2, 5\]"):
        P.assemble_b200(mesh, P.StiffnessKernel(mesh))


def test_device_volumes_close_to_numpy_det(cuda_ok):
    from oracle import oracle as O

    for d, n in [(1, 50), (2, 60), (3, 12)]:
        q, me = P.hypercube_arrays(d, n)
        q = P.jitter_interior(q, n, 0.15, 2)
        v = P.device_volumes(q, me)
        ref = O.volumes(q, me)
        assert np.max(np.abs(v - ref) / ref) < 1e-14


def test_full_size_c2_properties(cuda_ok):
    """configs[1] (2D N=2000, 8M triangles) at full size: pattern and values
    vs the threaded oracle, plus size-independent invariants."""
    mesh = _jittered(2, 2000, 14013302)
    mass, stiff = P.assemble_many_b200(mesh, [P.MassKernel(mesh), P.StiffnessKernel(mesh)])
    assert_csr_equal(stiff, *_oracle(mesh, "stiffness"))
    assert_csr_equal(mass, *_oracle(mesh, "mass", w=np.ones(mesh.q.shape[1])))
    assert abs(mass.vals.sum() - 1.0) < 1e-12           # total mass = |domain|
    rows = np.repeat(np.arange(stiff.nrows), np.diff(stiff.row_ptr))
    rs = np.bincount(rows, weights=stiff.vals, minlength=stiff.nrows)
    assert np.max(np.abs(rs)) < 1e-9                    # constants are in the kernel


@pytest.mark.parametrize("kernel", ["twopass", "rowgather"])
@pytest.mark.parametrize("name", golden_cases())
def test_golden_bitwise_kernels(cuda_ok, name, kernel, monkeypatch):
    # every numeric kernel is bitwise (general operator: exact=True): the
    # two-pass element-rows kernel, the one-pass row gather
    tune(monkeypatch, kernel=kernel)
    g = load_golden(name)
    mesh = golden_mesh(g)
    k = device_kernel_for(name, g, mesh)
    got = P.assemble_vector_b200(mesh, k) if k.m > 1 else P.assemble_b200(mesh, k)
    assert_csr_equal(got, g["row_ptr"], g["col_idx"], g["vals"])


@pytest.mark.parametrize("kernel", ["rowgather", "twopass"])
def test_unstructured_delaunay_mesh(cuda_ok, kernel, monkeypatch):
    # random points, Delaunay triangulation: irregular valence
    tune(monkeypatch, kernel=kernel)
    from scipy.spatial import Delaunay

    from paper_1401_3301_b200.device import DeviceMesh
    from oracle import oracle as O

    for d, npts in ((2, 4000), (3, 1500)):
        rng = np.random.default_rng(d)
        pts = rng.random((npts, d))
        tri = Delaunay(pts)
        q = np.ascontiguousarray(pts.T)
        me = np.ascontiguousarray(tri.simplices.T.astype(np.int64))
        try:
            vols = O.volumes(q, me)
        except O.OracleDegenerate:
            continue
        keep = vols > 1e-10
        me = np.ascontiguousarray(me[:, keep])
        mesh = P.Mesh(q, me, O.volumes(q, me))
        st = DeviceMesh(mesh.q, mesh.me, mesh.vols).plan(1).stats()
        assert st["max_row_nodes"] > 7, st
        mass, stiff = P.assemble_many_b200(mesh, [P.MassKernel(mesh, 1.0 + mesh.q[0]), P.StiffnessKernel(mesh)])
        assert_csr_equal(stiff, *_oracle(mesh, "stiffness", nthreads=4))
        assert_csr_equal(mass, *_oracle(mesh, "mass", nthreads=4, w=1.0 + mesh.q[0]))


@pytest.mark.parametrize("k", [40, 70, 400])
def test_high_valence_node(cuda_ok, k):
    # a fan of k triangles around node 0 (k incidences, k+1 neighbours; 400:
    # beyond the 8-bit column ranks -- the reference has no valence limit,
    # sparse.py:85-115)
    from oracle import oracle as O

    ang = np.linspace(0, 2 * np.pi, k, endpoint=False)
    q = np.vstack([np.concatenate([[0.0], np.cos(ang)]), np.concatenate([[0.0], np.sin(ang)])])
    me = np.array([[0] * k, [1 + i for i in range(k)], [1 + (i + 1) % k for i in range(k)]])
    mesh = P.Mesh(q, me, O.volumes(q, me))
    got = P.assemble_b200(mesh, P.StiffnessKernel(mesh))
    assert_csr_equal(got, *_oracle(mesh, "stiffness", nthreads=1))


@pytest.mark.parametrize("d,n,parts", [(2, 40, 3), (3, 9, 2)])
def test_block_e2e_slabs_stitch_bitwise(cuda_ok, d, n, parts):
    # the public per-rank call (assemble_block_b200: connectivity first,
    # coordinates uploaded during the symbolic phase, pattern downloaded
    # during the numeric phase, int32 indices widened on the host) on each
    # rank's slab stitches to the full oracle matrices, bitwise
    from oracle import oracle as O
    from paper_1401_3301_b200 import parallel
    from paper_1401_3301_b200.assembly import assemble_block_b200

    mesh = _jittered(d, n, 21)
    nq = mesh.q.shape[1]
    blocks_m, blocks_s = [], []
    for rb, re_ in parallel.row_blocks(nq, 1, parts):
        sl = parallel.slab(mesh.q, mesh.me, 1, rb, re_, mesh.vols)
        smesh = P.Mesh(sl.q, sl.me, sl.vols)
        ms, st = assemble_block_b200(smesh, [P.MassKernel(smesh), P.StiffnessKernel(smesh)], sl.row_begin,
                                     sl.row_end, col_offset=sl.col_offset)
        assert ms.col_idx.dtype == np.int64
        blocks_m.append((rb, re_, ms.row_ptr, ms.col_idx, ms.vals))
        blocks_s.append((rb, re_, st.row_ptr, st.col_idx, st.vals))
    assert_csr_equal(P.SparseMatrix(nq, nq, *parallel.stitch(blocks_m, nq, nq)),
                     *_oracle(mesh, "mass", w=np.ones(nq)))
    assert_csr_equal(P.SparseMatrix(nq, nq, *parallel.stitch(blocks_s, nq, nq)), *_oracle(mesh, "stiffness"))


def test_numeric_graph_replay_bitwise(cuda_ok):
    # the CUDA-graph replay of the numeric phase (bench.py's step) writes the
    # same values as a direct call, for the one-pass and the two-pass kernels
    import torch

    from paper_1401_3301_b200.device import OP_BITS, DeviceMesh

    for d, n, ks in ((2, 60, ("mass", "stiffness")), (3, 10, ("general",))):
        mesh = _jittered(d, n, 5)
        nq = mesh.q.shape[1]
        rng = np.random.default_rng(1)
        kern = {"mass": lambda: P.MassKernel(mesh), "stiffness": lambda: P.StiffnessKernel(mesh),
                "general": lambda: P.GeneralKernel(mesh, A=np.eye(3)[None] + 0.1 * rng.random((nq, 3, 3)),
                                                   b=rng.random((nq, 3)), c=rng.random((nq, 3)),
                                                   a0=rng.random(nq))}
        kernels = [kern[k]() for k in ks]
        plan = DeviceMesh(mesh.q, mesh.me, mesh.vols).plan(1)
        ref, _ = plan.numeric(kernels)
        ref = [r.clone() for r in ref]
        out = [torch.full((plan.nnz,), float("nan"), dtype=torch.float64, device="cuda") for _ in kernels]
        g = plan.numeric_graph(kernels, out, plan.resident_coeffs(kernels))
        for o in out:
            o.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert g.sa_kernels_per_replay >= 1
        order = sorted(range(len(kernels)), key=lambda i: OP_BITS[kernels[i].op])
        for j, i in enumerate(order):
            assert torch.equal(out[j], ref[i])


@pytest.mark.parametrize("d,n,seed", [(1, 37, 3), (2, 25, 14013302), (2, 1, None), (3, 7, 14013305), (3, 12, None)])
def test_device_mesh_generator_bitwise(cuda_ok, d, n, seed):
    # sa_kuhn_mesh (Kuhn cube + numpy-PCG64 jitter restated with jump-ahead)
    # equals the host generator (mesh.py:104-140 + SURVEY 8(d) jitter) bit for bit
    q_h, me_h = P.hypercube_arrays(d, n)
    if seed is not None:
        q_h = P.jitter_interior(q_h, n, 0.2 if d <= 2 else 0.15, seed)
    q_d, me_d = P.device_hypercube_arrays(d, n, seed=seed, host=True)
    assert np.array_equal(me_d, me_h)
    assert np.array_equal(q_d.view(np.int64), q_h.view(np.int64))


@pytest.mark.parametrize("name", golden_cases("pk_"))
def test_pk_mass_golden_bitwise(cuda_ok, name):
    # Pk mass on the B200 vs the reference's assemble_mass_pk, bitwise, with
    # the lattice mesh and table from this package's host restatements
    from paper_1401_3301_b200 import pk

    g = load_golden(name)
    d, k = g["q"].shape[0], int(g["k"])
    pm = pk.build_pk_mesh(P.Mesh(g["p1_q"], g["p1_me"], g["vols"]), k)
    got = P.assemble_mass_pk_b200(pm, pk.pk_mass_coeffs(d, k))
    assert got.shape == tuple(g["shape"])
    assert_csr_equal(got, g["row_ptr"], g["col_idx"], g["vals"])


def test_pk_mass_larger_mesh_vs_oracle(cuda_ok):
    # P2 on a 3D jittered cube (exact-zero table entries, skipped/dropped as
    # the reference does) and P3 in 2D, against the oracle restatement
    from oracle import oracle as O
    from paper_1401_3301_b200 import pk

    for d, n, k in ((3, 8, 2), (2, 20, 3)):
        mesh = _jittered(d, n, 4)
        pm = pk.build_pk_mesh(mesh, k)
        C = pk.pk_mass_coeffs(d, k)
        got = P.assemble_mass_pk_b200(pm, C)
        assert_csr_equal(got, *O.assemble_mass_pk(pm.me, pm.vols, C.C, d, pm.nq))
    with pytest.raises(ValueError):
        P.assemble_mass_pk_b200(pm, pk.pk_mass_coeffs(d, 2))


@pytest.mark.parametrize("kernel", ["rowgather", "twopass"])
def test_haswell_core_vs_oracle(cuda_ok, kernel, monkeypatch):
    # the OpenBLAS Haswell kernel family (unfused getrf/getrs updates,
    # SURVEY.md Appendix A): GPU gradients and the oracle agree bitwise, so
    # the value-dependent pattern (exact zeros) matches under that core too
    from oracle import oracle as O
    from paper_1401_3301_b200.assembly import to_host
    from paper_1401_3301_b200.device import DeviceMesh

    tune(monkeypatch, kernel=kernel)
    mesh = _jittered(3, 9, 17)
    nq = mesh.q.shape[1]
    for kind in ("stiffness", "general"):
        kw = {}
        kern = P.StiffnessKernel(mesh)
        if kind == "general":
            rng = np.random.default_rng(2)
            kw = dict(A=np.eye(3)[None] + 0.1 * rng.random((nq, 3, 3)), b=rng.random((nq, 3)),
                      c=rng.random((nq, 3)), a0=rng.random(nq))
            kern = P.GeneralKernel(mesh, exact=True, **kw)
        plan = DeviceMesh(mesh.q, mesh.me, mesh.vols, core="Haswell").plan(1)
        (csr,) = plan.assemble([kern])
        got = to_host(csr)
        op = O.OracleOp(kind, 3, mesh.vols, core="Haswell", **kw)
        assert_csr_equal(got, *O.assemble(mesh.q, mesh.me, op, nthreads=4))


@pytest.mark.parametrize("kernel", ["rowgather", "twopass"])
def test_edge_cases_empty_and_isolated(cuda_ok, kernel, monkeypatch):
    # reference edge cases: a zero kernel gives an empty matrix
    # (test_assembly.py:99-102, sparse.py:91-95/108-111); nodes no element
    # references give empty rows; a mesh without elements; a row block of
    # isolated nodes only
    from oracle import oracle as O
    from paper_1401_3301_b200.device import DeviceMesh

    tune(monkeypatch, kernel=kernel)
    mesh = _jittered(2, 6, 3)
    nq = mesh.q.shape[1]
    z = P.assemble_b200(mesh, P.MassKernel(mesh, np.zeros(nq)))
    assert z.nnz == 0 and np.array_equal(z.row_ptr, np.zeros(nq + 1, dtype=np.int64))
    # 5 isolated nodes appended (never referenced)
    q2 = np.hstack([mesh.q, np.full((2, 5), 0.5)])
    mesh2 = P.Mesh(q2, mesh.me, mesh.vols)
    got = P.assemble_b200(mesh2, P.StiffnessKernel(mesh2))
    rp, ci, va = O.assemble(q2, mesh.me, O.OracleOp("stiffness", 2, mesh.vols), nthreads=2)
    assert_csr_equal(got, rp, ci, va)
    assert np.all(np.diff(got.row_ptr)[nq:] == 0)
    # a row block holding only the isolated nodes
    (csr,) = DeviceMesh(q2, mesh.me, mesh.vols).plan(1, nq, nq + 5).assemble([P.StiffnessKernel(mesh2)])
    assert csr.nnz == 0 and csr.indptr.cpu().numpy().tolist() == [0] * 6
    # no elements at all
    for d in (1, 2, 3):
        e = P.Mesh(np.zeros((d, 4)), np.zeros((d + 1, 0), dtype=np.int64), np.zeros(0))
        m0 = P.assemble_b200(e, P.StiffnessKernel(e))
        assert m0.nnz == 0 and m0.shape == (4, 4)


@pytest.mark.parametrize("d,n,parts", [(1, 30, 3), (2, 13, 4), (3, 7, 3)])
def test_device_slab_generator(cuda_ok, d, n, parts):
    # sa_kuhn_slab windows are bitwise slices of the full generated mesh,
    # cover every element touching the block, and the blocks assembled from
    # them stitch to the full oracle matrix
    from oracle import oracle as O
    from paper_1401_3301_b200 import parallel
    from paper_1401_3301_b200.device import DeviceMesh

    seed = 99
    q, me = P.device_hypercube_arrays(d, n, seed=seed, host=True)
    nq = q.shape[1]
    vols = O.volumes(q, me)
    blocks = []
    for rb, re_ in parallel.row_blocks(nq, 1, parts):
        sl = P.device_hypercube_slab(d, n, 1, rb, re_, seed=seed)
        e = sl.elements
        assert np.array_equal(sl.q.view(np.int64), q[:, sl.node_lo:sl.node_lo + sl.q.shape[1]].view(np.int64))
        assert np.array_equal(sl.me + sl.node_lo, me[:, e])
        touching = parallel.slab(q, me, 1, rb, re_).elements
        assert np.all(np.isin(touching, e))
        (csr,) = DeviceMesh(sl.q, sl.me, vols[e]).plan(1, sl.row_begin, sl.row_end).assemble(
            [P.StiffnessKernel(P.Mesh(sl.q, sl.me, vols[e]))])
        blocks.append((rb, re_, csr.indptr.cpu().numpy(), csr.indices.cpu().numpy().astype(np.int64) + sl.col_offset,
                       csr.vals.cpu().numpy()))
    rp, ci, va = parallel.stitch(blocks, nq, nq)
    assert_csr_equal(P.SparseMatrix(nq, nq, rp, ci, va),
                     *O.assemble(q, me, O.OracleOp("stiffness", d, vols), nthreads=4))



@pytest.mark.parametrize("name", ["elastic_d3_n6_jit", "elastic_d2_n15_jit", "elastic_d3_n5_kuhn", "elasticc_d3_n8_jit"])
def test_reference_elastic_kernel_object(cuda_ok, name):
    # the reference's own ElasticKernel keeps only per-element lambs/mus
    # (kernels.py:354-356); an object carrying exactly those arrays (as the
    # reference computes them) goes through the drop-in driver bitwise
    g = load_golden(name) if name in golden_cases() else None
    if g is None:
        pytest.skip(f"no fixture {name}")
    mesh = golden_mesh(g)
    d = g["q"].shape[0]
    nq = g["q"].shape[1]
    lam = g["lamb"] if "lamb" in g else np.full(nq, 1.0)
    mu = g["mu"] if "mu" in g else np.full(nq, 0.5)
    scale = mesh.vols / (d + 1)

    class ElasticKernel:   # the reference class's data members (kernels.py:343-356)
        symmetric = True

        def __init__(self):
            self.d = self.m = d
            self.lambs = lam[mesh.me].sum(axis=0) * scale
            self.mus = mu[mesh.me].sum(axis=0) * scale

    got = P.assemble_vector_b200(mesh, ElasticKernel())
    assert_csr_equal(got, g["row_ptr"], g["col_idx"], g["vals"])


FULL = {  # BASELINE.json configs at full size; exact-zero drops the reference makes
    "C1": None, "C2": None, "C3": 8 * 160 - 4, "C4": 24 * 100 + 16, "C5": 0}


@pytest.mark.parametrize("name", sorted(FULL))
def test_full_size_config(cuda_ok, name):
    """Every BASELINE config at full size against the threaded C oracle:
    pattern bit-exact, values bitwise (the fast general operator of C5:
    within 1e-12 of the row max), the reference's exact-zero drops, and
    run-to-run determinism (SHA-256 of two numeric passes)."""
    import hashlib

    import bench
    from oracle import oracle as O
    from paper_1401_3301_b200.assembly import to_host
    from paper_1401_3301_b200.device import DeviceMesh

    cfg = bench.CONFIGS[name]
    q, me = bench.make_mesh(cfg)
    vols = O.volumes(q, me)
    mesh = P.Mesh(q, me, vols)
    kernels = bench.make_kernels(cfg, mesh)
    dm = DeviceMesh(q, me, vols)
    plan = dm.plan(kernels[0].m)
    vals1, z1 = plan.numeric(kernels)
    sha1 = [hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest() for v in vals1]
    vals2, z2 = plan.numeric(kernels)
    sha2 = [hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest() for v in vals2]
    assert sha1 == sha2 and z1 == z2, "numeric phase not deterministic run to run"
    nthreads = 16
    for k, v, z in zip(kernels, vals1, z1):
        got = to_host(plan.compact(v, z))
        nq = q.shape[1]
        if k.op == "mass":
            op = O.OracleOp("mass", cfg["d"], vols, w=np.ones(nq))
        elif k.op == "stiffness":
            op = O.OracleOp("stiffness", cfg["d"], vols)
        elif k.op == "elastic":
            op = O.OracleOp("elastic", cfg["d"], vols, lamb=np.ones(nq), mu=np.full(nq, 0.5))
        else:
            op = O.OracleOp("general", cfg["d"], vols, A=k.A, b=k.b, c=k.c, a0=k.a0)
        rp, ci, va = O.assemble(q, me, op, nthreads=nthreads)
        assert_csr_equal(got, rp, ci, va, bitwise=not (k.op == "general" and not k.exact))
        if k.op != "mass" and FULL[name] is not None:
            assert plan.nnz - len(va) == z == FULL[name]
    dm.close()


@pytest.mark.parametrize("tool", ["racecheck", "memcheck"])
def test_compute_sanitizer(cuda_ok, tool):
    # shared-memory hazards (the cp.async element stage, the row
    # accumulators) and out-of-bounds / misaligned accesses on every path
    import shutil
    import subprocess
    import sys

    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    script = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "sanitize_case.py")
    r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "9", sys.executable, script],
                       capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    if "closed on this pool" in tail:   # the pool's compute-sanitizer wrapper refuses to run
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, tail
    assert "sanitize case ok" in r.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr, tail



def _dist_gpu_worker(rank, world, port, name, result_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist

    import paper_1401_3301_b200 as P
    from conftest import device_kernel_for as dk, load_golden as lg
    from paper_1401_3301_b200 import device, parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)   # one GPU here: both ranks on cuda:0, gloo collectives (functional check)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = lg(name)
        mesh = P.Mesh(g["q"], g["me"], g["vols"])
        device.launch_count(reset=True)
        res = parallel.assemble_distributed(mesh, [dk(name, g, mesh)])
        launched = device.launch_count()
        if rank == 0:
            a = res.matrices[0]
            ok = (np.array_equal(a.row_ptr, g["row_ptr"]) and np.array_equal(a.col_idx, g["col_idx"])
                  and np.array_equal(a.vals, g["vals"]) and res.totals[0] == len(g["vals"]) and launched > 0)
            result_q.put(bool(ok))
        else:
            result_q.put(res.matrices is None and res.offsets[0] > 0 and launched > 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["stiff_d3_n8_jit", "general_d3_n8_jit", "elastic_d3_n6_jit", "mass_d2_n15_jit"])
def test_distributed_driver_two_ranks_gpu(cuda_ok, name):
    # parallel.assemble_distributed through the product block assembler on
    # the GPU, two ranks (both on cuda:0 -- the pool has one GPU per call):
    # slabs, per-rank symbolic + numeric, offsets, gather, stitch == the
    # reference's matrix bitwise
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_gpu_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    results = [q.get(timeout=10) for _ in range(2)]
    assert all(results), results
    assert all(p.exitcode == 0 for p in procs)



@pytest.mark.parametrize("kind", ["elastic", "stiffness", "general"])
def test_3d_hub_node(cuda_ok, kind):
    # a hub node joined to 120 points on a sphere (cone over the convex hull):
    # its rows are heavy (k_heavy_rows), the other rows keep small
    # accumulators; bitwise against the oracle
    from scipy.spatial import ConvexHull

    from oracle import oracle as O
    from paper_1401_3301_b200.device import DeviceMesh

    rng = np.random.default_rng(7)
    p = rng.standard_normal((120, 3))
    p /= np.linalg.norm(p, axis=1)[:, None]
    hull = ConvexHull(p)
    q = np.ascontiguousarray(np.vstack([np.zeros((1, 3)), p]).T)
    tri = hull.simplices + 1
    me = np.ascontiguousarray(np.vstack([np.zeros(len(tri), dtype=np.int64), tri.T.astype(np.int64)]))
    mesh = P.Mesh(q, me, O.volumes(q, me))
    nq = q.shape[1]
    if kind == "elastic":
        lam, mu = 1.0 + q[0] ** 2, 0.5 + 0.1 * q[1]
        got = P.assemble_vector_b200(mesh, P.ElasticKernel(mesh, lam, mu))
        ref = _oracle(mesh, "elastic", nthreads=2, lamb=lam, mu=mu)
        m = 3
    elif kind == "stiffness":
        got = P.assemble_b200(mesh, P.StiffnessKernel(mesh))
        ref = _oracle(mesh, "stiffness", nthreads=2)
        m = 1
    else:
        f = _c5_fields(nq, 3)
        got = P.assemble_b200(mesh, P.GeneralKernel(mesh, exact=True, **f))
        ref = _oracle(mesh, "general", nthreads=2, **f)
        m = 1
    assert_csr_equal(got, *ref)
    st = DeviceMesh(mesh.q, mesh.me, mesh.vols).plan(m).stats()
    assert st["max_row_nodes"] == 121 and st["heavy_rows"] == 1 and st["light_row_nodes"] < 40, st



@pytest.mark.parametrize("core", ["SkylakeX", "Haswell"])
def test_general_fast_unstructured_and_cores(cuda_ok, core):
    # the fast general operator on an unstructured Delaunay tet mesh (valence
    # 10-30, irregular element batches) under both OpenBLAS kernel families:
    # pattern exact, values within 1e-12 of the row max; exact mode bitwise
    from scipy.spatial import Delaunay

    from oracle import oracle as O
    from paper_1401_3301_b200.assembly import to_host
    from paper_1401_3301_b200.device import DeviceMesh

    rng = np.random.default_rng(11)
    pts = rng.random((3000, 3))
    me = np.ascontiguousarray(Delaunay(pts).simplices.T.astype(np.int64))
    q = np.ascontiguousarray(pts.T)
    vols = O.volumes(q, me)
    me = np.ascontiguousarray(me[:, vols > 1e-9])
    mesh = P.Mesh(q, me, O.volumes(q, me))
    f = _c5_fields(q.shape[1], 12)
    op = O.OracleOp("general", 3, mesh.vols, core=core, **f)
    rp, ci, va = O.assemble(q, mesh.me, op, nthreads=8)
    for exact in (False, True):
        plan = DeviceMesh(mesh.q, mesh.me, mesh.vols, core=core).plan(1)
        (csr,) = plan.assemble([P.GeneralKernel(mesh, exact=exact, **f)])
        assert_csr_equal(to_host(csr), rp, ci, va, bitwise=exact)


def test_general_fast_row_blocks_stitch(cuda_ok):
    # fast general operator on row-block slabs (parallel.slab: local node
    # window, shifted columns, coefficient windows) stitches to the full
    # oracle matrix within north_star's bar, pattern exact
    from oracle import oracle as O
    from paper_1401_3301_b200 import kernels as K
    from paper_1401_3301_b200 import parallel
    from paper_1401_3301_b200.assembly import assemble_block_b200

    mesh = _jittered(3, 12, 31)
    nq = mesh.q.shape[1]
    f = _c5_fields(nq, 31)
    full = P.GeneralKernel(mesh, **f)
    blocks = []
    for rb, re_ in parallel.row_blocks(nq, 1, 3):
        sl = parallel.slab(mesh.q, mesh.me, 1, rb, re_, mesh.vols)
        smesh = P.Mesh(sl.q, sl.me, sl.vols)
        kk = K.restrict(full, smesh, slice(sl.node_lo, sl.node_lo + sl.q.shape[1]), sl.elements)
        (b,) = assemble_block_b200(smesh, [kk], sl.row_begin, sl.row_end, col_offset=sl.col_offset, ncols=nq)
        assert b.ncols == nq
        blocks.append((rb, re_, b.row_ptr, b.col_idx, b.vals))
    rp, ci, va = parallel.stitch(blocks, nq, nq)
    assert_csr_equal(P.SparseMatrix(nq, nq, rp, ci, va), *_oracle(mesh, "general", **f), bitwise=False)


def test_mesh_validate_on_device(cuda_ok):
    # Mesh.validate (reference mesh.py:72-101): same checks, order and
    # messages, index range and volume recomputation on the device
    from paper_1401_3301_b200.errors import IndexRangeError, MeshValidationError

    mesh = _jittered(3, 6, 11)
    mesh.validate()
    _jittered(2, 9, 12).validate()
    P.Mesh(*P.hypercube_arrays(1, 7), np.full(7, 1.0 / 7)).validate()
    me = mesh.me.copy()
    me[2, 17] = mesh.q.shape[1]
    me[3, 5] = -1
    with pytest.raises(IndexRangeError, match=r"me\[2, 17\] out of range \[0, 343\)"):
        P.Mesh(mesh.q, me, mesh.vols).validate()
    with pytest.raises(MeshValidationError, match=r"connectivity shape \(3, 1296\) does not match \(4, nme\)"):
        P.Mesh(mesh.q, mesh.me[:3], mesh.vols).validate()
    with pytest.raises(MeshValidationError, match=r"volume array shape \(5,\) does not match \(nme,\)"):
        P.Mesh(mesh.q, mesh.me, mesh.vols[:5]).validate()
    v = mesh.vols.copy()
    v[40] = 0.0
    v[77] = -v[77]
    with pytest.raises(MeshValidationError, match="volume of simplex 40 is not positive"):
        P.Mesh(mesh.q, mesh.me, v).validate()
    v = mesh.vols.copy()
    v[123] *= 1.0 + 3e-12
    v[500] *= 2.0
    with pytest.raises(MeshValidationError, match="stored volume of simplex 123 disagrees with its coordinates"):
        P.Mesh(mesh.q, mesh.me, v).validate()
    v = mesh.vols.copy()
    v[9] *= 1.0 + 2e-13    # inside the tolerance
    P.Mesh(mesh.q, mesh.me, v).validate()


def test_block_upload_narrows_connectivity_on_the_host(cuda_ok, monkeypatch):
    # assemble_block_b200 narrows the int64 connectivity to int32 on the host
    # while uploading (sa_host_narrow_upload): same matrices from pageable,
    # page-locked, read-only and non-contiguous arrays; a bad index -- also
    # one whose low 32 bits look valid -- raises the reference's IndexRangeError
    import torch

    from paper_1401_3301_b200.assembly import assemble_block_b200
    from paper_1401_3301_b200.device import connectivity_split
    from paper_1401_3301_b200.errors import IndexRangeError

    from paper_1401_3301_b200 import device as D

    monkeypatch.setattr(D, "_NARROW_MIN_ENTRIES", 0)   # (small arrays normally upload as they are)
    mesh = _jittered(3, 9, 21)
    nq = mesh.q.shape[1]
    k = P.StiffnessKernel(mesh)
    want = P.assemble_b200(mesh, k)
    pinned = torch.from_numpy(mesh.me.copy()).pin_memory().numpy()
    ro = mesh.me.copy()
    ro.setflags(write=False)
    fortran = np.asfortranarray(mesh.me)
    assert connectivity_split(pinned, 3) == 3 and connectivity_split(mesh.me.copy(), 3) == 4
    assert connectivity_split(fortran, 3) == 0 and connectivity_split(mesh.me.astype(np.int32), 3) == 0
    for me in (mesh.me.copy(), pinned, ro, fortran):
        (b,) = assemble_block_b200(P.Mesh(mesh.q, me, mesh.vols), [k], 0, nq)
        assert_csr_equal(b, want.row_ptr, want.col_idx, want.vals)
    for bad_val in (nq, -1, (1 << 32) + 5):
        for src in (mesh.me.copy(), pinned.copy()):
            src[1, 77] = bad_val
            src[3, 5] = -7
            with pytest.raises(IndexRangeError, match=rf"me\[1, 77\] out of range \[0, {nq}\)"):
                assemble_block_b200(P.Mesh(mesh.q, src, mesh.vols), [k], 0, nq)
