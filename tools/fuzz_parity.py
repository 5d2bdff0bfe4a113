"""Randomised parity sweep against the C oracle (test infrastructure): random
dimension, mesh kind (jittered Kuhn, unjittered Kuhn, Delaunay, shuffled
numbering), size, operator, coefficients and row blocks; bitwise for mass /
stiffness / elastic / exact general, pattern-exact + 1e-12 of the row max for
the fast general operator, through the end-to-end block driver.

    python tools/fuzz_parity.py [seconds] [seed]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1401_3301_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1401_3301_b200 import parallel  # noqa: E402
from paper_1401_3301_b200.assembly import assemble_block_b200  # noqa: E402


def make_mesh(rng):
    d = int(rng.integers(1, 4))
    kind = rng.choice(["jitter", "kuhn", "delaunay", "shuffle"]) if d > 1 else rng.choice(["jitter", "kuhn"])
    if kind == "delaunay":
        from scipy.spatial import Delaunay

        npts = int(rng.integers(30, 3000 if d == 2 else 1200))
        pts = rng.random((npts, d))
        me = np.ascontiguousarray(Delaunay(pts).simplices.T.astype(np.int64))
        q = np.ascontiguousarray(pts.T)
        vols = np.abs(np.array([np.linalg.det((q[:, me[1:, e]] - q[:, me[:1, e]]).T) for e in range(me.shape[1])]))
        me = np.ascontiguousarray(me[:, vols > 1e-9])
    else:
        n = int(rng.integers(1, {1: 4000, 2: 120, 3: 24}[d]))
        q, me = P.hypercube_arrays(d, n)
        if kind != "kuhn":
            q = P.jitter_interior(q, n, float(rng.uniform(0.01, 0.3 if d < 3 else 0.15)), int(rng.integers(1 << 30)))
        if kind == "shuffle":
            nq = q.shape[1]
            perm = rng.permutation(nq)
            inv = np.empty_like(perm)
            inv[perm] = np.arange(nq)
            q, me = np.ascontiguousarray(q[:, perm]), np.ascontiguousarray(inv[me])
            me = np.ascontiguousarray(me[:, rng.permutation(me.shape[1])])
    return d, str(kind), q, me


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rng = np.random.default_rng(seed)
    t0 = time.time()
    n = 0
    stats = {}
    biggest = 0
    while time.time() - t0 < budget:
        d, kind, q, me = make_mesh(rng)
        try:
            vols = O.volumes(q, me)
        except O.OracleDegenerate:
            continue
        nq = q.shape[1]
        mesh = P.Mesh(q, me, vols)
        op = str(rng.choice(["mass", "stiffness", "ms", "elastic", "general", "general_exact"]))
        if op == "elastic" and d == 1:
            op = "stiffness"
        exact = True
        if op == "mass":
            w = rng.uniform(0.5, 2.0, nq)
            ks, ops = [P.MassKernel(mesh, w)], [O.OracleOp("mass", d, vols, w=w)]
        elif op == "stiffness":
            ks, ops = [P.StiffnessKernel(mesh)], [O.OracleOp("stiffness", d, vols)]
        elif op == "ms":
            ks = [P.MassKernel(mesh), P.StiffnessKernel(mesh)]
            ops = [O.OracleOp("mass", d, vols, w=np.ones(nq)), O.OracleOp("stiffness", d, vols)]
        elif op == "elastic":
            lam, mu = rng.uniform(0.5, 2.0, nq), rng.uniform(0.1, 1.0, nq)
            ks, ops = [P.ElasticKernel(mesh, lam, mu)], [O.OracleOp("elastic", d, vols, lamb=lam, mu=mu)]
        else:
            R = rng.standard_normal((nq, d, d))
            f = dict(A=np.eye(d)[None] + np.einsum("nij,nkj->nik", R, R) / 6.0, b=rng.standard_normal((nq, d)),
                     c=rng.standard_normal((nq, d)), a0=rng.uniform(0, 1, nq))
            if rng.random() < 0.3:   # exact cancellations: the guard's case
                f = dict(A=np.broadcast_to(np.eye(d), (nq, d, d)).copy(), b=np.zeros((nq, d)), c=np.zeros((nq, d)),
                         a0=np.zeros(nq))
            exact = op == "general_exact"
            ks, ops = [P.GeneralKernel(mesh, exact=exact, **f)], [O.OracleOp("general", d, vols, **f)]
        m = ks[0].m
        nparts = int(rng.integers(1, 4))
        cuts = sorted(set([0, nq] + [int(x) for x in rng.integers(0, nq + 1, nparts - 1)]))
        blocks = [[] for _ in ks]
        for a, b in zip(cuts[:-1], cuts[1:]):
            out = assemble_block_b200(mesh, ks, m * a, m * b)
            for i, blk in enumerate(out):
                blocks[i].append((m * a, m * b, blk.row_ptr, blk.col_idx, blk.vals))
        for i, oop in enumerate(ops):
            rp, ci, va = parallel.stitch(blocks[i], m * nq, m * nq)
            erp, eci, eva = O.assemble(q, me, oop, nthreads=8)
            tag = f"case {n} seed {seed}: d={d} {kind} nq={nq} nme={me.shape[1]} op={op} cuts={cuts}"
            assert np.array_equal(rp, erp) and np.array_equal(ci, eci), "PATTERN " + tag
            if exact:
                assert np.array_equal(va.view(np.int64), eva.view(np.int64)), "VALUES " + tag
            else:
                rows = np.repeat(np.arange(len(erp) - 1), np.diff(erp))
                rmax = np.zeros(len(erp) - 1)
                np.maximum.at(rmax, rows, np.abs(eva))
                assert np.all(np.abs(va - eva) <= 1e-12 * rmax[rows]), "VALUES " + tag
        n += 1
        stats[(d, kind, op)] = stats.get((d, kind, op), 0) + 1
        biggest = max(biggest, me.shape[1])
    by_kind, by_op = {}, {}
    for (d, kind, op), c in stats.items():
        by_kind[f"{d}D {kind}"] = by_kind.get(f"{d}D {kind}", 0) + c
        by_op[op] = by_op.get(op, 0) + c
    print(f"fuzz ok: {n} cases in {time.time() - t0:.0f} s (seed {seed}); largest mesh {biggest} elements")
    print("  by mesh:", dict(sorted(by_kind.items())))
    print("  by operator:", dict(sorted(by_op.items())))


if __name__ == "__main__":
    main()
