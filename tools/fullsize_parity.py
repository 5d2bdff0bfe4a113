"""Full-size parity of the B200 path against the threaded CPU oracle on the
BASELINE.json configs (run on the GPU box; writes one JSON line per config).

    python tools/fullsize_parity.py C3 C4 C5

Checks: CSR pattern bit-exact (row_ptr, col_idx), values bitwise and within
1e-12 of each row's max, and run-to-run determinism (SHA-256 of two numeric
passes).  Volumes are the oracle's (glibc numpy-det) so both sides see the
same Mesh.vols, as the reference drivers would."""

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1401_3301_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def oracle_op(cfg, mesh, kernel):
    d, nq = cfg["d"], mesh.q.shape[1]
    if kernel.op == "mass":
        return O.OracleOp("mass", d, mesh.vols, w=np.ones(nq))
    if kernel.op == "stiffness":
        return O.OracleOp("stiffness", d, mesh.vols)
    if kernel.op == "elastic":
        return O.OracleOp("elastic", d, mesh.vols, lamb=np.full(nq, 1.0), mu=np.full(nq, 0.5))
    A = kernel.A if kernel.A is not None else np.broadcast_to(kernel.A_const, (nq, d, d))
    return O.OracleOp("general", d, mesh.vols, A=A, b=kernel.b, c=kernel.c, a0=kernel.a0)


def check(name):
    import torch

    from paper_1401_3301_b200.device import DeviceMesh

    cfg = bench.CONFIGS[name]
    t0 = time.time()
    q, me = bench.make_mesh(cfg)
    vols = O.volumes(q, me)
    mesh = P.Mesh(q, me, vols)
    kernels = bench.make_kernels(cfg, mesh)
    dm = DeviceMesh(q, me, vols)
    plan = dm.plan(kernels[0].m)
    vals1, z1 = plan.numeric(kernels)
    sha1 = [hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest() for v in vals1]
    vals2, _ = plan.numeric(kernels)
    sha2 = [hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest() for v in vals2]
    res = []
    for k, v, z in zip(kernels, vals1, z1):
        from paper_1401_3301_b200.assembly import to_host

        got = to_host(plan.compact(v, z))
        t1 = time.time()
        rp, ci, va = O.assemble(q, me, oracle_op(cfg, mesh, k), nthreads=os.cpu_count() or 1)
        t_or = time.time() - t1
        rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
        rowmax = np.zeros(len(rp) - 1)
        np.maximum.at(rowmax, rows, np.abs(va))
        pattern = bool(np.array_equal(got.row_ptr, rp) and np.array_equal(got.col_idx, ci))
        bitwise = pattern and bool(np.array_equal(got.vals, va))
        rel = float(np.max(np.abs(got.vals - va) / np.maximum(rowmax[rows], 1e-300))) if pattern else None
        res.append({"op": k.op, "nnz": int(len(va)), "exact_zeros_dropped": int(z), "pattern_bit_exact": pattern,
                    "values_bitwise": bitwise, "max_rel_err_vs_rowmax": rel, "oracle_s": round(t_or, 1)})
    line = {"config": name, "nme": int(me.shape[1]), "nq": int(q.shape[1]), "results": res,
            "deterministic": sha1 == sha2, "seconds": round(time.time() - t0, 1)}
    print(json.dumps(line), flush=True)
    dm.close()
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for n in sys.argv[1:]:
        check(n)
