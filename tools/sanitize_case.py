"""Small assemblies on every numeric path, for compute-sanitizer
(tests/test_gpu_parity.py::test_compute_sanitizer): the two-pass general
operator (cp.async pipeline, fast and exact), the row gather (mass +
stiffness 2D/3D, elastic), the guard fix-up, the compaction."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_3301_b200 as P  # noqa: E402


def main():
    for d, n in ((2, 12), (3, 6)):
        q, me = P.hypercube_arrays(d, n)
        q = P.jitter_interior(q, n, 0.2 if d == 2 else 0.15, 3)
        mesh = P.Mesh(q, me, P.device_volumes(q, me))
        nq = q.shape[1]
        P.assemble_many_b200(mesh, [P.MassKernel(mesh), P.StiffnessKernel(mesh)])
        rng = np.random.default_rng(1)
        f = dict(A=np.eye(d)[None] + 0.1 * rng.random((nq, d, d)), b=rng.random((nq, d)), c=rng.random((nq, d)),
                 a0=rng.random(nq))
        P.assemble_b200(mesh, P.GeneralKernel(mesh, **f))
        P.assemble_b200(mesh, P.GeneralKernel(mesh, exact=True, **f))
        P.assemble_vector_b200(mesh, P.ElasticKernel(mesh, 1.0, 0.5))
    q, me = P.hypercube_arrays(3, 4)   # unjittered: guarded rows + exact zeros
    mesh = P.Mesh(q, me, P.device_volumes(q, me))
    P.assemble_b200(mesh, P.GeneralKernel(mesh, A=np.eye(3)))
    print("sanitize case ok")


if __name__ == "__main__":
    main()
