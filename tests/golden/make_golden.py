"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container only (it imports /root/reference):
    OPENBLAS_CORETYPE=SkylakeX python tests/golden/make_golden.py
Writes tests/golden/*.npz.  Each fixture holds the mesh (q, me, vols as the
reference's Mesh.from_arrays computed them), the coefficients, and the CSR
(row_ptr, col_idx, vals) that the reference's assemble_optv2 /
assemble_vector_optv2 returned.  The general operator (absent from the
reference) is assembled by the reference drivers with the numpy kernel class
below, and its closed forms are checked here against the
reference's own quadrature oracle (pkg/tests/oracles.py).
"""

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")
import simplex_asm as sa  # noqa: E402
import oracles as ro  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def jittered(d, n, amp, seed):
    m = sa.generate_hypercube_mesh(d, n)
    if amp == 0:
        return m
    q = m.q.copy()
    h = 1.0 / n
    interior = np.all((q > 0) & (q < 1), axis=0)
    rng = np.random.default_rng(seed)
    q[:, interior] += rng.uniform(-amp * h, amp * h, size=(d, int(interior.sum())))
    return sa.Mesh.from_arrays(q, m.me)


class NumpyGeneralKernel:
    """General operator kernel in the reference kernel protocol (batched),
    arithmetic order of DESIGN.md 3.4 (no fma)."""

    symmetric = False

    def __init__(self, mesh, A, b, c, a0):
        d = mesh.d
        self.mesh, self.d = mesh, d
        me = mesh.me
        self.G = sa.compute_gradients(mesh)
        self.vol = mesh.vols
        self.Av = A[me]          # (d+1, nme, d, d)
        self.bv = b[me]          # (d+1, nme, d)
        self.cv = c[me]
        self.a0v = a0[me]        # (d+1, nme)
        As = self.Av[0].copy(); bs = self.bv[0].copy(); cs = self.cv[0].copy(); a0s = self.a0v[0].copy()
        for g in range(1, d + 1):
            As = As + self.Av[g]; bs = bs + self.bv[g]; cs = cs + self.cv[g]; a0s = a0s + self.a0v[g]
        self.As, self.bs, self.cs, self.a0s = As, bs, cs, a0s
        self.s1 = self.vol / (d + 1)
        self.s2 = self.vol / ((d + 1) * (d + 2))
        self.den = (d + 1) * (d + 2) * (d + 3)

    def batched(self, alpha, beta):
        d, G = self.d, self.G
        ga, gb = G[:, alpha, :], G[:, beta, :]
        AG = []
        for i in range(d):
            t = self.As[:, i, 0] * gb[:, 0]
            for j in range(1, d):
                t = t + self.As[:, i, j] * gb[:, j]
            AG.append(t)
        diff = ga[:, 0] * AG[0]
        conv = (self.bs[:, 0] + self.bv[beta][:, 0]) * ga[:, 0]
        tran = (self.cs[:, 0] + self.cv[alpha][:, 0]) * gb[:, 0]
        for i in range(1, d):
            diff = diff + ga[:, i] * AG[i]
            conv = conv + (self.bs[:, i] + self.bv[beta][:, i]) * ga[:, i]
            tran = tran + (self.cs[:, i] + self.cv[alpha][:, i]) * gb[:, i]
        coef = (2.0 if alpha == beta else 1.0) / self.den
        rea = (coef * self.vol) * ((self.a0s + self.a0v[alpha]) + self.a0v[beta])
        return ((diff * self.s1 - conv * self.s2) + tran * self.s2) + rea

    def single(self, alpha, beta, k):
        return float(self.batched(alpha, beta)[k])


def general_fields(mesh, seed):
    """C5 recipe: A = I + 0.5 R R^T / 3, b, c ~ N(0,1), a0 ~ U[0,1)."""
    d, nq = mesh.d, mesh.nq
    rng = np.random.default_rng(seed)
    R = rng.standard_normal((nq, d, d))
    A = np.eye(d)[None] + 0.5 * np.einsum("nij,nkj->nik", R, R) / 3.0
    b = rng.standard_normal((nq, d))
    c = rng.standard_normal((nq, d))
    a0 = rng.uniform(0.0, 1.0, nq)
    return A, b, c, a0


def save(name, mesh, mat, **extra):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), q=mesh.q, me=mesh.me, vols=mesh.vols,
                        row_ptr=mat.row_ptr, col_idx=mat.col_idx, vals=mat.vals,
                        shape=np.array(mat.shape), **extra)


def check_general_quadrature():
    """Closed forms vs the reference's collapsed-Gauss quadrature (oracles.py:16-63)."""
    worst = 0.0
    for d in (1, 2, 3):
        rng = np.random.default_rng(100 + d)
        verts = rng.random((d, d + 1)) * 2 - 0.5
        mesh = sa.Mesh.from_arrays(verts, np.arange(d + 1).reshape(d + 1, 1))
        A = rng.standard_normal((d + 1, d, d)); b = rng.standard_normal((d + 1, d))
        c = rng.standard_normal((d + 1, d)); a0 = rng.random(d + 1)
        K = NumpyGeneralKernel(mesh, A, b, c, a0)
        pts, w = ro.simplex_quadrature(d, 6)
        phys = verts[:, :1].T + pts @ (verts[:, 1:] - verts[:, :1]).T
        lam = ro.barycentric_at(verts, phys)            # (d+1, N)
        scale = abs(np.linalg.det(verts[:, 1:] - verts[:, :1]))
        G = sa.compute_gradients(mesh)[0]                # (d+1, d)
        Aq = np.einsum("gn,gij->nij", lam, A); bq = lam.T @ b; cq = lam.T @ c; a0q = lam.T @ a0
        for al in range(d + 1):
            for be in range(d + 1):
                integrand = (np.einsum("i,nij,j->n", G[al], Aq, G[be]) - lam[be] * (bq @ G[al])
                             + (cq @ G[be]) * lam[al] + a0q * lam[be] * lam[al])
                exact = float(np.dot(w, integrand) * scale)
                got = float(K.batched(al, be)[0])
                worst = max(worst, abs(got - exact) / max(1.0, abs(exact)))
    return worst


def main():
    manifest = {"numpy": np.__version__, "openblas_coretype": os.environ.get("OPENBLAS_CORETYPE", "auto"),
                "cases": []}
    cases = [(1, 40, 0.0, 0), (1, 40, 0.2, 5), (2, 12, 0.0, 0), (2, 15, 0.2, 11), (3, 5, 0.0, 0),
             (3, 6, 0.15, 13), (3, 8, 0.15, 14)]
    for d, n, amp, seed in cases:
        mesh = jittered(d, n, amp, seed)
        tag = f"d{d}_n{n}_{'jit' if amp else 'kuhn'}"
        w = 1.0 + mesh.q[0] ** 2 + 0.5 * mesh.q[-1]
        m = sa.assemble_optv2(mesh, sa.MassKernel(mesh, lambda q: 1.0 + q[0] ** 2 + 0.5 * q[-1]))
        save(f"mass_{tag}", mesh, m, w=w)
        m1 = sa.assemble_optv2(mesh, sa.MassKernel(mesh))
        save(f"mass1_{tag}", mesh, m1)
        s = sa.assemble_optv2(mesh, sa.StiffnessKernel(mesh))
        save(f"stiff_{tag}", mesh, s)
        manifest["cases"] += [f"mass_{tag}", f"mass1_{tag}", f"stiff_{tag}"]
        if d >= 2:
            lam = 1.0 + mesh.q[0]
            mu = 0.5 + mesh.q[-1] ** 2
            e = sa.assemble_vector_optv2(mesh, sa.ElasticKernel(mesh, lambda q: 1.0 + q[0], lambda q: 0.5 + q[-1] ** 2))
            save(f"elastic_{tag}", mesh, e, lamb=lam, mu=mu)
            ec = sa.assemble_vector_optv2(mesh, sa.ElasticKernel(mesh, 1.0, 0.5))
            save(f"elasticc_{tag}", mesh, ec)
            manifest["cases"] += [f"elastic_{tag}", f"elasticc_{tag}"]
        A, b, c, a0 = general_fields(mesh, seed + 1000)
        g = sa.assemble_optv2(mesh, NumpyGeneralKernel(mesh, A, b, c, a0))
        save(f"general_{tag}", mesh, g, A=A, b=b, c=c, a0=a0)
        manifest["cases"].append(f"general_{tag}")
    manifest["general_quadrature_max_rel_err"] = check_general_quadrature()
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
