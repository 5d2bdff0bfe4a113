"""Kernel descriptors with the reference constructors' signatures.

Reference kernel objects (kernels.py:258-387) precompute per-element data on
the CPU (gradients, W = w[me], lambs/mus).  These descriptors only evaluate
the nodal coefficients (``_nodal_values``, kernels.py:268-278) and run the
reference's argument checks; everything per element happens on the B200
inside the numeric phase.
"""

from __future__ import annotations

import numpy as np

from .errors import RangeGuardError


def nodal_values(value, q: np.ndarray):
    """Constant -> (None, float); callable f(q) -> ((nq,) f64, None), with the
    reference's shape check (kernels.py:268-278)."""
    if callable(value):
        out = np.asarray(value(q), dtype=np.float64)
        if out.shape != (q.shape[1],):
            raise ValueError(f"coefficient returned shape {out.shape}, expected ({q.shape[1]},)")
        return np.ascontiguousarray(out), None
    if isinstance(value, np.ndarray):
        out = np.asarray(value, dtype=np.float64)
        if out.shape != (q.shape[1],):
            raise ValueError(f"coefficient has shape {out.shape}, expected ({q.shape[1]},)")
        return np.ascontiguousarray(out), None
    return None, float(value)


class MassKernel:
    """Weighted mass matrix, weight interpolated at the vertices
    (MassKernel, kernels.py:281-303)."""

    symmetric = True
    op = "mass"
    m = 1

    def __init__(self, mesh, weight=1.0):
        self.mesh = mesh
        self.w, self.w_const = nodal_values(weight, mesh.q)


class StiffnessKernel:
    """Scalar stiffness (Laplacian) matrix (StiffnessKernel, kernels.py:306-329)."""

    symmetric = True
    op = "stiffness"
    m = 1

    def __init__(self, mesh):
        self.mesh = mesh


class ElasticKernel:
    """Isotropic linear elasticity, m = d unknowns per node, interleaved dofs
    (ElasticKernel, kernels.py:332-387)."""

    symmetric = True
    op = "elastic"

    def __init__(self, mesh, lamb=1.0, mu=1.0):
        d = mesh.q.shape[0]
        if d not in (2, 3):
            raise ValueError(f"elastic tables are defined for d in {{2, 3}}, got {d}")
        self.mesh = mesh
        self.d = self.m = d
        self.lamb, self.lamb_const = nodal_values(lamb, mesh.q)
        self.mu, self.mu_const = nodal_values(mu, mesh.q)
        lam_n = self.lamb if self.lamb is not None else np.full(mesh.q.shape[1], self.lamb_const)
        mu_n = self.mu if self.mu is not None else np.full(mesh.q.shape[1], self.mu_const)
        bad = lam_n + mu_n <= 0.0
        if np.any(bad):
            node = int(np.flatnonzero(bad)[0])
            raise ValueError(f"Lame parameters must satisfy lamb + mu > 0; violated at node {node}")
        self.lambs_e = self.mus_e = None

    @classmethod
    def per_element(cls, mesh, lambs, mus):
        """Descriptor from per-element Lame sums already scaled by
        vols/(d+1) -- exactly the ``lambs``/``mus`` arrays the reference's
        ElasticKernel keeps (kernels.py:354-356); the device uses them as
        given, so the values are bitwise the reference's."""
        self = cls.__new__(cls)
        d = mesh.q.shape[0]
        if d not in (2, 3):
            raise ValueError(f"elastic tables are defined for d in {{2, 3}}, got {d}")
        nme = mesh.me.shape[1]
        self.mesh = mesh
        self.d = self.m = d
        self.lamb = self.mu = None
        self.lamb_const = self.mu_const = 1.0
        self.lambs_e = np.ascontiguousarray(np.asarray(lambs, dtype=np.float64))
        self.mus_e = np.ascontiguousarray(np.asarray(mus, dtype=np.float64))
        if self.lambs_e.shape != (nme,) or self.mus_e.shape != (nme,):
            raise ValueError(f"lambs/mus must have shape ({nme},), got {self.lambs_e.shape} and {self.mus_e.shape}")
        return self


def _field(value, q, shape_tail, name):
    """Nodal field of shape (nq, *shape_tail): constant array of shape
    shape_tail, callable f(q) -> (*shape_tail, nq) like the reference
    coefficient convention, or an explicit (nq, *shape_tail) array."""
    nq = q.shape[1]
    if value is None:
        return None, np.zeros(shape_tail)
    if callable(value):
        out = np.asarray(value(q), dtype=np.float64)
        if out.shape != tuple(shape_tail) + (nq,):
            raise ValueError(f"{name} returned shape {out.shape}, expected {tuple(shape_tail) + (nq,)}")
        return np.ascontiguousarray(np.moveaxis(out, -1, 0)), None
    arr = np.asarray(value, dtype=np.float64)
    if arr.shape == tuple(shape_tail) or (arr.ndim == 0 and not shape_tail):
        return None, arr.reshape(shape_tail)
    if arr.shape == (nq,) + tuple(shape_tail):
        return np.ascontiguousarray(arr), None
    raise ValueError(f"{name} has shape {arr.shape}; expected {tuple(shape_tail)} or {(nq,) + tuple(shape_tail)}")


class GeneralKernel:
    """General second-order operator -div(A grad u) + div(b u) + c.grad u + a0 u
    (weak form and quadrature in DESIGN.md 3.4).  Row = test
    function, as in the reference.  Not symmetric in general.  ``exact``
    selects bitwise reference-order element arithmetic (see below).

    A: (d, d) constant, (nq, d, d) nodal array or callable q -> (d, d, nq);
    b, c: (d,) constant, (nq, d) nodal or callable q -> (d, nq); a0: scalar,
    (nq,) nodal or callable q -> (nq,).  Missing terms are zero."""

    op = "general"
    m = 1

    def __init__(self, mesh, A=None, b=None, c=None, a0=None, exact=False):
        q = mesh.q
        d = q.shape[0]
        if d not in (1, 2, 3):
            raise RangeGuardError(f"dimension must be 1, 2 or 3, got {d}")
        self.mesh = mesh
        self.A, self.A_const = _field(A, q, (d, d), "A")
        self.b, b_const = _field(b, q, (d,), "b")
        self.c, c_const = _field(c, q, (d,), "c")
        if self.b is None and np.any(b_const != 0):
            self.b = np.ascontiguousarray(np.broadcast_to(b_const, (q.shape[1], d)))
        if self.c is None and np.any(c_const != 0):
            self.c = np.ascontiguousarray(np.broadcast_to(c_const, (q.shape[1], d)))
        if a0 is None:
            self.a0, self.a0_const = None, 0.0
        else:
            self.a0, self.a0_const = nodal_values(a0, q)
        self.symmetric = False
        # exact=True: element values in the reference's operation order
        # (bitwise the oracle).  Default: fused multiply-adds in the local
        # matrix (values within a few ulp of the contributions, far inside the
        # 1e-12-of-row-max bar); the exact-zero pattern is the reference's in
        # both modes (guarded rows are recomputed in reference order).
        self.exact = bool(exact)
        self._packed = None
        self._cols = None

    def packed(self) -> np.ndarray:
        """Nodal coefficients as one 128-byte record per node,
        [A (3x3, zero-padded) | b (3) | c (3) | a0] -- the device layout
        (one cache line per vertex gather instead of 16 scattered loads)."""
        if self._packed is None:
            q = self.mesh.q
            d, nq = q.shape
            p = np.zeros((nq, 16))
            A = self.A if self.A is not None else np.broadcast_to(self.A_const, (nq, d, d))
            for i in range(d):
                p[:, 3 * i:3 * i + d] = A[:, i, :]
            if self.b is not None:
                p[:, 9:9 + d] = self.b
            if self.c is not None:
                p[:, 12:12 + d] = self.c
            p[:, 15] = self.a0 if self.a0 is not None else self.a0_const
            self._packed = p
        return self._packed

    def packed_columns(self):
        """(cols (nq, nv) f64, colmap (16,) int32, consts (16,) f64): the
        record of ``packed()`` with the columns that are constant over the
        nodes (zero padding, absent terms, constant fields) or repeat an
        earlier column (a symmetric A) left out -- what crosses PCIe;
        ``sa_unpack_columns`` rebuilds the 128-byte records on the device,
        bit for bit.  Computed once per coefficient set."""
        if getattr(self, "_cols", None) is None:
            p = self.packed()
            colmap = np.full(16, -1, dtype=np.int32)
            consts = np.zeros(16)
            keep = []
            mirror = {3: 1, 6: 2, 7: 5}   # A[1][0] ~ A[0][1], A[2][0] ~ A[0][2], A[2][1] ~ A[1][2]
            for j in range(16):
                col = p[:, j]
                if col.size == 0 or np.all(col == col[0]):
                    consts[j] = col[0] if col.size else 0.0
                    continue
                k = mirror.get(j)
                if k is not None and colmap[k] >= 0 and np.array_equal(col, p[:, k]):
                    colmap[j] = colmap[k]
                    continue
                colmap[j] = len(keep)
                keep.append(j)
            self._cols = (np.ascontiguousarray(p[:, keep]), colmap, consts)
        return self._cols


def restrict(kernel, mesh_local, nodes: slice, elements):
    """The descriptor ``kernel`` on a sub-mesh (a rank's slab,
    parallel.slab): nodal coefficient arrays cut to the node window
    ``nodes``, per-element arrays to ``elements`` (ascending global ids);
    constants unchanged.  Used by the distributed driver."""
    import copy

    k = copy.copy(kernel)
    k.mesh = mesh_local
    k.__dict__.pop("_pinned_cache", None)
    k.__dict__.pop("_packed", None)
    k.__dict__.pop("_cols", None)
    for name in ("w", "lamb", "mu", "A", "b", "c", "a0"):
        v = getattr(kernel, name, None)
        if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == kernel.mesh.q.shape[1]:
            setattr(k, name, np.ascontiguousarray(v[nodes]))
    for name in ("lambs_e", "mus_e"):
        v = getattr(kernel, name, None)
        if v is not None:
            setattr(k, name, np.ascontiguousarray(np.asarray(v)[elements]))
    if getattr(kernel, "op", None) == "general":
        k._packed = None
    return k
