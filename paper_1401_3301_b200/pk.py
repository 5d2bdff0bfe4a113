"""Order-k node lattices and the Pk mass matrix.

Host side, restating the reference's element-independent Pk machinery so the
package stands alone (the reference is not present on a GPU box):

* ``multi_index_lattice(d, k)`` -- exponent tuples of length d+1 summing to
  k, descending lexicographic (mesh.py:147-164): the local node numbering.
* ``pk_mass_coeffs(d, k)`` -- the exact-rational table C with the local mass
  matrix d! |K| C (kernels.py:178-255, paper Eq. 4 moments
  (prod n_i!)/(d + sum n_i)!), rounded once to float.
* ``build_pk_mesh(mesh, k)`` -- the lattice over a simplicial mesh
  (mesh.py:195-243): vertices keep their ids, added nodes are keyed by their
  exact (vertex, integer weight) pairs and numbered in first-seen order
  (element-major, local-minor); vectorised here.

The assembly itself (``assemble_mass_pk_b200``, assembly.py) runs on the
B200: sa_pk_* in csrc/sa_pk.cu.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .errors import RangeGuardError


def multi_index_lattice(d: int, k: int) -> list[tuple[int, ...]]:
    out: list[tuple[int, ...]] = []

    def rec(prefix, left, slots):
        if slots == 1:
            out.append(prefix + (left,))
            return
        for head in range(left, -1, -1):
            rec(prefix + (head,), left - head, slots - 1)

    rec((), k, d + 1)
    return out


def _poly_mul_linear(poly: dict, slot: int, a: Fraction, b: Fraction) -> dict:
    """poly * (a * x_slot + b) over exponent-tuple monomials."""
    res: dict = {}
    for mono, c in poly.items():
        up = mono[:slot] + (mono[slot] + 1,) + mono[slot + 1:]
        res[up] = res.get(up, Fraction(0)) + c * a
        if b:
            res[mono] = res.get(mono, Fraction(0)) + c * b
    return res


def _lattice_basis(alpha: tuple[int, ...], k: int) -> dict:
    """prod_slots prod_{j < alpha_s} (k x_s - j) / (j + 1) in barycentric
    monomials: 1 at the lattice point alpha/k, 0 at the others."""
    poly = {(0,) * len(alpha): Fraction(1)}
    for s, a_s in enumerate(alpha):
        for j in range(a_s):
            poly = _poly_mul_linear(poly, s, Fraction(k, j + 1), Fraction(-j, j + 1))
    return poly


def _moment(d: int, expo: tuple[int, ...]) -> Fraction:
    return Fraction(math.prod(math.factorial(e) for e in expo), math.factorial(d + sum(expo)))


@dataclass(frozen=True, eq=False)
class PkCoeffTable:
    """Local mass matrix of any d-simplex K is d! |K| C (lattice order)."""

    d: int
    k: int
    ndfe: int
    lattice: tuple
    C: np.ndarray
    exact: tuple


def pk_mass_coeffs(d: int, k: int) -> PkCoeffTable:
    if not 1 <= d <= 3:
        raise RangeGuardError(f"mass coefficients support 1 <= d <= 3, got d={d}")
    if not 1 <= k <= 6:
        raise RangeGuardError(f"mass coefficients support 1 <= k <= 6, got k={k}")
    lat = multi_index_lattice(d, k)
    basis = [list(_lattice_basis(a, k).items()) for a in lat]
    n = len(lat)
    ex = [[Fraction(0)] * n for _ in range(n)]
    for a in range(n):
        for b in range(a, n):
            s = Fraction(0)
            for mu, cm in basis[a]:
                for nu, cn in basis[b]:
                    s += cm * cn * _moment(d, tuple(x + y for x, y in zip(mu, nu)))
            ex[a][b] = ex[b][a] = s
    return PkCoeffTable(d, k, n, tuple(lat), np.array([[float(x) for x in row] for row in ex]),
                        tuple(tuple(r) for r in ex))


@dataclass(frozen=True, eq=False)
class PkMesh:
    d: int
    k: int
    q: np.ndarray     # (d, nq) node coordinates
    me: np.ndarray    # (ndfe, nme) node connectivity
    vols: np.ndarray  # (nme,) simplex volumes of the source mesh

    @property
    def ndfe(self) -> int:
        return self.me.shape[0]

    @property
    def nq(self) -> int:
        return self.q.shape[1]

    @property
    def nme(self) -> int:
        return self.me.shape[1]


def build_pk_mesh(mesh, k: int) -> PkMesh:
    if k < 1:
        raise ValueError(f"polynomial order must be >= 1, got {k}")
    q0, me0 = np.asarray(mesh.q), np.asarray(mesh.me, dtype=np.int64)
    d, nq0, nme = q0.shape[0], q0.shape[1], me0.shape[1]
    lat = multi_index_lattice(d, k)
    ndfe = len(lat)
    me = np.empty((ndfe, nme), dtype=np.int64)
    # keys of the non-vertex lattice points: (vertex id, weight) pairs of the
    # nonzero slots sorted by vertex id, padded with -1 to 2(d+1) columns
    keys, where = [], []
    for loc, a in enumerate(lat):
        if max(a) == k:
            me[loc] = me0[a.index(k)]
            continue
        nz = [s for s in range(d + 1) if a[s]]
        ids = me0[nz].T                                   # (nme, len(nz))
        w = np.array([a[s] for s in nz], dtype=np.int64)
        order = np.argsort(ids, axis=1, kind="stable")
        kk = np.full((nme, 2 * (d + 1)), -1, dtype=np.int64)
        kk[:, 0:2 * len(nz):2] = np.take_along_axis(ids, order, axis=1)
        kk[:, 1:2 * len(nz):2] = w[order]
        keys.append(kk)
        where.append(loc)
    if not keys:
        return PkMesh(d, k, q0, me, np.asarray(mesh.vols))
    # first-seen order over (element, local point): element-major
    allk = np.stack(keys, axis=1).reshape(-1, 2 * (d + 1))  # row = e * nl + j
    uniq, first, inv = np.unique(allk, axis=0, return_index=True, return_inverse=True)
    rank = np.empty(len(uniq), dtype=np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(len(uniq))
    node = (nq0 + rank[inv.reshape(-1)]).reshape(nme, len(where))
    alphas = np.array(lat, dtype=np.float64).T / k          # (d+1, ndfe)
    newq = np.empty((d, len(uniq)))
    for j, loc in enumerate(where):
        me[loc] = node[:, j]
    # coordinates of each new node from its first-seen (element, local point),
    # as the reference computes them: q[:, verts] @ alphas[:, local]
    for u, f in enumerate(first):
        e, j = divmod(int(f), len(where))
        newq[:, u] = q0[:, me0[:, e]] @ alphas[:, where[j]]
    q = np.hstack([q0, newq[:, np.argsort(rank)]]) if len(uniq) else q0
    return PkMesh(d, k, q, me, np.asarray(mesh.vols))
