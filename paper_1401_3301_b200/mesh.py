"""Simplicial meshes: the input side of the assembly path.

``Mesh`` mirrors the reference type (mesh.py:46-101): ``q`` (d, nq) f64,
``me`` (d+1, nme) int64, ``vols`` (nme,) f64, immutable.  The drivers accept
any object with those three attributes, in particular the reference's own
``simplex_asm.Mesh``.

``generate_hypercube_mesh`` restates the reference's Kuhn generator
(mesh.py:104-140) and ``jittered_hypercube_mesh`` adds the seeded interior
jitter of SURVEY.md 8(d) used for every benchmark configuration.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np

from .errors import CapacityError

_MAX_INDEX = np.iinfo(np.int64).max


@dataclass(frozen=True, eq=False)
class Mesh:
    q: np.ndarray     # (d, nq) vertex coordinates
    me: np.ndarray    # (d+1, nme) zero-based connectivity
    vols: np.ndarray  # (nme,) simplex volumes

    @classmethod
    def from_arrays(cls, q, me, vols=None) -> "Mesh":
        """Cast like the reference (mesh.py:54-58).  Volumes, when not given,
        are computed on the B200 from the numpy-det factorisation
        (``device.device_volumes``); the reference computes them with numpy
        on the host, which agrees to a few ulp."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        me = np.ascontiguousarray(me, dtype=np.int64)
        if vols is None:
            from .device import device_volumes

            vols = device_volumes(q, me)
        return cls(q, me, np.ascontiguousarray(vols, dtype=np.float64))

    def validate(self) -> None:
        """The reference's structural checks (mesh.py:72-101), same order and
        messages; the index range check and the volume recomputation run on
        the B200 (sa_mesh_create / sa_mesh_validate), so a 100 M element mesh
        validates in milliseconds.  The recomputed volumes follow the
        numpy-det factorisation and agree with ``compute_volumes`` to ~1e-14
        relative, far inside the 1e-12 tolerance being tested."""
        from .device import DeviceMesh
        from .errors import MeshValidationError

        d = self.d
        me = np.asarray(self.me)
        if me.shape != (d + 1, self.nme):
            raise MeshValidationError(f"connectivity shape {me.shape} does not match ({d + 1}, nme)")
        vols = np.asarray(self.vols)
        # (IndexRangeError naming me[a, k] comes from the device mesh)
        dm = DeviceMesh(self.q, me, None if vols.shape != (self.nme,) else vols)
        try:
            if vols.shape != (self.nme,):
                raise MeshValidationError(f"volume array shape {vols.shape} does not match (nme,)")
            nonpos, mismatch = dm.validate_vols(vols)
        finally:
            dm.close()
        if nonpos >= 0:
            raise MeshValidationError(f"volume of simplex {nonpos} is not positive")
        if mismatch >= 0:
            raise MeshValidationError(f"stored volume of simplex {mismatch} disagrees with its coordinates")

    @property
    def d(self) -> int:
        return self.q.shape[0]

    @property
    def nq(self) -> int:
        return self.q.shape[1]

    @property
    def nme(self) -> int:
        return self.me.shape[1]


def hypercube_arrays(d: int, n: int):
    """(q, me) of the Kuhn triangulation of [0,1]^d with n cells per axis:
    row-major grid points, d! simplices per cell (one per axis permutation),
    the simplices of a cell adjacent (mesh.py:104-140)."""
    if d < 1:
        raise ValueError(f"dimension must be >= 1, got {d}")
    if n < 1:
        raise ValueError(f"subdivision count must be >= 1, got {n}")
    nq = (n + 1) ** d
    nme = math.factorial(d) * n ** d
    if nq > _MAX_INDEX or (d + 1) * nme > _MAX_INDEX:
        raise CapacityError(f"hypercube mesh d={d}, n={n} exceeds the platform index range")
    grid = np.indices((n + 1,) * d).reshape(d, -1)
    q = grid / float(n)
    strides = (n + 1) ** np.arange(d - 1, -1, -1, dtype=np.int64)
    cells = np.indices((n,) * d, dtype=np.int64).reshape(d, -1)
    base = strides @ cells
    me = np.empty((nme, d + 1), dtype=np.int64)
    for p, perm in enumerate(itertools.permutations(range(d))):
        rows = me[p::math.factorial(d)]
        rows[:, 0] = base
        acc = base.copy()
        for j, axis in enumerate(perm):
            acc = acc + strides[axis]
            rows[:, j + 1] = acc
    return q, np.ascontiguousarray(me.T)


def jitter_interior(q: np.ndarray, n: int, amplitude: float, seed: int) -> np.ndarray:
    """interior nodes (all coordinates strictly inside (0,1))
    move by rng.uniform(-a*h, a*h) per coordinate, h = 1/n."""
    q = q.copy()
    h = 1.0 / n
    interior = np.all((q > 0) & (q < 1), axis=0)
    rng = np.random.default_rng(seed)
    q[:, interior] += rng.uniform(-amplitude * h, amplitude * h, size=(q.shape[0], int(interior.sum())))
    return q


def generate_hypercube_mesh(d: int, n: int, vols=None) -> Mesh:
    q, me = hypercube_arrays(d, n)
    return Mesh.from_arrays(q, me, vols)


def jittered_hypercube_mesh(d: int, n: int, seed: int, amplitude: float | None = None, vols=None) -> Mesh:
    """The benchmark meshes: Kuhn cube + seeded interior jitter
    (a = 0.2 in 2D, 0.15 in 3D unless given)."""
    if amplitude is None:
        amplitude = 0.2 if d <= 2 else 0.15
    q, me = hypercube_arrays(d, n)
    q = jitter_interior(q, n, amplitude, seed)
    return Mesh.from_arrays(q, me, vols)


def device_hypercube_arrays(d: int, n: int, seed: int | None = None, amplitude: float | None = None,
                            device=None, host: bool = False):
    """The benchmark mesh generated on the B200 (sa_kuhn_mesh): bitwise the
    arrays of ``hypercube_arrays`` (+ ``jitter_interior`` when ``seed`` is
    given; a = 0.2 in 2D, 0.15 in 3D unless given).  Returns CUDA tensors
    (q (d, nq) f64, me (d+1, nme) int64), or numpy arrays when ``host``
    (one device->host copy instead of the host generator)."""
    import ctypes

    import torch

    from . import _lib
    from .device import _require_cuda, _stream_ptr

    if d < 1 or d > 3:
        raise ValueError(f"dimension must be 1, 2 or 3, got {d}")
    if n < 1:
        raise ValueError(f"subdivision count must be >= 1, got {n}")
    dev = _require_cuda(device)
    nq, nme = (n + 1) ** d, math.factorial(d) * n ** d
    q = torch.empty((d, nq), dtype=torch.float64, device=dev)
    me = torch.empty((d + 1, nme), dtype=torch.int64, device=dev)
    lo = rg = 0.0
    s_hi = s_lo = i_hi = i_lo = 0
    if seed is not None:
        if amplitude is None:
            amplitude = 0.2 if d <= 2 else 0.15
        h = 1.0 / n
        lo, hi = -amplitude * h, amplitude * h     # numpy: uniform(lo, hi) = lo + (hi - lo) u
        rg = hi - lo
        st = np.random.PCG64(seed).state["state"]  # default_rng(seed)'s seeded generator
        s_hi, s_lo = st["state"] >> 64, st["state"] & ((1 << 64) - 1)
        i_hi, i_lo = st["inc"] >> 64, st["inc"] & ((1 << 64) - 1)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().sa_kuhn_mesh(d, n, 1 if seed is not None else 0, lo, rg, s_hi, s_lo, i_hi, i_lo,
                                            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(me.data_ptr()),
                                            _stream_ptr()))
    if host:
        return q.cpu().numpy(), me.cpu().numpy()
    return q, me


def kuhn_slab_window(d: int, n: int, nb0: int, nb1: int) -> tuple[int, int, int, int]:
    """Node window [v0, v1) and element window [e0, e1) of the Kuhn mesh
    (mesh.py:104-140: nodes row-major with the first coordinate slowest,
    cells likewise, d! simplices per cell) that hold every element touching
    nodes [nb0, nb1): the node planes i0-1 .. i1+1 around the block and the
    cells between them."""
    P, C, dfact = (n + 1) ** (d - 1), n ** (d - 1), math.factorial(d)
    if nb1 <= nb0:
        return nb0, nb0, 0, 0
    i0, i1 = nb0 // P, (nb1 - 1) // P
    c_lo, c_hi = max(i0 - 1, 0), min(i1, n - 1)
    return max(i0 - 1, 0) * P, (min(i1 + 1, n) + 1) * P, c_lo * C * dfact, (c_hi + 1) * C * dfact


def device_hypercube_slab(d: int, n: int, m: int, row_begin: int, row_end: int, seed: int | None = None,
                          amplitude: float | None = None, device=None):
    """A rank's slab of the (jittered) Kuhn mesh generated directly on the
    B200 (sa_kuhn_slab), without the global mesh: the node planes around
    dof rows [row_begin, row_end) and the cells between them (first
    coordinate slowest, mesh.py:123-139), node ids relative to the window.
    A superset of parallel.slab's elements in the same (ascending) order --
    elements that touch no row of the block contribute nothing to it -- so
    the block assembles bitwise the rows of the full mesh.  Returns a
    parallel.Slab with host arrays (vols None: computed by the device mesh)."""
    import ctypes

    import torch

    from . import _lib
    from .device import _require_cuda, _stream_ptr
    from .parallel import Slab

    dev = _require_cuda(device)
    nb0, nb1 = row_begin // m, row_end // m
    v0, v1, e0, e1 = kuhn_slab_window(d, n, nb0, nb1)
    q = torch.empty((d, v1 - v0), dtype=torch.float64, device=dev)
    me = torch.empty((d + 1, e1 - e0), dtype=torch.int64, device=dev)
    lo = rg = 0.0
    s_hi = s_lo = i_hi = i_lo = 0
    if seed is not None:
        if amplitude is None:
            amplitude = 0.2 if d <= 2 else 0.15
        h = 1.0 / n
        lo, hi = -amplitude * h, amplitude * h
        rg = hi - lo
        st = np.random.PCG64(seed).state["state"]
        s_hi, s_lo = st["state"] >> 64, st["state"] & ((1 << 64) - 1)
        i_hi, i_lo = st["inc"] >> 64, st["inc"] & ((1 << 64) - 1)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().sa_kuhn_slab(d, n, 1 if seed is not None else 0, lo, rg, s_hi, s_lo, i_hi, i_lo,
                                            v0, v1, e0, e1, ctypes.c_void_p(q.data_ptr()),
                                            ctypes.c_void_p(me.data_ptr()), _stream_ptr()))
    return Slab(q=q.cpu().numpy(), me=me.cpu().numpy(), vols=None, node_lo=v0, row_begin=m * (nb0 - v0),
                row_end=m * (nb1 - v0), col_offset=m * v0, elements=np.arange(e0, e1))
