"""CPU oracle for the P1 assembly path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` (as the checker) and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
module.  The product package (``paper_1401_3301_b200``) never does.

It wraps ``p1_oracle.c`` (a C restatement of the reference's numerics,
see that file's header for the file:line map) with ctypes.  The oracle is
pinned against the live reference by ``tests/golden/make_golden.py``
(bitwise CSR equality on the committed fixtures).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")

CORES = {"SkylakeX": 0, "Haswell": 1}
OPS = {"mass": 0, "stiffness": 1, "elastic": 2, "general": 3}

OR_OK, OR_DEGENERATE, OR_BAD_ARG, OR_NOMEM = 0, 1, 2, 3


class OracleDegenerate(Exception):
    def __init__(self, element):
        self.element = element
        super().__init__(f"simplex {element} is degenerate (zero volume)")


def build() -> str:
    """Compile p1_oracle.c with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "p1_oracle.c"))
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        dp = ctypes.POINTER(ctypes.c_double)
        L.or_volumes.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, dp, i64p,
                                 ctypes.c_int, dp, i64p]
        L.or_gradients.argtypes = L.or_volumes.argtypes
        L.or_assemble_block.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, dp, i64p,
                                        ctypes.c_int64, ctypes.c_int64,
                                        ctypes.POINTER(i64p), ctypes.POINTER(i64p),
                                        ctypes.POINTER(dp), i64p]
        L.or_assemble_threaded.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, dp, i64p,
                                           ctypes.c_int, i64p, ctypes.POINTER(i64p),
                                           ctypes.POINTER(i64p), ctypes.POINTER(dp)]
        L.or_free.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


class _OrOp(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int), ("d", ctypes.c_int), ("m", ctypes.c_int),
                ("core", ctypes.c_int)] + [
        (name, ctypes.POINTER(ctypes.c_double))
        for name in ("w", "lamb", "mu", "tabQ", "tabS", "A", "b", "c", "a0", "vols")
    ]


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None


def _i64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _prep(q, me):
    q = np.ascontiguousarray(q, dtype=np.float64)
    me = np.ascontiguousarray(me, dtype=np.int64)
    return q, me


def volumes(q, me, core="SkylakeX") -> np.ndarray:
    """mesh.py:29-43 restated (numpy det path, glibc log/exp)."""
    q, me = _prep(q, me)
    d, nq = q.shape
    nme = me.shape[1]
    out = np.empty(nme)
    bad = np.zeros(1, dtype=np.int64)
    rc = lib().or_volumes(d, nq, nme, _dp(q), _i64p(me), CORES[core], _dp(out), _i64p(bad))
    if rc == OR_DEGENERATE:
        raise OracleDegenerate(int(bad[0]))
    if rc:
        raise RuntimeError(f"or_volumes rc={rc}")
    return out


def gradients(q, me, core="SkylakeX") -> np.ndarray:
    """kernels.py:49-65 restated (OpenBLAS dgesv operation order)."""
    q, me = _prep(q, me)
    d, nq = q.shape
    nme = me.shape[1]
    out = np.empty((nme, d + 1, d))
    bad = np.zeros(1, dtype=np.int64)
    rc = lib().or_gradients(d, nq, nme, _dp(q), _i64p(me), CORES[core], _dp(out), _i64p(bad))
    if rc == OR_DEGENERATE:
        raise OracleDegenerate(int(bad[0]))
    if rc:
        raise RuntimeError(f"or_gradients rc={rc}")
    return out


def elastic_tables(d: int):
    """Q[n][l] = Bl[n]^T C0 Bl[l], S[n][l] = Bl[n]^T C1 Bl[l]
    (restates kernels.py:114-138 from the Voigt definitions)."""
    nv = 3 * (d - 1)
    shear = [(0, 1)] if d == 2 else [(0, 1), (1, 2), (0, 2)]
    bl = []
    for l in range(d):
        b = np.zeros((nv, d))
        b[l, l] = 1.0
        for row, (i, j) in enumerate(shear, start=d):
            if l == i:
                b[row, j] = 1.0
            elif l == j:
                b[row, i] = 1.0
        bl.append(b)
    c0 = np.zeros((nv, nv))
    c0[:d, :d] = 1.0
    c1 = np.eye(nv)
    c1[:d, :d] *= 2.0
    Q = np.empty((d, d, d, d))
    S = np.empty((d, d, d, d))
    for n in range(d):
        for l in range(d):
            Q[n, l] = bl[n].T @ c0 @ bl[l]
            S[n, l] = bl[n].T @ c1 @ bl[l]
    return Q, S


class OracleOp:
    """Operator + nodal coefficients, in the form the C oracle consumes."""

    def __init__(self, kind, d, vols, *, w=None, lamb=None, mu=None, A=None, b=None, c=None,
                 a0=None, core="SkylakeX"):
        self.kind = kind
        self.d = d
        self.m = d if kind == "elastic" else 1
        self.keep = []
        arr = lambda x: None if x is None else self._keep(np.ascontiguousarray(x, dtype=np.float64))
        self.s = _OrOp()
        self.s.op = OPS[kind]
        self.s.d = d
        self.s.m = self.m
        self.s.core = CORES[core]
        self.s.vols = _dp(arr(vols))
        if kind == "mass":
            self.s.w = _dp(arr(w))
        if kind == "elastic":
            Q, S = elastic_tables(d)
            self.s.tabQ = _dp(arr(Q.reshape(-1)))
            self.s.tabS = _dp(arr(S.reshape(-1)))
            self.s.lamb = _dp(arr(lamb))
            self.s.mu = _dp(arr(mu))
        if kind == "general":
            self.s.A = _dp(arr(A))
            self.s.b = _dp(arr(b))
            self.s.c = _dp(arr(c))
            self.s.a0 = _dp(arr(a0))

    def _keep(self, a):
        self.keep.append(a)
        return a


def _take(ptr, n, dtype):
    if n == 0:
        out = np.empty(0, dtype=dtype)
    else:
        ctype = ctypes.c_int64 if dtype == np.int64 else ctypes.c_double
        buf = ctypes.cast(ptr, ctypes.POINTER(ctype * n)).contents
        out = np.frombuffer(buf, dtype=dtype).copy()
    lib().or_free(ptr)
    return out


def assemble_block(q, me, op: OracleOp, row_begin=0, row_end=None):
    """Row block [row_begin, row_end) of the optv2 CSR: (row_ptr, col_idx, vals)
    with row_ptr relative to the block."""
    q, me = _prep(q, me)
    nq = q.shape[1]
    nme = me.shape[1]
    ndof = op.m * nq
    if row_end is None:
        row_end = ndof
    i64p = ctypes.POINTER(ctypes.c_int64)
    dp = ctypes.POINTER(ctypes.c_double)
    rp, ci, va = i64p(), i64p(), dp()
    nnz = ctypes.c_int64(0)
    rc = lib().or_assemble_block(ctypes.byref(op.s), nq, nme, _dp(q), _i64p(me), row_begin, row_end,
                                 ctypes.byref(rp), ctypes.byref(ci), ctypes.byref(va),
                                 ctypes.byref(nnz))
    if rc:
        raise RuntimeError(f"or_assemble_block rc={rc}")
    n = nnz.value
    return (_take(rp, row_end - row_begin + 1, np.int64), _take(ci, n, np.int64),
            _take(va, n, np.float64))


def assemble(q, me, op: OracleOp, nthreads: int = 1):
    """Full optv2 CSR (row_ptr, col_idx, vals), rows split over nthreads."""
    q, me = _prep(q, me)
    nq = q.shape[1]
    nme = me.shape[1]
    ndof = op.m * nq
    i64p = ctypes.POINTER(ctypes.c_int64)
    dp = ctypes.POINTER(ctypes.c_double)
    rp, ci, va = i64p(), i64p(), dp()
    nnz = ctypes.c_int64(0)
    rc = lib().or_assemble_threaded(ctypes.byref(op.s), nq, nme, _dp(q), _i64p(me), nthreads,
                                    ctypes.byref(nnz), ctypes.byref(rp), ctypes.byref(ci),
                                    ctypes.byref(va))
    if rc:
        raise RuntimeError(f"or_assemble_threaded rc={rc}")
    n = nnz.value
    return _take(rp, ndof + 1, np.int64), _take(ci, n, np.int64), _take(va, n, np.float64)


def assemble_mass_pk(me, vols, C, d: int, nq: int):
    """Pk mass matrix, CPU restatement of assemble_mass_pk (assembly.py:265-292)
    and its canonical constructor (sparse.py:85-133): element-major triplets
    (beta outer, alpha inner within an element), value (d! * C[a, b]) * vol,
    exact zeros skipped, stable sort by (row, col), left-to-right sums,
    exact-zero sums dropped.  Returns (row_ptr, col_idx, vals).  Test
    infrastructure only (numpy; small meshes)."""
    me = np.asarray(me, dtype=np.int64)
    vols = np.asarray(vols, dtype=np.float64)
    ndfe, nme = me.shape
    dfact = float(math.factorial(d))
    vals = np.empty((ndfe * ndfe, nme))
    rows = np.empty((ndfe * ndfe, nme), dtype=np.int64)
    cols = np.empty((ndfe * ndfe, nme), dtype=np.int64)
    l = 0
    for b in range(ndfe):
        for a in range(ndfe):
            vals[l] = dfact * C[a, b] * vols
            rows[l] = me[a]
            cols[l] = me[b]
            l += 1
    v, r, c = vals.ravel(order="F"), rows.ravel(order="F"), cols.ravel(order="F")
    keep = v != 0.0
    v, r, c = v[keep], r[keep], c[keep]
    order = np.lexsort((c, r))
    v, r, c = v[order], r[order], c[order]
    if len(v):
        start = np.ones(len(v), dtype=bool)
        start[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        seg = np.cumsum(start) - 1
        sums = np.bincount(seg, weights=v)
        r, c = r[start], c[start]
        nzs = sums != 0.0
        r, c, sums = r[nzs], c[nzs], sums[nzs]
    else:
        sums = v
    row_ptr = np.zeros(nq + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=nq), out=row_ptr[1:])
    return row_ptr, c, sums
