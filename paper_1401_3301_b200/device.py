"""Device layer: torch CUDA buffers around the C ABI (include/simplex_asm_b200.h).

PyTorch is used for device memory, streams and transfers only; every
numeric step runs in the sm_100a library.  There is no CPU fallback: without
CUDA or the library these classes raise ExtensionMissingError.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ExtensionMissingError

try:
    import torch
except Exception as exc:  # pragma: no cover
    raise ExtensionMissingError(f"torch is required for device buffers: {exc}") from exc

OP_BITS = {"mass": _lib.SA_OP_MASS, "stiffness": _lib.SA_OP_STIFF, "elastic": _lib.SA_OP_ELASTIC,
           "general": _lib.SA_OP_GENERAL}


def _require_cuda(device):
    if not torch.cuda.is_available():
        raise ExtensionMissingError("no CUDA device: the B200 assembly path has no CPU fallback")
    return torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _to_dev(x, dtype, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype, non_blocking=True).contiguous()
    t = torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device=device, dtype=dtype, non_blocking=True).contiguous()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


class DeviceMesh:
    """A mesh resident on one B200: q (padded AoS f64), me (int32 AoS), vols.

    ``q`` (d, nq) and ``me`` (d+1, nme) are host arrays (numpy, the reference
    layout) or CUDA tensors.  ``vols=None`` computes volumes on the device.
    """

    def __init__(self, q, me, vols=None, *, core: str = "SkylakeX", device=None, stream=None, nq: int | None = None,
                 me32=None):
        dev = _require_cuda(device)
        L = _lib.load()
        self.device = dev
        self.core = core
        with torch.cuda.device(dev):
            # q=None (with nq): connectivity only; set_coords() later -- the
            # symbolic phase can run while the coordinates upload
            qd = _to_dev(q, torch.float64, dev) if q is not None else None
            # me32: the first rows of the connectivity already on the device
            # as int32 (upload_connectivity); ``me`` then holds the remaining
            # int64 rows (or None)
            med = _to_dev(me, torch.int64, dev) if me is not None else None
            rows32 = int(me32.shape[0]) if me32 is not None else 0
            rows = rows32 + (int(med.shape[0]) if med is not None and med.dim() == 2 else 0)
            vd = _to_dev(vols, torch.float64, dev) if vols is not None else None
            self.d = rows - 1 if qd is None else int(qd.shape[0])
            self.nq = int(nq) if qd is None else int(qd.shape[1])
            some = me32 if me32 is not None else med
            self.nme = int(some.shape[1]) if some is not None and some.dim() == 2 else 0
            if rows != self.d + 1:
                raise ValueError(f"connectivity with {rows} rows does not match ({self.d + 1}, nme)")
            h = ctypes.c_void_p()
            if me32 is not None:
                rc = L.sa_mesh_create_split(self.d, self.nq, self.nme, _ptr(qd), _ptr(me32), rows32, _ptr(med), _ptr(vd),
                                            _lib.SA_CORE[core], dev.index, _stream_ptr(stream), ctypes.byref(h))
            else:
                rc = L.sa_mesh_create(self.d, self.nq, self.nme, _ptr(qd), _ptr(med), _ptr(vd), _lib.SA_CORE[core],
                                      dev.index, _stream_ptr(stream), ctypes.byref(h))
            _lib.check(rc)
        self._h = h
        self._plans = {}

    @property
    def handle(self):
        return self._h

    def set_coords(self, q, vols=None, stream=None):
        """Coordinates (and volumes; computed on the device when None) of a
        mesh created with q=None (sa_mesh_set_coords)."""
        with torch.cuda.device(self.device):
            qd = _to_dev(q, torch.float64, self.device)
            vd = _to_dev(vols, torch.float64, self.device) if vols is not None else None
            _lib.check(_lib.load().sa_mesh_set_coords(self._h, _ptr(qd), _ptr(vd), _stream_ptr(stream)))

    def vols(self, stream=None) -> "torch.Tensor":
        out = torch.empty(self.nme, dtype=torch.float64, device=self.device)
        _lib.check(_lib.load().sa_mesh_vols(self._h, _ptr(out), _stream_ptr(stream)))
        return out

    def validate_vols(self, vols, stream=None) -> tuple[int, int]:
        """(first element with a non-positive stored volume, first element
        whose stored volume disagrees with its coordinates by more than 1e-12
        relative); -1 = none.  The volumes are recomputed on the device
        (sa_mesh_validate; reference mesh.py:92-101)."""
        with torch.cuda.device(self.device):
            vd = _to_dev(vols, torch.float64, self.device)
            a, b = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(_lib.load().sa_mesh_validate(self._h, _ptr(vd), ctypes.byref(a), ctypes.byref(b),
                                                    _stream_ptr(stream)))
        return a.value, b.value

    def plan(self, m: int = 1, row_begin: int = 0, row_end: int | None = None, stream=None) -> "Plan":
        if row_end is None:
            row_end = m * self.nq
        key = (m, row_begin, row_end)
        p = self._plans.get(key)
        if p is None:
            p = Plan(self, m, row_begin, row_end, stream)
            self._plans[key] = p
        return p

    def close(self):
        for p in self._plans.values():
            p.close()
        self._plans.clear()
        if getattr(self, "_h", None):
            _lib.load().sa_mesh_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:
            pass


@dataclass
class DeviceCSR:
    """Block CSR on the device: indptr int64 (relative), indices int32 (global
    column dofs), vals f64; rows [row_begin, row_end) of an ncols matrix."""

    row_begin: int
    row_end: int
    ncols: int
    indptr: "torch.Tensor"
    indices: "torch.Tensor"
    vals: "torch.Tensor"

    @property
    def nnz(self) -> int:
        return int(self.vals.numel())


class Plan:
    """Symbolic phase of one dof-row block (sa_plan)."""

    def __init__(self, dmesh: DeviceMesh, m: int, row_begin: int, row_end: int, stream=None):
        L = _lib.load()
        self.dmesh = dmesh
        self.m = m
        self.row_begin, self.row_end = row_begin, row_end
        h = ctypes.c_void_p()
        with torch.cuda.device(dmesh.device):
            _lib.check(L.sa_plan_create(dmesh.handle, m, row_begin, row_end, _stream_ptr(stream), ctypes.byref(h)))
        self._h = h
        nr, nnz, md = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(L.sa_plan_info(h, ctypes.byref(nr), ctypes.byref(nnz), ctypes.byref(md)))
        self.nrows, self.nnz, self.max_row_nodes = nr.value, nnz.value, md.value
        self._pattern = None

    @property
    def handle(self):
        return self._h

    def stats(self) -> dict:
        out = (ctypes.c_int64 * 11)()
        _lib.check(_lib.load().sa_plan_stats(self._h, out, 11))
        keys = ("incidences", "max_row_nodes", "nodes", "nnz", "warp_records", "twopass_slots",
                "element_batches_staged", "max_batch_vertices", "device_bytes", "light_row_nodes", "heavy_rows")
        return dict(zip(keys, [int(x) for x in out]))

    def pattern(self, stream=None):
        """Structural (indptr int64 relative, indices int32) of the block."""
        if self._pattern is None:
            dev = self.dmesh.device
            ip = torch.empty(self.nrows + 1, dtype=torch.int64, device=dev)
            ix = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
            _lib.check(_lib.load().sa_plan_pattern(self._h, _ptr(ip), _ptr(ix), _stream_ptr(stream)))
            self._pattern = (ip, ix[: self.nnz])
        return self._pattern

    def coeffs(self, kernels, stream=None) -> tuple[_lib.SaCoeffs, list]:
        """Pack the kernels' nodal coefficients into an sa_coeffs (device)."""
        return upload_coeffs(kernels, self.dmesh.device, self.dmesh.d, stream)

    def prepare(self, kernels, stream=None):
        """Build the per-plan structures the numeric kernel for these
        kernels needs (two-pass slot map / row buffer / element batches)
        now, so they count as symbolic work (sa_plan_prepare)."""
        ops = 0
        for k in kernels:
            ops |= OP_BITS[k.op]
        with torch.cuda.device(self.dmesh.device):
            _lib.check(_lib.load().sa_plan_prepare(self._h, ops, _stream_ptr(stream)))

    def resident_coeffs(self, kernels):
        """Upload the kernels' nodal coefficients once and keep them in HBM;
        pass the result as ``numeric(..., coeffs=...)`` to re-assemble without
        re-uploading (the coefficient arrays must not change meanwhile)."""
        order = sorted(kernels, key=lambda k: OP_BITS[k.op])
        return self.coeffs(order)

    def numeric(self, kernels, out=None, stream=None, sync: bool = True, coeffs=None):
        """Values of every structural entry for each kernel (ascending op-bit
        order).  Returns (list of vals tensors, list of exact-zero counts or
        None when sync=False).  ``coeffs`` = ``resident_coeffs(kernels)`` skips
        the host->device upload of the nodal coefficients."""
        ops = 0
        for k in kernels:
            ops |= OP_BITS[k.op]
            if getattr(k, "exact", False):
                ops |= _lib.SA_OP_EXACT
        order = sorted(kernels, key=lambda k: OP_BITS[k.op])
        n = len(order)
        dev = self.dmesh.device
        if out is None:
            out = [torch.empty(max(self.nnz, 1), dtype=torch.float64, device=dev) for _ in range(n)]
        cf, keep = self.coeffs(order) if coeffs is None else coeffs
        ptrs = (ctypes.c_void_p * 4)(*[o.data_ptr() for o in out] + [0] * (4 - n))
        nz = (ctypes.c_int64 * 4)()
        with torch.cuda.device(dev):
            rc = _lib.load().sa_numeric(self._h, ops, ctypes.byref(cf), ptrs,
                                        nz if sync else None, _stream_ptr(stream))
        _lib.check(rc)
        del keep
        vals = [o[: self.nnz] for o in out]
        by_kernel = {id(k): v for k, v in zip(order, vals)}
        zeros = {id(k): int(nz[i]) for i, k in enumerate(order)} if sync else None
        return ([by_kernel[id(k)] for k in kernels],
                [zeros[id(k)] for k in kernels] if sync else None)

    def numeric_graph(self, kernels, out, coeffs):
        """Capture one re-assembly (sa_numeric: counter resets + the numeric
        kernel launches, no host sync) in a CUDA graph; ``g.replay()`` then
        re-assembles into ``out`` with one launch from the host, so small
        meshes are not bound by per-launch host overhead.  The plan's
        kernel-specific data must exist first (prepare() or one numeric call);
        zero counts / degenerate checks need a regular numeric(sync=True)."""
        self.prepare(kernels)
        torch.cuda.synchronize(self.dmesh.device)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.dmesh.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.numeric(kernels, out=out, sync=False, coeffs=coeffs)   # warm (module loads, attributes)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize(self.dmesh.device)
        n0 = launch_count()
        with torch.cuda.graph(g):
            self.numeric(kernels, out=out, sync=False, coeffs=coeffs)
        g.sa_kernels_per_replay = launch_count() - n0   # library kernels inside the graph
        return g

    def compact(self, vals: "torch.Tensor", n_zero: int, stream=None) -> DeviceCSR:
        """Canonical block CSR: exact-zero sums dropped (sparse.py:108-111)."""
        ip, ix = self.pattern(stream)
        ncols = self.m * self.dmesh.nq
        if n_zero == 0:
            return DeviceCSR(self.row_begin, self.row_end, ncols, ip, ix, vals)
        dev = self.dmesh.device
        nnz = self.nnz - n_zero
        nip = torch.empty(self.nrows + 1, dtype=torch.int64, device=dev)
        nix = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        nva = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        _lib.check(_lib.load().sa_compact(self._h, _ptr(vals), _ptr(nip), _ptr(nix), _ptr(nva),
                                          _stream_ptr(stream)))
        return DeviceCSR(self.row_begin, self.row_end, ncols, nip, nix[:nnz], nva[:nnz])

    def assemble(self, kernels, stream=None, coeffs=None) -> list[DeviceCSR]:
        vals, zeros = self.numeric(kernels, stream=stream, sync=True, coeffs=coeffs)
        return [self.compact(v, z, stream) for v, z in zip(vals, zeros)]

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().sa_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _pinned(k, name, arr):
    """A page-locked host copy of a kernel's coefficient array, cached on the
    descriptor (built once per coefficient set, like the reference's kernel
    construction), so every assembly uploads it at full PCIe rate and
    asynchronously."""
    cache = k.__dict__.setdefault("_pinned_cache", {})
    t = cache.get(name)
    if t is None or t.numel() != np.asarray(arr).size:
        t = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1))
        if torch.cuda.is_available():
            t = t.pin_memory()
        cache[name] = t
    return t


def upload_coeffs(kernels, device, d, stream=None) -> tuple[_lib.SaCoeffs, list]:
    """sa_coeffs for ``kernels`` (ascending op-bit order) with their nodal /
    per-element arrays uploaded to ``device`` on ``stream`` (asynchronous from
    pinned copies; the caller orders the numeric phase after the stream)."""
    c = _lib.SaCoeffs()
    c.w_const = c.lamb_const = c.mu_const = 1.0
    keep = []
    s = stream if stream is not None else torch.cuda.current_stream(device)

    def up(k, name, a):
        with torch.cuda.stream(s):
            t = _pinned(k, name, a).to(device=device, dtype=torch.float64, non_blocking=True)
        keep.append(t)
        return _ptr(t)

    for k in kernels:
        if k.op == "mass":
            if k.w is not None:
                c.w = up(k, "w", k.w)
            else:
                c.w_const = k.w_const
        elif k.op == "elastic" and getattr(k, "lambs_e", None) is not None:
            c.lambs_e = up(k, "lambs_e", k.lambs_e)
            c.mus_e = up(k, "mus_e", k.mus_e)
        elif k.op == "elastic":
            if k.lamb is not None:
                c.lamb = up(k, "lamb", k.lamb)
            else:
                c.lamb_const = k.lamb_const
            if k.mu is not None:
                c.mu = up(k, "mu", k.mu)
            else:
                c.mu_const = k.mu_const
        elif k.op == "general":
            # only the varying, distinct columns of the records cross PCIe
            # (C5: 13 of 16 -- A is symmetric); rebuilt on the device
            cols, colmap, consts = k.packed_columns()
            nq = int(cols.shape[0])
            with torch.cuda.stream(s):
                rec = torch.empty((nq, 16), dtype=torch.float64, device=device)
                src = _pinned(k, "cols", cols).to(device=device, non_blocking=True) if cols.shape[1] else None
                cm = np.ascontiguousarray(colmap, dtype=np.int32)
                cs = np.ascontiguousarray(consts, dtype=np.float64)
                with torch.cuda.device(device):
                    _lib.check(_lib.load().sa_unpack_columns(_ptr(src), int(cols.shape[1]), ctypes.c_void_p(cm.ctypes.data),
                                                             ctypes.c_void_p(cs.ctypes.data), nq, _ptr(rec),
                                                             ctypes.c_void_p(s.cuda_stream)))
            keep.append(rec)
            keep.append(src)
            c.gen_packed = _ptr(rec)
    return c, keep


# page-locked int32 staging buffer of upload_connectivity: grow-only and
# reused across calls (a fresh pinned allocation per call costs more than
# the upload it serves)
_STAGING: dict = {}
_STAGING_LOCK = __import__("threading").Lock()   # one upload at a time fills the buffer
_NARROW_MIN_ENTRIES = 48 << 20


def _staging_buffer(n: int) -> "torch.Tensor":
    ev = _STAGING.get("event")
    if ev is not None:
        ev.synchronize()
    buf = _STAGING.get("buf")
    if buf is None or buf.numel() < n:
        _STAGING["buf"] = None
        buf = torch.empty(max(n, 1), dtype=torch.int32, pin_memory=True)
        _STAGING["buf"] = buf
    return buf[:n]


def _host_threads() -> int:
    """Host threads for the narrowing pass: the CPUs this process may run on
    (affinity mask, capped by a cgroup CPU quota when one is set)."""
    import os

    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        n = os.cpu_count() or 1
    try:
        with open("/sys/fs/cgroup/cpu.max") as f:
            quota, period = f.read().split()[:2]
        if quota != "max":
            n = max(1, min(n, int(int(quota) / int(period))))
    except Exception:
        pass
    # several ranks on one host (torchrun): share the CPUs
    try:
        n = max(1, n // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1"))))
    except ValueError:
        pass
    return int(os.environ.get("SA_UPLOAD_THREADS", n))


def connectivity_split(me, d: int) -> int:
    """How many leading rows of a host connectivity array upload_connectivity
    narrows to int32 on the host (the others cross PCIe as int64): all but
    the last when the array is page-locked (the int64 row's DMA keeps PCIe
    busy while the host threads narrow), every row otherwise, 0 when the
    array cannot be narrowed in place (not int64 / not C-contiguous)."""
    a = np.asarray(me)
    if a.dtype != np.int64 or a.ndim != 2 or not a.flags.c_contiguous or a.shape[1] == 0:
        return 0
    # small arrays: waking the host threads costs more than the PCIe bytes
    # saved (measured: C2, 24 M entries, 20.1 vs 18.6 ms end to end)
    if a.size < _NARROW_MIN_ENTRIES:
        return 0
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")   # read-only arrays (frozen meshes)
        pinned = torch.cuda.is_available() and torch.from_numpy(a).is_pinned()
    return d if (pinned and d >= 1) else d + 1


def upload_connectivity(me, nq: int, device, stream=None):
    """Host (d+1, nme) int64 connectivity -> (me32 device (rows32, nme) int32,
    me64 device (d+1-rows32, nme) int64 or None).  The host threads narrow
    and range-check the first rows (sa_host_narrow_upload) while the copies
    run; raises IndexRangeError naming me[a, k] like the reference."""
    from .errors import IndexRangeError

    a = np.asarray(me)
    d = a.shape[0] - 1
    rows32 = connectivity_split(a, d)
    if rows32 == 0:
        return None, _to_dev(a, torch.int64, device)
    nme = a.shape[1]
    s = stream if stream is not None else torch.cuda.current_stream(device)
    with _STAGING_LOCK, torch.cuda.device(device), torch.cuda.stream(s):
        import warnings

        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            me64 = torch.from_numpy(a[rows32:]).to(device, non_blocking=True) if rows32 <= d else None
        staging = _staging_buffer(rows32 * nme).view(rows32, nme)
        me32 = torch.empty((rows32, nme), dtype=torch.int32, device=device)
        bad = ctypes.c_int64(-1)
        nthreads = _host_threads()
        rc = _lib.load().sa_host_narrow_upload(ctypes.c_void_p(a.ctypes.data), rows32 * nme, int(nq),
                                               _ptr(staging), _ptr(me32), nthreads, device.index,
                                               ctypes.c_void_p(s.cuda_stream), ctypes.byref(bad))
        _lib.check(rc)
        ev = torch.cuda.Event()
        ev.record(s)
        _STAGING["event"] = ev   # the next upload waits for these copies before reusing the buffer
    if bad.value >= 0:
        ev.synchronize()
        raise IndexRangeError(f"connectivity entry me[{bad.value // nme}, {bad.value % nme}] out of range [0, {nq})")
    return me32, me64


def device_volumes(q, me, core: str = "SkylakeX") -> np.ndarray:
    """Simplex volumes computed on the B200 (numpy-det factorisation,
    mesh.py:38-43); raises DegenerateSimplexError like compute_volumes."""
    dm = DeviceMesh(q, me, None, core=core)
    try:
        return dm.vols().cpu().numpy()
    finally:
        dm.close()


def launch_count(reset: bool = False) -> int:
    return int(_lib.load().sa_launch_count(1 if reset else 0))
