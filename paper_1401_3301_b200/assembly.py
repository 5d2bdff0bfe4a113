"""Drop-in assembly drivers (the reference's plugin API, assembly.py:295-308).

``assemble_b200(mesh, kernel) -> SparseMatrix`` has the signature of every
reference scalar driver; ``assemble_vector_b200`` that of the vector
drivers.  They return the canonical CSR the reference's ``assemble_optv2``
returns -- bitwise: same row_ptr, col_idx and vals.
``register()`` adds them to the reference's own SCALAR_DRIVERS /
VECTOR_DRIVERS dicts (and bench.VARIANTS_FOR) when simplex_asm is importable,
so ``simplex_asm.bench`` and its CLI dispatch to the B200 as variant "b200".
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import kernels as _k
from .device import upload_connectivity, OP_BITS, DeviceCSR, DeviceMesh, upload_coeffs
from .sparse import SparseMatrix

_MESH_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_ID_CACHE: dict = {}


def device_mesh_for(mesh, core: str = "SkylakeX", cache: bool = True) -> DeviceMesh:
    """Upload (once per mesh object; meshes are immutable, mesh.py:46-52)."""
    if cache:
        try:
            dm = _MESH_CACHE.get(mesh)
        except TypeError:
            dm = None
        if dm is not None and dm.core == core:
            return dm
    dm = DeviceMesh(mesh.q, mesh.me, getattr(mesh, "vols", None), core=core)
    if cache:
        try:
            _MESH_CACHE[mesh] = dm
        except TypeError:
            pass
    return dm


def _as_descriptor(mesh, kernel):
    """Accept our descriptors, or the reference's kernel objects where the
    nodal data can be recovered exactly."""
    if hasattr(kernel, "op"):
        return kernel
    name = type(kernel).__name__
    if name == "StiffnessKernel":
        return _k.StiffnessKernel(mesh)
    if name == "MassKernel" and hasattr(kernel, "W"):
        # reference MassKernel keeps W = w_nodal[me] (kernels.py:287); scatter back
        w = np.empty(mesh.q.shape[1])
        for a in range(kernel.W.shape[0]):
            w[np.asarray(mesh.me[a])] = kernel.W[a]
        return _k.MassKernel(mesh, w)
    if name == "ElasticKernel" and hasattr(kernel, "lambs") and hasattr(kernel, "mus"):
        # reference ElasticKernel keeps only the per-element scaled Lame sums
        # (kernels.py:354-356): pass them through unchanged (bitwise)
        return _k.ElasticKernel.per_element(mesh, kernel.lambs, kernel.mus)
    if name == "ScalarAsVectorKernel":
        return _as_descriptor(mesh, kernel._kernel)
    raise TypeError(f"assemble_b200 cannot use a {name}; build the kernel with "
                    "paper_1401_3301_b200.{MassKernel,StiffnessKernel,ElasticKernel,GeneralKernel}")


class _PatternDownload:
    """Asynchronous device->host copy of one block pattern: indptr (int64)
    and the column indices as int32 (half the PCIe bytes of int64; widened
    on the host, sparse.py:53-55 stores int64), on a side stream so it can
    overlap the numeric phase.  ``col_offset`` shifts a slab's local columns
    to global dofs on the device first."""

    def __init__(self, indptr, indices, col_offset: int = 0, local_ncols: int | None = None):
        import torch

        self.key = (indptr.data_ptr(), indices.data_ptr(), indices.numel())
        self.stream = torch.cuda.Stream(device=indptr.device)
        self.stream.wait_stream(torch.cuda.current_stream())
        # global dofs fit int32 (CapacityError otherwise, sa_plan_create); the
        # shift is done on the device in int32 only when it cannot wrap
        self.host_offset = 0
        if col_offset and (local_ncols is None or int(col_offset) + int(local_ncols) >= (1 << 31)):
            self.host_offset, col_offset = int(col_offset), 0
        with torch.cuda.stream(self.stream):
            ix = indices + col_offset if col_offset else indices
            self.ip = torch.empty(indptr.shape, dtype=torch.int64, pin_memory=True)
            self.ix32 = torch.empty(ix.shape, dtype=torch.int32, pin_memory=True)
            self.ip.copy_(indptr, non_blocking=True)
            self.ix32.copy_(ix, non_blocking=True)
            self.done = torch.cuda.Event()
            self.done.record(self.stream)
        self._host = None

    def host(self):
        """(row_ptr int64, col_idx int64) numpy arrays; waits for this copy
        only, then widens on the host (torch's parallel CPU copy) while other
        transfers continue."""
        import torch

        if self._host is None:
            self.done.synchronize()
            ix64 = torch.empty(self.ix32.shape, dtype=torch.int64, pin_memory=True)
            # widened on the library's own parked host threads (a torch CPU op
            # would leave its OpenMP workers spinning into the next upload)
            from . import _lib
            from .device import _host_threads

            _lib.check(_lib.load().sa_host_widen_i32(ctypes.c_void_p(self.ix32.data_ptr()), self.ix32.numel(),
                                                     int(self.host_offset), ctypes.c_void_p(ix64.data_ptr()),
                                                     _host_threads()))
            self._host = (self.ip.numpy(), ix64.numpy())
        return self._host


def to_host(csr: DeviceCSR, nrows_total: int | None = None) -> SparseMatrix:
    """Download a full-matrix device CSR into the reference's SparseMatrix
    (int64 indices, as sparse.py:53-55)."""
    return to_host_many([csr], nrows_total)[0]


def to_host_many(csrs, nrows_total=None, col_offset: int = 0, patterns=(), ncols: int | None = None) -> list[SparseMatrix]:
    """Download several results; fused outputs that share one pattern (no
    exact-zero entries dropped) share the host row_ptr/col_idx arrays, so the
    pattern crosses PCIe once (as int32 indices, widened on the host while
    the values transfer).  ``col_offset`` is added to the column indices on
    the device (a slab's local columns -> global dofs).  ``patterns``:
    downloads already in flight (_PatternDownload)."""
    import torch

    cache = {p.key: p for p in patterns}
    for c in csrs:
        key = (c.indptr.data_ptr(), c.indices.data_ptr(), c.indices.numel())
        if key not in cache:
            cache[key] = _PatternDownload(c.indptr, c.indices, col_offset, c.ncols)
    vals = []
    for c in csrs:
        v = torch.empty(c.vals.shape, dtype=c.vals.dtype, pin_memory=True)
        v.copy_(c.vals, non_blocking=True)
        vals.append(v)
    res = []
    hosts = [cache[(c.indptr.data_ptr(), c.indices.data_ptr(), c.indices.numel())].host() for c in csrs]
    torch.cuda.current_stream().synchronize()
    for c, (ip, ix), v in zip(csrs, hosts, vals):
        nrows = c.row_end - c.row_begin if nrows_total is None else nrows_total
        # global column count: a slab's local columns were shifted by col_offset
        res.append(SparseMatrix(nrows, ncols if ncols is not None else c.ncols + col_offset, ip, ix, v.numpy()))
    return res


def assemble_device(mesh, kernels, core: str = "SkylakeX", cache: bool = True) -> list[DeviceCSR]:
    """Fused assembly of one or more kernels sharing a plan (e.g. mass +
    stiffness); results stay on the device."""
    kernels = [_as_descriptor(mesh, k) for k in kernels]
    m = kernels[0].m
    if any(k.m != m for k in kernels):
        raise ValueError("fused kernels must have the same number of unknowns per node")
    dm = device_mesh_for(mesh, core, cache)
    return dm.plan(m).assemble(kernels)


def assemble_many_b200(mesh, kernels, core: str = "SkylakeX", cache: bool = True) -> list[SparseMatrix]:
    """Fused drop-in assembly of several kernels on one mesh (e.g. mass +
    stiffness): one upload, one symbolic phase, one numeric pass."""
    return to_host_many(assemble_device(mesh, kernels, core, cache))


def assemble_block_b200(mesh, kernels, row_begin: int, row_end: int, core: str = "SkylakeX",
                        timings: dict | None = None, col_offset: int = 0, ncols: int | None = None):
    """Rows [row_begin, row_end) of the fused assembly, end to end from host
    arrays (the per-rank call of the row-block data-parallel path): upload,
    symbolic, numeric, exact-zero compaction, download.  Returns one
    (indptr, indices, vals) host block per kernel.  For a rank's slab
    (parallel.slab) pass its local rows and ``col_offset`` to get global
    column dofs, and ``ncols`` the global column count of the matrix the
    block belongs to (default: the slab's columns + col_offset)."""
    import time

    import torch

    kernels = [_as_descriptor(mesh, k) for k in kernels]
    t = time.perf_counter()
    # connectivity and volumes first (the symbolic phase needs the former;
    # uploading the volumes on the side stream instead measured slower: C5
    # e2e 315 vs 215 ms); coordinates and coefficients follow on a side
    # stream while the symbolic phase runs
    main = torch.cuda.current_stream()
    # connectivity: narrowed to int32 by the host threads while it uploads
    # (half the PCIe bytes of the reference's int64 array for those rows)
    nq_ = int(np.asarray(mesh.q).shape[1])
    me32, med = upload_connectivity(mesh.me, nq_, main.device)
    vols = getattr(mesh, "vols", None)
    # the fast general operator (values within 1e-12, exact pattern) does not
    # need the host volumes bit for bit: they are recomputed on the device
    # from the coordinates (numpy-det factorisation, a few ulp from
    # mesh.vols) instead of crossing PCIe
    if all(k.op == "general" and not getattr(k, "exact", False) for k in kernels):
        vols = None
    vd = torch.as_tensor(np.asarray(vols)).to(main.device, non_blocking=True) if vols is not None else None
    me_done = torch.cuda.Event()
    me_done.record(main)
    side = torch.cuda.Stream(device=main.device)
    side.wait_event(me_done)
    with torch.cuda.stream(side):
        qd = torch.as_tensor(np.asarray(mesh.q)).to(main.device, non_blocking=True)
    # nodal coefficients (pinned copies cached on the descriptors) upload on
    # the side stream too, behind the coordinates, during the symbolic phase
    order = sorted(kernels, key=lambda k: OP_BITS[k.op])
    coeffs = upload_coeffs(order, main.device, int(np.asarray(mesh.q).shape[0]), side)
    dm = DeviceMesh(None, med, vd, core=core, nq=nq_, me32=me32)
    t1 = time.perf_counter()
    plan = dm.plan(kernels[0].m, row_begin, row_end)
    # the kernel-specific plan data (two-pass slot map, element batches) needs
    # the connectivity only: built while the coefficients still upload
    if vd is not None or kernels[0].op == "general":
        plan.prepare(kernels)
    main.wait_stream(side)
    dm.set_coords(qd)
    # the structural pattern downloads while the numeric phase runs
    pat = _PatternDownload(*plan.pattern(), col_offset, kernels[0].m * dm.nq)
    t2 = time.perf_counter()
    csrs = plan.assemble(kernels, coeffs=coeffs)
    torch.cuda.current_stream().synchronize()
    del coeffs
    t3 = time.perf_counter()
    out = to_host_many(csrs, col_offset=col_offset, patterns=(pat,), ncols=ncols)
    t4 = time.perf_counter()
    dm.close()
    if timings is not None:
        for k, v in (("upload_ms", t1 - t), ("symbolic_ms", t2 - t1), ("numeric_ms", t3 - t2),
                     ("download_ms", t4 - t3), ("free_ms", time.perf_counter() - t4)):
            timings[k] = timings.get(k, 0.0) + 1e3 * v
    return out


def assemble_b200(mesh, kernel) -> SparseMatrix:
    """Scalar driver: same contract as assemble_optv2 (assembly.py:92-111)."""
    k = _as_descriptor(mesh, kernel)
    if k.m != 1:
        raise ValueError("assemble_b200 takes scalar kernels; use assemble_vector_b200")
    return to_host(assemble_device(mesh, [k])[0])


def assemble_vector_b200(mesh, kernel) -> SparseMatrix:
    """Vector driver: same contract as assemble_vector_optv2 (assembly.py:188-209);
    dofs interleaved r = m*i + l."""
    k = _as_descriptor(mesh, kernel)
    return to_host(assemble_device(mesh, [k])[0])


def assemble_mass_pk_b200(pkmesh, coeffs) -> SparseMatrix:
    """Pk mass matrix, same contract as assemble_mass_pk (assembly.py:265-292):
    every local entry is (d! C[a][b]) |K|; canonical CSR, each entry summed in
    ascending element order (bitwise the reference's values), exact-zero sums
    dropped.  Accepts the reference's PkMesh / PkCoeffTable or this package's
    (pk.build_pk_mesh, pk.pk_mass_coeffs)."""
    import ctypes
    import math

    import torch

    from . import _lib
    from .device import DeviceCSR, _ptr, _require_cuda, _stream_ptr, _to_dev

    if (pkmesh.d, pkmesh.k) != (coeffs.d, coeffs.k):
        raise ValueError(
            f"coefficient table (d={coeffs.d}, k={coeffs.k}) does not match "
            f"lattice mesh (d={pkmesh.d}, k={pkmesh.k})"
        )
    dev = _require_cuda(None)
    L = _lib.load()
    me = np.asarray(pkmesh.me)
    ndfe, nme = int(me.shape[0]), int(me.shape[1])
    nq = int(np.asarray(pkmesh.q).shape[1])
    # d! * C[a, b] exactly as the reference forms it (a float64 product)
    cs = float(math.factorial(pkmesh.d)) * np.asarray(coeffs.C, dtype=np.float64)
    with torch.cuda.device(dev):
        med = _to_dev(me, torch.int64, dev)
        vd = _to_dev(np.asarray(pkmesh.vols), torch.float64, dev)
        csd = _to_dev(np.ascontiguousarray(cs), torch.float64, dev)
        h = ctypes.c_void_p()
        _lib.check(L.sa_pk_plan_create(ndfe, nq, nme, _ptr(med), dev.index, _stream_ptr(), ctypes.byref(h)))
        try:
            nnz, md = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(L.sa_pk_plan_info(h, ctypes.byref(nnz), ctypes.byref(md)))
            n = nnz.value
            ip = torch.empty(nq + 1, dtype=torch.int64, device=dev)
            ix = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            va = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
            _lib.check(L.sa_pk_plan_pattern(h, _ptr(ip), _ptr(ix), _stream_ptr()))
            nz = ctypes.c_int64()
            _lib.check(L.sa_pk_mass(h, _ptr(csd), _ptr(vd), _ptr(va), ctypes.byref(nz), _stream_ptr()))
            if nz.value:
                m = n - nz.value
                nip = torch.empty(nq + 1, dtype=torch.int64, device=dev)
                nix = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
                nva = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
                _lib.check(L.sa_pk_compact(h, _ptr(va), _ptr(nip), _ptr(nix), _ptr(nva), _stream_ptr()))
                csr = DeviceCSR(0, nq, nq, nip, nix[:m], nva[:m])
            else:
                csr = DeviceCSR(0, nq, nq, ip, ix[:n], va[:n])
            return to_host(csr)
        finally:
            torch.cuda.current_stream().synchronize()
            L.sa_pk_plan_destroy(h)


SCALAR_DRIVERS = {"b200": assemble_b200}
VECTOR_DRIVERS = {"b200": assemble_vector_b200}


def register() -> bool:
    """Plug the B200 variant into the reference's registries (assembly.py:295-308,
    bench.py:31-36) if the reference package is importable."""
    try:
        import simplex_asm.assembly as ra  # type: ignore
        import simplex_asm.bench as rb  # type: ignore
    except Exception:
        return False
    ra.SCALAR_DRIVERS["b200"] = assemble_b200
    ra.VECTOR_DRIVERS["b200"] = assemble_vector_b200
    for key in ("mass", "stiffness", "elastic"):
        if "b200" not in rb.VARIANTS_FOR[key]:
            rb.VARIANTS_FOR[key] = tuple(rb.VARIANTS_FOR[key]) + ("b200",)
    return True
