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

import weakref

import numpy as np

from . import kernels as _k
from .device import DeviceCSR, DeviceMesh
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
    if name == "ScalarAsVectorKernel":
        return _as_descriptor(mesh, kernel._kernel)
    raise TypeError(f"assemble_b200 cannot use a {name}; build the kernel with "
                    "paper_1401_3301_b200.{MassKernel,StiffnessKernel,ElasticKernel,GeneralKernel}")


def to_host(csr: DeviceCSR, nrows_total: int | None = None) -> SparseMatrix:
    """Download a full-matrix device CSR into the reference's SparseMatrix
    (int64 indices, as sparse.py:53-55)."""
    import torch

    nrows = csr.row_end - csr.row_begin if nrows_total is None else nrows_total
    # int32 -> int64 on the device (SparseMatrix stores int64, sparse.py:53-55),
    # then one asynchronous copy per array into pinned host buffers
    srcs = (csr.indptr, csr.indices.to(torch.int64), csr.vals)
    outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in srcs]
    for o, t in zip(outs, srcs):
        o.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    row_ptr, col_idx, vals = (o.numpy() for o in outs)
    return SparseMatrix(nrows, csr.ncols, row_ptr, col_idx, vals)


def to_host_many(csrs, nrows_total=None, col_offset: int = 0) -> list[SparseMatrix]:
    """Download several results; fused outputs that share one pattern (no
    exact-zero entries dropped) share the host row_ptr/col_idx arrays, so the
    pattern crosses PCIe once.  ``col_offset`` is added to the column indices
    on the device (a slab's local columns -> global dofs)."""
    import torch

    cache = {}
    out = []
    for c in csrs:
        key = (c.indptr.data_ptr(), c.indices.data_ptr(), c.indices.numel())
        if key not in cache:
            ix = c.indices.to(torch.int64)
            if col_offset:
                ix += col_offset
            srcs = (c.indptr, ix)
            pinned = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in srcs]
            for o, t in zip(pinned, srcs):
                o.copy_(t, non_blocking=True)
            cache[key] = pinned
        v = torch.empty(c.vals.shape, dtype=c.vals.dtype, pin_memory=True)
        v.copy_(c.vals, non_blocking=True)
        out.append((c, cache[key], v))
    torch.cuda.current_stream().synchronize()
    res = []
    for c, (ip, ix), v in out:
        nrows = c.row_end - c.row_begin if nrows_total is None else nrows_total
        res.append(SparseMatrix(nrows, c.ncols, ip.numpy(), ix.numpy(), v.numpy()))
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
                        timings: dict | None = None, col_offset: int = 0):
    """Rows [row_begin, row_end) of the fused assembly, end to end from host
    arrays (the per-rank call of the row-block data-parallel path): upload,
    symbolic, numeric, exact-zero compaction, download.  Returns one
    (indptr, indices, vals) host block per kernel.  For a rank's slab
    (parallel.slab) pass its local rows and ``col_offset`` to get global
    column dofs."""
    import time

    import torch

    kernels = [_as_descriptor(mesh, k) for k in kernels]
    t = time.perf_counter()
    dm = DeviceMesh(mesh.q, mesh.me, getattr(mesh, "vols", None), core=core)
    torch.cuda.current_stream().synchronize()
    t1 = time.perf_counter()
    plan = dm.plan(kernels[0].m, row_begin, row_end)
    t2 = time.perf_counter()
    csrs = plan.assemble(kernels)
    torch.cuda.current_stream().synchronize()
    t3 = time.perf_counter()
    out = to_host_many(csrs, col_offset=col_offset)
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
