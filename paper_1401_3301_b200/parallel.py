"""Row-block data parallelism.

Rows are split into P contiguous node blocks; rank p assembles the rows of
block p from the elements touching it, with no inter-GPU traffic on the hot
path.  The row-block optv2 is bitwise the corresponding rows of the full
optv2, so stitching the blocks gives exactly the single-GPU matrix.  The only
collectives are an all-gather of the P block nnz counts (global row offsets)
and, for validation, a gather of the blocks to rank 0.  Both run over
torch.distributed (NCCL on the B200 box, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def row_blocks(nq: int, m: int, nparts: int) -> list[tuple[int, int]]:
    """Contiguous dof-row blocks aligned to nodes (rows m*i .. m*i+m-1 stay
    together), balanced by node count."""
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    cuts = [(nq * p) // nparts for p in range(nparts + 1)]
    return [(m * cuts[p], m * cuts[p + 1]) for p in range(nparts)]


@dataclass
class Slab:
    """The part of a mesh one rank needs for its row block: the elements
    touching the block's nodes, in their original (ascending) order, over the
    window [node_lo, node_lo + nq_local) of nodes they reference, renumbered
    from 0.  Rows [row_begin, row_end) of the local problem are the block's
    rows; local column dof c is global column dof c + col_offset.  Because
    the element order is kept, the block assembled from the slab is bitwise
    the block of the full mesh (same contributions, same fold order)."""

    q: np.ndarray          # (d, nq_local) f64
    me: np.ndarray         # (d+1, nme_local) int64, local node ids
    vols: np.ndarray | None
    node_lo: int
    row_begin: int         # local dof rows of the block
    row_end: int
    col_offset: int        # m * node_lo
    elements: np.ndarray   # global ids of the slab's elements (ascending)

    def nodal(self, a):
        """Window of a per-node array (nq, ...) or None."""
        return None if a is None else np.ascontiguousarray(np.asarray(a)[self.node_lo:self.node_lo + self.q.shape[1]])


def slab(q, me, m: int, row_begin: int, row_end: int, vols=None) -> Slab:
    """Slab of dof rows [row_begin, row_end) (node aligned) of mesh (q, me)."""
    if row_begin % m or row_end % m:
        raise ValueError("row block must be node aligned")
    nb0, nb1 = row_begin // m, row_end // m
    me = np.asarray(me)
    touch = np.zeros(me.shape[1], dtype=bool)
    for a in range(me.shape[0]):
        touch |= (me[a] >= nb0) & (me[a] < nb1)
    sel = np.flatnonzero(touch)
    mes = me[:, sel]
    lo, hi = nb0, nb1
    if sel.size:
        lo, hi = min(lo, int(mes.min())), max(hi, int(mes.max()) + 1)
    return Slab(q=np.ascontiguousarray(np.asarray(q)[:, lo:hi]), me=np.ascontiguousarray(mes - lo),
                vols=None if vols is None else np.ascontiguousarray(np.asarray(vols)[sel]),
                node_lo=lo, row_begin=m * (nb0 - lo), row_end=m * (nb1 - lo), col_offset=m * lo, elements=sel)


def global_offsets(local_nnz: int, group=None, device=None) -> tuple[int, int, list[int]]:
    """All-gather the per-rank block nnz; return (offset of this rank's first
    entry in the global CSR, total nnz, all counts)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = torch.tensor([local_nnz], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    counts = [int(x.item()) for x in out]
    return int(sum(counts[:rank])), int(sum(counts)), counts


def stitch(blocks, nrows: int, ncols: int):
    """Concatenate row blocks (row_begin, row_end, indptr_rel, indices, vals)
    given in row order into one CSR (row_ptr, col_idx, vals) (host numpy)."""
    row_ptr = np.zeros(nrows + 1, dtype=np.int64)
    cols, vals = [], []
    off = 0
    expect = 0
    for rb, re, ip, ix, va in blocks:
        if rb != expect:
            raise ValueError(f"row blocks are not contiguous: expected {expect}, got {rb}")
        ip = np.asarray(ip, dtype=np.int64)
        row_ptr[rb + 1:re + 1] = off + ip[1:]
        off += int(ip[-1])
        cols.append(np.asarray(ix, dtype=np.int64))
        vals.append(np.asarray(va, dtype=np.float64))
        expect = re
    if expect != nrows:
        raise ValueError(f"row blocks cover {expect} of {nrows} rows")
    return row_ptr, np.concatenate(cols) if cols else np.empty(0, np.int64), \
        np.concatenate(vals) if vals else np.empty(0)


def gather_blocks_to_root(block, group=None, root: int = 0):
    """Gather (row_begin, row_end, indptr, indices, vals) host-numpy blocks to
    ``root`` (validation only, off the timed path)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [None] * world if dist.get_rank(group) == root else None
    if dist.get_backend(group) == "nccl":
        # gather_object over NCCL needs the rank's device set; objects are
        # pickled through it
        import torch

        torch.cuda.set_device(torch.cuda.current_device())
    dist.gather_object(block, out, dst=root, group=group)
    return out


@dataclass
class DistributedResult:
    """One rank's share of a distributed assembly: its row block per kernel
    (host CSR: indptr relative, global int64 columns, values), the global
    offset of its first entry, the global nnz, and -- on the root rank when
    gathered -- the stitched matrices."""

    row_begin: int
    row_end: int
    blocks: list
    offsets: list
    totals: list
    matrices: list | None


def assemble_distributed(mesh, kernels, group=None, gather: bool = True, root: int = 0, core: str = "SkylakeX",
                         timings: dict | None = None) -> DistributedResult:
    """Rank-aware driver of the row-block data-parallel path,
    one process per GPU (torchrun; torch.distributed initialised, NCCL on
    B200s, gloo in tests; a single process without a process group is world
    size 1).  Each rank takes the node-aligned row block ``row_blocks(nq, m,
    P)[rank]``, cuts its slab (the elements touching its rows, in ascending
    order, over their node window) and assembles it on its current CUDA
    device with ``assemble_block_b200`` -- no inter-GPU traffic on the data
    path.  The only collectives: an all-gather of the block nnz (global
    offsets) and, with ``gather``, a gather of the blocks to ``root``, which
    stitches them into the full matrices (bitwise the single-GPU result:
    same contributions, same fold order)."""
    import torch.distributed as dist

    from .assembly import _as_descriptor, assemble_block_b200
    from .kernels import restrict
    from .mesh import Mesh

    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    else:
        world, rank = 1, 0
    kernels = [_as_descriptor(mesh, k) for k in kernels]
    m = kernels[0].m
    nq = np.asarray(mesh.q).shape[1]
    rb, re_ = row_blocks(nq, m, world)[rank]
    sl = slab(mesh.q, mesh.me, m, rb, re_, getattr(mesh, "vols", None))
    smesh = Mesh(sl.q, sl.me, sl.vols) if sl.vols is not None else Mesh.from_arrays(sl.q, sl.me)
    window = slice(sl.node_lo, sl.node_lo + sl.q.shape[1])
    skernels = [restrict(k, smesh, window, sl.elements) for k in kernels]
    out = assemble_block_b200(smesh, skernels, sl.row_begin, sl.row_end, core=core, timings=timings,
                              col_offset=sl.col_offset, ncols=m * nq)
    blocks = [(rb, re_, b.row_ptr, b.col_idx, b.vals) for b in out]
    offsets, totals, matrices = [], [], None
    for b in out:
        if world > 1:
            off, tot, _ = global_offsets(b.nnz, group=group, device=_coll_device(group))
        else:
            off, tot = 0, b.nnz
        offsets.append(off)
        totals.append(tot)
    if gather:
        from .sparse import SparseMatrix

        gathered = gather_blocks_to_root(blocks, group=group, root=root) if world > 1 else [blocks]
        if rank == root:
            matrices = []
            for ki in range(len(kernels)):
                rp, ci, va = stitch([g[ki] for g in gathered], m * nq, m * nq)
                matrices.append(SparseMatrix(m * nq, m * nq, rp, ci, va))
    return DistributedResult(rb, re_, blocks, offsets, totals, matrices)


def _coll_device(group=None):
    """Device for small collective tensors: the current CUDA device under
    NCCL, the CPU under gloo."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")
