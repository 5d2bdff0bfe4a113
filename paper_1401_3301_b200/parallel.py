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
    dist.gather_object(block, out, dst=root, group=group)
    return out
