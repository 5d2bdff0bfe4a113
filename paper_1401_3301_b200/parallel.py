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

import numpy as np


def row_blocks(nq: int, m: int, nparts: int) -> list[tuple[int, int]]:
    """Contiguous dof-row blocks aligned to nodes (rows m*i .. m*i+m-1 stay
    together), balanced by node count."""
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    cuts = [(nq * p) // nparts for p in range(nparts + 1)]
    return [(m * cuts[p], m * cuts[p + 1]) for p in range(nparts)]


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
