"""World-size-2 gloo test of the row-block data-parallel path (host logic).

Each rank assembles its node-aligned row block (here with the CPU oracle as
the block assembler -- the GPU block assembler is exercised by the -m gpu
tests), all-gathers the block nnz for the global offsets and gathers the
blocks to rank 0, which stitches them and compares with the single-process
matrix bitwise."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, load_golden, oracle_op_for


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, result_q, use_slab=False):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from conftest import load_golden as lg, oracle_op_for as oo
    from oracle import oracle as O
    from paper_1401_3301_b200 import parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = lg(name)
        op = oo(name, g)
        nq = g["q"].shape[1]
        rb, re_ = parallel.row_blocks(nq, op.m, world)[rank]
        if use_slab:
            # the rank only holds its slab: elements touching its rows, local
            # node numbering; columns shifted back to global dofs
            sl = parallel.slab(g["q"], g["me"], op.m, rb, re_, g["vols"])
            gl = dict(g, q=sl.q, me=sl.me, vols=sl.vols)
            for key in ("w", "lamb", "mu", "A", "b", "c", "a0"):
                if key in g:
                    gl[key] = sl.nodal(g[key])
            ip, ix, va = O.assemble_block(sl.q, sl.me, oo(name, gl), sl.row_begin, sl.row_end)
            ix = ix + sl.col_offset
        else:
            ip, ix, va = O.assemble_block(g["q"], g["me"], op, rb, re_)
        off, total, counts = parallel.global_offsets(len(va))
        blocks = parallel.gather_blocks_to_root((rb, re_, ip, ix, va))
        if rank == 0:
            rp, ci, vv = parallel.stitch(blocks, op.m * nq, op.m * nq)
            ok = (np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])
                  and np.array_equal(vv, g["vals"]) and total == len(g["vals"]) and off == 0)
            result_q.put(bool(ok))
        else:
            result_q.put(off == counts[0])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("use_slab", [False, True])
@pytest.mark.parametrize("name", ["stiff_d3_n6_jit", "elastic_d2_n15_jit", "general_d2_n15_jit"])
def test_two_rank_row_blocks_stitch_to_full_matrix(name, use_slab):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q, use_slab)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    results = [q.get(timeout=10) for _ in range(2)]
    assert all(results), results
    assert all(p.exitcode == 0 for p in procs)



def _driver_worker(rank, world, port, name, result_q):
    # the product's distributed driver (parallel.assemble_distributed): slab
    # cut, coefficient restriction, offsets, gather, stitch -- with the block
    # assembler swapped for the oracle (no GPU here; the -m gpu test runs the
    # real one)
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import paper_1401_3301_b200 as P
    from conftest import device_kernel_for as dk, load_golden as lg, oracle_op_for as oo
    from oracle import oracle as O
    from paper_1401_3301_b200 import assembly, parallel

    def fake_block(mesh, kernels, row_begin, row_end, core="SkylakeX", timings=None, col_offset=0, ncols=None):
        out = []
        for k in kernels:
            g = {"q": mesh.q, "me": mesh.me, "vols": mesh.vols}
            if k.op == "mass":
                g["w"] = k.w if k.w is not None else np.full(mesh.q.shape[1], k.w_const)
            if k.op == "elastic":
                g["lamb"], g["mu"] = k.lamb, k.mu
            if k.op == "general":
                g.update(A=k.A, b=k.b, c=k.c, a0=k.a0)
            ip, ix, va = O.assemble_block(mesh.q, mesh.me, oo(name, g), row_begin, row_end)
            out.append(P.SparseMatrix(row_end - row_begin, ncols, ip, ix + col_offset, va))
        return out

    assembly.assemble_block_b200 = fake_block
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = lg(name)
        mesh = P.Mesh(g["q"], g["me"], g["vols"])
        res = parallel.assemble_distributed(mesh, [dk(name, g, mesh)])
        if rank == 0:
            a = res.matrices[0]
            ok = (np.array_equal(a.row_ptr, g["row_ptr"]) and np.array_equal(a.col_idx, g["col_idx"])
                  and np.array_equal(a.vals, g["vals"]) and res.totals[0] == len(g["vals"]) and res.offsets[0] == 0)
            result_q.put(bool(ok))
        else:
            result_q.put(res.matrices is None and res.offsets[0] > 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["stiff_d3_n6_jit", "mass_d2_n15_jit", "elastic_d3_n6_jit", "general_d3_n6_jit"])
def test_distributed_driver_two_ranks(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_driver_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    results = [q.get(timeout=10) for _ in range(2)]
    assert all(results), results
    assert all(p.exitcode == 0 for p in procs)
