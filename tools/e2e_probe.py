"""Fine-grained timing of one assemble_block_b200 call (C5 by default):
each stage synchronised, to see where the end-to-end time goes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1401_3301_b200 as P  # noqa: E402
from paper_1401_3301_b200 import device as D  # noqa: E402
from paper_1401_3301_b200.assembly import _PatternDownload, to_host_many  # noqa: E402


def main(name="C5"):
    cfg = bench.CONFIGS[name]
    q, me = bench.make_mesh(cfg)
    vols = P.device_volumes(q, me)
    mesh0 = P.Mesh(q, me, vols)
    kernels = bench.make_kernels(cfg, mesh0)
    pq, pme, pv = (torch.from_numpy(x).pin_memory() for x in (q, me, np.asarray(vols)))
    for it in range(4):
        T = {}
        dev = torch.device("cuda", 0)
        main_s = torch.cuda.current_stream()

        def mark(k, t0=[time.perf_counter()]):
            torch.cuda.synchronize()
            t = time.perf_counter()
            T[k] = round(1e3 * (t - t0[0]), 1)
            t0[0] = t

        mark("start")
        med = pme.to(dev, non_blocking=True)
        vd = pv.to(dev, non_blocking=True)
        mark("up_me_vols")
        qd = pq.to(dev, non_blocking=True)
        order = sorted(kernels, key=lambda k: D.OP_BITS[k.op])
        coeffs = D.upload_coeffs(order, dev, q.shape[0])
        mark("up_q_coeffs")
        dm = D.DeviceMesh(None, med, vd, nq=q.shape[1])
        mark("mesh_create")
        plan = dm.plan(kernels[0].m)
        mark("symbolic")
        dm.set_coords(qd)
        mark("set_coords")
        plan.prepare(kernels)
        mark("prepare")
        pat = _PatternDownload(*plan.pattern(), 0, kernels[0].m * q.shape[1])
        mark("pattern_dl")
        vals, zeros = plan.numeric(kernels, coeffs=coeffs)
        mark("numeric")
        csrs = [plan.compact(v, z) for v, z in zip(vals, zeros)]
        mark("compact")
        out = to_host_many(csrs, patterns=(pat,))
        mark("download")
        dm.close()
        del out, csrs, vals, coeffs
        mark("free")
        print(it, T, flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
