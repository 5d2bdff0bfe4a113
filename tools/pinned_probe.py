"""Do torch's pinned allocations inside repeated end-to-end calls ever miss the host cache? (times every pin_memory allocation)"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1401_3301_b200 as P
from paper_1401_3301_b200.assembly import assemble_block_b200
_empty = torch.empty
slow = []
def timed_empty(*a, **k):
    t0 = time.perf_counter(); r = _empty(*a, **k); dt = 1e3 * (time.perf_counter() - t0)
    if k.get("pin_memory") and dt > 5: slow.append((round(dt, 1), tuple(r.shape), str(r.dtype)))
    return r
torch.empty = timed_empty
cfg = bench.CONFIGS["C5"]
q, me = bench.make_mesh(cfg)
vols = P.device_volumes(q, me)
pq, pme, pv = (torch.from_numpy(x).pin_memory() for x in (q, me, np.asarray(vols)))
mesh = P.Mesh(pq.numpy(), pme.numpy(), pv.numpy())
kernels = bench.make_kernels(cfg, mesh)
for i in range(14):
    slow.clear(); st = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    blocks = assemble_block_b200(mesh, kernels, 0, q.shape[1], timings=st)
    torch.cuda.synchronize(); dt = 1e3 * (time.perf_counter() - t0)
    del blocks
    print(i, round(dt, 1), {k: round(v, 1) for k, v in st.items()}, "slow pinned allocs:", slow, flush=True)
