"""Timing of device.upload_connectivity (host narrowing + chunked upload) against the plain int64 upload."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1401_3301_b200 import device as D
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
q, me = bench.make_mesh(cfg)
pme = torch.from_numpy(me).pin_memory()
dev = torch.device("cuda", 0)
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    a, b = D.upload_connectivity(pme.numpy(), q.shape[1], dev)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    x = pme.to(dev, non_blocking=True); torch.cuda.synchronize(); t3 = time.perf_counter()
    print("narrow+upload: call %.1f ms, done %.1f ms | plain int64 upload %.1f ms" % (1e3*(t1-t0), 1e3*(t2-t0), 1e3*(t3-t2)), flush=True)
    del a, b, x
