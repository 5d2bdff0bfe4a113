"""Tiled two-pass plan statistics of the C5 mesh for several ring budgets:
tiles, virtual elements / elements (halo recomputation), largest batch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_3301_b200 as P  # noqa: E402
from paper_1401_3301_b200.device import DeviceMesh  # noqa: E402

n = int(os.environ.get("N", 256))
q, me = P.device_hypercube_arrays(3, n, seed=14013305, amplitude=0.15, host=True)
mesh = P.Mesh(q, me, None)
k = P.GeneralKernel(mesh, A=np.eye(3))
for kb in sys.argv[1:]:
    os.environ["SA_TUNE"] = kb
    dm = DeviceMesh(q, me, None)
    plan = dm.plan(1)
    plan.prepare([k])
    st = plan.stats()
    print(kb, "tiles", st["tiles"], "factor", round(st["tile_elements"] / me.shape[1], 4), "maxbatch",
          st["max_batch_vertices"], flush=True)
    dm.close()
