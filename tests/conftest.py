import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a library")


def golden_cases(prefix=""):
    """P1 fixtures (make_golden.py); prefix "pk_" selects the Pk mass ones
    (make_golden_pk.py)."""
    names = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))
    return names if prefix.startswith("pk_") else [n for n in names if not n.startswith("pk_")]


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def oracle_op_for(name, g):
    """OracleOp matching a golden fixture name."""
    from oracle import oracle as O

    d = g["q"].shape[0]
    kind = name.split("_")[0]
    if kind == "mass":
        return O.OracleOp("mass", d, g["vols"], w=g["w"])
    if kind == "mass1":
        return O.OracleOp("mass", d, g["vols"], w=np.ones(g["q"].shape[1]))
    if kind == "stiff":
        return O.OracleOp("stiffness", d, g["vols"])
    if kind == "elastic":
        return O.OracleOp("elastic", d, g["vols"], lamb=g["lamb"], mu=g["mu"])
    if kind == "elasticc":
        nq = g["q"].shape[1]
        return O.OracleOp("elastic", d, g["vols"], lamb=np.full(nq, 1.0), mu=np.full(nq, 0.5))
    if kind == "general":
        return O.OracleOp("general", d, g["vols"], A=g["A"], b=g["b"], c=g["c"], a0=g["a0"])
    raise KeyError(name)


def device_kernel_for(name, g, mesh):
    """Product kernel descriptor matching a golden fixture name."""
    import paper_1401_3301_b200 as P

    kind = name.split("_")[0]
    if kind == "mass":
        return P.MassKernel(mesh, g["w"])
    if kind == "mass1":
        return P.MassKernel(mesh)
    if kind == "stiff":
        return P.StiffnessKernel(mesh)
    if kind == "elastic":
        return P.ElasticKernel(mesh, g["lamb"], g["mu"])
    if kind == "elasticc":
        return P.ElasticKernel(mesh, 1.0, 0.5)
    if kind == "general":
        return P.GeneralKernel(mesh, A=g["A"], b=g["b"], c=g["c"], a0=g["a0"], exact=True)
    raise KeyError(name)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
