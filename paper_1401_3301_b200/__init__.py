"""B200-native P1 finite-element assembly (arXiv 1401.3301, vectorised OptV2
semantics) behind the reference ``simplex_asm`` driver API.

    from paper_1401_3301_b200 import assemble_b200, StiffnessKernel
    A = assemble_b200(mesh, StiffnessKernel(mesh))     # canonical CSR, bitwise optv2

All numerics run in hand-written sm_100a CUDA (csrc/), reached through the C
ABI in include/simplex_asm_b200.h.  There is no CPU fallback.
"""

from .errors import (
    CapacityError,
    DegenerateSimplexError,
    ExtensionMissingError,
    IndexRangeError,
    NonSymmetricKernelError,
    SimplexAsmError,
)
from .kernels import ElasticKernel, GeneralKernel, MassKernel, StiffnessKernel
from .mesh import (
    Mesh,
    device_hypercube_arrays,
    device_hypercube_slab,
    generate_hypercube_mesh,
    hypercube_arrays,
    jitter_interior,
    jittered_hypercube_mesh,
)
from .pk import PkCoeffTable, PkMesh, build_pk_mesh, multi_index_lattice, pk_mass_coeffs
from .sparse import SparseMatrix, to_scipy, write_matrixmarket

__version__ = "0.1.0"


def __getattr__(name):
    # the device layer imports torch and loads the sm_100a library lazily
    if name in ("assemble_b200", "assemble_vector_b200", "assemble_many_b200", "assemble_device",
                "SCALAR_DRIVERS", "VECTOR_DRIVERS", "register", "to_host", "device_mesh_for",
                "assemble_mass_pk_b200"):
        from . import assembly

        return getattr(assembly, name)
    if name in ("DeviceMesh", "Plan", "DeviceCSR", "device_volumes", "launch_count"):
        from . import device

        return getattr(device, name)
    raise AttributeError(name)
