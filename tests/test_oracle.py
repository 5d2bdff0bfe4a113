"""The CPU oracle (test infrastructure) pinned against the reference's own
outputs: every committed golden fixture was produced by the reference
(tests/golden/make_golden.py); the C restatement must reproduce it bitwise."""

import numpy as np
import pytest

from conftest import golden_cases, load_golden, oracle_op_for
from oracle import oracle as O


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matches_reference_bitwise(name):
    g = load_golden(name)
    op = oracle_op_for(name, g)
    rp, ci, va = O.assemble(g["q"], g["me"], op, nthreads=2)
    assert np.array_equal(rp, g["row_ptr"])
    assert np.array_equal(ci, g["col_idx"])
    assert np.array_equal(va, g["vals"])


@pytest.mark.parametrize("name", golden_cases("stiff_"))
def test_oracle_volumes_match_mesh_from_arrays(name):
    g = load_golden(name)
    assert np.array_equal(O.volumes(g["q"], g["me"]), g["vols"])


@pytest.mark.parametrize("name", golden_cases("stiff_d3") + golden_cases("stiff_d2"))
def test_oracle_row_block_is_bitwise_the_full_rows(name):
    # a row block of optv2 is bitwise the same rows of the full optv2
    g = load_golden(name)
    op = oracle_op_for(name, g)
    nrows = len(g["row_ptr"]) - 1
    cuts = [0, nrows // 3, (2 * nrows) // 3, nrows]
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        rp, ci, va = O.assemble_block(g["q"], g["me"], op, r0, r1)
        s, e = g["row_ptr"][r0], g["row_ptr"][r1]
        assert np.array_equal(rp + s, g["row_ptr"][r0:r1 + 1])
        assert np.array_equal(ci, g["col_idx"][s:e])
        assert np.array_equal(va, g["vals"][s:e])


def test_known_answer_reference_triangle_stiffness():
    # test_kernels.py:186-191 / test_assembly.py:82-89 golden values
    q = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    me = np.array([[0], [1], [2]])
    vols = O.volumes(q, me)
    rp, ci, va = O.assemble(q, me, O.OracleOp("stiffness", 2, vols))
    dense = np.zeros((3, 3))
    for r in range(3):
        dense[r, ci[rp[r]:rp[r + 1]]] = va[rp[r]:rp[r + 1]]
    assert np.array_equal(dense, 0.5 * np.array([[2.0, -1, -1], [-1, 1, 0], [-1, 0, 1]]))


def test_degenerate_element_named():
    q = np.array([[0.0, 1.0, 2.0, 0.0], [0.0, 1.0, 2.0, 1.0]])
    me = np.array([[0, 0], [3, 1], [1, 2]])  # element 1 is collinear
    with pytest.raises(O.OracleDegenerate) as ei:
        O.gradients(q, me)
    assert ei.value.element == 1


def test_pk_host_restatements_and_oracle_match_reference_goldens():
    # lattice, coefficient table, lattice mesh (host restatements in the
    # package) and the Pk mass oracle (oracle/) against fixtures the reference
    # itself produced (tests/golden/make_golden_pk.py) -- bitwise
    import paper_1401_3301_b200 as P
    from oracle import oracle as O
    from paper_1401_3301_b200 import pk

    names = golden_cases("pk_")
    assert len(names) >= 6
    for name in names:
        g = load_golden(name)
        d, k = g["q"].shape[0], int(g["k"])
        C = pk.pk_mass_coeffs(d, k)
        assert np.array_equal(C.C, g["C"]) and C.lattice == tuple(map(tuple, g["lattice"]))
        pm = pk.build_pk_mesh(P.Mesh(g["p1_q"], g["p1_me"], g["vols"]), k)
        assert np.array_equal(pm.me, g["me"]) and np.array_equal(pm.q, g["q"])
        rp, ci, va = O.assemble_mass_pk(g["me"], g["vols"], g["C"], d, g["q"].shape[1])
        assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])
        assert np.array_equal(va, g["vals"])
