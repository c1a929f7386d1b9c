"""uniform_refine / export_mesh on the device (mesh.py:157-218) vs the reference."""

import numpy as np
import numpy.testing as npt
import pytest

from conftest import golden, to_np

import oracle as o

pytestmark = pytest.mark.gpu


def test_refine_reproduces_generator(gpu):
    import paper_1911_03973_b200 as eb
    for level in range(4):
        fine = eb.uniform_refine(eb.build_unit_square_mesh(level))
        direct = eb.build_unit_square_mesh(level + 1)
        npt.assert_array_equal(to_np(fine.nodes), to_np(direct.nodes))
        npt.assert_array_equal(to_np(fine.elements), to_np(direct.elements))
        npt.assert_array_equal(to_np(fine.boundary_nodes), to_np(direct.boundary_nodes))
        assert fine.level == level + 1


def test_refine_unstructured_matches_reference(gpu):
    import paper_1911_03973_b200 as eb
    g = golden("refine")
    fine = eb.uniform_refine(eb.Mesh(g["nodes"], g["elements"], g["boundary"]))
    npt.assert_array_equal(to_np(fine.nodes), g["fine_nodes"])
    npt.assert_array_equal(to_np(fine.elements), g["fine_elements"])
    npt.assert_array_equal(to_np(fine.boundary_nodes), g["fine_boundary"])
    assert fine.level is None


def test_refine_single_triangle_and_area(gpu):
    import paper_1911_03973_b200 as eb
    m = eb.Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]]),
                np.array([0, 1, 2]))
    fine = eb.uniform_refine(m)
    assert fine.level is None and fine.n_nodes == 6 and fine.n_elements == 4
    assert np.all(to_np(eb.signed_areas(fine.nodes, conn=fine.conn)) == 0.125)
    m = eb.build_unit_square_mesh(2)
    for _ in range(2):
        m = eb.uniform_refine(m)
        assert float(eb.signed_areas(m.nodes, conn=m.conn).sum()) == 1.0
    small = eb.build_unit_square_mesh(1)
    at_cap = eb.Mesh(small.nodes, small.elements, small.boundary_nodes, level=eb.MAX_LEVEL)
    with pytest.raises(ValueError):
        eb.uniform_refine(at_cap)


def test_export_mesh_roundtrip(gpu, tmp_path):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(2)
    eb.export_mesh(m, tmp_path)
    npt.assert_array_equal(np.loadtxt(tmp_path / "nodes.txt"), to_np(m.nodes))
    npt.assert_array_equal(np.loadtxt(tmp_path / "elements.txt", dtype=np.int64), to_np(m.elements))


def test_refine_is_native_and_large(gpu):
    """ebs_refine_tri (libebs) at size: level 9 -> 10 equals the generator bit for bit, and
    a jittered + permuted (unstructured numbering) mesh refines like the oracle restatement
    of mesh.py:157-208."""
    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200._lib import launch_count
    n0 = launch_count()
    fine = eb.uniform_refine(eb.build_unit_square_mesh(9))
    assert launch_count() > n0  # device kernels, not host code
    direct = eb.build_unit_square_mesh(10)
    npt.assert_array_equal(to_np(fine.nodes), to_np(direct.nodes))
    npt.assert_array_equal(to_np(fine.conn), to_np(direct.conn))
    inp = o.config_inputs(4, seed=3, size=5)
    m = eb.Mesh(inp["nodes"], inp["elements"], inp["dirichlet"])
    fine = eb.uniform_refine(m)
    ref_nodes, ref_elements = o.uniform_refine(inp["nodes"], inp["elements"])
    npt.assert_array_equal(to_np(fine.nodes), ref_nodes)
    npt.assert_array_equal(to_np(fine.elements), ref_elements)
