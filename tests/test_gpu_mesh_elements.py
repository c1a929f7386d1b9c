"""GPU parity: mesh generation and batched assembly vs the reference (golden) and the
oracle restatement -- bit for bit."""

import numpy as np
import numpy.testing as npt
import pytest

from conftest import golden, to_np

import oracle as o

pytestmark = pytest.mark.gpu


def test_grid_mesh_matches_reference(gpu):
    import paper_1911_03973_b200 as eb
    g = golden("mesh2d")
    for level in range(4):
        m = eb.build_unit_square_mesh(level)
        assert m.level == level and m.n_nodes == (2**level + 1) ** 2
        assert m.n_elements == 2 * 4**level
        npt.assert_array_equal(to_np(m.nodes), g[f"nodes_l{level}"])
        npt.assert_array_equal(to_np(m.elements), g[f"elements_l{level}"])
        npt.assert_array_equal(to_np(m.boundary_nodes), g[f"boundary_l{level}"])
    npt.assert_array_equal(to_np(eb.build_grid_mesh(2).elements), [[0, 1, 3], [0, 3, 2]])
    for level in (5, 7):
        nodes, elements, boundary = o.unit_square_mesh(level)
        m = eb.build_unit_square_mesh(level)
        npt.assert_array_equal(to_np(m.nodes), nodes)
        npt.assert_array_equal(to_np(m.elements), elements)
        npt.assert_array_equal(to_np(m.boundary_nodes), boundary)
        assert len(boundary) == 4 * 2**level


def test_mesh_guards_and_validation(gpu):
    import paper_1911_03973_b200 as eb
    with pytest.raises(ValueError):
        eb.build_unit_square_mesh(-1)
    with pytest.raises(ValueError):
        eb.build_unit_square_mesh(eb.MAX_LEVEL + 1)
    with pytest.raises(ValueError):
        eb.build_grid_mesh(1)
    nodes = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    with pytest.raises(ValueError):  # clockwise
        eb.Mesh(nodes, np.array([[0, 2, 1]]), np.array([0]))
    with pytest.raises(ValueError):  # out of range
        eb.Mesh(nodes, np.array([[0, 1, 3]]), np.array([0]))
    with pytest.raises(ValueError):
        eb.Mesh(nodes, np.array([[0, 1, 2]]), np.array([7]))
    with pytest.raises(ValueError):
        eb.Mesh(nodes[:, :1], np.array([[0, 1, 2]]), np.array([0]))


@pytest.mark.parametrize("N", [1, 2, 3, 5])
def test_kuhn_mesh_matches_oracle(gpu, N):
    import paper_1911_03973_b200 as eb
    nodes, elements, face = o.kuhn_cube_mesh(N)
    m = eb.build_unit_cube_mesh(N)
    npt.assert_array_equal(to_np(m.nodes), nodes)
    npt.assert_array_equal(to_np(m.elements), elements)
    npt.assert_array_equal(to_np(eb.face_z0_nodes(m)), face)
    npt.assert_array_equal(to_np(m.boundary_nodes), o.detect_boundary(nodes))
    vol = to_np(eb.signed_areas(m.nodes, conn=m.conn))
    npt.assert_array_equal(vol, o.signed_measure(nodes, elements))


@pytest.mark.parametrize("config,size", [(2, 3), (2, 5), (4, 4), (4, 6)])
def test_seeded_recipes_match_oracle(gpu, config, size):
    from paper_1911_03973_b200.inputs import config_problem
    ref = o.config_inputs(config, seed=0, size=size)
    got = config_problem(config, seed=0, size=size, assemble=False)
    npt.assert_array_equal(got["perm"], ref["perm"])
    npt.assert_array_equal(to_np(got["mesh"].nodes), ref["nodes"])
    npt.assert_array_equal(to_np(got["mesh"].elements), ref["elements"])
    npt.assert_array_equal(to_np(got["dirichlet"].nd), ref["dirichlet"])
    if config == 2:
        npt.assert_array_equal(got["x"], ref["x"])


@pytest.mark.parametrize("nu", [0.0, 1.0, 2.5])
def test_element_batch_matches_reference(gpu, nu):
    import paper_1911_03973_b200 as eb
    g = golden("batch2d_l3")
    m = eb.build_unit_square_mesh(3)
    batch = eb.build_element_batch(m, nu=nu)
    npt.assert_array_equal(to_np(batch.K_e), g[f"K_e_nu{nu}"])
    npt.assert_array_equal(to_np(batch.M_e), g[f"M_e_nu{nu}"])
    npt.assert_array_equal(to_np(batch.A_e), g[f"A_e_nu{nu}"])
    npt.assert_array_equal(to_np(batch.b_e), g[f"b_e_nu{nu}"])
    npt.assert_array_equal(to_np(eb.local_stiffness_batch(m)), g[f"K_e_nu{nu}"])
    npt.assert_array_equal(to_np(eb.local_mass_batch(m)), g[f"M_e_nu{nu}"])
    npt.assert_array_equal(to_np(eb.combine_system(batch.K_e, batch.M_e, nu)), g[f"A_e_nu{nu}"])
    with pytest.raises(ValueError):
        eb.combine_system(batch.K_e, batch.M_e, -0.5)


def test_element_known_answers(gpu):
    import paper_1911_03973_b200 as eb
    g = golden("batch2d_l3")
    K_REF = np.array([[1.0, -0.5, -0.5], [-0.5, 0.5, 0.0], [-0.5, 0.0, 0.5]])
    for h in (1.0, 0.5, 0.25, 0.0625):
        m = eb.Mesh(np.array([[0.0, 0.0], [h, 0.0], [0.0, h]]), np.array([[0, 1, 2]]),
                    np.array([0, 1, 2]))
        npt.assert_array_equal(to_np(eb.local_stiffness_batch(m))[:, :, 0], K_REF)
    m1 = eb.build_unit_square_mesh(1)
    npt.assert_array_equal(to_np(eb.local_load_batch(m1, lambda x, y: x + y)), g["b_e_xy"])
    npt.assert_array_equal(to_np(eb.local_load_batch(m1, 2.0)),
                           2.0 * to_np(eb.local_load_batch(m1, lambda x, y: np.ones_like(x))))
    with pytest.raises(ValueError):
        eb.local_load_batch(m1, lambda x, y: np.full_like(x, np.nan))
    sliver = eb.Mesh(np.array([[0.0, 0.0], [1e-7, 0.0], [0.0, 2e-7]]), np.array([[0, 1, 2]]),
                     np.array([0]))
    with pytest.raises(ValueError, match="degenerate"):
        eb.local_stiffness_batch(sliver)
    # stiffness row sums exactly zero on dyadic meshes (test_elements.py:40-45)
    K = to_np(eb.local_stiffness_batch(eb.build_unit_square_mesh(3)))
    assert np.all(K.sum(axis=1) == 0.0) and np.all(K.sum(axis=0) == 0.0)


def test_jittered_permuted_batch_matches_reference(gpu):
    import paper_1911_03973_b200 as eb
    g = golden("c4_l4_seed0")
    m = eb.Mesh(g["nodes"], g["elements"], g["dirichlet"])
    batch = eb.build_element_batch(m, nu=10.0, f=lambda x, y: np.sin(np.pi * x) * np.sin(np.pi * y))
    for k in ("K_e", "M_e", "A_e", "b_e"):
        npt.assert_array_equal(to_np(getattr(batch, k)), g[k])


@pytest.mark.parametrize("N", [2, 3])
def test_tet_batch_matches_oracle(gpu, N):
    import paper_1911_03973_b200 as eb
    g = golden("kuhn3d")
    m = eb.build_unit_cube_mesh(N)
    batch = eb.build_element_batch(m, nu=1.0)
    npt.assert_array_equal(to_np(batch.K_e), g[f"K_e_N{N}"])
    npt.assert_array_equal(to_np(batch.M_e), g[f"M_e_N{N}"])
    npt.assert_array_equal(to_np(batch.A_e), g[f"A_e_N{N}"])
    npt.assert_array_equal(to_np(batch.b_e), g[f"b_e_N{N}"])


def test_batch_validation(gpu):
    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(1)
    b = eb.build_element_batch(m)
    with pytest.raises(ValueError):
        eb.ElementBatch(K_e=b.K_e, M_e=b.M_e, A_e=b.A_e, b_e=b.b_e[:, :3], nu=0.0, index=b.index)
    with pytest.raises(ValueError):
        eb.ElementBatch(K_e=b.K_e, M_e=b.M_e, A_e=b.A_e, b_e=b.b_e, nu=-1.0, index=b.index)
