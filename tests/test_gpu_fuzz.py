"""Randomised user batches through the device operator, bitwise against the oracle's
(j, e)-ordered bincount (operators.py:72-107, spectrum.py:54-61): arbitrary connectivity,
repeated nodes inside one element, hub nodes of valence in the thousands (rows spanning
many chunks), id spans beyond the delta-packing range (absolute-id fallback), untouched
trailing nodes, random A_e that is neither symmetric nor definite."""

import numpy as np
import numpy.testing as npt
import pytest

from conftest import to_np

import oracle as o

pytestmark = pytest.mark.gpu


def _batch(eb, A, b_e, indt):
    nb, n_e = indt.shape
    return eb.ElementBatch(K_e=A, M_e=np.zeros_like(A), A_e=A, b_e=b_e, nu=0.0,
                           index=eb.IndexArrays(indt.reshape(nb, 1, n_e), indt))


def _case(rng, nb, n_e, n_n, kind):
    if kind == "uniform":          # ids spread over the whole range: no locality
        indt = rng.integers(0, n_n, size=(nb, n_e))
    elif kind == "hub":            # a few nodes shared by thousands of elements
        indt = rng.integers(0, n_n, size=(nb, n_e))
        hubs = rng.integers(0, n_n, size=3)
        sel = rng.random(n_e) < 0.6
        indt[0, sel] = hubs[rng.integers(0, 3, size=int(sel.sum()))]
    elif kind == "repeat":         # the same node twice or more inside one element
        indt = rng.integers(0, n_n, size=(nb, n_e))
        rep = rng.random(n_e) < 0.3
        indt[1, rep] = indt[0, rep]
        if nb == 4:
            indt[3, rep[::-1]] = indt[2, rep[::-1]]
    elif kind == "local":          # mesh-like locality with a long tail of untouched nodes
        base = np.sort(rng.integers(0, n_n // 2, size=n_e))
        indt = (base[None, :] + rng.integers(0, 40, size=(nb, n_e))) % (n_n // 2)
    else:
        raise AssertionError(kind)
    A = rng.standard_normal((nb, nb, n_e))
    b_e = rng.standard_normal((nb, n_e))
    return A, b_e, indt.astype(np.int64)


@pytest.mark.parametrize("nb", [3, 4])
@pytest.mark.parametrize("kind", ["uniform", "hub", "repeat", "local"])
def test_random_batches_bitwise(gpu, nb, kind):
    import paper_1911_03973_b200 as eb
    rng = np.random.default_rng([nb, sum(kind.encode())])  # reproducible (str hashes are salted)
    for n_e, n_n in ((1, 5), (37, 50), (5000, 3000), (40000, 200000)):
        A, b_e, indt = _case(rng, nb, n_e, n_n, kind)
        batch = _batch(eb, A, b_e, indt)
        x = rng.uniform(-1, 1, n_n)
        npt.assert_array_equal(to_np(eb.residual(batch, x)), o.residual(A, b_e, indt, x),
                               err_msg=f"{kind} nb={nb} n_e={n_e}")
        nd = np.unique(rng.integers(0, n_n, size=max(1, n_n // 10)))
        d = eb.DirichletData(nd, np.zeros(len(nd)))
        npt.assert_array_equal(to_np(eb.matvec(batch, x, d)), o.matvec_masked(A, indt, x, nd))
        npt.assert_array_equal(to_np(eb.diagonal(batch, n_n)), o.diagonal(A, indt, n_n))
        npt.assert_array_equal(to_np(eb.assemble_rhs(b_e, indt)),
                               np.bincount(indt.ravel(), b_e.ravel(), minlength=indt.max() + 1))
        fast = to_np(eb.residual(batch, x, deterministic=False))
        ref = o.residual(A, b_e, indt, x)
        assert np.max(np.abs(fast - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1.0)


def test_hub_valence_info(gpu):
    """One node in every element: its row is n_e slots long (spans many 32-row chunks)."""
    import paper_1911_03973_b200 as eb
    rng = np.random.default_rng(7)
    n_e, n_n = 20000, 30000
    indt = rng.integers(0, n_n, size=(3, n_e))
    indt[2, :] = 12345
    A = rng.standard_normal((3, 3, n_e))
    b_e = rng.standard_normal((3, n_e))
    batch = _batch(eb, A, b_e, indt)
    assert batch.operator(n_n).info()["max_valence"] >= n_e
    x = rng.uniform(-1, 1, n_n)
    npt.assert_array_equal(to_np(eb.residual(batch, x)), o.residual(A, b_e, indt, x))
