"""GPU parity of the narrow-row cell filter of f(C, X) (objective_rows.cuh, GRID variant: fp64 rows of
n <= 3 and fp32 rows of n = 2, kv <= 32): labels and counts bit-exact against the oracle's reference
argmin (core.hpp:146-157), the cost within the fp64 / fp32-mode tolerance. Cases: exact ties on
lattices (bisectors through cells), rows far from the origin, rows outside the grid, duplicate centres,
the kv = 32 limit and kv = 33 (the screen kernel), a config-3-shaped mixture."""
import numpy as np
import pytest

import paper_2311_04517_b200 as hp
from oracle_py import orc

pytestmark = pytest.mark.gpu

RTOL = 1e-12
FP32_RTOL = 1e-5


def rel(a, b):
    return abs(float(a) - float(b)) / max(abs(float(b)), 1e-300)


def check(X, C_):
    lab, cnt, cost, _ = orc().assign(np.asarray(X, np.float64), np.asarray(C_, np.float64))
    a, f = hp.final_assignment(X, C_)
    assert np.array_equal(a.labels, lab)
    assert np.array_equal(a.counts, cnt)
    assert rel(f, cost) <= (FP32_RTOL if np.asarray(X).dtype == np.float32 else RTOL)


@pytest.mark.parametrize("dtype,n", [(np.float64, 1), (np.float64, 2), (np.float64, 3), (np.float32, 2)])
def test_lattice_ties_lowest_index(dtype, n):
    # integer lattice rows and centres: many rows exactly on bisectors (exact fp64 ties)
    g = np.arange(-12, 13, dtype=np.float64)
    X = np.stack(np.meshgrid(*([g] * n), indexing="ij"), -1).reshape(-1, n)
    rs = np.random.default_rng(n)
    C_ = rs.integers(-6, 7, (9, n)).astype(np.float64)
    check(X.astype(dtype), C_)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_far_from_origin(n):
    # |x| ~ 1e6 with clusters 0.5 apart: the cell index and the drop test at large offsets
    rs = np.random.default_rng(10 + n)
    C_ = 1e6 + 0.5 * rs.standard_normal((12, n))
    X = C_[rs.integers(0, 12, 100001)] + 0.3 * rs.standard_normal((100001, n))
    check(X, C_)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_rows_outside_the_grid_and_duplicate_centres(n):
    rs = np.random.default_rng(20 + n)
    C_ = rs.uniform(-1, 1, (6, n))
    C_[5] = C_[2]  # duplicate centre: ties to the lower index
    X = np.concatenate([rs.uniform(-1, 1, (20000, n)), 50 * rs.standard_normal((20000, n))])
    check(X, C_)


@pytest.mark.parametrize("k", [32, 33])
def test_kv_limit(k):
    rs = np.random.default_rng(k)
    C_ = rs.uniform(0, 255, (k, 3))
    X = C_[rs.integers(0, k, 60000)] + 8 * rs.standard_normal((60000, 3))
    check(X, C_)


def test_config3_shaped_mixture():
    rs = np.random.default_rng(2314)
    means = rs.uniform(0, 255, (25, 3))
    X = means[rs.integers(0, 25, 400000)] + 8 * rs.standard_normal((400000, 3))
    noise = rs.random(400000) < 0.01
    X[noise] = rs.uniform(0, 255, (int(noise.sum()), 3))
    check(X, means + 0.3 * rs.standard_normal(means.shape))
