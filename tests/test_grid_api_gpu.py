"""BlockGrid's public search API (grid.py:297-394 of the reference) on the
device: search_into, neighbors, count_missing_neighbors against the oracle
grid, including stale-grid two-layer queries and table overflow (the
reference's test_grid.py strategy)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _grids(pts, n_fluid, lo, hi, bs):
    from oracle import sph as O
    from paper_2009_14514_b200.grid import BlockGrid
    g = BlockGrid(lo, hi, bs)
    o = O.OracleGrid(lo, hi, bs)
    g.rebuild(pts, n_fluid)
    o.rebuild(pts.astype(np.float64), n_fluid)
    return g, o


def test_search_into_matches_oracle_rows_and_order():
    rng = np.random.default_rng(3)
    lo, hi, h = (0.0, 0.0, 0.0), (0.5, 0.4, 0.3), 0.04
    pts = rng.uniform(0.01, 0.29, (3000, 3)).astype(np.float32)
    g, o = _grids(pts, 2500, lo, hi, h)
    idx = np.arange(2500)
    nbr_d = np.full((3000, 128), -7, dtype=np.int64)
    cnt_d = np.zeros(3000, dtype=np.int64)
    nbr_o, cnt_o = nbr_d.copy(), cnt_d.copy()
    g.search_into(pts, idx, np.ones(2500, dtype=np.int64), h, nbr_d, cnt_d)
    o.search_into(pts.astype(np.float64), idx, np.ones(2500, dtype=np.int64), h, nbr_o, cnt_o)
    assert np.array_equal(cnt_d, cnt_o)
    for i in idx:
        assert np.array_equal(nbr_d[i, : cnt_d[i]], nbr_o[i, : cnt_o[i]]), i
    # stale grid, displaced queries, two layers
    moved = (pts + rng.uniform(-0.01, 0.01, pts.shape)).astype(np.float32)
    moved[2500:] = pts[2500:]
    lay = np.full(2500, 2, dtype=np.int64)
    g.search_into(moved, idx, lay, h, nbr_d, cnt_d)
    o.search_into(moved.astype(np.float64), idx, lay, h, nbr_o, cnt_o)
    assert np.array_equal(cnt_d, cnt_o)
    for i in idx:
        assert np.array_equal(nbr_d[i, : cnt_d[i]], nbr_o[i, : cnt_o[i]]), i
    # candidate superset of one particle: every member of the 27 blocks, CSR order
    cx, cy, cz = o.cell_coords(pts[17:18].astype(np.float64))[0]
    nx, ny, nz = o.dims
    want = []
    for ax in range(max(0, cx - 1), min(nx, cx + 2)):
        for ay in range(max(0, cy - 1), min(ny, cy + 2)):
            for az in range(max(0, cz - 1), min(nz, cz + 2)):
                c = (ax * ny + ay) * nz + az
                want.append(o.order[o.starts[c]:o.starts[c + 1]])
    assert np.array_equal(g.neighbors(pts, 17, 1), np.concatenate(want))


def test_count_missing_and_overflow():
    from paper_2009_14514_b200 import NumericalError
    rng = np.random.default_rng(4)
    lo, hi, h = (0.0, 0.0, 0.0), (0.3, 0.3, 0.3), 0.05
    pts = rng.uniform(0.02, 0.28, (2000, 3)).astype(np.float32)
    g, _ = _grids(pts, 2000, lo, hi, h)
    idx = np.arange(2000)
    nbr = np.zeros((2000, 128), dtype=np.int64)
    cnt = np.zeros(2000, dtype=np.int64)
    g.search_into(pts, idx, np.ones(2000, dtype=np.int64), h, nbr, cnt)
    assert g.count_missing_neighbors(pts, 2000, idx, h, nbr, cnt) == 0
    cnt2 = cnt.copy()
    cnt2[::2] -= 1  # drop the last entry of every other row
    assert g.count_missing_neighbors(pts, 2000, idx, h, nbr, cnt2) == 1000
    dense = rng.uniform(0.1, 0.12, (400, 3)).astype(np.float32)
    gd, _ = _grids(dense, 400, lo, hi, 0.08)
    small = np.zeros((400, 16), dtype=np.int64)
    with pytest.raises(NumericalError, match="neighbor table overflow"):
        gd.search_into(dense, np.arange(400), np.ones(400, dtype=np.int64), 0.08, small,
                       np.zeros(400, dtype=np.int64))
