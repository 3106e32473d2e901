"""Seeded random sweep of the imaging kernel against the oracle: antenna
count, channel population, record length (ragged, not multiples of 4),
window start/length (inside, straddling and beyond the record, 32- and
48-sample chunks), interpolation, stride, region, mask and kind.  Also the
largest supported geometry (64 antennas, 4032 directed channels)."""

import numpy as np
import pytest

import paper_1709_02549_b200 as mw
from oracle import mwbeam_oracle as orc

pytestmark = pytest.mark.gpu


def _oracle(ds, pts, kind, interp, window):
    g = ds.geometry
    if window is None:
        return orc.multistatic_energies(g.antennas, g.propagation_speed, g.sample_interval, ds.signals, pts, kind,
                                        interp)
    k0, w = window
    return orc.windowed_energies_direct(g.antennas, g.propagation_speed, g.sample_interval, ds.signals, pts, kind,
                                        k0, w, interp)


@pytest.mark.parametrize("case", range(24))
def test_random_configuration(case):
    rng = np.random.default_rng(9000 + case)
    m = int(rng.integers(2, 9))
    n = int(rng.integers(5, 200))
    radius = float(rng.uniform(0.03, 0.08))
    geom = mw.ring_array(m, radius, propagation_speed=float(rng.uniform(0.6e8, 3e8)),
                         sample_interval=float(rng.uniform(5e-12, 4e-11)))
    sig = np.zeros((m, m, n))
    pop = rng.uniform(size=(m, m)) < rng.uniform(0.3, 1.0)
    sig[pop] = rng.normal(size=(int(pop.sum()), n))
    ds = mw.BackscatterDataset(geom, sig)
    res = float(rng.uniform(0.002, 0.01))
    side = 2 * radius
    grid = mw.ImagingGrid((-radius, -radius), (side, side), res)
    nx, ny = grid.dims
    stride = int(rng.integers(1, 4))
    x0, x1 = sorted(int(v) for v in rng.integers(0, nx, 2))
    y0, y1 = sorted(int(v) for v in rng.integers(0, ny, 2))
    region = mw.Region((x0, y0), (x1, y1))
    mask = rng.uniform(size=grid.dims) < 0.8 if case % 3 == 0 else None
    interp = "nearest" if case % 4 == 1 else "linear"
    choice = case % 5
    if choice == 0:
        window = None
    elif choice == 1:
        window = (int(rng.integers(0, n)), 48)
    elif choice == 2:
        window = (int(rng.integers(0, max(1, n // 2))), int(rng.integers(1, 40)))
    elif choice == 3:
        window = (n + 3, 32)  # entirely past the record: all zeros
    else:
        window = (int(rng.integers(0, n)), 96)
    kind = ("das", "dmas")[case % 2]
    em = mw.image(ds, kind, grid, region=region, stride=stride, mask=mask, interpolation=interp, window=window)
    ix, iy = orc.region_cells(grid.dims, (region.min_cell, region.max_cell), stride, mask)
    assert list(em.entries) == list(zip(ix.tolist(), iy.tolist()))
    if len(ix) == 0:
        return
    pts = np.array([grid.cell_center(a, b) for a, b in zip(ix.tolist(), iy.tolist())])
    want = _oracle(ds, pts, kind, interp, window)
    got = np.array(list(em.entries.values()))
    scale = np.abs(want).max()
    if scale == 0:
        assert (got == 0).all()
    else:
        assert np.abs(got - want).max() <= 1e-4 * scale, (m, n, window, interp, kind)
    # the same points through the point-list path give identical bits
    pt = mw.energies(ds, pts, kind, interp, window=window)
    assert np.array_equal(pt.astype(np.float32), got.astype(np.float32))


def test_largest_geometry_64_antennas():
    rng = np.random.default_rng(64)
    m, n = 64, 96
    geom = mw.ring_array(m, 0.06, propagation_speed=1e8, sample_interval=2e-11)
    sig = rng.normal(size=(m, m, n))
    ds = mw.BackscatterDataset(geom, sig)
    pts = rng.uniform(-0.04, 0.04, (40, 2))
    for kind in ("das", "dmas"):
        got = mw.energies(ds, pts, kind, window=(5, 32))
        want = orc.windowed_energies(geom.antennas, 1e8, 2e-11, sig, pts, kind, 5, 32)
        assert np.abs(got - want).max() <= 1e-4 * np.abs(want).max()
