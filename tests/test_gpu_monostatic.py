"""Monostatic DAS (reference beamform.py:215-261) — mirrors
/root/reference/pkg/tests/test_beamform.py:109-144 plus golden vectors."""

import numpy as np
import pytest

import paper_1709_02549_b200 as mw
from _mwb_helpers import dataset, load_json, peak_err, unit_geometry
from oracle import mwbeam_oracle as orc

pytestmark = pytest.mark.gpu


def test_zero_dataset():
    ds = dataset(unit_geometry([[1, 0, 0], [-1, 0, 0]]), np.zeros((2, 2, 16)))
    assert mw.das_energy_monostatic(ds, (0.0, 0.0)) == 0.0


def test_single_active_channel_squares():
    sig = np.zeros((2, 2, 8))
    sig[0, 0] = np.arange(8.0)
    ds = dataset(unit_geometry([[1, 0, 0], [-1, 0, 0]]), sig)
    assert mw.das_energy_monostatic(ds, (1.0, 0.0)) == float((sig[0, 0] ** 2).sum())


def test_cross_check_against_multistatic_kernel():
    geom = unit_geometry([[4, 0, 0], [0, 8, 0]])
    mono = np.zeros((2, 2, 32))
    mono[0, 0, 5] = 1.0
    mono[1, 1, 7] = 1.0
    multi = np.zeros((2, 2, 32))
    multi[0, 0, 11] = 1.0
    multi[1, 1, 19] = 1.0
    assert mw.das_energy_monostatic(dataset(geom, mono), (0.0, 0.0)) == mw.das_energy(dataset(geom, multi), (0.0, 0.0)) == 4.0


def test_rejects_multistatic_dataset():
    sig = np.zeros((2, 2, 8))
    sig[0, 1, 0] = 1.0
    with pytest.raises(ValueError, match="monostatic"):
        mw.das_energy_monostatic(dataset(unit_geometry([[1, 0, 0], [-1, 0, 0]]), sig), (0.0, 0.0))


def test_golden_and_image():
    for case in load_json("monostatic.json"):
        geom = mw.ring_array(case["m"], 1.0, propagation_speed=1.0, sample_interval=case["dt"])
        ds = dataset(geom, np.array(case["signals"]))
        got = np.array([mw.das_energy_monostatic(ds, r) for r in case["points"]])
        want = np.array(case["das"])
        assert np.abs(got - want).max() <= 2e-5 * max(np.abs(want).max(), 1.0)
    grid = mw.ImagingGrid((-0.8, -0.8), (1.6, 1.6), 0.1)
    em = mw.image_monostatic(ds, grid)
    cells = sorted(em.entries)
    pts = np.array([grid.cell_center(*c) for c in cells])
    ref = orc.monostatic_energies(geom.antennas, 1.0, case["dt"], ds.signals, pts)
    assert peak_err([em.entries[c] for c in cells], ref) <= 1e-4
    assert all(mw.das_energy_monostatic(ds, grid.cell_center(*c)) == em.entries[c] for c in cells[:10])
