"""Shared test inputs.  Reference-style datasets come from the oracle's
restatement of the reference simulator (simulate.py:111-162, presets.py);
BASELINE-config scans come from paper_1709_02549_b200.synth."""

from __future__ import annotations

import hashlib
import json

import numpy as np

import paper_1709_02549_b200 as mw
from oracle import mwbeam_oracle as orc
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def unit_geometry(positions):
    """v = dt = 1 so delays equal plain distance sums (test_beamform.py:20-22)."""
    return mw.ArrayGeometry(np.asarray(positions, dtype=float), 1.0, 1.0)


def dataset(geom, signals):
    return mw.BackscatterDataset(geom, np.asarray(signals, dtype=float))


def grid_for_geometry(geom, resolution) -> mw.ImagingGrid:
    origin, extent, res = orc.grid_for_antennas(geom.antennas, resolution)
    return mw.ImagingGrid(origin, extent, res)


def sim_small(radius=0.05, tumor=(0.01, -0.005), n_ant=8, n=256, noise_std=0.0, seed=0):
    """test_beamform.py:29-32 / test_coarse2fine.py:23-26."""
    geom = mw.ring_array(n_ant, radius, sample_interval=1e-11)
    sig = orc.simulate(geom.antennas, geom.propagation_speed, geom.sample_interval, n, [(tumor, 1.0)],
                       noise_std=noise_std, seed=seed)
    return tumor, mw.BackscatterDataset(geom, sig)


def preset(name: str, noise_std: float = 0.0, seed: int = 0, tumor_free: bool = False):
    """presets.py:22-55 (dataset1 / dataset2), 12-antenna ring on the phantom boundary."""
    radius, tumour = {"dataset1": (0.10, (-0.02, -0.03)), "dataset2": (0.05, (0.02, 0.0))}[name]
    geom = mw.ring_array(12, radius, sample_interval=1e-11)
    scat = [] if tumor_free else [(tumour, 1.0)]
    sig = orc.simulate(geom.antennas, geom.propagation_speed, geom.sample_interval, 256, scat,
                       noise_std=noise_std, seed=seed)
    return tumour, mw.BackscatterDataset(geom, sig)


def load_json(name):
    return json.loads((GOLDEN / name).read_text())


def peak_err(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.abs(got - want).max() / np.abs(want).max())


def masked_rel_err(got, want, frac=1e-2) -> float:
    """Per-pixel relative error on pixels with |ref| >= frac * peak."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    keep = np.abs(want) >= frac * np.abs(want).max()
    return float((np.abs(got - want)[keep] / np.abs(want)[keep]).max())
