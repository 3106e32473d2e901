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


# ---------------------------------------------------------------------------
# near-tie excuse for selection traces
# ---------------------------------------------------------------------------
NEAR = 1e-4


def _rec(r, key):
    """Field of a trace record given as a dict (oracle / golden) or an object (GPU)."""
    if isinstance(r, dict):
        return r[{"w": "W", "b": "B"}.get(key, key)]
    return getattr(r, key)


def _close(a, b, tol=NEAR) -> bool:
    return abs(a - b) <= tol * max(abs(a), abs(b), 1e-300)


def _scores_tied(r) -> bool:
    sc = sorted([s for s in _rec(r, "scores") if s != float("-inf")], reverse=True)
    return len(sc) >= 2 and _close(sc[0], sc[1])


def _satisfied_fragile(r, prev) -> bool:
    """Could the W/B test of record r (coarse2fine.py:235, ``B > B_prev or
    W < W_prev``) flip under a relative perturbation of NEAR?  With it
    satisfied, every clause that holds must be a near-tie; with it failed,
    one near-tie clause suffices."""
    if prev is None:
        return False  # the first iteration is satisfied unconditionally
    b, w, pb, pw = _rec(r, "b"), _rec(r, "w"), _rec(prev, "b"), _rec(prev, "w")
    clauses = [(b > pb, _close(b, pb)), (w < pw, _close(w, pw))]
    if any(ok for ok, _ in clauses):
        return all(tie for ok, tie in clauses if ok)
    return any(tie for _, tie in clauses)


def divergence_excused(got_records, got_term, want_records, want_term) -> tuple[bool, bool, str]:
    """(same, excused, why) for a GPU selection trace against the oracle's.

    The traces are compared record by record.  At the FIRST iteration where
    they differ (selected child, W/B verdict, or one trace ending), the
    difference is excused only if that iteration is a near-tie: the oracle's
    top-two child scores within NEAR, or its W/B verdict fragile within NEAR
    (the GPU record stands in where the oracle stopped without a record, e.g.
    an n-min termination).  A divergence at any other iteration is not
    excused, whatever happens elsewhere in the trace.
    """
    n = max(len(got_records), len(want_records))
    for i in range(n):
        g = got_records[i] if i < len(got_records) else None
        w = want_records[i] if i < len(want_records) else None
        if g is not None and w is not None and _rec(g, "selected") == _rec(w, "selected") \
                and bool(_rec(g, "satisfied")) == bool(_rec(w, "satisfied")):
            continue
        r = w if w is not None else g
        prev_list = want_records if w is not None else got_records
        prev = prev_list[i - 1] if i > 0 else None
        if _scores_tied(r):
            return False, True, f"iteration {i + 1}: top-two scores within {NEAR}"
        if g is not None and w is not None and _rec(g, "selected") == _rec(w, "selected") \
                and _satisfied_fragile(r, prev):
            return False, True, f"iteration {i + 1}: W/B verdict within {NEAR}"
        return False, False, f"iteration {i + 1}: diverges without a near-tie"
    if got_term != want_term:
        # same records, different stop: decided by the iteration after the
        # last record (n-min / region-floor are exact integer tests)
        return False, False, f"termination {got_term!r} != {want_term!r}"
    return True, False, ""
