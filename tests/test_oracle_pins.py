"""The oracle against the reference's own known-answer tests (CPU).

Restates, for ``oracle.mwbeam_oracle``, the hand values and properties the
reference asserts for its kernel and framework helpers
(/root/reference/pkg/tests/test_beamform.py:86-239,
test_coarse2fine.py:29-85, test_acceptance.py:143-176).  Together with the
golden vectors from the real reference (test_oracle_golden.py) they pin the
oracle that the GPU parity tests compare against.
"""

import math

import numpy as np
import pytest

from oracle import mwbeam_oracle as orc

UNIT = np.array([[1.0, 0, 0], [-1.0, 0, 0]])  # v = dt = 1: delays are distance sums


def e(ants, sig, r, kind, interp="linear"):
    return float(orc.multistatic_energies(ants, 1.0, 1.0, sig, np.array([r], dtype=float), kind, interp)[0])


def ring(m, radius=1.0):
    return np.asarray(orc.ring_antennas(m, radius), dtype=float)


def aligned(ants, sig, i, j, r):
    """One channel aligned to r by linear interpolation, zero past the record
    (the reference's aligned_channel, beamform.py:136-166, restated)."""
    d = lambda a: math.sqrt((r[0] - a[0]) ** 2 + (r[1] - a[1]) ** 2 + a[2] ** 2)  # noqa: E731
    n = d(ants[i]) + d(ants[j])
    i0 = math.floor(n)
    f = n - i0
    y = np.concatenate([sig[i, j], np.zeros(i0 + 2)])
    k = np.arange(sig.shape[2])
    return (1 - f) * y[k + i0] + f * y[k + i0 + 1]


def brute_force_dmas(ants, sig, r):
    """O(M^4) pairwise sum over all directed channels (test_beamform.py:147-157)."""
    m = sig.shape[0]
    al = [aligned(ants, sig, i, j, r) for i in range(m) for j in range(m)]
    return sum(float((al[k] * al[l]).sum()) for k in range(len(al)) for l in range(k + 1, len(al)))


def test_zero_dataset_and_unit_impulse():
    assert e(UNIT, np.zeros((2, 2, 16)), (0.0, 0.0), "das") == 0.0
    sig = np.zeros((2, 2, 16))
    sig[0, 1, 4] = 1.0  # aligned by delay 2 -> lands at sample 2
    assert e(UNIT, sig, (0.0, 0.0), "das") == 1.0


def test_dmas_hand_values():
    sig = np.zeros((2, 2, 16))
    sig[0, 1, 5] = 2.5
    assert e(UNIT, sig, (0.3, -0.2), "dmas") == 0.0  # one channel: no pairs
    sig = np.zeros((2, 2, 16))
    sig[0, 0, 6] = 3.0
    sig[0, 1, 6] = 4.0
    assert e(UNIT, sig, (0.0, 0.0), "dmas") == 12.0  # ((3 + 4)^2 - (9 + 16)) / 2


def test_dmas_identity_matches_brute_force():
    rng = np.random.default_rng(123)
    for _ in range(10):
        ants = ring(4)
        sig = rng.normal(size=(4, 4, 64))
        r = rng.uniform(-0.8, 0.8, 2)
        assert e(ants, sig, r, "dmas") == pytest.approx(brute_force_dmas(ants, sig, r), rel=1e-9, abs=1e-12)


def test_kernel_properties():
    rng = np.random.default_rng(1)
    ants = ring(3)
    sig = rng.normal(size=(3, 3, 48))
    r = (0.3, 0.1)
    for kind in ("das", "dmas"):
        assert e(ants, 2.0 * sig, r, kind) == 4.0 * e(ants, sig, r, kind)  # exact
        assert e(ants, 1.7 * sig, r, kind) == pytest.approx(1.7**2 * e(ants, sig, r, kind), rel=1e-12)
    ants4 = ring(4)
    sig4 = np.random.default_rng(3).normal(size=(4, 4, 48))
    perm = np.array([2, 0, 3, 1])
    for seed in range(5):
        r = np.random.default_rng(seed).uniform(-0.8, 0.8, 2)
        for kind in ("das", "dmas"):
            assert e(ants4[perm], sig4[np.ix_(perm, perm)], r, kind) == pytest.approx(e(ants4, sig4, r, kind),
                                                                                     rel=1e-12)
    for seed in range(10):
        g = np.random.default_rng(seed)
        s = g.normal(size=(3, 3, 48))
        for _ in range(5):
            assert e(ants, s, g.uniform(-1.5, 1.5, 2), "das") >= 0.0


def test_nearest_equals_rounded_delays():
    """interpolation='nearest' rounds the delay (beamform.py:187-188): the energy
    equals the linear one of a signal shifted by whole samples."""
    sig = np.zeros((2, 2, 16))
    sig[0, 1, 7] = 1.0
    r = (0.25, 0.0)  # on the antenna axis: delay 0.75 + 1.25 = 2 exactly
    assert math.sqrt((0.25 - 1) ** 2) + math.sqrt((0.25 + 1) ** 2) == 2.0
    assert e(UNIT, sig, r, "das", "nearest") == e(UNIT, sig, r, "das") == 1.0
    r = (0.0, 0.3)  # delay 2 * sqrt(1.09) = 2.088 -> rounds to 2
    assert e(UNIT, sig, r, "das", "nearest") == 1.0
    assert e(UNIT, sig, r, "das") < 1.0


def test_framework_helpers_hand_values():
    # auto decimation factor (test_coarse2fine.py:29-41)
    assert orc.auto_decimation_factor(0.01, 0.001) == 7
    assert orc.auto_decimation_factor(0.001, 0.001) == 1
    assert orc.auto_decimation_factor(0.02, 0.001) == 14
    # Eq. (5) (test_coarse2fine.py:44-62, acceptance criterion 5)
    assert orc.metric_parts(np.array([1.0, 3.0]), 1.0)[0] == 2.0  # Delta = 0 -> mean
    assert orc.metric_parts(np.array([0.0, 4.0]), 0.0)[0] == 4.0  # Delta = 1 -> variance
    assert orc.metric_parts(np.array([2.0, 2.0]), 5.0)[0] == 2.0  # sigma^2 = 0 -> mean
    # W / B distances (test_coarse2fine.py:82-85)
    assert orc.class_distances([1.0, 3.0], [2.0, 6.0]) == (10.0, 4.0)
