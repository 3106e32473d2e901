"""Host-side logic (CPU only): geometry types, framework helpers, EnergyMap
semantics, trace decoding and the synthetic generator — mirroring
/root/reference/pkg/tests/test_geometry.py and test_coarse2fine.py:29-97."""

import json
import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1709_02549_b200 as mw
from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import _native as nat
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.coarse2fine import decode_trace


class TestGeometry:
    def test_ring_array_first_antenna_on_x(self):
        g = mw.ring_array(4, 2.0, center=(1.0, -1.0))
        np.testing.assert_allclose(g.antennas[0], [3.0, -1.0, 0.0])
        np.testing.assert_allclose(g.antennas[1], [1.0, 1.0, 0.0], atol=1e-12)
        assert not g.antennas.flags.writeable

    def test_geometry_validation(self):
        with pytest.raises(ValueError):
            mw.ArrayGeometry(np.zeros((3, 2)))
        with pytest.raises(ValueError):
            mw.ArrayGeometry(np.zeros((1, 3)))
        with pytest.raises(ValueError):
            mw.ArrayGeometry(np.array([[0, 0, 0], [0, 0, 0.0]]))
        with pytest.raises(ValueError):
            mw.ArrayGeometry(np.array([[0, 0, 0], [1, 0, 0.0]]), propagation_speed=0.0)
        with pytest.raises(ValueError):
            mw.ArrayGeometry(np.array([[0, 0, np.nan], [1, 0, 0.0]]))

    def test_delays_hand_values(self):  # test_geometry.py hand values
        g = mw.ArrayGeometry(np.array([[3.0, 0, 0], [0, 4.0, 0]]), 1.0, 1.0)
        assert mw.distance(g, 0, (0.0, 0.0)) == 3.0
        assert mw.delay_monostatic(g, 1, (0.0, 0.0)) == 2.0
        assert mw.delay_multistatic(g, 0, 1, (0.0, 0.0)) == 7.0
        assert mw.delay_multistatic(g, 0, 0, (0.0, 0.0)) == 4 * mw.delay_monostatic(g, 0, (0.0, 0.0))

    def test_grid_dims_and_centres(self):
        g = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
        assert g.dims == (100, 100)
        assert g.cell_center(0, 0) == (-0.05 + 0.5e-3, -0.05 + 0.5e-3)
        assert g.point_to_cell(0.0, 0.0) == (50, 50)
        assert mw.ImagingGrid((0, 0), (0.0105, 0.01), 1e-3).dims == (11, 10)
        with pytest.raises(ValueError):
            mw.ImagingGrid((0, 0), (0.01, 0.01), 0.0)

    @settings(max_examples=200)
    @given(x0=st.integers(0, 20), y0=st.integers(0, 20), w=st.integers(1, 30), h=st.integers(1, 30))
    def test_quadrants_partition_exactly(self, x0, y0, w, h):  # test_geometry.py:153-174
        r = mw.Region((x0, y0), (x0 + w - 1, y0 + h - 1))
        q = r.quadrants()
        if w < 2 or h < 2:
            assert q is None
            return
        assert sum(x.n_cells for x in q) == r.n_cells
        cells = set()
        for x in q:
            assert r.contains_region(x)
            for ix in range(x.min_cell[0], x.max_cell[0] + 1):
                for iy in range(x.min_cell[1], x.max_cell[1] + 1):
                    cells.add((ix, iy))
        assert len(cells) == r.n_cells
        assert q[0].width >= q[1].width and q[0].height >= q[2].height
        assert [(a.min_cell, a.max_cell) for a in q] == [tuple(map(tuple, z)) for z in
                                                         orc.quadrants((r.min_cell, r.max_cell))]

    def test_expand_and_intersection(self):
        parent = mw.Region((0, 0), (19, 19))
        r = mw.Region((5, 5), (9, 9)).expand(0.25, parent)
        assert r == mw.Region((3, 3), (11, 11))
        assert mw.Region((0, 0), (3, 3)).expand(0.5, parent) == mw.Region((0, 0), (5, 5))
        assert mw.Region((0, 0), (2, 2)).intersection(mw.Region((3, 3), (4, 4))) is None
        assert mw.Region((0, 0), (5, 5)).intersection(mw.Region((3, 2), (9, 4))) == mw.Region((3, 2), (5, 4))
        assert mw.Region.from_dict(r.to_dict()) == r


class TestFrameworkHelpers:  # test_coarse2fine.py:29-97
    def test_auto_factor(self):
        assert mw.auto_decimation_factor(0.01, 0.001) == 7
        assert mw.auto_decimation_factor(0.001, 0.001) == 1
        assert mw.auto_decimation_factor(0.02, 0.001) == 14
        with pytest.raises(ValueError):
            mw.auto_decimation_factor(0.0, 0.001)

    def test_decision_metric_hand_values(self):
        assert mw.decision_metric([1.0, 3.0], 1.0) == 2.0
        assert mw.decision_metric([0.0, 4.0], 0.0) == 4.0
        assert mw.decision_metric([0.0, 4.0], 2.0) == 3.0
        assert mw.decision_metric([5.0, 5.0, 5.0], 3.0) == 5.0
        with pytest.raises(ValueError):
            mw.decision_metric([], 1.0)

    @settings(max_examples=200)
    @given(vals=st.lists(st.floats(-1e6, 1e6), min_size=1, max_size=12), prev=st.floats(0, 1e9))
    def test_metric_between_mean_and_variance(self, vals, prev):
        arr = np.asarray(vals)
        mu, var = float(arr.mean()), float(arr.var())
        out = mw.decision_metric(vals, prev)
        lo, hi = min(mu, var), max(mu, var)
        span = max(abs(lo), abs(hi), 1.0)
        assert lo - 1e-9 * span <= out <= hi + 1e-9 * span

    def test_class_distances(self):
        assert mw.class_distances([5.0, 5.0], [5.0, 5.0]) == (0.0, 0.0)
        assert mw.class_distances([1.0, 3.0], [2.0, 6.0]) == (10.0, 4.0)
        w1, b1 = mw.class_distances([1.0, 3.0, 7.0], [2.0, 6.0])
        w2, b2 = mw.class_distances([2.0, 6.0], [1.0, 3.0, 7.0])
        assert w1 == w2 and b1 == pytest.approx(b2, rel=1e-12)
        with pytest.raises(ValueError):
            mw.class_distances([], [1.0])

    def test_config_validation(self):
        with pytest.raises(ValueError):
            mw.FrameworkConfig(frame_fraction=1.0)
        with pytest.raises(ValueError):
            mw.FrameworkConfig(n_min=0)
        with pytest.raises(ValueError):
            mw.Manual(0)
        with pytest.raises(ValueError):
            mw.Automatic(0.0)

    def test_breast_mask(self):  # test_coarse2fine.py:252-260
        grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 0.001)
        mask = mw.breast_mask(grid)
        assert mask[50, 50] and not mask[0, 0] and not mask[99, 99]
        assert mask.sum() == pytest.approx(np.pi * 50**2, rel=0.02)
        np.testing.assert_array_equal(mask, orc.breast_mask(grid.origin, grid.resolution, grid.dims))


class TestEnergyMapHost:  # test_beamform.py:312-329
    def test_rejects_nonfinite(self):
        grid = mw.ImagingGrid((0, 0), (0.01, 0.01), 0.001)
        with pytest.raises(ValueError):
            mw.EnergyMap(grid, {(0, 0): float("nan")})

    def test_argmax_ties(self):
        grid = mw.ImagingGrid((0, 0), (0.01, 0.01), 0.001)
        assert mw.EnergyMap(grid, {(3, 4): 1.0, (1, 2): 1.0, (5, 0): 0.5}).argmax_cell() == (1, 2)

    def test_dense_holds_blocks(self):
        grid = mw.ImagingGrid((0, 0), (0.006, 0.006), 0.001)
        dense = mw.EnergyMap(grid, {(0, 0): 2.0, (3, 3): 5.0, (1, 1): 9.0}, stride=3).dense()
        assert dense[2, 2] == 2.0 and dense[4, 5] == 5.0 and dense[1, 1] == 9.0

    def test_dense_backed_equals_dict_backed(self):
        grid = mw.ImagingGrid((0, 0), (0.011, 0.009), 0.001)
        rng = np.random.default_rng(0)
        vals = rng.normal(size=grid.dims).astype(np.float32)
        valid = rng.uniform(size=grid.dims) < 0.6
        valid[::3, ::3] = True
        a = mw.EnergyMap._from_dense(grid, vals, valid, stride=3, split=3)
        b = mw.EnergyMap(grid, dict(a.entries), stride=3)
        keys = list(a.entries)
        lat = [k for k in keys if k[0] % 3 == 0 and k[1] % 3 == 0]
        assert keys[: len(lat)] == lat  # coarse entries first, as in the composite
        assert a == b and len(a) == len(b) == int(valid.sum())
        assert a.argmax_cell() == b.argmax_cell()
        np.testing.assert_array_equal(a.dense(), b.dense())
        r = mw.Region((2, 1), (8, 7))
        assert sorted(a.values_in(r)) == sorted(b.values_in(r))


class TestTraceDecoding:
    def test_decode_round_trip(self):
        tr = nat.Trace()
        tr.termination = 3
        tr.n_records = 1
        tr.final_region[:] = [1, 2, 0, 30, 40, 0]
        r = tr.records[0]
        r.iteration = 1
        r.n_children = 4
        r.counts[:4] = [5, 0, 7, 9]
        r.selected = 3
        r.satisfied = 1
        r.has_stats[:4] = [1, 0, 1, 1]
        r.scores[:4] = [1.5, -math.inf, 2.0, 4.0]
        r.mu[:4] = [1.0, 0.0, 2.0, 3.0]
        r.var[:4] = [1.5, 0.0, 2.0, 4.0]
        r.selected_region[:] = [10, 10, 0, 20, 20, 0]
        r.expanded_region[:] = [8, 8, 0, 22, 22, 0]
        r.w, r.b = 3.25, 1.5
        final, trace, code = decode_trace(bytes(tr))
        assert code == 3 and trace.termination == "n-min" and final == mw.Region((1, 2), (30, 40))
        rec = trace.records[0]
        assert rec.stats[1] is None and rec.stats[0] == {"mu": 1.0, "var": 1.5}
        assert rec.scores[1] == -math.inf and rec.selected_region == mw.Region((10, 10), (20, 20))
        assert len(rec.scores) == 4 and rec.quadrant_counts == [5, 0, 7, 9]
        json.dumps(trace.to_dict())

    def test_decode_errors(self):
        tr = nat.Trace()
        tr.termination = -1
        with pytest.raises(ValueError, match="no entries"):
            decode_trace(bytes(tr))
        tr.termination = -2
        with pytest.raises(RuntimeError):
            decode_trace(bytes(tr))


class TestSynth:
    def test_deterministic_and_pairs_only(self):
        m = synth.ScanModel(n_samples=256)
        a, ta = synth.dataset_2d(m, 4)
        b, tb = synth.dataset_2d(m, 4)
        assert np.array_equal(a.signals, b.signals) and ta == tb
        il = np.tril_indices(12)
        assert not a.signals[il].any()
        assert m.pairs().shape == (66, 2) and m.k0 == 8
        assert math.hypot(*ta) < 0.05

    def test_pulse_peak_and_snr(self):
        u = np.linspace(-5, 5, 100001) * 60e-12
        assert np.abs(synth.diff_gaussian(u, 60e-12)).max() == pytest.approx(1.0, rel=1e-6)
        m = synth.ScanModel()
        sig, _ = synth.scan_2d(m, 1, snr_db=20.0)
        clean = synth.clean_pairs(m, m.geometry().antennas, [(synth.scan_2d(m, 1)[1], 1.0)], m.pairs())
        sigma = (sig - clean).std()
        assert sigma == pytest.approx(np.abs(clean).max() / 10.0, rel=0.02)

    def test_hemisphere(self):
        a = synth.hemisphere_antennas(32, 0.08)
        assert a.shape == (32, 3) and (a[:, 2] >= 0).all()
        np.testing.assert_allclose(np.linalg.norm(a, axis=1), 0.08)
        assert synth.VolumeModel().pairs().shape == (496, 2)

    def test_compaction(self):
        from paper_1709_02549_b200._device import compact_channels

        sig = np.zeros((3, 3, 5))
        sig[0, 2, 1] = 1.0
        sig[2, 1, 4] = -2.0
        comp, pairs = compact_channels(sig)
        assert pairs.tolist() == [[0, 2], [2, 1]]
        assert comp.dtype == np.float32 and comp[1, 4] == -2.0
        comp0, pairs0 = compact_channels(np.zeros((2, 2, 4)))
        assert pairs0.tolist() == [[0, 0]] and not comp0.any()


def test_kind_parsing():
    assert mw.BeamformerKind.parse("DAS") is mw.BeamformerKind.DAS
    assert mw.BeamformerKind.parse(" dmas ") is mw.BeamformerKind.DMAS
    with pytest.raises(ValueError):
        mw.BeamformerKind.parse("mvdr")


def test_near_tie_excuse_is_tied_to_the_first_divergence():
    """_mwb_helpers.divergence_excused: a differing selection is excused only
    by a near-tie AT the iteration where the traces first differ."""
    from _mwb_helpers import divergence_excused

    def rec(sel, scores, w=1.0, b=1.0, sat=True):
        return {"selected": sel, "scores": scores, "W": w, "B": b, "satisfied": sat}

    clear = [1.0, 0.5, 0.2, 0.1]
    tied = [1.0, 1.0 - 1e-6, 0.2, 0.1]
    want = [rec(0, clear), rec(1, tied), rec(2, clear, w=0.5, b=2.0)]
    # identical traces
    assert divergence_excused(want, "n-min", want, "n-min")[:2] == (True, False)
    # diverges at the tied iteration -> excused
    got = [want[0], rec(0, tied)]
    assert divergence_excused(got, "n-min", want, "n-min")[:2] == (False, True)
    # a tie elsewhere does not excuse a divergence at a clear iteration
    got = [want[0], want[1], rec(1, clear, w=0.5, b=2.0)]
    assert divergence_excused(got, "n-min", want, "n-min")[:2] == (False, False)
    # W/B clause: same child, verdict flipped, B within 1e-4 of B_prev and W not improving
    w2 = [rec(0, clear, w=1.0, b=1.0), rec(1, clear, w=1.5, b=1.0 + 1e-6, sat=True)]
    g2 = [w2[0], rec(1, clear, w=1.5, b=1.0 - 1e-6, sat=False)]
    assert divergence_excused(g2, "distance-metrics", w2, "n-min")[:2] == (False, True)
    # verdict flipped with clear margins -> not excused
    w3 = [rec(0, clear, w=1.0, b=1.0), rec(1, clear, w=1.5, b=2.0, sat=True)]
    g3 = [w3[0], rec(1, clear, w=1.5, b=2.0, sat=False)]
    assert divergence_excused(g3, "distance-metrics", w3, "n-min")[:2] == (False, False)
    # same records, different termination -> never excused
    assert divergence_excused(want, "n-min", want, "region-floor")[:2] == (False, False)
