"""GPU parity of the imaging kernel (through libmwb.so) — mirrors the reference's
/root/reference/pkg/tests/test_beamform.py case by case, plus golden-vector
parity against the real reference on the BASELINE cfg0/cfg1 scans.

Tolerances: arithmetic is fp32 (delays fp64).  Hand-value tests whose inputs
are small integers stay exact.  Reference tests that assert rel 1e-12 on
fp64 values are re-stated at the fp32 tolerance and marked as such.  Energy
maps use the BASELINE bound: max |gpu - ref| / max |ref| <= 1e-4
(peak-normalised).
"""

import numpy as np
import pytest

import paper_1709_02549_b200 as mw
from _mwb_helpers import (
    GOLDEN,
    dataset,
    grid_for_geometry,
    load_json,
    masked_rel_err,
    peak_err,
    sha,
    sim_small,
    unit_geometry,
)
from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import synth

pytestmark = pytest.mark.gpu

TOL = 1e-4  # BASELINE: energy maps within 1e-4 (peak-normalised), fp32
FP32_REL = 2e-5  # stand-in for the reference's fp64 rel=1e-12 point checks


def as_dense(emap, dims):
    out = np.full(dims, np.nan)
    for (ix, iy), v in emap.entries.items():
        out[ix, iy] = v
    return out


class TestDasEnergy:  # test_beamform.py:87-106
    def test_zero_dataset(self):
        ds = dataset(unit_geometry([[1, 0, 0], [-1, 0, 0]]), np.zeros((2, 2, 16)))
        assert mw.das_energy(ds, (0.0, 0.0)) == 0.0

    def test_single_unit_impulse(self):
        sig = np.zeros((2, 2, 16))
        sig[0, 1, 4] = 1.0  # aligned by delay 2 -> lands at sample 2
        ds = dataset(unit_geometry([[1, 0, 0], [-1, 0, 0]]), sig)
        assert mw.das_energy(ds, (0.0, 0.0)) == 1.0

    def test_argmax_on_fine_grid_hits_tumor(self):
        tumour, ds = sim_small()
        grid = grid_for_geometry(ds.geometry, 0.002)
        got = mw.image(ds, mw.BeamformerKind.DAS, grid, mask=mw.breast_mask(grid)).argmax_cell()
        want = grid.point_to_cell(*tumour)
        assert max(abs(got[0] - want[0]), abs(got[1] - want[1])) <= 1


class TestDmasEnergy:  # test_beamform.py:160-187
    def test_single_channel_gives_zero(self):
        sig = np.zeros((2, 2, 16))
        sig[0, 1, 5] = 2.5
        ds = dataset(unit_geometry([[1, 0, 0], [-1, 0, 0]]), sig)
        assert mw.dmas_energy(ds, (0.3, -0.2)) == 0.0

    def test_two_aligned_values_multiply(self):
        sig = np.zeros((2, 2, 16))
        sig[0, 0, 6] = 3.0
        sig[0, 1, 6] = 4.0
        ds = dataset(unit_geometry([[1, 0, 0], [-1, 0, 0]]), sig)
        assert mw.dmas_energy(ds, (0.0, 0.0)) == 12.0

    def test_identity_matches_brute_force(self):
        """O(M^4) pairwise sum (test_beamform.py:147-157) at the fp32 tolerance."""
        rng = np.random.default_rng(123)
        for _ in range(10):
            geom = mw.ring_array(4, 1.0, propagation_speed=1.0, sample_interval=1.0)
            ds = dataset(geom, rng.normal(size=(4, 4, 64)))
            r = rng.uniform(-0.8, 0.8, 2)
            aligned = [mw.aligned_channel(ds, i, j, r) for i in range(4) for j in range(4)]
            slow = sum(float((aligned[k] * aligned[l]).sum()) for k in range(16) for l in range(k + 1, 16))
            scale = sum(float((a * a).sum()) for a in aligned)
            assert abs(mw.dmas_energy(ds, r) - slow) <= FP32_REL * scale

    def test_acceptance_criterion_4_at_fp32(self):
        """test_acceptance.py:143-161 (criterion 4) on its own 100 random
        datasets (seed 2024), with the fp32 bound relative to the channel
        self-energy sum instead of the fp64 rel 1e-9 on the (zero-crossing)
        DMAS value itself."""
        rng = np.random.default_rng(2024)
        worst = 0.0
        for _ in range(100):
            geom = mw.ring_array(4, 1.0, propagation_speed=1.0, sample_interval=1.0)
            ds = dataset(geom, rng.normal(size=(4, 4, 64)))
            r = rng.uniform(-0.8, 0.8, 2)
            aligned = [mw.aligned_channel(ds, i, j, r) for i in range(4) for j in range(4)]
            slow = sum(float((aligned[k] * aligned[l]).sum()) for k in range(16) for l in range(k + 1, 16))
            scale = sum(float((a * a).sum()) for a in aligned)
            worst = max(worst, abs(mw.dmas_energy(ds, r) - slow) / scale)
        assert worst <= FP32_REL, worst


class TestKernelProperties:  # test_beamform.py:190-239
    def make_random(self, seed, m=3, n=48):
        rng = np.random.default_rng(seed)
        geom = mw.ring_array(m, 1.0, propagation_speed=1.0, sample_interval=1.0)
        return dataset(geom, rng.normal(size=(m, m, n))), rng

    def test_scaling_by_two_is_exact(self):
        ds, _ = self.make_random(1)
        scaled = mw.BackscatterDataset(ds.geometry, 2.0 * ds.signals)
        r = (0.3, 0.1)
        assert mw.das_energy(scaled, r) == 4.0 * mw.das_energy(ds, r)
        assert mw.dmas_energy(scaled, r) == 4.0 * mw.dmas_energy(ds, r)

    def test_scaling_general_alpha(self):  # rel 1e-12 in fp64 -> fp32 tolerance
        ds, _ = self.make_random(2)
        scaled = mw.BackscatterDataset(ds.geometry, 1.7 * ds.signals)
        r = (-0.2, 0.4)
        assert mw.das_energy(scaled, r) == pytest.approx(1.7**2 * mw.das_energy(ds, r), rel=FP32_REL)
        assert mw.dmas_energy(scaled, r) == pytest.approx(1.7**2 * mw.dmas_energy(ds, r), rel=FP32_REL)

    def test_antenna_relabeling_invariance(self):
        ds, _ = self.make_random(3, m=4)
        perm = np.array([2, 0, 3, 1])
        ds2 = dataset(mw.ArrayGeometry(ds.geometry.antennas[perm], 1.0, 1.0), ds.signals[np.ix_(perm, perm)])
        for seed in range(5):
            r = np.random.default_rng(seed).uniform(-0.8, 0.8, 2)
            a, b = mw.das_energy(ds2, r), mw.das_energy(ds, r)
            assert a == pytest.approx(b, rel=FP32_REL)
            c, d = mw.dmas_energy(ds2, r), mw.dmas_energy(ds, r)
            assert abs(c - d) <= FP32_REL * max(abs(a), 1e-30)

    def test_das_never_negative(self):
        for seed in range(10):
            ds, rng = self.make_random(seed)
            pts = rng.uniform(-1.5, 1.5, (5, 2))
            assert (mw.energies(ds, pts, "das") >= 0.0).all()

    def test_das_dmas_argmax_agree_on_clean_data(self):
        _, ds = sim_small()
        grid = grid_for_geometry(ds.geometry, 0.0025)
        mask = mw.breast_mask(grid)
        a = mw.image(ds, mw.BeamformerKind.DAS, grid, mask=mask).argmax_cell()
        b = mw.image(ds, mw.BeamformerKind.DMAS, grid, mask=mask).argmax_cell()
        assert max(abs(a[0] - b[0]), abs(a[1] - b[1])) <= 1


class TestNearest:  # test_beamform.py:62-84
    def test_nearest_consistent_with_aligned_channels(self):
        geom = unit_geometry([[0.3, 0, 0], [-0.45, 0, 0]])
        rng = np.random.default_rng(8)
        ds = dataset(geom, rng.normal(size=(2, 2, 24)))
        r = (0.1, 0.05)
        manual = sum(mw.aligned_channel(ds, i, j, r, interpolation="nearest") for i in range(2) for j in range(2))
        assert mw.das_energy(ds, r, interpolation="nearest") == pytest.approx(float((manual**2).sum()), rel=FP32_REL)

    def test_bad_interpolation(self):
        ds = dataset(unit_geometry([[1, 0, 0], [-1, 0, 0]]), np.zeros((2, 2, 4)))
        with pytest.raises(ValueError):
            mw.das_energy(ds, (0, 0), interpolation="cubic")


class TestImageOperation:  # test_beamform.py:242-309
    def small_ds(self):
        geom = mw.ring_array(3, 0.05, propagation_speed=1.0, sample_interval=0.01)
        return dataset(geom, np.random.default_rng(0).normal(size=(3, 3, 32)))

    def grid(self, n=20, res=0.005):
        return mw.ImagingGrid((-n * res / 2, -n * res / 2), (n * res, n * res), res)

    def test_decimated_point_count(self):
        emap = mw.image(self.small_ds(), mw.BeamformerKind.DAS, self.grid(), stride=7)
        assert len(emap) == 9
        assert all(ix % 7 == 0 and iy % 7 == 0 for ix, iy in emap.entries)

    def test_shared_cells_identical_across_strides(self):
        ds, grid = self.small_ds(), self.grid()
        full = mw.image(ds, mw.BeamformerKind.DAS, grid, stride=1)
        dec = mw.image(ds, mw.BeamformerKind.DAS, grid, stride=7)
        for cell, val in dec.entries.items():
            assert full.entries[cell] == val

    def test_matches_per_point_kernel_exactly(self):
        ds, grid = self.small_ds(), self.grid()
        for kind, single in ((mw.BeamformerKind.DAS, mw.das_energy), (mw.BeamformerKind.DMAS, mw.dmas_energy)):
            emap = mw.image(ds, kind, grid, stride=3)
            for (ix, iy), val in list(emap.entries.items())[:12]:
                assert single(ds, grid.cell_center(ix, iy)) == val

    def test_counter_accounting(self):
        before = mw.EVAL_COUNTER.value
        emap = mw.image(self.small_ds(), mw.BeamformerKind.DAS, self.grid(), stride=2)
        assert mw.EVAL_COUNTER.value - before == len(emap)

    def test_thread_count_does_not_change_values(self):
        _, ds = sim_small(n_ant=5, n=128)
        grid = grid_for_geometry(ds.geometry, 0.004)
        mask = mw.breast_mask(grid)
        one = mw.image(ds, mw.BeamformerKind.DMAS, grid, mask=mask, threads=1)
        four = mw.image(ds, mw.BeamformerKind.DMAS, grid, mask=mask, threads=4)
        assert one.entries == four.entries

    def test_skip_cells(self):
        ds, grid = self.small_ds(), self.grid()
        full = mw.image(ds, mw.BeamformerKind.DAS, grid, stride=2)
        some = set(list(full.entries)[:5])
        rest = mw.image(ds, mw.BeamformerKind.DAS, grid, stride=2, skip=some)
        assert set(rest.entries) == set(full.entries) - some
        for cell, val in rest.entries.items():
            assert full.entries[cell] == val

    def test_bad_arguments(self):
        ds, grid = self.small_ds(), self.grid()
        with pytest.raises(ValueError):
            mw.image(ds, mw.BeamformerKind.DAS, grid, stride=0)
        with pytest.raises(ValueError):
            mw.image(ds, mw.BeamformerKind.DAS, grid, region=mw.Region((0, 0), (25, 25)))

    def test_region_subset_and_order(self):
        ds, grid = self.small_ds(), self.grid()
        reg = mw.Region((3, 5), (17, 11))
        em = mw.image(ds, "dmas", grid, region=reg, stride=3)
        ref = orc.region_cells(grid.dims, (reg.min_cell, reg.max_cell), 3)
        assert list(em.entries) == list(zip(ref[0].tolist(), ref[1].tolist()))


class TestEdgeCases:
    def test_empty_mask_gives_empty_map(self):
        _, ds = sim_small(n_ant=4)
        grid = grid_for_geometry(ds.geometry, 0.01)
        em = mw.image(ds, "das", grid, mask=np.zeros(grid.dims, dtype=bool))
        assert len(em) == 0 and em.entries == {}
        with pytest.raises(ValueError):
            em.argmax_cell()

    def test_all_zero_dataset(self):
        geom = mw.ring_array(5, 0.05)
        ds = dataset(geom, np.zeros((5, 5, 40)))
        grid = grid_for_geometry(geom, 0.01)
        for kind in ("das", "dmas"):
            em = mw.image(ds, kind, grid)
            assert set(em.entries.values()) == {0.0}
            assert em.argmax_cell() == (0, 0)  # all ties -> lowest (ix, iy)

    @pytest.mark.parametrize("n", [1, 3, 5, 7, 33])
    def test_ragged_record_lengths(self, n):
        rng = np.random.default_rng(n)
        geom = mw.ring_array(3, 1.0, propagation_speed=1.0, sample_interval=0.1)
        sig = rng.normal(size=(3, 3, n))
        ds = dataset(geom, sig)
        pts = rng.uniform(-1.2, 1.2, (40, 2))
        for kind in ("das", "dmas"):
            got = mw.energies(ds, pts, kind)
            want = orc.multistatic_energies(geom.antennas, 1.0, 0.1, sig, pts, kind)
            assert np.abs(got - want).max() <= 1e-5 * max(np.abs(want).max(), 1e-30) + 1e-6

    def test_points_beyond_the_record_are_zero(self):
        geom = mw.ring_array(4, 0.05)
        sig = np.random.default_rng(1).normal(size=(4, 4, 16))
        ds = dataset(geom, sig)
        far = np.array([[3.0, 3.0], [-5.0, 2.0]])  # delays >> N
        assert (mw.energies(ds, far, "das") == 0.0).all()
        assert (mw.energies(ds, far, "dmas") == 0.0).all()

    def test_wide_spread_tile_uses_channel_groups_or_gather(self):
        """Points spread over metres -> per-tile spans exceed the stage buffer."""
        rng = np.random.default_rng(5)
        geom = mw.ring_array(8, 0.5, propagation_speed=1.0, sample_interval=0.002)
        sig = rng.normal(size=(8, 8, 600))
        ds = dataset(geom, sig)
        pts = rng.uniform(-1.0, 1.0, (300, 2))
        for kind in ("das", "dmas"):
            a = mw.energies(ds, pts, kind)
            b = mw.energies(ds, pts, kind, mode="gather")
            assert np.array_equal(a, b)
            want = orc.multistatic_energies(geom.antennas, 1.0, 0.002, sig, pts, kind)
            assert peak_err(a, want) <= TOL

    def test_smem_and_gather_bit_identical(self):
        model = synth.ScanModel(n_samples=256)
        ds, _ = synth.dataset_2d(model, seed=11)
        grid = synth.grid_square(0.1, 50)
        for kind in ("das", "dmas"):
            for window in (None, (model.k0, 32), (3, 50)):
                a = mw.image(ds, kind, grid, window=window)
                b = mw.image(ds, kind, grid, window=window, mode="gather")
                assert a.entries == b.entries

    def test_window_beyond_record(self):
        model = synth.ScanModel(n_samples=128)
        ds, _ = synth.dataset_2d(model, seed=2)
        grid = synth.grid_square(0.1, 10)
        em = mw.image(ds, "das", grid, window=(500, 32))
        assert set(em.entries.values()) == {0.0}
        em0 = mw.image(ds, "das", grid, window=(0, 0))
        assert set(em0.entries.values()) == {0.0}


class TestEnergyMap:  # test_beamform.py:312-329 on GPU-produced maps
    def test_dense_backed_matches_dict_semantics(self):
        _, ds = sim_small(n_ant=5, n=128)
        grid = grid_for_geometry(ds.geometry, 0.004)
        em = mw.image(ds, "das", grid, stride=3, mask=mw.breast_mask(grid))
        plain = mw.EnergyMap(grid, dict(em.entries), 3)
        assert em.argmax_cell() == plain.argmax_cell()
        np.testing.assert_array_equal(em.dense(), plain.dense())
        reg = mw.Region((5, 5), (20, 30))
        np.testing.assert_array_equal(em.values_in(reg), plain.values_in(reg))


class TestGoldenBaselineScans:
    """cfg0 (100x100, DAS/DMAS) and cfg1 (200x200 DMAS) against reference output."""

    @pytest.fixture(scope="class")
    @classmethod
    def scan(cls):
        z = np.load(GOLDEN / "scan_cfg0.npz")
        model = synth.ScanModel()
        ds, tumour = synth.dataset_2d(model, seed=0)
        assert sha(ds.signals) == str(z["sig_sha"]), "synthetic scan differs from the golden input"
        return z, ds, model

    @pytest.mark.parametrize("kind", ["das", "dmas"])
    def test_cfg0_full_record(self, scan, kind):
        z, ds, _ = scan
        grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
        em = mw.image(ds, kind, grid)
        got = as_dense(em, grid.dims)
        want = z[f"cfg0_{kind}_full"]
        assert peak_err(got, want) <= TOL
        assert masked_rel_err(got, want) <= 1e-3
        assert tuple(em.argmax_cell()) == tuple(z[f"cfg0_{kind}_full_argmax"])

    @pytest.mark.parametrize("kind", ["das", "dmas"])
    def test_cfg0_window(self, scan, kind):
        z, ds, model = scan
        grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
        em = mw.image(ds, kind, grid, window=(model.k0, model.window))
        got = as_dense(em, grid.dims)
        want = z[f"cfg0_{kind}_win"]
        assert peak_err(got, want) <= TOL
        assert em.argmax_cell() == np.unravel_index(np.argmax(want), want.shape)

    def test_cfg1_dmas_window(self, scan):
        z, ds, model = scan
        grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 5e-4)
        em = mw.image(ds, "dmas", grid, window=(model.k0, model.window))
        got = as_dense(em, grid.dims)
        want = z["cfg1_dmas_win"]
        assert peak_err(got, want) <= TOL
        assert em.argmax_cell() == np.unravel_index(np.argmax(want), want.shape)


class TestGoldenPoints:
    def test_small_random_datasets(self):
        for case in load_json("points_small.json"):
            m = case["m"]
            geom = mw.ring_array(m, 1.0, propagation_speed=1.0, sample_interval=1.0)
            ds = dataset(geom, np.array(case["signals"]))
            pts = np.array(case["points"])
            for kind in ("das", "dmas"):
                got = mw.energies(ds, pts, kind, case["interp"])
                want = np.array(case[kind])
                scale = max(np.abs(want).max(), 1.0)
                assert np.abs(got - want).max() <= 1e-5 * scale, (case["m"], case["n"], kind)


def test_lattice_cache_hit_is_identical():
    """Repeated image() calls on one geometry/grid reuse the cached lattice and
    delay table: maps, counts and argmax are identical to the uncached call."""
    from paper_1709_02549_b200.beamform import _LATTICE_CACHE

    model = synth.ScanModel()
    ds1, _ = synth.dataset_2d(model, seed=11)
    ds2, _ = synth.dataset_2d(model, seed=12)
    grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
    mask = mw.breast_mask(grid)
    import paper_1709_02549_b200.beamform as bf

    _LATTICE_CACHE.clear()
    first = mw.images(ds1, ("das", "dmas"), grid, mask=mask, window=(model.k0, model.window))
    real = bf.lattice_pass

    def no_enumeration(*a, **k):  # a hit must not enumerate again
        raise AssertionError("cache miss")

    bf.lattice_pass = no_enumeration
    try:
        before = mw.EVAL_COUNTER.value
        again = mw.images(ds1, ("das", "dmas"), grid, mask=mask, window=(model.k0, model.window))  # cache hit
        assert mw.EVAL_COUNTER.value - before == 2 * int(mask.sum())
        other = mw.images(ds2, ("das", "dmas"), grid, mask=mask, window=(model.k0, model.window))  # hit, new scan
    finally:
        bf.lattice_pass = real
    _LATTICE_CACHE.clear()
    fresh = mw.images(ds2, ("das", "dmas"), grid, mask=mask, window=(model.k0, model.window))
    for k in ("das", "dmas"):
        assert np.array_equal(first[k].dense(fill=np.nan), again[k].dense(fill=np.nan), equal_nan=True)
        assert np.array_equal(other[k].dense(fill=np.nan), fresh[k].dense(fill=np.nan), equal_nan=True)
        assert other[k].argmax_cell() == fresh[k].argmax_cell()
        assert len(other[k]) == len(fresh[k]) == int(mask.sum())


def test_image_plan_replay_matches_first_pass_across_datasets():
    """image() replays a captured energy launch once a lattice is cached: maps of
    several datasets (same scanner; one with a different record length) equal
    the first, uncached evaluation of each."""
    from paper_1709_02549_b200 import beamform as bf
    from paper_1709_02549_b200 import synth

    grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
    dss = [synth.dataset_2d(synth.ScanModel(n_samples=n), seed=s)[0] for n, s in ((1024, 1), (1024, 2), (512, 3))]
    fresh = []
    for ds in dss:
        bf._LATTICE_CACHE.clear()
        fresh.append(mw.images(ds, ("das", "dmas"), grid))
    for _ in range(2):
        for ds, want in zip(dss, fresh):
            got = mw.images(ds, ("das", "dmas"), grid)
            for k in ("das", "dmas"):
                assert got[k].entries == want[k].entries
