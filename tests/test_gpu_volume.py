"""3-D voxel imaging and octant segmentation (BASELINE configs[4]).

Energies are pinned to the reference through the exact z-shift adapter
(golden vectors from the real reference in tests/golden/volume_cfg4.json and
the oracle's volume_energies); the octant control flow is checked against
the oracle's restatement (no reference counterpart exists)."""

import numpy as np
import pytest

import paper_1709_02549_b200 as mw
from _mwb_helpers import load_json, peak_err
from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.volume import Box, VolumeGrid, hemisphere_mask, image_volume, run_framework_volume

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vol():
    vm = synth.VolumeModel()
    spec = load_json("volume_cfg4.json")
    sig, tum = synth.scan_3d(vm, seed=spec["seed"])
    ds = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
    return vm, spec, ds, tum


def test_golden_voxels(vol):
    vm, spec, ds, _ = vol
    for sl in spec["slices"]:
        xy = np.array(sl["xy"])
        pts = np.concatenate([xy, np.full((len(xy), 1), sl["z"])], axis=1)
        got = mw.energies(ds, pts, "dmas", window=(spec["k0"], spec["window"]))
        assert peak_err(got, sl["dmas"]) <= 1e-4, sl["z"]


def test_image_volume_vs_oracle_and_point_path(vol):
    vm, _, ds, tum = vol
    g = ds.geometry
    grid = VolumeGrid((-0.012, -0.012, 0.0), (0.024, 0.024, 0.012), 0.002)
    both = image_volume(ds, ("das", "dmas"), grid, window=(vm.k0, vm.window))
    cells = [(ix, iy, iz) for ix in range(0, 12, 3) for iy in range(1, 12, 4) for iz in range(0, 6, 2)]
    pts = np.array([grid.cell_center(*c) for c in cells])
    for kind in ("das", "dmas"):
        want = orc.volume_energies(g.antennas, g.propagation_speed, g.sample_interval, ds.signals, pts, kind,
                                   vm.k0, vm.window)
        got = np.array([both[kind].values[c] for c in cells])
        assert peak_err(got, want) <= 1e-4
        # the point-list path gives the same fp32 bits
        pt = mw.energies(ds, pts, kind, window=(vm.k0, vm.window))
        assert np.array_equal(pt.astype(np.float32), got.astype(np.float32))
    assert len(both["das"]) == np.prod(grid.dims)


def test_strided_masked_volume():
    vm = synth.VolumeModel(n_samples=512)
    sig, _ = synth.scan_3d(vm, seed=2)
    ds = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
    grid = VolumeGrid((-0.03, -0.03, 0.0), (0.06, 0.06, 0.03), 0.003)
    mask = hemisphere_mask(grid, 0.03)
    m = image_volume(ds, "das", grid, stride=2, mask=mask, window=(vm.k0, vm.window))["das"]
    want = {(ix, iy, iz) for ix in range(0, 20, 2) for iy in range(0, 20, 2) for iz in range(0, 10, 2)
            if mask[ix, iy, iz]}
    assert set(m.entries) == want


def test_octant_framework_vs_oracle():
    vm = synth.VolumeModel(n_samples=1024)
    g = vm.geometry()
    rng = np.random.default_rng(11)
    for seed in range(3):
        tumour = np.array([rng.uniform(-0.015, 0.015), rng.uniform(-0.015, 0.015), rng.uniform(0.004, 0.02)])
        clean = synth.clean_pairs(vm, g.antennas, [(tumour, 1.0)], vm.pairs())
        sig = synth.add_noise(clean, 25.0, np.random.default_rng(seed))
        ds = mw.BackscatterDataset(g, synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
        grid = VolumeGrid((-0.024, -0.024, 0.0), (0.048, 0.048, 0.024), 0.002)
        comp, rep = run_framework_volume(ds, "dmas", grid, mw.Manual(3), phantom_radius=0.024,
                                         window=(vm.k0, vm.window))
        oc, orep = orc.run_framework_3d(g.antennas, vm.v, vm.dt, ds.signals, "dmas", grid.origin, grid.resolution,
                                        grid.dims, 3, 0.024, window=(vm.k0, vm.window))
        assert rep.final_region.bounds() == (*orep["final_region"][0], *orep["final_region"][1])
        assert [r.selected for r in rep.trace.records] == [r["selected"] for r in orep["trace"]["records"]]
        assert rep.trace.termination == orep["trace"]["termination"]
        assert rep.argmax_cell == orep["argmax_cell"]
        assert rep.coarse_points_evaluated == orep["coarse"] and rep.fine_points_evaluated == orep["fine"]
        assert rep.final_region.contains_cell(*grid.point_to_cell(*tumour)) or rep.trace.termination == "degenerate"


def test_box_octants_partition():
    b = Box((1, 2, 3), (6, 4, 9))
    kids = b.octants()
    assert sum(k.n_cells for k in kids) == b.n_cells
    assert [(k.min_cell, k.max_cell) for k in kids] == orc.octants((b.min_cell, b.max_cell))
    assert Box((0, 0, 0), (3, 3, 0)).octants() is None


def test_volume_cache_hit_is_identical(vol):
    """image_volume caches the voxel enumeration and delay table per geometry:
    a hit (same or a different dataset of the same scanner) equals a fresh run."""
    from paper_1709_02549_b200 import volume as vmod

    vm, _, ds, _ = vol
    sig2, _ = synth.scan_3d(vm, seed=77)
    ds2 = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig2))
    grid = VolumeGrid((-0.02, -0.02, 0.0), (0.04, 0.04, 0.02), 0.001)
    mask = hemisphere_mask(grid, 0.018)
    win = (vm.k0, vm.window)
    vmod._VOLUME_CACHE.clear()
    fresh = [image_volume(d, ("das", "dmas"), grid, mask=mask, window=win) for d in (ds, ds2)]
    vmod._VOLUME_CACHE.clear()
    image_volume(ds, "dmas", grid, mask=mask, window=win)  # populates the cache
    before = mw.EVAL_COUNTER.value
    hits = [image_volume(d, ("das", "dmas"), grid, mask=mask, window=win) for d in (ds, ds2)]
    assert mw.EVAL_COUNTER.value - before == 2 * 2 * int(mask.sum())
    for f, h in zip(fresh, hits):
        for k in ("das", "dmas"):
            assert np.array_equal(f[k].valid, h[k].valid)
            assert np.array_equal(f[k].values[f[k].valid], h[k].values[h[k].valid])


def test_octant_framework_replay_and_dataset_switch():
    """run_framework_volume replays one graph per scanner geometry: a second
    call on a dataset equals the first, after another dataset ran in between."""
    vm = synth.VolumeModel(n_samples=1024)
    g = vm.geometry()
    grid = VolumeGrid((-0.024, -0.024, 0.0), (0.048, 0.048, 0.024), 0.002)
    dss = []
    for seed in (21, 22):
        sig, _ = synth.scan_3d(vm, seed=seed)
        dss.append(mw.BackscatterDataset(g, synth.embed_pairs(vm.n_ant, vm.pairs(), sig)))
    win = (vm.k0, vm.window)
    first = [run_framework_volume(ds, "das", grid, mw.Manual(3), phantom_radius=0.024, window=win) for ds in dss]
    again = [run_framework_volume(ds, "das", grid, mw.Manual(3), phantom_radius=0.024, window=win)
             for ds in (dss[1], dss[0])]
    for (c0, r0), (c1, r1) in zip(first, again[::-1]):
        assert np.array_equal(c0.valid, c1.valid)
        assert np.array_equal(c0.values[c0.valid], c1.values[c1.valid])
        assert r0.final_region == r1.final_region and r0.argmax_cell == r1.argmax_cell


def test_octant_framework_argument_errors():
    vm = synth.VolumeModel(n_samples=256)
    sig, _ = synth.scan_3d(vm, seed=3)
    ds = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
    grid = VolumeGrid((-0.012, -0.012, 0.0), (0.024, 0.024, 0.012), 0.002)
    with pytest.raises(ValueError):  # mask of the wrong shape
        run_framework_volume(ds, "das", grid, mw.Manual(3), mask=np.ones((3, 3, 3), dtype=bool))
    with pytest.raises(ValueError):  # no coarse point inside the mask
        run_framework_volume(ds, "das", grid, mw.Manual(3), mask=np.zeros(grid.dims, dtype=bool))
    with pytest.raises(ValueError):
        run_framework_volume(ds, "das", grid, mw.Manual(3), interpolation="cubic")


def test_octant_framework_sees_in_place_mask_edits():
    """A writable mask edited in place between calls must not replay the plan
    of its old contents (volume._mask_key hashes writable masks every call)."""
    vm = synth.VolumeModel(n_samples=1024)
    g = vm.geometry()
    sig, _ = synth.scan_3d(vm, seed=31)
    ds = mw.BackscatterDataset(g, synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
    grid = VolumeGrid((-0.024, -0.024, 0.0), (0.048, 0.048, 0.024), 0.002)
    mask = np.array(hemisphere_mask(grid, 0.024))  # writable copy
    win = (vm.k0, vm.window)
    _, rep_a = run_framework_volume(ds, "dmas", grid, mw.Manual(3), mask=mask, window=win)
    mask[:, :, 6:] = False  # in place: the upper half of the volume leaves the phantom
    _, rep_b = run_framework_volume(ds, "dmas", grid, mw.Manual(3), mask=mask, window=win)
    fresh = np.array(mask)
    _, rep_c = run_framework_volume(ds, "dmas", grid, mw.Manual(3), mask=fresh, window=win)
    assert rep_b.full_equivalent_points == int(mask.sum()) != rep_a.full_equivalent_points
    assert rep_b.to_dict() | {"elapsed": None} == rep_c.to_dict() | {"elapsed": None}


def test_degenerate_octant_run_uses_the_overflow_copy():
    """An all-zero volume is degenerate: the final box is the whole grid and
    the composite comes back through the overflow path of the result block."""
    vm = synth.VolumeModel(n_samples=1024)
    g = vm.geometry()
    zero = mw.BackscatterDataset(g, np.zeros((vm.n_ant, vm.n_ant, vm.n_samples)))
    grid = VolumeGrid((-0.048, -0.048, 0.0), (0.096, 0.096, 0.048), 0.0015)  # 64 x 64 x 32 > the box budget
    mask = hemisphere_mask(grid, 0.048)
    comp, rep = run_framework_volume(zero, "dmas", grid, mw.Manual(4), mask=mask, window=(vm.k0, vm.window))
    assert rep.trace.termination == "degenerate"
    assert rep.final_region.bounds() == (0, 0, 0, *(n - 1 for n in grid.dims))
    assert comp.valid.sum() == int(mask.sum()) == rep.coarse_points_evaluated + rep.fine_points_evaluated
    assert not comp.values[comp.valid].any()
