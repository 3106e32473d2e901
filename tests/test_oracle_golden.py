"""Pin the CPU oracle to the real reference (CPU-only, no GPU needed).

The golden vectors under tests/golden/ were produced by running
/root/reference/pkg/src/mwbeam itself (tests/golden/make_golden.py).  The
oracle restates the same numpy algorithm, so full-record values must match
bit for bit; windowed values (suffix-difference adapter, truncation point
chosen from the evaluated points) match to fp64 rounding.
"""

import numpy as np
import pytest

from _mwb_helpers import GOLDEN, load_json, sha
from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import synth


@pytest.fixture(scope="module")
def cfg0():
    z = np.load(GOLDEN / "scan_cfg0.npz")
    model = synth.ScanModel()
    ds, tumour = synth.dataset_2d(model, seed=0)
    assert sha(ds.signals) == str(z["sig_sha"])
    return z, ds, model


def test_generator_reproduces_golden_input(cfg0):
    z, ds, _ = cfg0
    assert tuple(z["tumour"]) == pytest.approx(tuple(synth.scan_2d(synth.ScanModel(), 0)[1]))


@pytest.mark.parametrize("kind", ["das", "dmas"])
def test_oracle_full_record_bit_exact(cfg0, kind):
    z, ds, _ = cfg0
    g = ds.geometry
    origin, res = (-0.05, -0.05), 1e-3
    cells = [(ix, iy) for ix in range(0, 100, 9) for iy in range(3, 100, 11)]
    pts = np.array([(origin[0] + (ix + 0.5) * res, origin[1] + (iy + 0.5) * res) for ix, iy in cells])
    got = orc.multistatic_energies(g.antennas, g.propagation_speed, g.sample_interval, ds.signals, pts, kind)
    want = np.array([z[f"cfg0_{kind}_full"][c] for c in cells])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("kind", ["das", "dmas"])
def test_oracle_window_adapter(cfg0, kind):
    z, ds, model = cfg0
    g = ds.geometry
    origin, res = (-0.05, -0.05), 1e-3
    cells = [(ix, iy) for ix in range(1, 100, 13) for iy in range(0, 100, 7)]
    pts = np.array([(origin[0] + (ix + 0.5) * res, origin[1] + (iy + 0.5) * res) for ix, iy in cells])
    got = orc.windowed_energies(g.antennas, g.propagation_speed, g.sample_interval, ds.signals, pts, kind,
                                model.k0, model.window)
    want = np.array([z[f"cfg0_{kind}_win"][c] for c in cells])
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    direct = orc.windowed_energies_direct(g.antennas, g.propagation_speed, g.sample_interval, ds.signals,
                                          pts[:6], kind, model.k0, model.window)
    assert np.abs(direct - want[:6]).max() <= 1e-12 * np.abs(want).max()


def test_oracle_points_small():
    for case in load_json("points_small.json")[:8]:
        ants = orc.ring_antennas(case["m"], 1.0)
        sig = np.array(case["signals"])
        pts = np.array(case["points"])
        for kind in ("das", "dmas"):
            got = orc.multistatic_energies(ants, 1.0, 1.0, sig, pts, kind, case["interp"])
            np.testing.assert_allclose(got, case[kind], rtol=1e-12, atol=1e-12)


def test_oracle_select_roi_maps():
    for case in load_json("select_roi_maps.json"):
        entries = {tuple(c): v for c, v in zip(case["cells"], case["values"])}
        n = case["n"]
        final, trace = orc.select_roi(entries, ((0, 0), (n - 1, n - 1)), case["frame_fraction"], case["n_min"])
        assert [list(final[0]), list(final[1])] == [case["final"]["min_cell"], case["final"]["max_cell"]]
        assert trace["termination"] == case["trace"]["termination"]
        assert [r["selected"] for r in trace["records"]] == [r["selected"] for r in case["trace"]["records"]]
        for a, b in zip(trace["records"], case["trace"]["records"]):
            assert a["W"] == b["W"] and a["B"] == b["B"] and a["scores"] == b["scores"]


def test_oracle_framework_presets():
    cases = load_json("framework_presets.json")
    seen = 0
    for case in cases:
        if case["resolution"] != 0.002:
            continue
        radius, tumour = {"dataset1": (0.10, (-0.02, -0.03)), "dataset2": (0.05, (0.02, 0.0))}[case["preset"]]
        ants = orc.ring_antennas(12, radius)
        sig = orc.simulate(ants, orc.SPEED_OF_LIGHT, 1e-11, 256, [(tumour, 1.0)], case["noise_std"], case["seed"])
        assert sha(sig) == case["sig_sha"]
        origin, extent, res = orc.grid_for_antennas(ants, case["resolution"])
        dims = orc.grid_dims(extent, res)
        mode = case["mode"]
        d = (orc.auto_decimation_factor(float(mode.split(":")[1]), res) if mode.startswith("auto")
             else int(mode.split(":")[1]))
        comp, rep = orc.run_framework(ants, orc.SPEED_OF_LIGHT, 1e-11, sig, case["kind"], origin, res, dims, d)
        want = case["report"]
        assert [list(rep["final_region"][0]), list(rep["final_region"][1])] == [
            want["final_region"]["min_cell"], want["final_region"]["max_cell"]]
        assert list(rep["argmax_cell"]) == want["argmax_cell"]
        assert rep["coarse_points_evaluated"] == want["coarse_points_evaluated"]
        assert rep["fine_points_evaluated"] == want["fine_points_evaluated"]
        assert rep["trace"]["termination"] == want["trace"]["termination"]
        golden_vals = dict(zip(map(tuple, case["cells"]), case["values"]))
        assert comp == golden_vals
        seen += 1
    assert seen >= 4


def test_oracle_volume_z_shift():
    spec = load_json("volume_cfg4.json")
    vm = synth.VolumeModel()
    sig, tum = synth.scan_3d(vm, seed=spec["seed"])
    z = np.load(GOLDEN / "volume_cfg4.npz")
    assert sha(sig) == str(z["sig_sha"])
    full = synth.embed_pairs(vm.n_ant, vm.pairs(), sig)
    ants = vm.geometry().antennas
    sl = spec["slices"][0]
    shifted = ants - np.array([0.0, 0.0, sl["z"]])
    xy = np.array(sl["xy"])[:6]
    got = orc.windowed_energies(shifted, vm.v, vm.dt, full, xy, "dmas", spec["k0"], spec["window"])
    want = np.array(sl["dmas"])[:6]
    assert np.abs(got - want).max() <= 1e-12 * np.abs(np.array(sl["dmas"])).max()


def test_oracle_monostatic():
    for case in load_json("monostatic.json"):
        ants = orc.ring_antennas(case["m"], 1.0)
        got = orc.monostatic_energies(ants, 1.0, case["dt"], np.array(case["signals"]), np.array(case["points"]))
        np.testing.assert_allclose(got, case["das"], rtol=1e-12, atol=1e-12)
