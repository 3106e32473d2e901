"""Parity report: the GPU path against every golden fixture produced by the
real reference (tests/golden) and against the oracle on the BASELINE configs.
Prints a markdown table (committed as profiles/<round>_parity.md)."""

import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

import numpy as np

import paper_1709_02549_b200 as mw
from _mwb_helpers import GOLDEN, grid_for_geometry, load_json, preset, sha
from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.segment import segment
from paper_1709_02549_b200.volume import VolumeGrid, run_framework_volume

rows = []


def peak(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def masked(got, want, frac=1e-2):
    got, want = np.asarray(got, float), np.asarray(want, float)
    keep = np.abs(want) >= frac * np.abs(want).max()
    return float((np.abs(got - want)[keep] / np.abs(want)[keep]).max())


def add(case, source, n, err, err2, same):
    rows.append((case, source, n, err, err2, same))


# configs[0] / [1] maps vs the reference's own image() output
z = np.load(GOLDEN / "scan_cfg0.npz")
model = synth.ScanModel()
ds, _ = synth.dataset_2d(model, seed=0)
assert sha(ds.signals) == str(z["sig_sha"])
g0 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
g1 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 5e-4)
for kind in ("das", "dmas"):
    for tag, win in (("full record", None), ("W=32", (model.k0, 32))):
        em = mw.image(ds, kind, g0, window=win)
        want = z[f"cfg0_{kind}_full" if win is None else f"cfg0_{kind}_win"]
        got = em.dense(fill=np.nan)
        am = np.unravel_index(np.nanargmax(want), want.shape)
        add(f"configs[0] {kind.upper()} 100x100 {tag}", "reference image()", want.size, peak(got, want),
            masked(got, want), em.argmax_cell() == tuple(int(v) for v in am))
em = mw.image(ds, "dmas", g1, window=(model.k0, 32))
want = z["cfg1_dmas_win"]
got = em.dense(fill=np.nan)
add("configs[1] DMAS 200x200 W=32", "reference (suffix adapter)", want.size, peak(got, want), masked(got, want),
    em.argmax_cell() == tuple(int(v) for v in np.unravel_index(np.argmax(want), want.shape)))

# point values (linear + nearest) on random small datasets
errs = []
for case in load_json("points_small.json"):
    geom = mw.ring_array(case["m"], 1.0, propagation_speed=1.0, sample_interval=1.0)
    dsx = mw.BackscatterDataset(geom, np.array(case["signals"]))
    for kind in ("das", "dmas"):
        got = mw.energies(dsx, np.array(case["points"]), kind, case["interp"])
        errs.append(np.abs(got - case[kind]).max() / max(np.abs(case[kind]).max(), 1.0))
add("das/dmas_energy, 24 random datasets (linear+nearest)", "reference das/dmas_energy", 240, max(errs), None, True)

errs = []
for case in load_json("monostatic.json"):
    geom = mw.ring_array(case["m"], 1.0, propagation_speed=1.0, sample_interval=case["dt"])
    dsx = mw.BackscatterDataset(geom, np.array(case["signals"]))
    got = [mw.das_energy_monostatic(dsx, r) for r in case["points"]]
    errs.append(peak(got, case["das"]))
add("das_energy_monostatic, 8 datasets", "reference", 48, max(errs), None, True)

# select_roi on random lattice maps
same = 0
cases = load_json("select_roi_maps.json")
for case in cases:
    n = case["n"]
    grid = mw.ImagingGrid((0, 0), (n * 1e-3, n * 1e-3), 1e-3)
    emap = mw.EnergyMap(grid, {tuple(c): v for c, v in zip(case["cells"], case["values"])}, case["stride"])
    final, trace = mw.select_roi(emap, grid.full_region(), mw.FrameworkConfig(case["frame_fraction"], case["n_min"]))
    same += (final.to_dict() == case["final"] and trace.termination == case["trace"]["termination"]
             and [r.selected for r in trace.records] == [r["selected"] for r in case["trace"]["records"]])
add("select_roi, 16 random lattice maps", "reference select_roi", len(cases), None, None, f"{same}/{len(cases)}")

# framework runs
for name, fname in (("preset datasets (reference simulator)", "framework_presets.json"),
                    ("configs[2] runs (N=2048, 0.25 mm, Manual(nx//32))", "framework_cfg2.json")):
    same, errs, tot = 0, [], 0
    m2 = synth.ScanModel(n_samples=2048)
    for case in load_json(fname):
        if "preset" in case:
            _, dsx = preset(case["preset"], case["noise_std"], case["seed"])
            grid = grid_for_geometry(dsx.geometry, case["resolution"])
            mode = case["mode"]
            md = mw.Automatic(float(mode.split(":")[1])) if mode.startswith("auto") else mw.Manual(int(mode.split(":")[1]))
        else:
            dsx, _ = synth.dataset_2d(m2, seed=case["seed"], phantom_radius=case["radius"])
            r = case["radius"]
            grid = mw.ImagingGrid((-r, -r), (2 * r, 2 * r), 2.5e-4)
            md = mw.Manual(case["d"])
        comp, rep = mw.run_framework(dsx, case["kind"], grid, md)
        want = case["report"]
        ok = (rep.final_region.to_dict() == want["final_region"] and list(rep.argmax_cell) == want["argmax_cell"]
              and rep.trace.termination == want["trace"]["termination"]
              and [x.selected for x in rep.trace.records] == [x["selected"] for x in want["trace"]["records"]]
              and rep.coarse_points_evaluated == want["coarse_points_evaluated"]
              and rep.fine_points_evaluated == want["fine_points_evaluated"])
        same += ok
        tot += 1
        golden = dict(zip(map(tuple, case["cells"]), case["values"]))
        errs.append(peak([comp.entries[k] for k in golden], list(golden.values())))
    add(f"run_framework, {name}", "reference run_framework", tot, max(errs), None, f"{same}/{tot}")

# BASELINE segmentation variant and 3-D octants vs the oracle
same, tot = 0, 0
for seed in range(4):
    rng = np.random.default_rng(700 + seed)
    radius = float(rng.uniform(0.04, 0.06))
    dsx, _ = synth.dataset_2d(m2, seed=700 + seed, phantom_radius=radius)
    grid = mw.ImagingGrid((-radius, -radius), (2 * radius, 2 * radius), 2.5e-4)
    for kind in ("das", "dmas"):
        fine, rep = segment(dsx, kind, grid, 16, 0.01, window=(m2.k0, 32))
        g = dsx.geometry
        want = orc.segment_baseline(g.antennas, g.propagation_speed, g.sample_interval, dsx.signals, kind, grid.origin,
                                    grid.resolution, grid.dims, 16, rep.stop_cells, window=(m2.k0, 32),
                                    mask=mw.breast_mask(grid))
        same += ([r.selected for r in rep.records] == [r["selected"] for r in want["records"]]
                 and rep.argmax_cell == want["argmax_cell"])
        tot += 1
add("BASELINE segmentation (16x16 max/mean, 1 cm, 0.25 mm)", "oracle (reference energies)", tot, None, None,
    f"{same}/{tot}")

vm = synth.VolumeModel(n_samples=1024)
g = vm.geometry()
same, tot = 0, 0
rng = np.random.default_rng(11)
for seed in range(3):
    tumour = np.array([rng.uniform(-0.015, 0.015), rng.uniform(-0.015, 0.015), rng.uniform(0.004, 0.02)])
    clean = synth.clean_pairs(vm, g.antennas, [(tumour, 1.0)], vm.pairs())
    sig = synth.add_noise(clean, 25.0, np.random.default_rng(seed))
    dsx = mw.BackscatterDataset(g, synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
    vg = VolumeGrid((-0.024, -0.024, 0.0), (0.048, 0.048, 0.024), 0.002)
    comp, rep = run_framework_volume(dsx, "dmas", vg, mw.Manual(3), phantom_radius=0.024, window=(vm.k0, vm.window))
    oc, orep = orc.run_framework_3d(g.antennas, vm.v, vm.dt, dsx.signals, "dmas", vg.origin, vg.resolution, vg.dims,
                                    3, 0.024, window=(vm.k0, vm.window))
    same += (rep.final_region.bounds() == (*orep["final_region"][0], *orep["final_region"][1])
             and rep.argmax_cell == orep["argmax_cell"])
    tot += 1
add("3-D octant framework (configs[4] geometry, 24x24x12)", "oracle (z-shift reference energies)", tot, None, None,
    f"{same}/{tot}")

# tensor-core batch path (K1-TC) vs the oracle and the fp32 CUDA-core kernel
import torch  # noqa: E402

from paper_1709_02549_b200.batch import BatchImager  # noqa: E402

for win_w in (32, 48):
    sig_b, _ = synth.batch_2d(model, list(range(16)))
    grid_b = synth.grid_square(0.06, 128)
    win_b = (model.k0, win_w)
    tcb = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid_b, window=win_b, mode="tc")
    ref = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid_b, window=win_b)
    sd = tcb.to_device_layout(sig_b)
    outs = {}
    for name, bi in (("tc", tcb), ("fp32", ref)):
        o = {k: torch.empty((16, 128 * 128), dtype=torch.float32, device="cuda") for k in ("das", "dmas")}
        kd = {k: torch.zeros(16, dtype=torch.int64, device="cuda") for k in ("das", "dmas")}
        bi.run_device(sd, o["das"], o["dmas"], kd["das"], kd["dmas"])
        outs[name] = ({k: v.cpu().numpy() for k, v in o.items()},
                      {k: bi.decode_keys(v.cpu().numpy().view(np.uint64)) for k, v in kd.items()})
    g = model.geometry()
    cells = [(ix, iy) for ix in range(0, 128, 11) for iy in range(5, 128, 13)]
    pts = np.array([grid_b.cell_center(*c) for c in cells])
    slots = np.array([ix * 128 + iy for ix, iy in cells])
    for kind in ("das", "dmas"):
        e_ref, e_fp32, same = [], [], 0
        for s_ in range(16):
            full = synth.embed_pairs(12, model.pairs(), sig_b[s_].astype(np.float64))
            want = orc.windowed_energies(g.antennas, g.propagation_speed, g.sample_interval, full, pts, kind,
                                         model.k0, win_w)
            e_ref.append(peak(outs["tc"][0][kind][s_][slots], want))
            e_fp32.append(peak(outs["tc"][0][kind][s_], outs["fp32"][0][kind][s_]))
            same += tuple(outs["tc"][1][kind][s_]) == tuple(outs["fp32"][1][kind][s_])
        add(f"K1-TC batch {kind.upper()} W={win_w} (16 scans, 128x128 at 0.47 mm)", "oracle (max over scans)", 16,
            max(e_ref), None, f"argmax vs fp32 K1: {same}/16")
        add(f"K1-TC batch {kind.upper()} W={win_w}: vs the fp32 CUDA-core kernel", "K1 (mode smem)", 16, max(e_fp32),
            None, "—")

# BASELINE segmentation at batch scale: SegmentBatch (region-tree plan) vs the
# oracle's composed rule and vs per-scan segment()
from paper_1709_02549_b200.segment import SegmentBatch, segment  # noqa: E402

m2 = synth.ScanModel(n_samples=2048)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
seeds2 = list(range(2000, 2008))
sig2, _ = synth.batch_2d(m2, seeds2, phantom_radius=(0.04, 0.05))
for kind in ("das", "dmas"):
    res = SegmentBatch(m2.geometry(), m2.pairs(), m2.n_samples, g2, kind, 16, 0.01, window=(m2.k0, 32)).run(
        torch.from_numpy(sig2).cuda())
    errs, same_o, same_s = [], 0, 0
    for s_ in range(len(seeds2)):
        ds_ = mw.BackscatterDataset(m2.geometry(), synth.embed_pairs(12, m2.pairs(), sig2[s_].astype(np.float64)))
        fine, rep = segment(ds_, kind, g2, 16, 0.01, window=(m2.k0, 32))
        same_s += (res.fine(s_).entries == fine.entries and res.final_region(s_) == rep.final_region
                   and tuple(res.argmax_cells[s_]) == rep.argmax_cell)
        g = m2.geometry()
        want = orc.segment_baseline(g.antennas, g.propagation_speed, g.sample_interval, ds_.signals, kind,
                                    g2.origin, g2.resolution, g2.dims, 16, 40, window=(m2.k0, 32),
                                    mask=mw.breast_mask(g2))
        ok = ([r["selected"] for r in want["records"]] == [r.selected for r in res.records(s_)]
              and tuple(res.argmax_cells[s_]) == tuple(want["argmax_cell"]))
        same_o += ok
        if ok:
            cells = list(want["fine"])
            got_f = res.fine(s_).entries
            errs.append(peak([got_f[c] for c in cells], [want["fine"][c] for c in cells]))
    add(f"SegmentBatch {kind.upper()} (8 configs[2] scans, region-tree plan)", "oracle (reference energies)", 8,
        max(errs) if errs else None, None, f"{same_o}/8; bit-identical to per-scan segment(): {same_s}/8")

# BASELINE configs[3] at full size (4096 scans x 256^2, tensor-core path): oracle spot checks
mdl = synth.ScanModel()
sig3, _ = synth.batch_2d_device(mdl, range(4096))
g3 = synth.grid_square(0.12, 256)
bi3 = BatchImager(mdl.geometry(), mdl.pairs(), mdl.n_samples, g3, window=(mdl.k0, mdl.window), mode="auto")
o3 = {k: torch.empty((4096, 256 * 256), dtype=torch.float32, device="cuda") for k in ("das", "dmas")}
bi3.run_device(sig3, o3["das"], o3["dmas"])
rng = np.random.default_rng(3)
cells3 = [(int(a), int(b)) for a, b in rng.integers(0, 256, size=(96, 2))]
pts3 = np.array([g3.cell_center(*c) for c in cells3])
slots3 = np.array([ix * 256 + iy for ix, iy in cells3])
picks = (0, 1777, 4095)
rows3 = sig3[list(picks)].cpu().numpy()
for kind in ("das", "dmas"):
    e3 = []
    for s_, row in zip(picks, rows3):
        full = synth.embed_pairs(12, mdl.pairs(), row[:, : mdl.n_samples].astype(np.float64))
        g = mdl.geometry()
        want = orc.windowed_energies(g.antennas, g.propagation_speed, g.sample_interval, full, pts3, kind,
                                     mdl.k0, mdl.window)
        got = o3[kind][s_].cpu().numpy()
        e3.append(float(np.abs(got[slots3] - want).max() / np.abs(got).max()))
    add(f"configs[3] full size {kind.upper()}: 4096 scans x 256^2, tensor cores", "oracle (96 px of scans 0, 1777, 4095)",
        288, max(e3), None, "—")
del sig3, o3

print("# Parity report (GPU vs reference / oracle)\n")
print("Energy error = max |gpu - ref| / max |ref| (BASELINE bound 1e-4); masked = max per-pixel relative error on "
      "pixels >= 1 % of peak.  'Same' = identical argmax / regions / selection sequence / termination / counts.\n")
print("| case | compared with | n | energy error | masked rel. error | same decisions |")
print("|---|---|---|---|---|---|")
for case, src, n, e, e2, same in rows:
    fe = f"{e:.2e}" if e is not None else "—"
    fe2 = f"{e2:.2e}" if e2 is not None else "—"
    print(f"| {case} | {src} | {n} | {fe} | {fe2} | {same} |")
