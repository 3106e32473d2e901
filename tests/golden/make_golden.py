"""Generate golden vectors by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

Every value stored here is computed by `mwbeam` itself (image, das_energy,
dmas_energy, run_framework, select_roi).  Inputs come from the repo's seeded
generator (paper_1709_02549_b200.synth) or from the reference simulator; each
fixture stores a sha256 of its input signals so a test can prove it rebuilt
the same input.  The fixtures are small .npz/.json files that travel to the
GPU box; the reference does not.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import mwbeam as R  # noqa: E402
from mwbeam import presets as RP  # noqa: E402

from paper_1709_02549_b200 import synth  # noqa: E402

THREADS = len(os.sched_getaffinity(0))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def ref_ds(geom_like, signals):
    g = R.ArrayGeometry(np.asarray(geom_like.antennas), geom_like.propagation_speed, geom_like.sample_interval)
    return R.BackscatterDataset(g, np.asarray(signals, dtype=np.float64))


def windowed(rds, pts, kind, k0, w):
    """Reference-only windowed energy: suffix difference of two reference calls
    on truncated records (see oracle.windowed_energies)."""
    sig = rds.signals
    n = sig.shape[2]
    ants = rds.geometry.antennas
    d = np.sqrt((pts[:, None, 0] - ants[None, :, 0]) ** 2 + (pts[:, None, 1] - ants[None, :, 1]) ** 2
                + ants[None, :, 2] ** 2)
    b = min(n, k0 + w + int(np.ceil(2 * d.max() / (rds.geometry.propagation_speed * rds.geometry.sample_interval))) + 4)
    head = R.BackscatterDataset(rds.geometry, np.ascontiguousarray(sig[..., k0:b]))
    kind_e = R.BeamformerKind(kind)
    e1 = np.concatenate([R.beamform._multistatic_energies(head, pts[i:i + 64], kind_e)
                         for i in range(0, len(pts), 64)])
    if k0 + w >= b:
        return e1
    tail = R.BackscatterDataset(rds.geometry, np.ascontiguousarray(sig[..., k0 + w:b]))
    e2 = np.concatenate([R.beamform._multistatic_energies(tail, pts[i:i + 64], kind_e) for i in range(0, len(pts), 64)])
    return e1 - e2


def dense_of(emap, dims):
    out = np.full(dims, np.nan)
    for (ix, iy), v in emap.entries.items():
        out[ix, iy] = v
    return out


def trace_json(trace):
    return trace.to_dict()


def main():
    t_start = time.time()
    meta = {"generated_by": "tests/golden/make_golden.py", "reference": "mwbeam 0.1.0 (/root/reference/pkg/src)",
            "numpy": np.__version__}

    # ---- cfg0 / cfg1 style scans (66 pairs, N=1024, v=c/3, dt=20ps) --------
    model = synth.ScanModel()
    ds, tumour = synth.dataset_2d(model, seed=0)
    rds = ref_ds(ds.geometry, ds.signals)
    grid0 = R.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
    maps = {}
    for kind in ("das", "dmas"):
        t = time.time()
        em = R.image(rds, R.BeamformerKind(kind), grid0, threads=THREADS)
        maps[f"cfg0_{kind}_full"] = dense_of(em, grid0.dims)
        maps[f"cfg0_{kind}_full_argmax"] = np.array(em.argmax_cell())
        print(f"cfg0 {kind} full: {time.time() - t:.1f}s")
        pts = np.array([grid0.cell_center(i, j) for i in range(100) for j in range(100)])
        t = time.time()
        e = windowed(rds, pts, kind, model.k0, model.window)
        maps[f"cfg0_{kind}_win"] = e.reshape(100, 100)
        print(f"cfg0 {kind} windowed: {time.time() - t:.1f}s")
    grid1 = R.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 5e-4)
    pts1 = np.array([grid1.cell_center(i, j) for i in range(200) for j in range(200)])
    t = time.time()
    maps["cfg1_dmas_win"] = windowed(rds, pts1, "dmas", model.k0, model.window).reshape(200, 200)
    print(f"cfg1 dmas windowed: {time.time() - t:.1f}s")
    np.savez_compressed(HERE / "scan_cfg0.npz", **maps, sig_sha=np.array(sha(ds.signals)),
                        tumour=np.array(tumour), k0=model.k0, window=model.window)

    # ---- point energies on small random datasets (test_beamform.py style) ---
    rng = np.random.default_rng(123)
    pts_cases = []
    for trial in range(12):
        m = int(rng.integers(2, 6))
        n = int(rng.integers(8, 80))
        geom = R.ring_array(m, 1.0, propagation_speed=1.0, sample_interval=1.0)
        sig = rng.normal(size=(m, m, n))
        rds_s = R.BackscatterDataset(geom, sig)
        rs = rng.uniform(-0.9, 0.9, (5, 2))
        for interp in ("linear", "nearest"):
            das = [R.das_energy(rds_s, r, interp) for r in rs]
            dmas = [R.dmas_energy(rds_s, r, interp) for r in rs]
            pts_cases.append({"m": m, "n": n, "signals": sig.tolist(), "points": rs.tolist(), "interp": interp,
                              "das": das, "dmas": dmas})
    (HERE / "points_small.json").write_text(json.dumps(pts_cases))

    # ---- monostatic DAS (beamform.py:215-261) on diagonal-only datasets -------
    mono = []
    for trial in range(8):
        m = int(rng.integers(2, 7))
        n = int(rng.integers(16, 120))
        geom = R.ring_array(m, 1.0, propagation_speed=1.0, sample_interval=float(rng.choice([0.05, 0.1])))
        sig = np.zeros((m, m, n))
        for i in range(m):
            sig[i, i] = rng.normal(size=n)
        rds_m = R.BackscatterDataset(geom, sig)
        rs = rng.uniform(-0.9, 0.9, (6, 2))
        mono.append({"m": m, "n": n, "dt": geom.sample_interval, "signals": sig.tolist(), "points": rs.tolist(),
                     "das": [R.das_energy_monostatic(rds_m, r) for r in rs]})
    (HERE / "monostatic.json").write_text(json.dumps(mono))

    # ---- reference-simulator framework runs (test_coarse2fine.py style) -----
    fw = []
    for name, res, modes in (("dataset2", 0.002, ("auto:0.01", "manual:3", "manual:1")),
                             ("dataset1", 0.004, ("auto:0.01", "manual:2"))):
        pds = RP.preset_dataset(name, noise_std=0.02, seed=5)
        grid = RP.grid_for_geometry(pds.geometry, res)
        for kind in ("das", "dmas"):
            for mode in modes:
                md = R.Automatic(float(mode.split(":")[1])) if mode.startswith("auto") else R.Manual(int(mode.split(":")[1]))
                comp, rep = R.run_framework(pds, R.BeamformerKind(kind), grid, md, threads=THREADS)
                cells = np.array(list(comp.entries.keys()), dtype=np.int64).reshape(-1, 2)
                fw.append({
                    "preset": name, "noise_std": 0.02, "seed": 5, "resolution": res, "kind": kind, "mode": mode,
                    "sig_sha": sha(pds.signals),
                    "report": {k: v for k, v in rep.to_dict().items() if k != "elapsed"},
                    "cells": cells.tolist(),
                    "values": list(comp.entries.values()),
                })
                print(f"framework {name} {kind} {mode}: {rep.trace.termination} {rep.final_region}")
    (HERE / "framework_presets.json").write_text(json.dumps(fw))

    # ---- cfg2 style: R ~ U(4,6) cm, N=2048, 0.25 mm, Manual(nx//32) ----------
    cfg2 = []
    m2 = synth.ScanModel(n_samples=2048)
    for seed in range(4):
        rng2 = np.random.default_rng(1000 + seed)
        radius = float(rng2.uniform(0.04, 0.06))
        ds2, tum2 = synth.dataset_2d(m2, seed=1000 + seed, phantom_radius=radius)
        rds2 = ref_ds(ds2.geometry, ds2.signals)
        grid2 = R.ImagingGrid((-radius, -radius), (2 * radius, 2 * radius), 2.5e-4)
        d = grid2.dims[0] // 32
        for kind in ("das", "dmas"):
            t = time.time()
            comp, rep = R.run_framework(rds2, R.BeamformerKind(kind), grid2, R.Manual(d), threads=THREADS)
            cells = np.array(list(comp.entries.keys()), dtype=np.int64).reshape(-1, 2)
            cfg2.append({"seed": 1000 + seed, "radius": radius, "kind": kind, "d": d, "sig_sha": sha(ds2.signals),
                         "tumour": list(tum2),
                         "report": {k: v for k, v in rep.to_dict().items() if k != "elapsed"},
                         "cells": cells.tolist(), "values": list(comp.entries.values())})
            print(f"cfg2 seed {seed} {kind}: dims {grid2.dims} D={d} {rep.trace.termination} {rep.final_region} "
                  f"{time.time() - t:.1f}s")
    (HERE / "framework_cfg2.json").write_text(json.dumps(cfg2))

    # ---- select_roi on hand-built lattice maps (test_coarse2fine.py:98-127) --
    sel = []
    rng3 = np.random.default_rng(77)
    for case in range(16):
        n = int(rng3.integers(8, 80))
        stride = int(rng3.integers(1, 5))
        grid = R.ImagingGrid((0, 0), (n * 1e-3, n * 1e-3), 1e-3)
        entries = {}
        for ix in range(0, n, stride):
            for iy in range(0, n, stride):
                entries[(ix, iy)] = float(rng3.exponential())
        hot = (int(rng3.integers(0, n)) // stride * stride, int(rng3.integers(0, n)) // stride * stride)
        entries[hot] = 20.0
        emap = R.EnergyMap(grid, entries, stride)
        ff = float(rng3.choice([0.0, 0.1, 0.25, 0.5]))
        nmin = int(rng3.integers(1, 8))
        final, trace = R.select_roi(emap, grid.full_region(), R.FrameworkConfig(frame_fraction=ff, n_min=nmin))
        sel.append({"n": n, "stride": stride, "cells": [list(k) for k in entries], "values": list(entries.values()),
                    "frame_fraction": ff, "n_min": nmin, "final": final.to_dict(), "trace": trace_json(trace)})
    (HERE / "select_roi_maps.json").write_text(json.dumps(sel))

    # ---- 3-D voxels via the exact z-shift adapter (SURVEY.md §8c adapter 3) --
    vm = synth.VolumeModel()
    sig3, tum3 = synth.scan_3d(vm, seed=9)
    geom3 = vm.geometry()
    full3 = synth.embed_pairs(vm.n_ant, vm.pairs(), sig3)
    vox = []
    rng4 = np.random.default_rng(4)
    zs = sorted(set([float(t[2]) for t in tum3] + [0.0, 0.02]))
    for z in zs:
        g_shift = R.ArrayGeometry(geom3.antennas - np.array([0.0, 0.0, z]), geom3.propagation_speed, geom3.sample_interval)
        rds3 = R.BackscatterDataset(g_shift, full3)
        xy = rng4.uniform(-0.05, 0.05, (24, 2))
        near = [t[:2] for t in tum3 if abs(t[2] - z) < 1e-12]
        if near:
            xy = np.concatenate([xy, np.array(near)])
        e = windowed(rds3, xy, "dmas", vm.k0, vm.window)
        vox.append({"z": z, "xy": xy.tolist(), "dmas": e.tolist()})
        print(f"3-D slice z={z:.4f}: {len(xy)} voxels")
    np.savez_compressed(HERE / "volume_cfg4.npz", sig_sha=np.array(sha(sig3)), tumours=tum3)
    (HERE / "volume_cfg4.json").write_text(json.dumps({"seed": 9, "k0": vm.k0, "window": vm.window, "slices": vox}))

    # ---- wire formats (io.py): a small .mwb container and one export ---------
    from mwbeam import io as RIO

    rng5 = np.random.default_rng(55)
    g5 = R.ring_array(4, 0.05, propagation_speed=1.2e8, sample_interval=2e-11)
    ds5 = R.BackscatterDataset(g5, rng5.normal(size=(4, 4, 48)), t0=1.5e-10)
    RIO.save_dataset(ds5, HERE / "small.mwb")
    grid5 = R.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 0.01)
    comp5, _ = R.run_framework(ds5, R.BeamformerKind.DAS, grid5, R.Manual(3))
    RIO.export_energy_map(comp5, HERE / "export_small")

    meta["seconds"] = time.time() - t_start
    (HERE / "META.json").write_text(json.dumps(meta, indent=2))
    print(f"done in {meta['seconds']:.0f}s")


if __name__ == "__main__":
    main()
