"""Quick GPU check: parity of image/das/framework vs the oracle, microbenchmarks,
and a first timing of the batched cfg3 kernel.  Development aid."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import ctypes

import numpy as np
import torch

import paper_1709_02549_b200 as mw
from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import _native as nat
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager


def pn(got, want):
    return float(np.abs(got - want).max() / np.abs(want).max())


def main():
    torch.cuda.init()
    print(torch.cuda.get_device_name(0))
    model = synth.ScanModel(n_samples=256)
    ds, tum = synth.dataset_2d(model, seed=3)
    g = ds.geometry
    grid = synth.grid_square(0.1, 40)
    for kind in ("das", "dmas"):
        for window in (None, (model.k0, 32)):
            for mode in ("smem", "gather"):
                t0 = time.perf_counter()
                em = mw.image(ds, kind, grid, window=window, mode=mode)
                t1 = time.perf_counter()
                ref = orc.image(g.antennas, g.propagation_speed, g.sample_interval, ds.signals, kind, grid.origin,
                                grid.resolution, grid.dims, window=window)
                cells = sorted(ref)
                got = np.array([em.entries[c] for c in cells])
                want = np.array([ref[c] for c in cells])
                print(f"{kind} window={window} mode={mode}: n={len(em)} err={pn(got, want):.2e} "
                      f"argmax {em.argmax_cell()} vs {orc.argmax_cell(ref)}  ({(t1 - t0) * 1e3:.1f} ms)")
        # point path == lattice path
        em = mw.image(ds, kind, grid, stride=3)
        cells = list(em.entries)[:20]
        f = mw.das_energy if kind == "das" else mw.dmas_energy
        ok = all(f(ds, grid.cell_center(*c)) == em.entries[c] for c in cells)
        print(kind, "point==lattice:", ok)
    # framework
    grid2 = synth.grid_square(0.1, 100)
    for kind in ("das", "dmas"):
        comp, rep = mw.run_framework(ds, kind, grid2, mw.Manual(4))
        oc, orep = orc.run_framework(g.antennas, g.propagation_speed, g.sample_interval, ds.signals, kind,
                                     grid2.origin, grid2.resolution, grid2.dims, 4)
        print(kind, "framework:", rep.final_region, orep["final_region"], rep.trace.termination,
              orep["trace"]["termination"], rep.argmax_cell, orep["argmax_cell"], rep.coarse_points_evaluated,
              orep["coarse_points_evaluated"], rep.fine_points_evaluated, orep["fine_points_evaluated"],
              rep.elapsed)
        cells = sorted(oc)
        print("  composite err", pn(np.array([comp.entries[c] for c in cells]), np.array([oc[c] for c in cells])),
              set(comp.entries) == set(oc))
    # microbenchmarks
    lib = nat.load()
    for which, name in ((0, "LDS.32 bytes"), (1, "FFMA2 flop"), (2, "FFMA flop")):
        work = ctypes.c_double()
        ms = ctypes.c_float()
        nat.check(lib.mwb_microbench(which, ctypes.byref(work), ctypes.byref(ms), None), "mb")
        print(f"microbench {name}: {work.value / ms.value / 1e9:.1f} G/ms -> {work.value / (ms.value * 1e-3) / 1e12:.2f} T/s")
    # batched cfg3-like timing
    m3 = synth.ScanModel()
    S = 512
    sig, tumours = synth.batch_2d(m3, range(S))
    grid3 = synth.grid_square(0.12, 256)
    bi = BatchImager(m3.geometry(), m3.pairs(), m3.n_samples, grid3, window=(m3.k0, 32))
    sig_d = bi.to_device_layout(sig)
    nxny = 256 * 256
    for kind in ("das", "dmas"):
        for mode in (0, 1):
            bi.mode = mode
            out = torch.empty((S, nxny), dtype=torch.float32, device="cuda")
            keys = torch.zeros(S, dtype=torch.int64, device="cuda")
            for _ in range(2):
                bi.run_device(sig_d, kind, out, keys)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 3
            for _ in range(reps):
                bi.run_device(sig_d, kind, out, keys)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            pps = S * bi.n_pts * bi.n_chan * 32 / (ms * 1e-3)
            print(f"batch {kind} mode={mode}: {ms:.2f} ms for {S} scans, {pps / 1e12:.2f} Tpps/s, "
                  f"{S * bi.n_pts * bi.n_chan / (ms * 1e-3) / 1e9:.1f} G pixel-pair/s")
        cells = bi.decode_keys(keys.cpu().numpy().view(np.uint64))
        hits = np.mean([np.abs(np.array(grid3.point_to_cell(*tumours[i])) - cells[i]).max() <= 2 for i in range(S)])
        print(f"  {kind} argmax within 2 cells of tumour: {hits:.3f}")
    # batch parity vs oracle for 2 scans
    bi.mode = 0
    for kind in ("das", "dmas"):
        out = torch.empty((S, nxny), dtype=torch.float32, device="cuda")
        bi.run_device(sig_d, kind, out)
        o = out.cpu().numpy()
        for s in (0, 7):
            ds_s = mw.BackscatterDataset(m3.geometry(), synth.embed_pairs(12, m3.pairs(), sig[s].astype(np.float64)))
            sub = synth.grid_square(0.12, 256)
            pts = np.array([sub.cell_center(i, j) for i in range(0, 256, 9) for j in range(0, 256, 11)])
            ref = orc.windowed_energies(ds_s.geometry.antennas, ds_s.geometry.propagation_speed,
                                        ds_s.geometry.sample_interval, ds_s.signals, pts, kind, m3.k0, 32)
            got = np.array([o[s, i * 256 + j] for i in range(0, 256, 9) for j in range(0, 256, 11)])
            print(f"  batch parity {kind} scan {s}: err {pn(got, ref):.2e}")


if __name__ == "__main__":
    main()
