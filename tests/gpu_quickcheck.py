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


if __name__ == "__main__":
    main()
