"""configs[4] octant framework: per-phase device time and wall.  Development aid."""
import sys
import statistics
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.volume import VolumeGrid, hemisphere_mask, image_volume, run_framework_volume

vm = synth.VolumeModel()
sig, _ = synth.scan_3d(vm, seed=9)
ds4 = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
g4 = VolumeGrid((-0.06, -0.06, 0.0), (0.12, 0.12, 0.12), 0.12 / 128)
mask = hemisphere_mask(g4, vm.phantom_radius)
win = (vm.k0, vm.window)
for _ in range(2):
    comp, rep = run_framework_volume(ds4, "dmas", g4, mw.Automatic(0.01), mask=mask, window=win)
torch.cuda.synchronize()
walls, els = [], []
for _ in range(5):
    t0 = time.perf_counter()
    comp, rep = run_framework_volume(ds4, "dmas", g4, mw.Automatic(0.01), mask=mask, window=win)
    walls.append((time.perf_counter() - t0) * 1e3)
    els.append(rep.elapsed)
print("octant wall ms", statistics.median(walls), {k: round(statistics.median(e[k] * 1e3 for e in els), 3)
                                                    for k in els[0]},
      "d", rep.decimation_factor, "coarse", rep.coarse_points_evaluated, "fine", rep.fine_points_evaluated,
      "iters", rep.iterations)
image_volume(ds4, "dmas", g4, window=win)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    image_volume(ds4, "dmas", g4, window=win)
    ts.append((time.perf_counter() - t0) * 1e3)
print("volume repeat wall ms", statistics.median(ts))
import cProfile
import pstats

pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    run_framework_volume(ds4, "dmas", g4, mw.Automatic(0.01), mask=mask, window=win)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
