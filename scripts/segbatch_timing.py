"""SegmentBatch (BASELINE configs[2] rule, 4096 scans): device-phase times and
single-call segment() latency breakdown.  Development aid."""
import sys
import statistics
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import time

import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.segment import SegmentBatch, segment

m2 = synth.ScanModel(n_samples=2048)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
sig2, _ = synth.batch_2d_device(m2, range(4096), phantom_radius=(0.04, 0.05))
for kind, tree in (("das", True), ("dmas", True), ("das", False)):
    sb = SegmentBatch(m2.geometry(), m2.pairs(), m2.n_samples, g2, kind, 16, 0.01, window=(m2.k0, 32), tree=tree)
    res = sb.run(sig2)
    torch.cuda.synchronize()
    walls, el = [], []
    for _ in range(5):
        t0 = time.perf_counter()
        res = sb.run(sig2)
        walls.append((time.perf_counter() - t0) * 1e3)
        el.append(res.elapsed)
    print(kind, "tree" if tree else "per-iteration", "wall ms", statistics.median(walls),
          {k: statistics.median(e[k] * 1e3 for e in el) for k in el[0]}, "iters", res.iterations[:8].tolist(),
          "fine pts mean", float(res.fine_points_evaluated.mean()))
ds2, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
for kind in ("das", "dmas"):
    segment(ds2, kind, g2, 16, 0.01, window=(m2.k0, 32))
    torch.cuda.synchronize()
    walls, el = [], []
    for _ in range(7):
        t0 = time.perf_counter()
        _, rep = segment(ds2, kind, g2, 16, 0.01, window=(m2.k0, 32))
        walls.append((time.perf_counter() - t0) * 1e3)
        el.append(rep.elapsed)
    print("single", kind, "wall ms", statistics.median(walls),
          {k: statistics.median(e[k] * 1e3 for e in el) for k in el[0]})
