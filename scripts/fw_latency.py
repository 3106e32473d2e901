import sys, time, statistics
sys.path.insert(0, '/root/repo')
import torch
import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
m2 = synth.ScanModel(n_samples=2048)
ds2, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
d = g2.dims[0] // 32
for kind in ("das", "dmas"):
    ts = []
    for i in range(30):
        t0 = time.perf_counter(); c, r = mw.run_framework(ds2, kind, g2, mw.Manual(d), window=(m2.k0, 32)); ts.append(time.perf_counter() - t0)
    print(kind, "first", ts[0]*1e3, "median", statistics.median(ts[5:])*1e3, "ms", r.elapsed, r.final_region, r.argmax_cell)
