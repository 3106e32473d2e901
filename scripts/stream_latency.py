"""Per-call wall latency of the drop-in API on (a) the same dataset repeatedly
and (b) a stream of distinct datasets of one geometry (each call uploads its
scan).  Development aid."""
import sys
import statistics
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.segment import segment


def wall(fn, reps):
    ts = []
    for r in range(reps):
        t0 = time.perf_counter()
        fn(r)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


m0 = synth.ScanModel()
win = (m0.k0, m0.window)
g1 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 5e-4)
dss = [synth.dataset_2d(m0, seed=s)[0] for s in range(40)]
mw.image(dss[0], "dmas", g1, window=win)
print("image cfg1 same  ms", wall(lambda r: mw.image(dss[0], "dmas", g1, window=win), 20))
print("image cfg1 stream ms", wall(lambda r: mw.image(dss[1 + r], "dmas", g1, window=win), 20))
m2 = synth.ScanModel(n_samples=2048)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
d = g2.dims[0] // 32
ds2 = [synth.dataset_2d(m2, seed=1000 + s, phantom_radius=0.05)[0] for s in range(40)]
w2 = (m2.k0, 32)
mw.run_framework(ds2[0], "das", g2, mw.Manual(d), window=w2)
print("run_framework same  ms", wall(lambda r: mw.run_framework(ds2[0], "das", g2, mw.Manual(d), window=w2), 20))
print("run_framework stream ms", wall(lambda r: mw.run_framework(ds2[1 + r], "das", g2, mw.Manual(d), window=w2), 19))
segment(ds2[0], "das", g2, 16, 0.01, window=w2)
print("segment same  ms", wall(lambda r: segment(ds2[0], "das", g2, 16, 0.01, window=w2), 20))
print("segment stream ms", wall(lambda r: segment(ds2[20 + r], "das", g2, 16, 0.01, window=w2), 19))
from paper_1709_02549_b200 import _device as dv

new = [synth.dataset_2d(m2, seed=3000 + s, phantom_radius=0.05)[0] for s in range(10)]
print("scan upload only (configs[2] dataset) ms", wall(lambda r: dv.scan_for(new[r]), 10))
