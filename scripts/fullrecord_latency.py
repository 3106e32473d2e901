"""Reference-semantics (full-record window) latency of the drop-in calls on a
configs[2] scan (2048 samples).  Development aid."""
import sys
import statistics
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.segment import segment

m2 = synth.ScanModel(n_samples=2048)
ds, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
d = g2.dims[0] // 32


def wall(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


print("run_framework full record ms", wall(lambda: mw.run_framework(ds, "das", g2, mw.Manual(d))))
print("segment full record ms", wall(lambda: segment(ds, "das", g2, 16, 0.01)))
print("segment tree=False full record ms", wall(lambda: segment(ds, "das", g2, 16, 0.01, tree=False)))
print("image masked full record ms", wall(lambda: mw.image(ds, "das", g2, mask=mw.breast_mask(g2))))
