"""Reference acceptance criterion 2 (test_acceptance.py:86-111) on the GPU:
point-count and wall-clock reduction of the framework vs the full masked DMAS
image, for one call and for a batch.  Development aid."""
import sys
import statistics
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager
from paper_1709_02549_b200.fwbatch import FrameworkBatch
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from _mwb_helpers import grid_for_geometry, preset


def ev_ms(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


_, ds1 = preset("dataset1")
grid = grid_for_geometry(ds1.geometry, 0.001)
mask = mw.breast_mask(grid)
t_full = ev_ms(lambda: mw.image(ds1, "dmas", grid, mask=mask))
fw = []
for _ in range(5):
    _, rep = mw.run_framework(ds1, "dmas", grid, mw.Automatic(0.01))
    fw.append(rep.elapsed["total"] * 1e3)
t_fw_wall = ev_ms(lambda: mw.run_framework(ds1, "dmas", grid, mw.Automatic(0.01)))
print("single dataset1: full image", t_full, "ms; framework device", statistics.median(fw), "ms, wall", t_fw_wall,
      "ms; reduction ratio", rep.reduction_ratio, "grid", grid.dims)
m = synth.ScanModel(n_samples=1024)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
for s in (256, 1024):
    sig, _ = synth.batch_2d_device(m, range(s), phantom_radius=(0.04, 0.05))
    bi = BatchImager(m.geometry(), m.pairs(), m.n_samples, g2, window=(m.k0, 32), mask=mw.breast_mask(g2),
                    mode="auto")
    out = torch.empty((s, g2.dims[0] * g2.dims[1]), dtype=torch.float32, device="cuda")
    t_b = ev_ms(lambda: bi.run_device(sig, out_dmas=out), reps=3)
    fb = FrameworkBatch(m.geometry(), m.pairs(), m.n_samples, g2, mw.Automatic(0.01), "dmas", window=(m.k0, 32))
    t_f = ev_ms(lambda: fb.run(sig), reps=3)
    res = fb.run(sig)
    print(f"batch {s}: full masked DMAS {t_b:.2f} ms (tc={bi.uses_tensor_cores}), FrameworkBatch {t_f:.2f} ms, "
          f"wall ratio {t_b / t_f:.1f}, mean point ratio {float(res.reduction_ratios.mean()):.1f}")
    del sig, out
