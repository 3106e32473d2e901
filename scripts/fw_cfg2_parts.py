"""configs[2] single-scan latency: run_framework vs the full masked image,
host/device breakdown (CUDA events + perf_counter).  Development aid; also the
target of an ncu launch list (--profile)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import coarse2fine as c2f
from paper_1709_02549_b200 import synth

m2 = synth.ScanModel(n_samples=2048)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
d = g2.dims[0] // 32
w2 = (m2.k0, 32)
ds, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
mask = mw.breast_mask(g2)
profile = "--profile" in sys.argv


def dev_ms(fn, n=20):
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def wall_us(fn, n=20):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return float(np.median(ts))


for kind in ("das", "dmas"):
    fw = lambda: mw.run_framework(ds, kind, g2, mw.Manual(d), window=w2)
    im = lambda: mw.image(ds, kind, g2, mask=mask, window=w2)
    fw(), im()
    if profile:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        fw(), im()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        continue
    _, rep = fw()
    plan, scan = c2f._plan_for(ds, kind, g2, d, c2f.FrameworkConfig(), "linear", w2, 0)

    def launch_sync():
        plan.launch(scan)
        torch.cuda.synchronize()

    from paper_1709_02549_b200.segment import segment

    sg = lambda: segment(ds, kind, g2, 16, 0.01, window=w2)
    sg()
    print(f"{kind}: segment wall {wall_us(sg):.1f} us (events {dev_ms(sg):.1f})", flush=True)
    print(f"{kind}: run_framework wall {wall_us(fw):.1f} us (events {dev_ms(fw):.1f}), "
          f"launch {wall_us(lambda: plan.launch(scan)):.1f}, launch+sync {wall_us(launch_sync):.1f}; "
          f"elapsed {', '.join(f'{k} {v * 1e6:.1f}' for k, v in rep.elapsed.items())} us; "
          f"coarse {rep.coarse_points_evaluated} fine {rep.fine_points_evaluated}; "
          f"image wall {wall_us(im):.1f} us (events {dev_ms(im):.1f})", flush=True)
