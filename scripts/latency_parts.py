"""Host-side breakdown of run_framework / scan upload latency.  Development aid."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import _device as dv
from paper_1709_02549_b200 import coarse2fine as c2f
from paper_1709_02549_b200 import synth

m2 = synth.ScanModel(n_samples=2048)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
d = g2.dims[0] // 32
w2 = (m2.k0, 32)
dss = [synth.dataset_2d(m2, seed=1000 + s, phantom_radius=0.05)[0] for s in range(30)]
mw.run_framework(dss[0], "das", g2, mw.Manual(d), window=w2)
torch.cuda.synchronize()


def tm(label, fn, n=20):
    ts = []
    for i in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(i)
        ts.append((time.perf_counter() - t0) * 1e6)
    print(f"{label:40s} median {np.median(ts):8.1f} us")


tm("run_framework same", lambda i: mw.run_framework(dss[0], "das", g2, mw.Manual(d), window=w2))
plan, scan = c2f._plan_for(dss[0], "das", g2, d, c2f.FrameworkConfig(), "linear", w2, 0)
tm("_plan_for", lambda i: c2f._plan_for(dss[0], "das", g2, d, c2f.FrameworkConfig(), "linear", w2, 0))
tm("geometry_key", lambda i: scan.geometry_key())
tm("slot copy", lambda i: plan.scan.sig.copy_(scan.sig, non_blocking=True))
tm("launch", lambda i: plan.launch(scan))
tm("launch+sync", lambda i: (plan.launch(scan), torch.cuda.synchronize()))


def lf(i):
    plan.launch(scan)
    plan.finish()


tm("launch+finish", lf)
tm("breast mask + factor", lambda i: (c2f.decimation_factor(mw.Manual(d), g2.resolution), c2f._breast_mask_device(g2)))
sig = np.asarray(dss[5].signals)
m, _, n = sig.shape
flat = sig.reshape(m * m, n)
tm("nonzero check", lambda i: np.flatnonzero(np.any(flat != 0.0, axis=1)))
keep = np.flatnonzero(np.any(flat != 0.0, axis=1))
tm("upload_rows", lambda i: dv.upload_rows(flat, keep, dv.round4(n)))
tm("pinned empty", lambda i: torch.empty((66, 2048), dtype=torch.float32, pin_memory=True))
tm("build_scan", lambda i: dv._build_scan(dss[10 + i % 10]))
