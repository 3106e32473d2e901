"""Tensor-core path vs the fp32 path: error statistics and configs[3] timing
(development aid).  Prints one JSON object."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager

model = synth.ScanModel()
grid = synth.grid_square(0.12, 256)
win = (model.k0, model.window)
n_scans = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
sig, _ = synth.batch_2d_device(model, list(range(n_scans)))
out = {}
res = {}
for mode in ("smem", "tc"):
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, mode=mode)
    n = grid.dims[0] * grid.dims[1]
    das = torch.empty((n_scans, n), dtype=torch.float32, device="cuda")
    dmas = torch.empty_like(das)
    kd = torch.zeros(n_scans, dtype=torch.int64, device="cuda")
    km = torch.zeros_like(kd)
    bi.run_device(sig, das, dmas, kd, km)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    reps = 3
    for _ in range(reps):
        bi.run_device(sig, das, dmas, kd, km)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    res[mode] = {"ms": ms, "pps_per_s": n_scans * n * bi.n_chan * model.window / (ms / 1e3)}
    cells = [bi.decode_keys(k.cpu().numpy().view(np.uint64)) for k in (kd, km)]
    out[mode] = (das[:256].cpu().numpy(), dmas[:256].cpu().numpy(), *cells)
a, b = out["tc"], out["smem"]
for i, k in enumerate(("das", "dmas")):
    errs = np.abs(a[i] - b[i]).max(axis=1) / np.abs(b[i]).max(axis=1)
    rel = (a[i] - b[i]) / np.abs(b[i]).max(axis=1, keepdims=True)
    res[f"{k}_peak_err_max"] = float(errs.max())
    res[f"{k}_peak_err_median"] = float(np.median(errs))
    res[f"{k}_mean_signed_err"] = float(rel.mean())
    res[f"{k}_argmax_agree"] = float((a[2 + i] == b[2 + i]).all(axis=1).mean())
print(json.dumps(res, indent=1))
