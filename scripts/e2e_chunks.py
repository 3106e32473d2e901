"""configs[3] end-to-end step time against the chunk size (BatchImager.__call__).  Development aid."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager

m = synth.ScanModel()
S = 4096
sig_d, _ = synth.batch_2d_device(m, range(S))
grid = synth.grid_square(0.12, 256)
bi = BatchImager(m.geometry(), m.pairs(), m.n_samples, grid, window=(m.k0, m.window), mode="auto")
host = sig_d[:, :, : m.n_samples].cpu().pin_memory()
out = {k: torch.empty((S, 65536), dtype=torch.float32, pin_memory=True) for k in ("das", "dmas")}
for chunk in (64, 96, 128, 192, 256, 384):
    bi(host, chunk=chunk, out=out)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bi(host, chunk=chunk, out=out)
        ts.append(time.perf_counter() - t0)
    print(chunk, f"{statistics.median(ts) * 1e3:.2f} ms", flush=True)
