"""configs[3] tensor-core step time (4096 scans, DAS + DMAS), median of 10.  Development aid."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager

m = synth.ScanModel()
S = 4096
sig, _ = synth.batch_2d_device(m, range(S))
bi = BatchImager(m.geometry(), m.pairs(), m.n_samples, synth.grid_square(0.12, 256), window=(m.k0, m.window),
                 mode="tc")
das, dmas = (torch.empty((S, 65536), device="cuda") for _ in range(2))
for _ in range(3):
    bi.run_device(sig, das, dmas)
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    bi.run_device(sig, das, dmas)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"tc step {statistics.median(ts):.2f} ms (min {min(ts):.2f})", flush=True)
