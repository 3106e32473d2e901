"""Device latency of a small K1 launch (one scan, 1024 points = 4 tiles,
W = 32) against the channel count, measured on 20 launches captured in a CUDA
graph (no host overhead); MWB_KSPLIT=1 disables the k-split.  Development aid."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager

m = synth.ScanModel()
sig, _ = synth.batch_2d_device(m, [0])
grid = synth.grid_square(0.03, int(sys.argv[1]) if len(sys.argv) > 1 else 32)
n = grid.dims[0] * grid.dims[1]
for nc in (66, 33, 16, 8):
    pairs = m.pairs()[:nc]
    bi = BatchImager(m.geometry(), pairs, m.n_samples, grid, window=(m.k0, m.window), mode="smem")
    s = sig[:, :nc].contiguous()
    out = torch.empty((1, n), device="cuda")
    for kind in ("das", "dmas"):
        kw = {f"out_{kind}": out}
        bi.run_device(s, **kw)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                bi.run_device(s, **kw)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        print(f"points={n} C={nc} {kind}: {a.elapsed_time(b) / 100 * 1e3:.1f} us per launch", flush=True)
