"""One FrameworkBatch run of 4096 configs[2]-shaped scans (for ncu launch lists; development aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.fwbatch import FrameworkBatch

model = synth.ScanModel(n_samples=2048)
grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
sig, _ = synth.batch_2d_device(model, range(4096), phantom_radius=(0.04, 0.05))
fb = FrameworkBatch(model.geometry(), model.pairs(), model.n_samples, grid, mw.Manual(grid.dims[0] // 32), "das",
                    window=(model.k0, 32))
for _ in range(2):
    res = fb.run(sig)
torch.cuda.synchronize()
print("ok", res.elapsed)
