"""A few configs[2] run_framework calls (DAS) for an ncu capture of the
framework's kernels (coarse K1, K2s select, region-filtered K1, gather).  Development aid."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth

m2 = synth.ScanModel(n_samples=2048)
ds2, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
for _ in range(3):
    mw.run_framework(ds2, "das", g2, mw.Manual(g2.dims[0] // 32), window=(m2.k0, 32))
torch.cuda.synchronize()
print("ok")
