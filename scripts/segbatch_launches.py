"""One SegmentBatch run (4096 scans, DAS) for an ncu launch list.  Development aid."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.segment import SegmentBatch

m2 = synth.ScanModel(n_samples=2048)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
sig2, _ = synth.batch_2d_device(m2, range(4096), phantom_radius=(0.04, 0.05))
sb = SegmentBatch(m2.geometry(), m2.pairs(), m2.n_samples, g2, "das", 16, 0.01, window=(m2.k0, 32))
torch.cuda.nvtx.range_push("segbatch")
res = sb.run(sig2)
torch.cuda.synchronize()
print("ok", res.elapsed)
