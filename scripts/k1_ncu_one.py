"""One warm-up and one profiled CUDA-core K1 launch at configs[3] shape (256 scans):
  ncu --set full -k regex:energy_kernel --launch-skip 1 -c 1 python scripts/k1_ncu_one.py dmas
Development aid."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager

kind = sys.argv[1] if len(sys.argv) > 1 else "both"
m = synth.ScanModel()
S = 256
sig, _ = synth.batch_2d_device(m, range(S))
grid = synth.grid_square(0.12, 256)
bi = BatchImager(m.geometry(), m.pairs(), m.n_samples, grid, window=(m.k0, m.window), mode="smem")
das = torch.empty((S, 256 * 256), device="cuda")
dmas = torch.empty((S, 256 * 256), device="cuda")
for _ in range(2):
    if kind == "das":
        bi.run_device(sig, out_das=das)
    elif kind == "dmas":
        bi.run_device(sig, out_dmas=dmas)
    else:
        bi.run_device(sig, das, dmas)
torch.cuda.synchronize()
