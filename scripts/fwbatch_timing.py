"""FrameworkBatch throughput on configs[2]-shaped scans (development aid)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.fwbatch import FrameworkBatch

model = synth.ScanModel(n_samples=2048)
grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
for S in (256, 1024, 4096):
    sig, _ = synth.batch_2d_device(model, range(S), phantom_radius=(0.04, 0.05))
    for kind in ("das", "dmas"):
        fb = FrameworkBatch(model.geometry(), model.pairs(), model.n_samples, grid, mw.Manual(grid.dims[0] // 32), kind,
                            window=(model.k0, 32))
        fb.run(sig)
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = fb.run(sig)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(S, kind, f"{dt*1e3:.1f} ms wall, device phases {res.elapsed}, {S/dt:.0f} segmented images/s, "
              f"fine pts mean {res.fine_points_evaluated.mean():.0f}, coarse {res.coarse_points_evaluated}")
    del sig
