"""Phase breakdown of run_framework on the reference's dataset1 preset."""
import sys
import statistics
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import torch

import paper_1709_02549_b200 as mw
from _mwb_helpers import grid_for_geometry, preset
from paper_1709_02549_b200 import _device as dv

_, ds1 = preset("dataset1")
grid = grid_for_geometry(ds1.geometry, 0.001)
scan = dv.scan_for(ds1)
print("channels", scan.n_chan, "samples", scan.n_samples, "grid", grid.dims)
for kind in ("das", "dmas"):
    els = []
    for _ in range(6):
        _, rep = mw.run_framework(ds1, kind, grid, mw.Automatic(0.01))
        els.append(rep.elapsed)
    print(kind, {k: round(statistics.median(e[k] for e in els[1:]) * 1e3, 3) for k in els[0]},
          "d", rep.decimation_factor, "coarse", rep.coarse_points_evaluated, "fine", rep.fine_points_evaluated,
          "iters", rep.iterations, "final", rep.final_region)
