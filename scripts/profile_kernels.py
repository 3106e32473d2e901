"""Launch each energy-kernel variant on a configs[3]-shaped batch (for ncu).

Launch order: DAS, DMAS, BOTH (smem), DAS, DMAS, BOTH (gather) — each once as a
warm-up and once more; with `-k regex:energy_kernel -s 6 -c 6` ncu captures
the second launch of every variant.
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager


def main(scans: int = 256):
    model = synth.ScanModel()
    sig, _ = synth.batch_2d(model, range(scans))
    grid = synth.grid_square(0.12, 256)
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(model.k0, model.window))
    sig_d = bi.to_device_layout(sig)
    out = [torch.empty((scans, 256 * 256), dtype=torch.float32, device="cuda") for _ in range(2)]
    for rep in range(2):
        for mode in (0, 1):
            bi.mode = mode
            bi.run_device(sig_d, out_das=out[0])
            bi.run_device(sig_d, out_dmas=out[1])
            bi.run_device(sig_d, out[0], out[1])
    torch.cuda.synchronize()
    print("ok", scans, bi.n_pts, bi.n_chan)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 256)
