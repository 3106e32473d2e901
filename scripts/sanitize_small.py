"""Small end-to-end run of every device path (for compute-sanitizer)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager
from paper_1709_02549_b200.segment import segment
from paper_1709_02549_b200.volume import VolumeGrid, image_volume, run_framework_volume

m = synth.ScanModel(n_samples=254)  # ragged record length (ld = 256)
ds, _ = synth.dataset_2d(m, seed=1)
grid = synth.grid_square(0.1, 40)
mw.images(ds, ("das", "dmas"), grid, window=(m.k0, 32))
mw.image(ds, "dmas", grid, stride=3, mask=mw.breast_mask(grid))
mw.image(ds, "das", grid, window=(240, 32))  # spans past the record (zero-fill path)
mw.image(ds, "das", grid, mode="gather")
mw.energies(ds, np.random.default_rng(0).uniform(-1, 1, (50, 2)), "dmas")  # wide tiles
mw.run_framework(ds, "dmas", grid, mw.Manual(3))
segment(ds, "das", synth.grid_square(0.1, 200), 16, 0.01, window=(m.k0, 32))
m3 = synth.ScanModel(n_samples=256)
sig, _ = synth.batch_2d(m3, range(6))
bi = BatchImager(m3.geometry(), m3.pairs(), m3.n_samples, grid, window=(m3.k0, 32))
bi(torch.from_numpy(sig), chunk=4)
vm = synth.VolumeModel(n_samples=512)
s3, _ = synth.scan_3d(vm, seed=2)
ds3 = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), s3))
vg = VolumeGrid((-0.02, -0.02, 0.0), (0.04, 0.04, 0.02), 0.002)
image_volume(ds3, ("das", "dmas"), vg, window=(vm.k0, 48))
run_framework_volume(ds3, "dmas", vg, mw.Manual(3), window=(vm.k0, 48))
torch.cuda.synchronize()
print("sanitize_small ok")
