"""configs[4] 128^3 DMAS voxel image once (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.volume import VolumeGrid, image_volume

vm = synth.VolumeModel()
sig, _ = synth.scan_3d(vm, seed=9)
ds = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
g = VolumeGrid((-0.06, -0.06, 0.0), (0.12, 0.12, 0.12), 0.12 / 128)
for _ in range(2):
    image_volume(ds, "dmas", g, window=(vm.k0, vm.window))
torch.cuda.synchronize()
print("ok")
