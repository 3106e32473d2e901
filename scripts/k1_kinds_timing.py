"""CUDA-core K1 (mode smem) at configs[3] shape: DAS, DMAS and fused BOTH step
times, and the configs[4] 128^3 volume.  Development aid."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager

m = synth.ScanModel()
S = 1024
sig, _ = synth.batch_2d_device(m, range(S))
grid = synth.grid_square(0.12, 256)
bi = BatchImager(m.geometry(), m.pairs(), m.n_samples, grid, window=(m.k0, m.window), mode="smem")
n = 256 * 256
das = torch.empty((S, n), device="cuda")
dmas = torch.empty((S, n), device="cuda")


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


pps = S * n * 66 * 32
for name, fn in (("das", lambda: bi.run_device(sig, out_das=das)), ("dmas", lambda: bi.run_device(sig, out_dmas=dmas)),
                 ("both", lambda: bi.run_device(sig, das, dmas))):
    ms = t(fn)
    print(f"{name}: {ms:.2f} ms, {pps / (ms * 1e-3):.3e} pps/s", flush=True)

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200.volume import VolumeGrid, image_volume

vm = synth.VolumeModel()
s3, _ = synth.scan_3d(vm, seed=9)
ds4 = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), s3))
g4 = VolumeGrid((-0.06, -0.06, 0.0), (0.12, 0.12, 0.12), 0.12 / 128)
print(f"volume dmas repeat: {t(lambda: image_volume(ds4, 'dmas', g4, window=(vm.k0, vm.window)), reps=3):.2f} ms")
