import cProfile, pstats, sys
sys.path.insert(0, ".")
import torch
import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
m2 = synth.ScanModel(n_samples=2048)
ds2, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
d = g2.dims[0] // 32
for _ in range(5):
    mw.run_framework(ds2, "das", g2, mw.Manual(d), window=(m2.k0, 32))
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    mw.run_framework(ds2, "das", g2, mw.Manual(d), window=(m2.k0, 32))
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
