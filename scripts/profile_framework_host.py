import cProfile, pstats, time, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
m2 = synth.ScanModel(n_samples=2048)
ds2, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
d = g2.dims[0] // 32
mask2 = mw.breast_mask(g2)
win = (m2.k0, 32)
fw = lambda: mw.run_framework(ds2, "das", g2, mw.Manual(d), window=win)
im = lambda: mw.image(ds2, "das", g2, mask=mask2, window=win)
for name, fn in (("framework", fw), ("image", im)):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000): fn()
    torch.cuda.synchronize()
    print(name, "wall us/call", (time.perf_counter() - t0) / 2000 * 1e6)
    pr = cProfile.Profile(); pr.enable()
    for _ in range(2000): fn()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
