"""cProfile of the host side of single-scan calls (configs[2] run_framework and
the full masked image).  Development aid."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth

m2 = synth.ScanModel(n_samples=2048)
g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
d = g2.dims[0] // 32
w2 = (m2.k0, 32)
ds, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
mask = mw.breast_mask(g2)
for name, fn in (("run_framework", lambda: mw.run_framework(ds, "das", g2, mw.Manual(d), window=w2)),
                 ("image", lambda: mw.image(ds, "das", g2, mask=mask, window=w2))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        fn()
    pr.disable()
    print("=" * 20, name)
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
