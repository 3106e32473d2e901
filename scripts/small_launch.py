"""K1 time vs tile count for one scan (W = 32 and full record): the fixed cost
of a small launch.  Development aid."""
import sys
import statistics
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1709_02549_b200 import _device as dv
from paper_1709_02549_b200 import _native as nat
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.beamform import build_table, launch_energies

model = synth.ScanModel(n_samples=1024)
sig_h, _ = synth.batch_2d(model, [0])
sig = torch.from_numpy(np.ascontiguousarray(sig_h[0])).cuda()
scan = dv.DeviceScan(sig=sig, chan=torch.from_numpy(model.pairs()).cuda(),
                     ant=torch.from_numpy(np.array(model.geometry().antennas)).cuda(),
                     inv_scale=1.0 / (model.v * model.dt), n_samples=1024, ld=1024, n_ant=12,
                     chan_host=model.pairs())
rng = np.random.default_rng(0)
for w, k0 in ((32, model.k0), (1024, 0)):
    for tiles in (1, 4, 16, 64, 148, 444):
        n = tiles * 256
        # a compact patch (pitch 0.5 mm) like a lattice tile set
        side = int(np.ceil(np.sqrt(n)))
        ix, iy = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
        p = np.zeros((n, 3))
        p[:, 0] = (ix.ravel()[:n] * 5e-4) - 0.02
        p[:, 1] = (iy.ravel()[:n] * 5e-4) - 0.02
        pts = torch.from_numpy(p).cuda()
        table = build_table(scan, pts, n, 0)
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        f = lambda: launch_energies(scan, pts, n, table, 0, k0, w, out, None)
        f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(9):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        us = statistics.median(ts)
        # device time alone: the same launch replayed from a CUDA graph
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        dev_us = a.elapsed_time(b) * 1e3 / 20
        pps = n * 66 * w / (dev_us * 1e-6)
        print(f"W={w:5d} tiles={tiles:4d} call {us:8.1f} us  device {dev_us:8.1f} us  {pps:.3e} pps/s")
