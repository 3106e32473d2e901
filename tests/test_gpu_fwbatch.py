"""FrameworkBatch: the framework for many scans at once must reproduce
run_framework scan by scan, bit for bit (regions, traces, argmax, values)."""

import numpy as np
import pytest
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.fwbatch import FrameworkBatch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["das", "dmas"])
def test_batch_equals_per_scan_run_framework(kind):
    model = synth.ScanModel(n_samples=1024)
    seeds = list(range(300, 312))
    sig, tum = synth.batch_2d(model, seeds, phantom_radius=(0.04, 0.05), snr_db=(15.0, 30.0))
    grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 5e-4)
    d = grid.dims[0] // 32
    fb = FrameworkBatch(model.geometry(), model.pairs(), model.n_samples, grid, mw.Manual(d), kind,
                        window=(model.k0, model.window))
    res = fb.run(torch.from_numpy(sig).cuda())
    for s in range(len(seeds)):
        ds = mw.BackscatterDataset(model.geometry(), synth.embed_pairs(12, model.pairs(), sig[s].astype(np.float64)))
        comp, rep = mw.run_framework(ds, kind, grid, mw.Manual(d), window=(model.k0, model.window))
        assert res.final_region(s) == rep.final_region
        assert tuple(res.argmax_cells[s]) == rep.argmax_cell
        assert res.fine_points_evaluated[s] == rep.fine_points_evaluated
        assert res.coarse_points_evaluated == rep.coarse_points_evaluated
        t = res.trace(s)
        assert [r.selected for r in t.records] == [r.selected for r in rep.trace.records]
        assert t.termination == rep.trace.termination
        assert [r.w for r in t.records] == [r.w for r in rep.trace.records]
        c = res.composite(s)
        assert c.entries == comp.entries
        assert res.reduction_ratios[s] == rep.reduction_ratio


def test_batch_throughput_smoke():
    model = synth.ScanModel(n_samples=1024)
    sig, _ = synth.batch_2d_device(model, range(256), phantom_radius=(0.04, 0.05))
    grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
    fb = FrameworkBatch(model.geometry(), model.pairs(), model.n_samples, grid, mw.Manual(grid.dims[0] // 32),
                        "dmas", window=(model.k0, model.window))
    res = fb.run(sig)
    assert res.n_scans == 256 and (res.fine_points_evaluated > 0).all()
    assert (res.reduction_ratios > 1).all()
