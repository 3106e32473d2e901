"""Per-configuration timings of the public API (BASELINE configs[0..4]).

Wall-clock medians include the host work of each call (enumeration launch,
delay table, energy launch, device->host copy of the map); device times are
CUDA events around the same calls.  Prints one JSON object.
"""

import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.segment import segment
from paper_1709_02549_b200.volume import VolumeGrid, hemisphere_mask, image_volume, run_framework_volume


def timed(fn, reps=10, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    walls, devs = [], []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
        devs.append(e0.elapsed_time(e1) / 1e3)
    return {"wall_ms": statistics.median(walls) * 1e3, "device_ms": statistics.median(devs) * 1e3}


def main():
    out = {}
    m0 = synth.ScanModel()
    ds, _ = synth.dataset_2d(m0, seed=0)
    win = (m0.k0, m0.window)
    g0 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
    g1 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 5e-4)
    out["cfg0_das_100x100"] = timed(lambda: mw.image(ds, "das", g0, window=win))
    out["cfg0_das+dmas_100x100"] = timed(lambda: mw.images(ds, ("das", "dmas"), g0, window=win))
    out["cfg1_dmas_200x200"] = timed(lambda: mw.image(ds, "dmas", g1, window=win))
    out["cfg1_dmas_200x200_full_record"] = timed(lambda: mw.image(ds, "dmas", g1))
    m2 = synth.ScanModel(n_samples=2048)
    ds2, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
    g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
    d = g2.dims[0] // 32
    for kind in ("das", "dmas"):
        out[f"cfg2_run_framework_{kind}"] = timed(lambda: mw.run_framework(ds2, kind, g2, mw.Manual(d),
                                                                           window=(m2.k0, 32)))
        _, rep = mw.run_framework(ds2, kind, g2, mw.Manual(d), window=(m2.k0, 32))
        out[f"cfg2_run_framework_{kind}"]["device_phases_ms"] = {k: v * 1e3 for k, v in rep.elapsed.items()}
        out[f"cfg2_segment_{kind}"] = timed(lambda: segment(ds2, kind, g2, 16, 0.01, window=(m2.k0, 32)))
        out[f"cfg2_full_image_{kind}"] = timed(lambda: mw.image(ds2, kind, g2, mask=mw.breast_mask(g2),
                                                               window=(m2.k0, 32)), reps=5)
    vm = synth.VolumeModel()
    sig, _ = synth.scan_3d(vm, seed=9)
    ds4 = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
    g4 = VolumeGrid((-0.06, -0.06, 0.0), (0.12, 0.12, 0.12), 0.12 / 128)  # 128^3, hemisphere in z < 6 cm
    out["cfg4_grid"] = list(g4.dims)
    out["cfg4_dmas_volume"] = timed(lambda: image_volume(ds4, "dmas", g4, window=(vm.k0, vm.window)), reps=3, warm=1)
    mask = hemisphere_mask(g4, vm.phantom_radius)
    out["cfg4_dmas_volume_hemisphere"] = timed(
        lambda: image_volume(ds4, "dmas", g4, mask=mask, window=(vm.k0, vm.window)), reps=3, warm=1)
    out["cfg4_octant_framework"] = timed(
        lambda: run_framework_volume(ds4, "dmas", g4, mw.Automatic(0.01), mask=mask, window=(vm.k0, vm.window)),
        reps=3, warm=1)
    _, rep4 = run_framework_volume(ds4, "dmas", g4, mw.Automatic(0.01), mask=mask, window=(vm.k0, vm.window))
    out["cfg4_octant_framework"]["report"] = {k: v for k, v in rep4.to_dict().items() if k != "trace"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
