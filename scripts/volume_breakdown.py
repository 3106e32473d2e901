"""configs[4] 128^3 DMAS volume: device time of each phase of image_volume
(enumeration, delay table, energy kernel, readback), CUDA events on the
launching stream, median of 10 calls.  Prints one JSON object."""
import json
import math
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes

import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import _device as dv
from paper_1709_02549_b200 import _native as nat
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.beamform import _Status, build_table, launch_energies
from paper_1709_02549_b200.volume import VolumeGrid

vm = synth.VolumeModel()
sig, _ = synth.scan_3d(vm, seed=9)
ds = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
g = VolumeGrid((-0.06, -0.06, 0.0), (0.12, 0.12, 0.12), 0.12 / 128)
scan = dv.scan_for(ds)
nx, ny, nz = g.dims
n = nx * ny * nz
dev = dv.device()
times = {k: [] for k in ("alloc", "enumerate", "table", "energy", "readback", "total")}
for it in range(12):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    dense = torch.zeros(n, dtype=torch.float32, device=dev)
    valid = torch.zeros(n, dtype=torch.uint8, device=dev)
    status = _Status()
    pts = torch.empty((n, 3), dtype=torch.float64, device=dev)
    oidx = torch.empty(n, dtype=torch.int32, device=dev)
    ws = torch.empty(int(nat.load().mwb_volume_workspace_bytes(nx, ny, nz, 1)), dtype=torch.uint8, device=dev)
    ev[1].record()
    box = (ctypes.c_int32 * 6)(*g.full_box().bounds())
    cp = status.count_ptr(0)
    nat.call("mwb_enumerate_volume", *g.origin, g.resolution, nx, ny, nz, ctypes.addressof(box), None, 1, None, 0,
             pts.data_ptr(), oidx.data_ptr(), cp, valid.data_ptr(), ws.data_ptr(), dv.stream_handle())
    ev[2].record()
    table = build_table(scan, pts, n, nat.INTERP["linear"], cp)
    ev[3].record()
    launch_energies(scan, pts, n, table, nat.INTERP["linear"], vm.k0, vm.window, None, dense, 0, oidx, cp,
                    status.key_ptr(0), status.key_ptr(1), status.flags_ptr, 0)
    ev[4].record()
    dv.to_host(status.t, valid, dense)
    ev[5].record()
    torch.cuda.synchronize()
    if it >= 2:
        for k, (a, b) in zip(times, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (0, 5)]):
            times[k].append(ev[a].elapsed_time(ev[b]))
print(json.dumps({k: statistics.median(v) for k, v in times.items()}))
