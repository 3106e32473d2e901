"""BASELINE configs[2] segmentation variant, device resident.

BASELINE.json describes the framework as: split the current region into 4
quadrants, score each on a 16 x 16 low-resolution sub-grid with the
max-to-mean energy metric, keep the argmax quadrant, stop at a 1 cm segment,
then refine that segment to 0.25 mm pixels while the rest of the image stays
at the low resolution.  The reference implements a different rule set
(single decimated pass + Eq. (5) + W/B, coarse2fine.py:169-350, available as
``run_framework``); this variant has no reference counterpart, so its oracle
composes reference energies with a restated control loop.

Choices recorded here (and in DESIGN.md):
* the quadrant split is the reference's Region.quadrants (geometry.py:225-242);
* sub-grid centres: corner + (i + 0.5) * side / n_sub per axis;
* DAS scores are max/mean of the sub-grid energies; DMAS energies can be
  negative, so they are shifted by the iteration's minimum first;
* ties go to the lowest quadrant index (np.argmax);
* the search stops when the kept segment's larger side is <= stop_size.

Every iteration (points, delay table, energies, score/argmax) stays on the
device; the host enqueues a fixed upper bound of iterations and reads the
result once.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _native as nat
from .beamform import EVAL_COUNTER, EnergyMap, _check_interpolation, _kind, _kind_code, _Status, _window, lattice_pass
from .coarse2fine import breast_mask
from .geometry import ImagingGrid, Region


@dataclass
class SegmentRecord:
    iteration: int
    parent: Region
    selected: int
    selected_region: Region
    scores: list[float]
    maxima: list[float]
    means: list[float]
    shift: float

    def to_dict(self) -> dict:
        return {
            "iteration": self.iteration,
            "parent": self.parent.to_dict(),
            "selected": self.selected,
            "selected_region": self.selected_region.to_dict(),
            "scores": self.scores,
            "maxima": self.maxima,
            "means": self.means,
            "shift": self.shift,
        }


@dataclass
class SegmentReport:
    kind: str
    n_sub: int
    stop_cells: int
    records: list[SegmentRecord]
    final_region: Region
    lowres: np.ndarray  # (2 n_sub, 2 n_sub) energies of the starting region
    subgrid_points_evaluated: int
    fine_points_evaluated: int
    full_equivalent_points: int
    argmax_cell: tuple[int, int]
    argmax_position: tuple[float, float]
    elapsed: dict

    @property
    def iterations(self) -> int:
        return len(self.records)

    def to_dict(self) -> dict:
        return {
            "kind": self.kind,
            "n_sub": self.n_sub,
            "stop_cells": self.stop_cells,
            "records": [r.to_dict() for r in self.records],
            "final_region": self.final_region.to_dict(),
            "subgrid_points_evaluated": self.subgrid_points_evaluated,
            "fine_points_evaluated": self.fine_points_evaluated,
            "full_equivalent_points": self.full_equivalent_points,
            "argmax_cell": list(self.argmax_cell),
            "argmax_position": list(self.argmax_position),
            "elapsed": self.elapsed,
        }


def _region(b) -> Region:
    return Region((int(b[0]), int(b[1])), (int(b[3]), int(b[4])))


def max_iterations(region: Region, stop_cells: int) -> int:
    """Upper bound on the iterations (the larger quadrant is kept every time)."""
    w, h = region.width, region.height
    n = 0
    while max(w, h) > stop_cells and w >= 2 and h >= 2:
        w, h = (w + 1) // 2, (h + 1) // 2
        n += 1
    return n


def segment(ds, kind, grid: ImagingGrid, n_sub: int = 16, stop_size: float = 0.01, *, region: Region | None = None,
            mask="breast", window=None, interpolation: str = "linear") -> tuple[EnergyMap, SegmentReport]:
    """Quadrant search scored on n_sub x n_sub sub-grids, then a full-resolution
    pass over the kept segment.  Returns (fine map of the segment, report)."""
    _check_interpolation(interpolation)
    if not stop_size > 0:
        raise ValueError("stop_size must be > 0")
    if not 1 <= n_sub <= 64:
        raise ValueError("n_sub must be in [1, 64]")
    region = grid.full_region() if region is None else region
    if not grid.full_region().contains_region(region):
        raise ValueError("region lies outside the grid")
    stop_cells = max(1, int(math.floor(stop_size / grid.resolution + 1e-9)))
    n_iter = max_iterations(region, stop_cells)
    if n_iter > nat.SEG_MAX_ITERS:
        raise ValueError("stop_size too small for the segment trace")
    kcode = _kind_code(kind)
    scan = dv.scan_for(ds)
    k0, w = _window(scan.n_samples, window)
    if w == 0:
        raise ValueError("the segmentation metric needs a non-empty energy window")
    interp = nat.INTERP[interpolation]
    nx, ny = grid.dims
    dev = dv.device()
    ws = torch.empty(int(nat.load().mwb_segment_workspace_bytes(n_sub, scan.n_chan)), dtype=torch.uint8, device=dev)
    region_t = torch.zeros(6, dtype=torch.int32, device=dev)
    lowres = torch.zeros((2 * n_sub) ** 2, dtype=torch.float32, device=dev)
    trace_t = torch.zeros(nat.SEG_TRACE_BYTES, dtype=torch.uint8, device=dev)
    m = breast_mask(grid) if isinstance(mask, str) and mask == "breast" else mask
    mask_t = dv.upload_mask(m, grid.dims) if m is not None else None
    dense = torch.zeros(nx * ny, dtype=torch.float32, device=dev)
    valid = torch.zeros(nx * ny, dtype=torch.uint8, device=dev)
    status = _Status()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    x0, y0, x1, y1 = region.bounds()
    ev[0].record()
    nat.call("mwb_segment", scan.sig.data_ptr(), scan.n_chan, scan.ld, scan.n_samples, scan.chan.data_ptr(),
             scan.ant.data_ptr(), scan.n_ant, scan.inv_scale, interp, k0, w, kcode, grid.origin[0], grid.origin[1],
             grid.resolution, nx, ny, x0, y0, x1, y1, n_sub, stop_cells, n_iter, region_t.data_ptr(),
             lowres.data_ptr(), trace_t.data_ptr(), ws.data_ptr(), dv.stream_handle())
    ev[1].record()
    lattice_pass(scan, grid, 1, mask_t, 0, (kcode,), interp, k0, w, {kcode: dense}, valid, status, 0,
                 d_region=region_t)
    ev[2].record()
    st, th, dh, vh, lh = dv.to_host(status.t, trace_t, dense.view(nx, ny), valid.view(nx, ny),
                                    lowres.view(2 * n_sub, 2 * n_sub))
    keys, counts, flags = status.read(st)
    if flags & 1:
        raise ValueError("energy map contains non-finite values")
    tr = nat.SegTrace.from_buffer_copy(th.tobytes())
    records = []
    for i in range(int(tr.n_records)):
        r = tr.records[i]
        records.append(SegmentRecord(
            iteration=int(r.iteration), parent=_region(r.parent), selected=int(r.selected),
            selected_region=_region(r.selected_region), scores=[float(v) for v in r.score],
            maxima=[float(v) for v in r.emax], means=[float(v) for v in r.emean], shift=float(r.shift)))
    final = _region(tr.final_region)
    n_fine = int(counts[0])
    EVAL_COUNTER.add(n_fine + 4 * n_sub * n_sub * len(records))
    fine = EnergyMap._from_dense(grid, dh, vh.view(bool), 1, roi=final)
    key = int(keys[0 if kcode == nat.MWB_DAS else 1])
    if key:
        slot = 0xFFFFFFFF - (key & 0xFFFFFFFF)
        cell = (slot // ny, slot % ny)
    else:
        cell = (final.min_cell[0], final.min_cell[1])
    full_eq = int(m.sum()) if m is not None else grid.dims[0] * grid.dims[1]
    report = SegmentReport(
        kind=_kind(kind).value, n_sub=n_sub, stop_cells=stop_cells, records=records, final_region=final,
        lowres=lh,
        subgrid_points_evaluated=4 * n_sub * n_sub * len(records), fine_points_evaluated=n_fine,
        full_equivalent_points=full_eq, argmax_cell=cell, argmax_position=grid.cell_center(*cell),
        elapsed={"search": ev[0].elapsed_time(ev[1]) / 1e3, "fine": ev[1].elapsed_time(ev[2]) / 1e3,
                 "total": ev[0].elapsed_time(ev[2]) / 1e3})
    return fine, report
