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

import ctypes as C
import functools
import hashlib
import math
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _native as nat
from .beamform import EVAL_COUNTER, EnergyMap, _check_interpolation, _kind, _kind_code, _Status, _window, lattice_pass
from .coarse2fine import _breast_mask_device
from .geometry import ArrayGeometry, ImagingGrid, Region, as_grid, as_region


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


_TREE_PLANS: "OrderedDict[tuple, tuple]" = OrderedDict()
_TREE_PLAN_CAPACITY = 4


def _tree_plan(scan: dv.DeviceScan, antennas, grid: ImagingGrid, region: Region, mask_key, mask_t, n_sub: int,
               stop_cells: int, n_iter: int, interp: int):
    """(plan tensor, fine tiles per scan) of the region tree for one geometry,
    grid, mask and search configuration, shared by every scan (LRU); None when
    the tree is too large for a plan."""
    ants = np.ascontiguousarray(np.asarray(antennas, dtype=np.float64)).tobytes()
    key = (torch.cuda.current_device(), ants, scan.chan_host.tobytes(), float(scan.inv_scale), tuple(grid.origin),
           float(grid.resolution), tuple(grid.dims), region.bounds(), mask_key, n_sub, stop_cells, n_iter, interp)
    if key in _TREE_PLANS:
        _TREE_PLANS.move_to_end(key)
        return _TREE_PLANS[key]
    lib = nat.load()
    nx, ny = grid.dims
    x0, y0, x1, y1 = region.bounds()
    info = (C.c_int64 * 4)()
    ent = None
    if lib.mwb_segment_plan_info(nx, ny, x0, y0, x1, y1, n_sub, stop_cells, n_iter, scan.n_chan, info) == 0:
        plan = torch.empty(int(info[0]), dtype=torch.uint8, device=dv.device())
        nat.call("mwb_segment_plan_prepare", scan.chan.data_ptr(), scan.n_chan, scan.ant.data_ptr(), scan.n_ant,
                 scan.inv_scale, interp, grid.origin[0], grid.origin[1], grid.resolution, nx, ny, x0, y0, x1, y1,
                 mask_t.data_ptr() if mask_t is not None else None, n_sub, stop_cells, n_iter, plan.data_ptr(),
                 dv.stream_handle())
        ent = (plan, int(info[3]))
    _TREE_PLANS[key] = ent
    while len(_TREE_PLANS) > _TREE_PLAN_CAPACITY:
        _TREE_PLANS.popitem(last=False)
    return ent


class _SegmentPlan(dv.GraphPlan):
    """One segment() configuration on one device scan, captured as a CUDA graph;
    later calls replay it and read the results back into pinned buffers with
    one synchronisation.  Buffers persist with the plan, so a replay allocates
    nothing (as coarse2fine._FrameworkPlan).

    With a region-tree plan (shared by every scan of the geometry and grid) the
    graph is one mwb_segment_run for this scan: two launches per iteration plus
    two for the fine pass, exactly SegmentBatch's routine for S = 1.  Without
    one (trees above 16384 regions) it is mwb_segment plus a lattice pass."""

    def __init__(self, scan: dv.DeviceScan, grid: ImagingGrid, region: Region, kcode: int, n_sub: int,
                 stop_cells: int, n_iter: int, interp: int, k0: int, w: int, mask_np, mask_t, tree):
        scan = self._init_slot(scan)
        self.scan, self.grid, self.region, self.kcode = scan, grid, region, kcode
        self.n_sub, self.stop_cells, self.n_iter = n_sub, stop_cells, n_iter
        self.interp, self.k0, self.w = interp, k0, w
        self.mask_np, self.mask_t = mask_np, mask_t
        self.tree = tree
        nx, ny = grid.dims
        dev = dv.device()
        n_low = (2 * n_sub) ** 2
        lib = nat.load()
        ws_bytes = (lib.mwb_segment_run_workspace_bytes(1, n_sub, tree[1], w) if tree is not None
                    else lib.mwb_segment_workspace_bytes(n_sub, scan.n_chan))
        self.ws = torch.empty(int(ws_bytes), dtype=torch.uint8, device=dev)
        self.region_t = torch.zeros(6, dtype=torch.int32, device=dev)
        self.lowres = torch.zeros(n_low, dtype=torch.float32, device=dev)
        self.trace_t = torch.zeros(nat.SEG_TRACE_BYTES, dtype=torch.uint8, device=dev)
        self.dense = torch.empty(nx * ny, dtype=torch.float32, device=dev)  # only valid cells are read
        self.valid = torch.empty(nx * ny, dtype=torch.uint8, device=dev)
        self.events = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]
        pin = torch.cuda.is_available()
        self._pin = pin
        self.full_eq = int(mask_np.sum()) if mask_np is not None else nx * ny
        # one result block read back with one copy per call (region-tree path):
        # [status | trace | low-res map | the final region's rectangle, row by
        # row (mwb_gather_composite)], sized for the worst case (the whole
        # start region); a call copies up to a budget of rectangle cells
        self._o_trace = _Status.BYTES
        self._o_low = (self._o_trace + nat.SEG_TRACE_BYTES + 15) // 16 * 16
        self._o_roi = self._o_low + 4 * n_low
        rx0, ry0, rx1, ry1 = region.bounds()
        cap = (rx1 - rx0 + 1) * (ry1 - ry0 + 1)
        self._res_full = self._o_roi + 4 * cap
        self._res_copy = self._o_roi + 4 * min(cap, self.ROI_BUDGET)
        self.res = torch.empty(self._res_full, dtype=torch.uint8, device=dev)
        self.status = _Status(self.res)
        self.roi_t = self.res[self._o_roi:].view(torch.float32)
        if tree is not None:
            self.trace_t = self.res[self._o_trace: self._o_trace + nat.SEG_TRACE_BYTES]
            self.lowres = self.res[self._o_low: self._o_roi].view(torch.float32)
        else:
            self.h_status = torch.empty_like(self.status.t, device="cpu", pin_memory=pin)
            self.h_trace = torch.empty(nat.SEG_TRACE_BYTES, dtype=torch.uint8, pin_memory=pin)
            self.h_lowres = torch.empty(n_low, dtype=torch.float32, pin_memory=pin)
        self._ms = (C.c_float * 2)()
        self._ev_handles = None

    ROI_BUDGET = 4096  # final-region cells read back with the result block (a 1 cm segment at 0.25 mm: 1600)

    def _enqueue(self) -> None:
        sc, grid = self.scan, self.grid
        nx, ny = grid.dims
        x0, y0, x1, y1 = self.region.bounds()
        ev = self.events
        self.status.t.zero_()
        self.lowres.zero_()
        if self.tree is not None:
            ev[0].record()
            das = self.kcode == nat.MWB_DAS
            nat.call("mwb_segment_run", self.tree[0].data_ptr(), sc.sig.data_ptr(), 1, sc.n_chan * sc.ld, sc.n_chan,
                     sc.ld, sc.n_samples, sc.chan.data_ptr(), sc.ant.data_ptr(), sc.n_ant, sc.inv_scale,
                     self.interp, self.k0, self.w, self.kcode, nx, ny, x0, y0, x1, y1, self.n_sub, self.stop_cells,
                     self.n_iter, self.region_t.data_ptr(), self.lowres.data_ptr(), self.trace_t.data_ptr(),
                     self.dense.data_ptr(), nx * ny, self.status.key_ptr(0 if das else 1), self.status.count_ptr(0),
                     self.status.flags_ptr, self.ws.data_ptr(), dv.stream_handle())
            ev[1].record()
            nat.call("mwb_gather_composite", self.dense.data_ptr(), ny, 1, None, 0, self.region_t.data_ptr(),
                     self.roi_t.data_ptr(), self.roi_t.numel(), dv.stream_handle())
            return
        self.valid.zero_()
        ev[0].record()
        nat.call("mwb_segment", sc.sig.data_ptr(), sc.n_chan, sc.ld, sc.n_samples, sc.chan.data_ptr(),
                 sc.ant.data_ptr(), sc.n_ant, sc.inv_scale, self.interp, self.k0, self.w, self.kcode, grid.origin[0],
                 grid.origin[1], grid.resolution, nx, ny, x0, y0, x1, y1, self.n_sub, self.stop_cells, self.n_iter,
                 self.region_t.data_ptr(), self.lowres.data_ptr(), self.trace_t.data_ptr(), self.ws.data_ptr(),
                 dv.stream_handle())
        ev[1].record()
        lattice_pass(sc, grid, 1, self.mask_t, 0, (self.kcode,), self.interp, self.k0, self.w,
                     {self.kcode: self.dense}, self.valid, self.status, 0, d_region=self.region_t)
        ev[2].record()

    def launch(self, scan: dv.DeviceScan) -> None:
        self.replay(scan)
        nx, ny = self.grid.dims
        if self.tree is not None:
            self.h_res = torch.empty(self._res_copy, dtype=torch.uint8, pin_memory=self._pin)
            nat.call("mwb_memcpy_async", self.h_res.data_ptr(), self.res.data_ptr(), self._res_copy,
                     dv.stream_handle())
            return
        self.h_dense = torch.empty(nx * ny, dtype=torch.float32, pin_memory=self._pin)
        if self.tree is None:
            self.h_valid = torch.empty(nx * ny, dtype=torch.uint8, pin_memory=self._pin)
        pairs = [(self.status.t, self.h_status), (self.trace_t, self.h_trace), (self.dense, self.h_dense),
                 (self.lowres, self.h_lowres)]
        if self.tree is None:
            pairs.append((self.valid, self.h_valid))
        for src, dst in pairs:
            dst.copy_(src, non_blocking=True)

    def _roi_arrays(self, block: np.ndarray, final: Region) -> tuple[np.ndarray, np.ndarray]:
        """(values, valid) of the fine map from the final region's rectangle:
        the region's cells that pass the mask."""
        nx, ny = self.grid.dims
        (x0, y0), (x1, y1) = final.min_cell, final.max_cell
        vals = np.zeros((nx, ny), dtype=np.float32)
        valid = np.zeros((nx, ny), dtype=bool)
        vals[x0: x1 + 1, y0: y1 + 1] = block.reshape(x1 - x0 + 1, y1 - y0 + 1)
        valid[x0: x1 + 1, y0: y1 + 1] = True
        if self.mask_np is not None:
            valid &= self.mask_np
        return vals, valid

    def finish(self, kind) -> tuple[EnergyMap, SegmentReport]:
        if self.tree is not None:
            return self._finish_block(kind)
        dv.sync_stream()
        grid = self.grid
        nx, ny = grid.dims
        keys, counts, flags = self.status.read(self.h_status.numpy())
        if flags & 1:
            raise ValueError("energy map contains non-finite values")
        records, final = _decode_seg_trace(self.h_trace.numpy().tobytes())
        n_fine = int(counts[0])
        n_sub = self.n_sub
        EVAL_COUNTER.add(n_fine + 4 * n_sub * n_sub * len(records))
        vals = self.h_dense.numpy().reshape(nx, ny)
        if self.tree is None:
            vmask = self.h_valid.numpy().reshape(nx, ny).view(bool)
        else:  # the final region's cells that pass the mask
            vmask = np.zeros((nx, ny), dtype=bool)
            (fx0, fy0), (fx1, fy1) = final.min_cell, final.max_cell
            vmask[fx0 : fx1 + 1, fy0 : fy1 + 1] = True
            if self.mask_np is not None:
                vmask &= self.mask_np
        fine = EnergyMap._from_dense(grid, vals, vmask, 1, roi=final, checked=True)
        key = int(keys[0 if self.kcode == nat.MWB_DAS else 1])
        if key:
            slot = 0xFFFFFFFF - (key & 0xFFFFFFFF)
            cell = (slot // ny, slot % ny)
        else:
            cell = (final.min_cell[0], final.min_cell[1])
        full_eq = self.full_eq
        ev = self.events
        if self.tree is None:
            t_s, t_f = ev[0].elapsed_time(ev[1]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3
            elapsed = {"search": t_s, "fine": t_f, "total": t_s + t_f}
        else:  # search and fine pass are one library call
            elapsed = {"total": ev[0].elapsed_time(ev[1]) / 1e3}
        report = SegmentReport(
            kind=_kind(kind).value, n_sub=n_sub, stop_cells=self.stop_cells, records=records, final_region=final,
            lowres=self.h_lowres.numpy().reshape(2 * n_sub, 2 * n_sub).copy(),
            subgrid_points_evaluated=4 * n_sub * n_sub * len(records), fine_points_evaluated=n_fine,
            full_equivalent_points=full_eq, argmax_cell=cell, argmax_position=grid.cell_center(*cell),
            elapsed=elapsed)
        return fine, report

    def _finish_block(self, kind) -> tuple[EnergyMap, SegmentReport]:
        """The region-tree path: everything from the one result block."""
        dv.sync_stream()
        grid = self.grid
        nx, ny = grid.dims
        blk = self.h_res.numpy()
        keys, counts, flags = _Status.decode(blk[: _Status.BYTES].view(np.int64))
        if flags & 1:
            raise ValueError("energy map contains non-finite values")
        records, final = _decode_seg_trace(blk[self._o_trace: self._o_trace + nat.SEG_TRACE_BYTES].tobytes())
        (x0, y0), (x1, y1) = final.min_cell, final.max_cell
        used = self._o_roi + 4 * (x1 - x0 + 1) * (y1 - y0 + 1)
        if used > self._res_copy:  # final region beyond the budget: copy the whole used block again
            self.h_res = torch.empty(used, dtype=torch.uint8, pin_memory=self._pin)
            nat.call("mwb_memcpy_async", self.h_res.data_ptr(), self.res.data_ptr(), used, dv.stream_handle())
            dv.sync_stream()
            blk = self.h_res.numpy()
        n_fine = int(counts[0])
        n_sub = self.n_sub
        EVAL_COUNTER.add(n_fine + 4 * n_sub * n_sub * len(records))
        block = blk[self._o_roi: used].view(np.float32)
        fine = EnergyMap._from_loader(grid, functools.partial(self._roi_arrays, block, final), 1, roi=final)
        key = int(keys[0 if self.kcode == nat.MWB_DAS else 1])
        if key:
            slot = 0xFFFFFFFF - (key & 0xFFFFFFFF)
            cell = (slot // ny, slot % ny)
        else:
            cell = (final.min_cell[0], final.min_cell[1])
        if self._ev_handles is None:
            self._ev_handles = (C.c_void_p * 2)(*[e.cuda_event for e in self.events[:2]])
        nat.call("mwb_elapsed_ms", self._ev_handles, 2, self._ms)
        report = SegmentReport(
            kind=_kind(kind).value, n_sub=n_sub, stop_cells=self.stop_cells, records=records, final_region=final,
            lowres=blk[self._o_low: self._o_roi].view(np.float32).reshape(2 * n_sub, 2 * n_sub).copy(),
            subgrid_points_evaluated=4 * n_sub * n_sub * len(records), fine_points_evaluated=n_fine,
            full_equivalent_points=self.full_eq, argmax_cell=cell, argmax_position=grid.cell_center(*cell),
            elapsed={"total": self._ms[0] / 1e3})
        return fine, report


_SEG_PLANS: "OrderedDict[tuple, _SegmentPlan]" = OrderedDict()
_SEG_PLAN_CAPACITY = 8


def _mask_for(grid: ImagingGrid, mask):
    """(host mask or None, device mask or None, cache key)."""
    if isinstance(mask, str):
        if mask != "breast":
            raise ValueError(f"unknown mask {mask!r}")
        m, mt = _breast_mask_device(grid)
        return m, mt, "breast"
    if mask is None:
        return None, None, None
    m = np.asarray(mask, dtype=bool)
    if m.shape != grid.dims:
        raise ValueError(f"mask shape {m.shape} != grid dims {grid.dims}")
    return m, dv.upload_mask(m, grid.dims), hashlib.sha1(np.packbits(m).tobytes()).hexdigest()


def segment(ds, kind, grid: ImagingGrid, n_sub: int = 16, stop_size: float = 0.01, *, region: Region | None = None,
            mask="breast", window=None, interpolation: str = "linear",
            tree: bool = True) -> tuple[EnergyMap, SegmentReport]:
    """Quadrant search scored on n_sub x n_sub sub-grids, then a full-resolution
    pass over the kept segment.  Returns (fine map of the segment, report).

    Calls with one configuration on scans of one geometry replay a captured
    CUDA graph that reads a signal slot each call refills (as run_framework's)."""
    _check_interpolation(interpolation)
    if not stop_size > 0:
        raise ValueError("stop_size must be > 0")
    if not 1 <= n_sub <= 64:
        raise ValueError("n_sub must be in [1, 64]")
    grid, region = as_grid(grid), as_region(region)
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
    m, mt, mkey = _mask_for(grid, mask)
    with dv.PLAN_LOCK:
        key = (scan.geometry_key(), grid.origin, grid.extent, grid.resolution, region.bounds(), kcode, n_sub,
               stop_cells, interp, k0, w, mkey, bool(tree))
        plan = _SEG_PLANS.get(key)
        if plan is None:
            tree = (_tree_plan(scan, ds.geometry.antennas, grid, region, mkey, mt, n_sub, stop_cells, n_iter, interp)
                    if tree else None)
            plan = _SegmentPlan(scan, grid, region, kcode, n_sub, stop_cells, n_iter, interp, k0, w, m, mt, tree)
            _SEG_PLANS[key] = plan
            while len(_SEG_PLANS) > _SEG_PLAN_CAPACITY:
                _SEG_PLANS.popitem(last=False)
        else:
            _SEG_PLANS.move_to_end(key)
        plan.launch(scan)
        return plan.finish(kind)


def _decode_seg_trace(raw: bytes) -> tuple[list[SegmentRecord], Region]:
    tr = nat.SegTrace.from_buffer_copy(raw)
    records = []
    for i in range(int(tr.n_records)):
        r = tr.records[i]
        records.append(SegmentRecord(
            iteration=int(r.iteration), parent=_region(r.parent), selected=int(r.selected),
            selected_region=_region(r.selected_region), scores=[float(v) for v in r.score],
            maxima=[float(v) for v in r.emax], means=[float(v) for v in r.emean], shift=float(r.shift)))
    return records, _region(tr.final_region)


@dataclass
class SegmentBatchResult:
    grid: ImagingGrid
    kind: str
    n_sub: int
    final_regions: np.ndarray  # (S, 4) x0, y0, x1, y1
    argmax_cells: np.ndarray  # (S, 2)
    iterations: np.ndarray  # (S,)
    fine_points_evaluated: np.ndarray  # (S,)
    full_equivalent_points: int
    dense: torch.Tensor  # (S, nx, ny) fine energies on the device (valid inside each final region only)
    lowres: torch.Tensor  # (S, 2 n_sub, 2 n_sub) on the device
    elapsed: dict
    _traces: torch.Tensor
    _mask: np.ndarray | None

    @property
    def n_scans(self) -> int:
        return int(self.final_regions.shape[0])

    def final_region(self, s: int) -> Region:
        x0, y0, x1, y1 = (int(v) for v in self.final_regions[s])
        return Region((x0, y0), (x1, y1))

    def records(self, s: int) -> list[SegmentRecord]:
        n = nat.SEG_TRACE_BYTES
        return _decode_seg_trace(self._traces[s * n : (s + 1) * n].cpu().numpy().tobytes())[0]

    def fine(self, s: int) -> EnergyMap:
        """Scan s's full-resolution map of its final segment, as ``segment`` returns it."""
        nx, ny = self.grid.dims
        x0, y0, x1, y1 = (int(v) for v in self.final_regions[s])
        valid = np.zeros((nx, ny), dtype=bool)
        valid[x0 : x1 + 1, y0 : y1 + 1] = True
        if self._mask is not None:
            valid &= self._mask
        # only the final segment's block comes back from the device
        values = np.zeros((nx, ny), dtype=np.float32)
        values[x0 : x1 + 1, y0 : y1 + 1] = self.dense[s, x0 : x1 + 1, y0 : y1 + 1].cpu().numpy()
        return EnergyMap._from_dense(self.grid, values, valid, 1, roi=self.final_region(s), checked=True)


class SegmentBatch:
    """``segment`` for S scans that share the antenna geometry, the grid and the
    start region (BASELINE configs[2] at batch throughput).

    The regions a search can visit depend only on the grid, start region and
    stop size, so the constructor builds a region-tree plan once
    (``mwb_segment_plan_prepare``): the sub-grid points and delay tables of
    every region that gets split, and the fine-pass cells and tables of every
    region a search can end in.  ``run`` is then one ``mwb_segment_run`` call:
    two launches per iteration for the whole batch and two for the fine pass,
    no host synchronisation until the results are read.

    When the tree is too large (tiny stop sizes), or with ``tree=False``, each
    iteration builds its own points and tables (``mwb_segment_batch``) and the
    fine pass is one packed launch (``mwb_enumerate_regions_*`` +
    ``mwb_delay_table_tiles`` + ``mwb_energies_tiles``, as in FrameworkBatch),
    with one host synchronisation to size the packed list.

    Either way, regions, traces, low-res images, fine energies and argmax cells
    are bit-identical to calling ``segment`` once per scan.
    """

    def __init__(self, geometry: ArrayGeometry, pairs, n_samples: int, grid: ImagingGrid, kind, n_sub: int = 16,
                 stop_size: float = 0.01, *, region: Region | None = None, mask="breast", window=None,
                 interpolation: str = "linear", tree: bool = True):
        _check_interpolation(interpolation)
        if not stop_size > 0:
            raise ValueError("stop_size must be > 0")
        if not 1 <= n_sub <= 64:
            raise ValueError("n_sub must be in [1, 64]")
        dev = dv.device()
        grid, region = as_grid(grid), as_region(region)
        self.grid = grid
        self.kind = _kind(kind)
        self.kcode = _kind_code(kind)
        self.n_sub = int(n_sub)
        self.region = grid.full_region() if region is None else region
        if not grid.full_region().contains_region(self.region):
            raise ValueError("region lies outside the grid")
        self.stop_cells = max(1, int(math.floor(stop_size / grid.resolution + 1e-9)))
        self.n_iter = max_iterations(self.region, self.stop_cells)
        if self.n_iter > nat.SEG_MAX_ITERS:
            raise ValueError("stop_size too small for the segment trace")
        self.interp = nat.INTERP[interpolation]
        self.n_samples = int(n_samples)
        self.ld = dv.round4(n_samples)
        self.k0, self.w = _window(self.n_samples, window)
        if self.w == 0:
            raise ValueError("the segmentation metric needs a non-empty energy window")
        pairs = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
        self.scan = dv.DeviceScan(
            sig=torch.empty(0, device=dev),
            chan=torch.from_numpy(pairs).to(dev),
            ant=torch.from_numpy(np.array(geometry.antennas, dtype=np.float64)).to(dev),
            inv_scale=1.0 / (float(geometry.propagation_speed) * float(geometry.sample_interval)),
            n_samples=self.n_samples, ld=self.ld, n_ant=geometry.n_antennas, chan_host=pairs)
        self.mask_np, self.mask_t, mkey = _mask_for(grid, mask)
        self._ws = None
        # region tree plan (search-node points/tables, terminal-node cells/tables),
        # unless the tree is too large: then every iteration builds its own table
        self.plan = None
        self.fine_tps = 0
        if tree:
            ent = _tree_plan(self.scan, geometry.antennas, grid, self.region, mkey, self.mask_t, self.n_sub,
                             self.stop_cells, self.n_iter, self.interp)
            if ent is not None:
                self.plan, self.fine_tps = ent

    @property
    def n_chan(self) -> int:
        return self.scan.n_chan

    def run(self, sig: torch.Tensor) -> SegmentBatchResult:
        """Segment S device-resident scans (S, C, ld) fp32."""
        s_n = int(sig.shape[0])
        if sig.dtype != torch.float32 or sig.shape[1:] != (self.n_chan, self.ld) or not sig.is_contiguous():
            raise ValueError(f"sig must be contiguous float32 (S, {self.n_chan}, {self.ld})")
        if s_n == 0 or s_n > 65535:
            raise ValueError("batch size must be in [1, 65535]")
        grid = self.grid
        nx, ny = grid.dims
        dev = dv.device()
        lib = nat.load()
        stream = dv.stream_handle()
        sc = self.scan
        n_low = (2 * self.n_sub) ** 2
        if self.plan is not None:
            ws_bytes = int(lib.mwb_segment_run_workspace_bytes(s_n, self.n_sub, self.fine_tps, self.w))
        else:
            ws_bytes = int(lib.mwb_segment_batch_workspace_bytes(s_n, self.n_sub, self.n_chan))
        if self._ws is None or self._ws.numel() < ws_bytes:
            self._ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        regions = torch.empty((s_n, 6), dtype=torch.int32, device=dev)
        traces = torch.empty(s_n * nat.SEG_TRACE_BYTES, dtype=torch.uint8, device=dev)
        lowres = torch.zeros((s_n, n_low), dtype=torch.float32, device=dev)
        dense = torch.empty((s_n, nx * ny), dtype=torch.float32, device=dev)
        keys = torch.zeros(s_n, dtype=torch.int64, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        das = self.kcode == nat.MWB_DAS
        x0, y0, x1, y1 = self.region.bounds()
        if self.plan is not None:
            return self._run_tree(sig, regions, traces, lowres, dense, keys, flags)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        nat.call("mwb_segment_batch", sig.data_ptr(), s_n, self.n_chan * self.ld, self.n_chan, self.ld,
                 self.n_samples, sc.chan.data_ptr(), sc.ant.data_ptr(), sc.n_ant, sc.inv_scale, self.interp, self.k0,
                 self.w, self.kcode, grid.origin[0], grid.origin[1], grid.resolution, nx, ny, x0, y0, x1, y1,
                 self.n_sub, self.stop_cells, self.n_iter, regions.data_ptr(), lowres.data_ptr(), traces.data_ptr(),
                 self._ws.data_ptr(), stream)
        ev[1].record()
        # fine pass over every scan's final segment: one packed list
        rws = torch.empty(int(lib.mwb_regions_workspace_bytes(s_n)), dtype=torch.uint8, device=dev)
        totals = torch.zeros(2, dtype=torch.int32, device=dev)
        mask_p = self.mask_t.data_ptr() if self.mask_t is not None else None
        nat.call("mwb_enumerate_regions_count", nx, ny, regions.data_ptr(), s_n, mask_p, 0, totals.data_ptr(),
                 rws.data_ptr(), stream)
        n_pts, n_tiles = (int(v) for v in totals.cpu().tolist())  # the one host sync: packed list size
        if n_pts > 0:
            f_pts = torch.empty((n_pts, 3), dtype=torch.float64, device=dev)
            f_idx = torch.empty(n_pts, dtype=torch.int32, device=dev)
            tile_info = torch.empty((n_tiles, 2), dtype=torch.int32, device=dev)
            nat.call("mwb_enumerate_regions_write", grid.origin[0], grid.origin[1], grid.resolution, nx, ny,
                     regions.data_ptr(), s_n, mask_p, 0, f_pts.data_ptr(), f_idx.data_ptr(), tile_info.data_ptr(),
                     rws.data_ptr(), stream)
            f_table = torch.empty(int(lib.mwb_delay_table_bytes(n_pts, self.n_chan)), dtype=torch.uint8, device=dev)
            nat.call("mwb_delay_table_tiles", f_pts.data_ptr(), n_pts, tile_info.data_ptr(), sc.chan.data_ptr(),
                     self.n_chan, sc.ant.data_ptr(), sc.n_ant, sc.inv_scale, self.interp, f_table.data_ptr(), stream)
            nat.call("mwb_energies_tiles", sig.data_ptr(), s_n, self.n_chan * self.ld, self.n_chan, self.ld,
                     self.n_samples, sc.chan.data_ptr(), sc.ant.data_ptr(), sc.n_ant, sc.inv_scale,
                     f_pts.data_ptr(), f_idx.data_ptr(), n_pts, tile_info.data_ptr(), f_table.data_ptr(),
                     self.interp, self.k0, self.w, dense.data_ptr() if das else None,
                     None if das else dense.data_ptr(), nx * ny, keys.data_ptr() if das else None,
                     None if das else keys.data_ptr(), flags.data_ptr(), 0, stream)
        ev[2].record()
        return self._result(s_n, rws.view(torch.int32)[:s_n], flags, regions, keys, traces, lowres, dense, ev)

    def _run_tree(self, sig, regions, traces, lowres, dense, keys, flags) -> SegmentBatchResult:
        s_n = int(sig.shape[0])
        grid = self.grid
        nx, ny = grid.dims
        sc = self.scan
        x0, y0, x1, y1 = self.region.bounds()
        counts = torch.empty(s_n, dtype=torch.int32, device=dv.device())
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        nat.call("mwb_segment_run", self.plan.data_ptr(), sig.data_ptr(), s_n, self.n_chan * self.ld, self.n_chan,
                 self.ld, self.n_samples, sc.chan.data_ptr(), sc.ant.data_ptr(), sc.n_ant, sc.inv_scale, self.interp,
                 self.k0, self.w, self.kcode, nx, ny, x0, y0, x1, y1, self.n_sub, self.stop_cells, self.n_iter,
                 regions.data_ptr(), lowres.data_ptr(), traces.data_ptr(), dense.data_ptr(), nx * ny,
                 keys.data_ptr(), counts.data_ptr(), flags.data_ptr(), self._ws.data_ptr(), dv.stream_handle())
        ev[1].record()
        return self._result(s_n, counts, flags, regions, keys, traces, lowres, dense, ev)

    def _result(self, s_n, counts_t, flags, regions, keys, traces, lowres, dense, ev) -> SegmentBatchResult:
        grid = self.grid
        nx, ny = grid.dims
        fine_counts, st, reg, k, n_rec = dv.to_host(counts_t, flags, regions, keys,
                                                     traces.view(s_n, -1)[:, :4].contiguous().view(torch.int32))
        if int(st[0]) & 1:
            raise ValueError("energy map contains non-finite values")
        fine_counts = fine_counts.astype(np.int64)
        k = k.view(np.uint64)
        slot = (0xFFFFFFFF - (k & np.uint64(0xFFFFFFFF))).astype(np.int64)
        cells = np.stack([slot // ny, slot % ny], axis=1)
        none = k == 0  # an empty final segment: segment() reports its first cell
        cells[none] = reg[none][:, [0, 1]]
        iters = n_rec.reshape(s_n).astype(np.int64)
        EVAL_COUNTER.add(int(fine_counts.sum()) + 4 * self.n_sub * self.n_sub * int(iters.sum()))
        full_eq = int(self.mask_np.sum()) if self.mask_np is not None else nx * ny
        if len(ev) == 3:
            elapsed = {"search": ev[0].elapsed_time(ev[1]) / 1e3, "fine": ev[1].elapsed_time(ev[2]) / 1e3}
            elapsed["total"] = elapsed["search"] + elapsed["fine"]
        else:  # tree plan: search and fine pass in one call
            elapsed = {"total": ev[0].elapsed_time(ev[1]) / 1e3}
        return SegmentBatchResult(
            grid=grid, kind=self.kind.value, n_sub=self.n_sub, final_regions=reg[:, [0, 1, 3, 4]],
            argmax_cells=cells, iterations=iters, fine_points_evaluated=fine_counts, full_equivalent_points=full_eq,
            dense=dense.view(s_n, nx, ny), lowres=lowres.view(s_n, 2 * self.n_sub, 2 * self.n_sub), elapsed=elapsed,
            _traces=traces, _mask=self.mask_np)
