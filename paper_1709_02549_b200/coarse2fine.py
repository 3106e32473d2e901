"""Coarse-to-fine segment-selection framework, device resident.

Drop-in for /root/reference/pkg/src/mwbeam/coarse2fine.py:

* ``run_framework`` (coarse2fine.py:301-350): coarse lattice pass -> device
  ``select_roi`` kernel -> fine pass over the ROI read from device memory ->
  composite argmax fused into the energy epilogue.  One host synchronisation,
  at the end, to fetch the map, the trace and the counters.
* ``select_roi`` (coarse2fine.py:169-256) on any ``EnergyMap``: uploads the map
  and runs the same device kernel.
* ``consistency_check`` (coarse2fine.py:353-402), ``breast_mask`` (259-268),
  ``decision_metric`` / ``class_distances`` (67-109), ``Manual`` /
  ``Automatic`` / ``auto_decimation_factor`` (24-64), ``FrameworkConfig``,
  ``IterationRecord``, ``MetricTrace``, ``FrameworkReport``, ``CheckVerdict``
  with the reference's fields and ``to_dict`` keys.

``elapsed`` timings are CUDA-event device times of the three phases.
"""

from __future__ import annotations

import ctypes
import functools

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from . import _native as nat
from .beamform import (
    EVAL_COUNTER,
    BeamformerKind,  # re-exported, as the reference's coarse2fine namespace has it
    EnergyMap,
    _check_interpolation,
    _kind_code,
    _Status,
    _window,
    build_table,
    launch_energies,
)
from .geometry import ImagingGrid, Region, as_grid, as_region


@dataclass(frozen=True)
class Manual:
    """Fixed spatial decimation factor."""

    factor: int

    def __post_init__(self):
        if self.factor < 1:
            raise ValueError("manual decimation factor must be >= 1")


@dataclass(frozen=True)
class Automatic:
    """Decimation derived from the smallest tumour diameter to detect."""

    min_tumor_diameter: float

    def __post_init__(self):
        if not self.min_tumor_diameter > 0:
            raise ValueError("min_tumor_diameter must be > 0")


DecimationMode = Manual | Automatic


def auto_decimation_factor(min_tumor_diameter: float, resolution: float) -> int:
    """Largest stride that keeps a coarse point inside the inscribed square
    (side d/sqrt 2) of any tumour of diameter d (coarse2fine.py:49-58)."""
    if not (min_tumor_diameter > 0 and resolution > 0):
        raise ValueError("min_tumor_diameter and resolution must be > 0")
    return max(1, math.floor((min_tumor_diameter / math.sqrt(2.0)) / resolution))


def decimation_factor(mode, resolution: float) -> int:
    if isinstance(mode, Manual) or hasattr(mode, "factor"):
        return int(mode.factor)
    return auto_decimation_factor(mode.min_tumor_diameter, resolution)


def _mean_var_parts(vals: np.ndarray, sigma_prev_sq: float) -> tuple[float, dict]:
    if vals.size == 0:
        raise ValueError("decision_metric needs a nonempty value set")
    mu = float(vals.mean())
    var = float(vals.var())
    if var == 0.0:
        return mu, {"mu": mu, "var": var, "delta_raw": 0.0, "delta": 0.0, "clamped": False}
    raw = (var - sigma_prev_sq) / var
    delta = min(max(raw, 0.0), 1.0)
    return (1.0 - delta) * mu + delta * var, {
        "mu": mu,
        "var": var,
        "delta_raw": raw,
        "delta": delta,
        "clamped": delta != raw,
    }


def decision_metric(energies_current, sigma_prev_sq: float) -> float:
    """Eq. (5): (1-Δ)μ + Δσ², Δ = clamp((σ² − σ²_prev)/σ², 0, 1); σ² = 0 -> μ."""
    value, _ = _mean_var_parts(np.asarray(energies_current, dtype=np.float64), sigma_prev_sq)
    return value


def class_distances(class_a, class_b) -> tuple[float, float]:
    """Eqs. (6)-(7) for scalar energies: within-class W and between-class B."""
    a = np.asarray(class_a, dtype=np.float64)
    b = np.asarray(class_b, dtype=np.float64)
    if a.size == 0 or b.size == 0:
        raise ValueError("class_distances needs nonempty classes")
    ma, mb = a.mean(), b.mean()
    w = float(((a - ma) ** 2).sum() + ((b - mb) ** 2).sum())
    g = np.concatenate([a, b]).mean()
    return w, float(a.size * (ma - g) ** 2 + b.size * (mb - g) ** 2)


@dataclass(frozen=True)
class FrameworkConfig:
    frame_fraction: float = 0.25
    n_min: int = 4
    min_tumor_diameter: float = 0.01

    def __post_init__(self):
        if not 0.0 <= self.frame_fraction < 1.0:
            raise ValueError("frame_fraction must be in [0, 1)")
        if self.n_min < 1:
            raise ValueError("n_min must be >= 1")
        if not self.min_tumor_diameter > 0:
            raise ValueError("min_tumor_diameter must be > 0")


@dataclass
class IterationRecord:
    iteration: int
    quadrant_counts: list[int]
    scores: list[float]
    stats: list[dict | None]
    selected: int
    selected_region: Region
    expanded_region: Region
    w: float
    b: float
    satisfied: bool

    def to_dict(self) -> dict:
        return {
            "iteration": self.iteration,
            "quadrant_counts": self.quadrant_counts,
            "scores": self.scores,
            "stats": self.stats,
            "selected": self.selected,
            "selected_region": self.selected_region.to_dict(),
            "expanded_region": self.expanded_region.to_dict(),
            "W": self.w,
            "B": self.b,
            "satisfied": self.satisfied,
        }


@dataclass
class MetricTrace:
    records: list[IterationRecord] = field(default_factory=list)
    termination: str = ""
    warning: str | None = None

    def to_dict(self) -> dict:
        return {
            "records": [r.to_dict() for r in self.records],
            "termination": self.termination,
            "warning": self.warning,
        }


def breast_mask(grid: ImagingGrid) -> np.ndarray:
    """Cells whose centres lie in the circle inscribed in the grid (coarse2fine.py:259-268)."""
    grid = as_grid(grid)
    nx, ny = grid.dims
    cx, cy = grid.center()
    radius = min(nx, ny) * grid.resolution / 2.0
    px = grid.origin[0] + (np.arange(nx) + 0.5) * grid.resolution
    py = grid.origin[1] + (np.arange(ny) + 0.5) * grid.resolution
    return (px[:, None] - cx) ** 2 + (py[None, :] - cy) ** 2 <= radius**2


_MASKS: dict[tuple, tuple[np.ndarray, torch.Tensor]] = {}


def _breast_mask_device(grid: ImagingGrid) -> tuple[np.ndarray, torch.Tensor]:
    key = (grid.origin, grid.extent, grid.resolution, torch.cuda.current_device())
    hit = _MASKS.get(key)
    if hit is None:
        m = breast_mask(grid)
        hit = (m, dv.upload_mask(m, grid.dims))
        if len(_MASKS) > 64:
            _MASKS.clear()
        _MASKS[key] = hit
    return hit


@dataclass
class FrameworkReport:
    decimation_factor: int
    iterations: int
    final_region: Region
    coarse_points_evaluated: int
    fine_points_evaluated: int
    full_equivalent_points: int
    reduction_ratio: float
    elapsed: dict[str, float]
    trace: MetricTrace
    argmax_cell: tuple[int, int]
    argmax_position: tuple[float, float]

    def to_dict(self) -> dict:
        return {
            "decimation_factor": self.decimation_factor,
            "iterations": self.iterations,
            "final_region": self.final_region.to_dict(),
            "coarse_points_evaluated": self.coarse_points_evaluated,
            "fine_points_evaluated": self.fine_points_evaluated,
            "full_equivalent_points": self.full_equivalent_points,
            "reduction_ratio": self.reduction_ratio,
            "elapsed": self.elapsed,
            "trace": self.trace.to_dict(),
            "argmax_cell": list(self.argmax_cell),
            "argmax_position": list(self.argmax_position),
        }


# ---------------------------------------------------------------------------
# trace decoding
# ---------------------------------------------------------------------------
def _region(b) -> Region:
    """2-D Region from a device box {x0, y0, z0, x1, y1, z1}."""
    return Region((int(b[0]), int(b[1])), (int(b[3]), int(b[4])))


class _DeviceTrace(MetricTrace):
    """A MetricTrace whose records are decoded from the device trace's bytes on
    first access.  run_framework's latency path reads only the termination
    and the final region; building ~7 records of Python objects per call
    (~60 us) is deferred until someone looks at them."""

    def __init__(self, raw_records: bytes, n: int, termination: str, warning, region):
        self._raw, self._n, self._region, self._records = raw_records, n, region, None
        self.termination, self.warning = termination, warning

    @property
    def records(self) -> list:
        if self._records is None:
            recs = (nat.IterRecord * self._n).from_buffer_copy(self._raw) if self._n else []
            self._records = [_record(recs[i], self._region) for i in range(self._n)]
        return self._records

    @records.setter
    def records(self, value) -> None:
        self._records = list(value)

    @property
    def n_records(self) -> int:
        return self._n if self._records is None else len(self._records)

    def __eq__(self, other) -> bool:
        if not isinstance(other, MetricTrace):
            return NotImplemented
        return (self.records, self.termination, self.warning) == (other.records, other.termination, other.warning)

    __hash__ = None


def _record(r, region) -> IterationRecord:
    stats: list[dict | None] = []
    nk = int(r.n_children)
    for k in range(nk):
        h = int(r.has_stats[k])
        if h == 0:
            stats.append(None)
        elif h == 1:
            stats.append({"mu": float(r.mu[k]), "var": float(r.var[k])})
        else:
            stats.append({
                "mu": float(r.mu[k]),
                "var": float(r.var[k]),
                "delta_raw": float(r.delta_raw[k]),
                "delta": float(r.delta[k]),
                "clamped": bool(r.clamped[k]),
            })
    return IterationRecord(
        iteration=int(r.iteration),
        quadrant_counts=[int(c) for c in r.counts[:nk]],
        scores=[float(x) for x in r.scores[:nk]],
        stats=stats,
        selected=int(r.selected),
        selected_region=region(r.selected_region),
        expanded_region=region(r.expanded_region),
        w=float(r.w),
        b=float(r.b),
        satisfied=bool(r.satisfied),
    )


_REC_OFFSET = None


def decode_trace_lazy(raw: np.ndarray, region=_region) -> tuple[Region, MetricTrace, int]:
    """decode_trace with the records deferred (_DeviceTrace): reads the header
    (termination, record count, final box) now and copies only the used
    records' bytes, so the source buffer may be reused at once."""
    import ctypes

    global _REC_OFFSET
    if _REC_OFFSET is None:
        _REC_OFFSET = nat.Trace.records.offset
    head = np.frombuffer(raw, dtype=np.int32, count=8)
    code, n = int(head[0]), int(head[1])
    if code == -1:
        raise ValueError("coarse map has no entries in the breast region")
    if code == -2:
        raise RuntimeError(f"select_roi exceeded {nat.MAX_ITERS} iterations")
    n = min(n, nat.MAX_ITERS)
    size = ctypes.sizeof(nat.IterRecord)
    body = bytes(memoryview(raw)[_REC_OFFSET: _REC_OFFSET + n * size])
    warning = "energy map has no discriminating signal" if code == 1 else None
    return region(head[2:8]), _DeviceTrace(body, n, nat.TERMINATION[code], warning, region), code


def decode_trace(raw, region=_region) -> tuple[Region, MetricTrace, int]:
    """Device trace (bytes, or a writable uint8 array decoded in place) ->
    (final region, MetricTrace, termination code); ``region`` converts a device
    box (2-D Region by default, volume.Box for 3-D)."""
    tr = nat.Trace.from_buffer_copy(raw) if isinstance(raw, (bytes, bytearray)) else nat.Trace.from_buffer(raw)
    code = int(tr.termination)
    if code == -1:
        raise ValueError("coarse map has no entries in the breast region")
    if code == -2:
        raise RuntimeError(f"select_roi exceeded {nat.MAX_ITERS} iterations")
    trace = MetricTrace()
    trace.termination = nat.TERMINATION[code]
    if code == 1:
        trace.warning = "energy map has no discriminating signal"
    for i in range(int(tr.n_records)):
        trace.records.append(_record(tr.records[i], region))
    return region(tr.final_region), trace, code


def _launch_select(dense: torch.Tensor, valid: torch.Tensor, grid: ImagingGrid, lattice: int, breast: Region,
                   cfg: FrameworkConfig, region_out: torch.Tensor, trace_buf: torch.Tensor) -> None:
    nx, ny = grid.dims
    x0, y0, x1, y1 = breast.bounds()
    nat.call("mwb_select_roi", dense.data_ptr(), valid.data_ptr(), nx, ny, lattice, x0, y0, x1, y1,
             float(cfg.frame_fraction), int(cfg.n_min), region_out.data_ptr(), trace_buf.data_ptr(),
             dv.stream_handle())


def select_roi(coarse: EnergyMap, breast_region: Region, cfg: FrameworkConfig = FrameworkConfig()) -> tuple[Region, MetricTrace]:
    """Iterative quadrant selection (coarse2fine.py:169-256), run by the device kernel."""
    grid = as_grid(coarse.grid)
    breast_region = as_region(breast_region)
    nx, ny = grid.dims
    if not grid.full_region().contains_region(breast_region):
        raise ValueError("breast region lies outside the grid")
    if getattr(coarse, "_entries", True) is None:  # dense-backed map from this package
        vals, valid = coarse._values.astype(np.float32), coarse._valid
    else:  # dict-backed (this package's or the reference's EnergyMap)
        vals = np.zeros((nx, ny), dtype=np.float32)
        valid = np.zeros((nx, ny), dtype=bool)
        for (ix, iy), v in coarse.entries.items():
            if 0 <= ix < nx and 0 <= iy < ny:
                vals[ix, iy] = v
                valid[ix, iy] = True
    (x0, y0), (x1, y1) = breast_region.min_cell, breast_region.max_cell
    if not valid[x0 : x1 + 1, y0 : y1 + 1].any():
        raise ValueError("coarse map has no entries in the breast region")
    d = max(1, int(coarse.stride))
    ix, iy = np.nonzero(valid)
    lattice = d if (d > 1 and not ((ix % d).any() or (iy % d).any())) else 1
    dev = dv.device()
    dense_t = torch.from_numpy(np.ascontiguousarray(vals).reshape(-1)).to(dev)
    valid_t = torch.from_numpy(np.ascontiguousarray(valid).view(np.uint8).reshape(-1)).to(dev)
    region_t = torch.zeros(6, dtype=torch.int32, device=dev)
    trace_t = torch.zeros(nat.TRACE_BYTES, dtype=torch.uint8, device=dev)
    _launch_select(dense_t, valid_t, grid, lattice, breast_region, cfg, region_t, trace_t)
    final, trace, _ = decode_trace(trace_t.cpu().numpy().tobytes())
    return final, trace


class _FrameworkPlan(dv.GraphPlan):
    """One framework configuration for one scanner geometry, captured as a CUDA graph.

    The coarse energy pass (its lattice and delay table are built once per
    plan), the select kernel and the ROI-driven fine pass are enqueued once
    eagerly, then captured; later
    calls replay the graph and read the results back into pinned buffers with
    a single synchronisation.  Buffers persist with the plan, so a replay
    allocates nothing.  The graph reads the plan's own signal slot: each call
    first copies its scan into the slot (device to device), so a stream of
    different scans of one geometry replays one graph.
    """

    def __init__(self, scan: dv.DeviceScan, grid: ImagingGrid, d: int, kcode: int, cfg: FrameworkConfig,
                 interp: int, k0: int, w: int, mode: int):
        scan = self._init_slot(scan)
        self.scan, self.grid, self.d, self.kcode, self.cfg = scan, grid, d, kcode, cfg
        self.interp, self.k0, self.w, self.mode = interp, k0, w, mode
        nx, ny = grid.dims
        self.mask_np, self.mask_t = _breast_mask_device(grid)
        self.full_equivalent = int(self.mask_np.sum())  # the report's full-resolution cell count (fixed per plan)
        dev = dv.device()
        # The kernels write a dense map and its valid mask; what a call reads
        # back is one result block [status | trace | compact values], the
        # compact values being the coarse lattice's followed by the final
        # ROI rectangle's, row by row (mwb_gather_composite): a few KB instead
        # of the whole map.  One copy per call into a fresh pinned block that
        # the returned map keeps; the host rebuilds the dense arrays only when
        # the map is first read (EnergyMap._from_loader).
        n = nx * ny
        self.dense = torch.empty(n, dtype=torch.float32, device=dev)  # only valid cells are read
        self.valid = torch.empty(n, dtype=torch.uint8, device=dev)
        self._o_trace = _Status.BYTES
        self._o_vals = (self._o_trace + nat.TRACE_BYTES + 15) // 16 * 16
        self._res_full = self._o_vals  # + 4 * (n_coarse + n), set below
        self.region_t = torch.empty(6, dtype=torch.int32, device=dev)
        # external events become timestamp nodes inside the captured graph
        self.events = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]
        self._ev_handles = None  # raw cudaEvent_t array for mwb_elapsed_ms (after the first record)
        self._ms = (ctypes.c_float * 3)()
        self._pin = torch.cuda.is_available()
        self.replays = 0
        # The coarse lattice and its delay table depend on the geometry, grid
        # and mask only: enumerated and tabled once here, outside the graph,
        # which then holds just the coarse energy launch.
        p_max = ((nx + d - 1) // d) * ((ny + d - 1) // d)
        self.c_pts = torch.empty((p_max, 3), dtype=torch.float64, device=dev)
        self.c_oidx = torch.empty(p_max, dtype=torch.int32, device=dev)
        self.c_valid = torch.zeros(nx * ny, dtype=torch.uint8, device=dev)
        self.c_count = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = torch.empty(int(nat.load().mwb_lattice_workspace_bytes(nx, ny, d)), dtype=torch.uint8, device=dev)
        nat.call("mwb_enumerate_lattice", grid.origin[0], grid.origin[1], grid.resolution, nx, ny, 0, 0, nx - 1,
                 ny - 1, None, d, self.mask_t.data_ptr(), 0, self.c_pts.data_ptr(), self.c_oidx.data_ptr(),
                 self.c_count.data_ptr(), self.c_valid.data_ptr(), ws.data_ptr(), dv.stream_handle())
        self.c_table = build_table(scan, self.c_pts, p_max, interp, self.c_count.data_ptr())
        self.n_coarse = int(self.c_count.item())
        self.c_slots = self.c_oidx[: self.n_coarse].clone()
        self.c_slots_host = self.c_slots.cpu().numpy()
        self.c_valid_host = self.c_valid.cpu().numpy().view(bool).reshape(nx, ny)
        self.lattice_host = np.zeros((nx, ny), dtype=bool)
        self.lattice_host[::d, ::d] = True
        # result block: device copy sized for the worst case (a degenerate run's
        # whole-grid ROI); a call copies the coarse values and ROI_BUDGET ROI
        # cells, and a second copy only when the ROI is larger
        cap = self.n_coarse + nx * ny
        self._res_full = self._o_vals + 4 * cap
        self._res_copy = self._o_vals + 4 * min(cap, self.n_coarse + self.ROI_BUDGET)
        self.res = torch.empty(self._res_full, dtype=torch.uint8, device=dev)
        self.status = _Status(self.res)
        self.trace_t = self.res[self._o_trace: self._o_trace + nat.TRACE_BYTES]
        self.compact = self.res[self._o_vals:].view(torch.float32)
        # Fine pass: every masked cell of the grid in the padded 16 x 16 tile
        # layout with its delay table, also built once here; each call's fine
        # launch (mwb_energies_region) evaluates just the tiles that meet the
        # ROI the select kernel left on the device, writing the ROI's
        # non-coarse cells.  No per-call enumeration, table or host sync.
        lib = nat.load()
        tiles = int(lib.mwb_lattice_tile_count(nx, ny, 1))
        self.f_n = 256 * tiles
        self.f_pts = torch.zeros((self.f_n, 3), dtype=torch.float64, device=dev)
        self.f_oidx = torch.zeros(self.f_n, dtype=torch.int32, device=dev)
        self.f_info = torch.zeros((tiles, 2), dtype=torch.int32, device=dev)
        f_count = torch.zeros(1, dtype=torch.int32, device=dev)
        f_valid = torch.zeros(nx * ny, dtype=torch.uint8, device=dev)
        ws = torch.empty(int(lib.mwb_lattice_workspace_bytes(nx, ny, 1)), dtype=torch.uint8, device=dev)
        nat.call("mwb_enumerate_lattice_padded", grid.origin[0], grid.origin[1], grid.resolution, nx, ny, 0, 0,
                 nx - 1, ny - 1, 1, self.mask_t.data_ptr(), 0, self.f_pts.data_ptr(), self.f_oidx.data_ptr(),
                 self.f_info.data_ptr(), f_count.data_ptr(), f_valid.data_ptr(), ws.data_ptr(), dv.stream_handle())
        self.f_table = torch.empty(int(lib.mwb_delay_table_bytes(self.f_n, scan.n_chan)), dtype=torch.uint8,
                                   device=dev)
        nat.call("mwb_delay_table_tiles", self.f_pts.data_ptr(), self.f_n, self.f_info.data_ptr(),
                 scan.chan.data_ptr(), scan.n_chan, scan.ant.data_ptr(), scan.n_ant, scan.inv_scale, interp,
                 self.f_table.data_ptr(), dv.stream_handle())
        # window-split partials for long windows (the reference's full record)
        need = int(lib.mwb_energies_split_bytes(self.f_n, 1, w)) if w > 48 else 0
        self.f_ws = torch.empty(need, dtype=torch.uint8, device=dev) if 0 < need <= (256 << 20) else None

    def _enqueue(self) -> None:
        g, d = self.grid, self.d
        ev = self.events
        self.valid.copy_(self.c_valid)
        self.status.t.zero_()
        st = self.status
        ev[0].record()
        launch_energies(self.scan, self.c_pts, self.c_pts.shape[0], self.c_table, self.interp, self.k0, self.w,
                        self.dense if self.kcode == nat.MWB_DAS else None,
                        self.dense if self.kcode == nat.MWB_DMAS else None, 0, self.c_oidx, self.c_count.data_ptr(),
                        st.key_ptr(0), st.key_ptr(1), st.flags_ptr, self.mode)
        ev[1].record()
        _launch_select(self.dense, self.valid, g, d, g.full_region(), self.cfg, self.region_t, self.trace_t)
        ev[2].record()
        sc, das = self.scan, self.kcode == nat.MWB_DAS
        nat.call("mwb_energies_region", sc.sig.data_ptr(), sc.n_chan, sc.ld, sc.n_samples, sc.chan.data_ptr(),
                 sc.ant.data_ptr(), sc.n_ant, sc.inv_scale, self.f_pts.data_ptr(), self.f_oidx.data_ptr(), self.f_n,
                 self.f_info.data_ptr(), self.f_table.data_ptr(), self.interp, self.k0, self.w,
                 self.dense.data_ptr() if das else None, None if das else self.dense.data_ptr(),
                 st.key_ptr(0), st.key_ptr(1), st.flags_ptr, self.region_t.data_ptr(), g.dims[1], d,
                 self.valid.data_ptr(), st.count_ptr(1), self.mode, nat.ptr(self.f_ws),
                 0 if self.f_ws is None else self.f_ws.numel(), dv.stream_handle())
        ev[3].record()
        nat.call("mwb_gather_composite", self.dense.data_ptr(), g.dims[1], 1, self.c_slots.data_ptr(), self.n_coarse,
                 self.region_t.data_ptr(), self.compact.data_ptr(), self.compact.numel(), dv.stream_handle())

    ROI_BUDGET = 16384  # ROI cells read back with the result block (64 KB)

    def _dense_arrays(self, comp: np.ndarray, final: Region) -> tuple[np.ndarray, np.ndarray]:
        """(values, valid) of a composite from its compact readback: coarse
        lattice cells from their fixed slots, fine cells = the ROI's masked
        non-lattice cells (the fine pass's filter, mwb_energies_region)."""
        nx, ny = self.grid.dims
        (x0, y0), (x1, y1) = final.min_cell, final.max_cell
        vals = np.zeros(nx * ny, dtype=np.float32)
        vals[self.c_slots_host] = comp[: self.n_coarse]
        vals = vals.reshape(nx, ny)
        valid = self.c_valid_host.copy()
        fine = self.mask_np[x0: x1 + 1, y0: y1 + 1] & ~self.lattice_host[x0: x1 + 1, y0: y1 + 1]
        block = comp[self.n_coarse:].reshape(x1 - x0 + 1, y1 - y0 + 1)
        vals[x0: x1 + 1, y0: y1 + 1][fine] = block[fine]
        valid[x0: x1 + 1, y0: y1 + 1] |= fine
        return vals, valid

    def launch(self, scan: dv.DeviceScan) -> None:
        """Enqueue one run on ``scan`` (graph replay after the first call) and the readback."""
        self.replay(scan)
        self.replays += 1
        self.h_res = torch.empty(self._res_copy, dtype=torch.uint8, pin_memory=self._pin)
        nat.call("mwb_memcpy_async", self.h_res.data_ptr(), self.res.data_ptr(), self._res_copy,
                 dv.stream_handle())

    def finish(self) -> tuple[EnergyMap, FrameworkReport]:
        dv.sync_stream()
        nx, ny = self.grid.dims
        blk = self.h_res.numpy()
        h = blk[: _Status.BYTES].view(np.int64)
        keys = h[:2].view(np.uint64)
        tail = h[2:].view(np.int32)
        counts, flags = tail[:2], int(tail[2])
        if flags & 1:
            raise ValueError("energy map contains non-finite values")
        final, trace, _ = decode_trace_lazy(blk[self._o_trace: self._o_trace + nat.TRACE_BYTES])
        n_coarse, n_fine = self.n_coarse, int(counts[1])
        EVAL_COUNTER.add(n_coarse)
        EVAL_COUNTER.add(n_fine)
        (x0, y0), (x1, y1) = final.min_cell, final.max_cell
        used = self._o_vals + 4 * (self.n_coarse + (x1 - x0 + 1) * (y1 - y0 + 1))
        if used > self._res_copy:  # ROI beyond the budget: copy the whole used block again
            self.h_res = torch.empty(used, dtype=torch.uint8, pin_memory=self._pin)
            nat.call("mwb_memcpy_async", self.h_res.data_ptr(), self.res.data_ptr(), used, dv.stream_handle())
            dv.sync_stream()
            blk = self.h_res.numpy()
        comp = blk[self._o_vals: used].view(np.float32)
        composite = EnergyMap._from_loader(self.grid, functools.partial(self._dense_arrays, comp, final),
                                           stride=self.d, roi=final, split=self.d)
        if self._ev_handles is None:
            self._ev_handles = (ctypes.c_void_p * 4)(*[e.cuda_event for e in self.events])
        nat.call("mwb_elapsed_ms", self._ev_handles, 4, self._ms)
        t_c, t_s, t_f = (self._ms[i] / 1e3 for i in range(3))
        full_equivalent = self.full_equivalent
        key = int(keys[0 if self.kcode == nat.MWB_DAS else 1])
        slot = 0xFFFFFFFF - (key & 0xFFFFFFFF)
        cell = (slot // ny, slot % ny) if key != 0 else composite.argmax_cell()
        report = FrameworkReport(
            decimation_factor=self.d,
            iterations=trace.n_records,
            final_region=final,
            coarse_points_evaluated=n_coarse,
            fine_points_evaluated=n_fine,
            full_equivalent_points=full_equivalent,
            reduction_ratio=full_equivalent / (n_coarse + n_fine),
            elapsed={"coarse": t_c, "select": t_s, "fine": t_f, "total": t_c + t_s + t_f},
            trace=trace,
            argmax_cell=cell,
            argmax_position=self.grid.cell_center(*cell),
        )
        return composite, report


_PLANS: "OrderedDict[tuple, _FrameworkPlan]" = None  # type: ignore[assignment]
_PLAN_CAPACITY = 8


def _plan_for(ds, kind, grid: ImagingGrid, d: int, cfg: FrameworkConfig, interpolation: str, window,
              mode: int) -> tuple[_FrameworkPlan, dv.DeviceScan]:
    """Cached plan per scanner geometry and configuration (not per dataset: the
    plan's graph reads a signal slot that every call refills)."""
    global _PLANS
    from collections import OrderedDict

    if _PLANS is None:
        _PLANS = OrderedDict()
    scan = dv.scan_for(ds)
    k0, w = _window(scan.n_samples, window)
    kcode = _kind_code(kind)
    interp = nat.INTERP[interpolation]
    key = (scan.geometry_key(), grid.origin, grid.extent, grid.resolution, d, kcode, cfg.frame_fraction, cfg.n_min,
           interp, k0, w, mode)
    plan = _PLANS.get(key)
    if plan is not None:
        _PLANS.move_to_end(key)
        return plan, scan
    plan = _FrameworkPlan(scan, grid, d, kcode, cfg, interp, k0, w, mode)
    _PLANS[key] = plan
    while len(_PLANS) > _PLAN_CAPACITY:
        _PLANS.popitem(last=False)
    return plan, scan


def run_framework(
    ds,
    kind,
    grid: ImagingGrid,
    mode,
    cfg: FrameworkConfig = FrameworkConfig(),
    threads: int = 1,
    *,
    interpolation: str = "linear",
    window=None,
    kernel_mode: str = "smem",
) -> tuple[EnergyMap, FrameworkReport]:
    """Coarse pass, ROI selection, fine pass, composite (coarse2fine.py:301-350)."""
    _check_interpolation(interpolation)
    grid = as_grid(grid)
    d = decimation_factor(mode, grid.resolution)
    mask_np, _ = _breast_mask_device(grid)
    if not mask_np[::d, ::d].any():
        raise ValueError("no coarse focal points inside the breast mask")
    with dv.PLAN_LOCK:
        plan, scan = _plan_for(ds, kind, grid, d, cfg, interpolation, window,
                               {"smem": 0, "gather": 1}[kernel_mode])
        plan.launch(scan)
        return plan.finish()


@dataclass
class CheckVerdict:
    """Outcome of running the framework with two decimation factors."""

    confirmed: bool
    overlap: Region | None
    region_a: Region
    region_b: Region

    def to_dict(self) -> dict:
        return {
            "confirmed": self.confirmed,
            "overlap": self.overlap.to_dict() if self.overlap else None,
            "region_a": self.region_a.to_dict(),
            "region_b": self.region_b.to_dict(),
        }


def consistency_check(
    ds,
    kind,
    grid: ImagingGrid,
    d1: int,
    d2: int,
    cfg: FrameworkConfig = FrameworkConfig(),
    threads: int = 1,
) -> tuple[CheckVerdict, FrameworkReport, FrameworkReport]:
    """Confirmed when the final regions of two decimation factors overlap
    (coarse2fine.py:371-402).  Both runs are enqueued back to back on the
    stream before the single synchronisation."""
    grid = as_grid(grid)
    if d1 == d2:
        raise ValueError("consistency check needs two different decimation factors")
    limit = auto_decimation_factor(cfg.min_tumor_diameter, grid.resolution)
    for dd in (d1, d2):
        if dd < 1 or dd > limit:
            raise ValueError(f"decimation factor {dd} outside acceptable range [1, {limit}]")
    mask, _ = _breast_mask_device(grid)
    for dd in (d1, d2):
        if not mask[::dd, ::dd].any():
            raise ValueError("no coarse focal points inside the breast mask")
    with dv.PLAN_LOCK:
        plans = [_plan_for(ds, kind, grid, dd, cfg, "linear", None, 0) for dd in (d1, d2)]
        for plan, scan in plans:
            plan.launch(scan)  # both runs are in flight before the first readback
        (_, rep_a), (_, rep_b) = (plan.finish() for plan, _ in plans)
    inter = rep_a.final_region.intersection(rep_b.final_region)
    return CheckVerdict(inter is not None, inter, rep_a.final_region, rep_b.final_region), rep_a, rep_b
