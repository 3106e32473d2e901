"""3-D voxel imaging and octant segmentation (BASELINE configs[4]).

The reference images the z = 0 slice only (geometry.py:17-19; 3-D is a
non-goal).  Its kernel already takes the antenna z into the
distance, so a voxel (x, y, z) has exactly the energy the reference assigns
to (x, y) with every antenna shifted by -z (SURVEY.md §8c adapter 3).  The
same device kernels therefore serve volumes: points carry a real z, the
lattice enumerator walks 8x8x4 voxel tiles, and the device selection splits
boxes into octants (index = xhigh + 2*yhigh + 4*zhigh, low half gets the odd
cell per axis, exactly Region.quadrants' rule, geometry.py:225-242) and
scores them with the reference's Eq. (5) / W-B / n_min control flow
(coarse2fine.py:169-256).
"""

from __future__ import annotations

import ctypes
import functools
import hashlib
import math
import weakref
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from . import _native as nat
from .beamform import (_MATERIALISE, EVAL_COUNTER, _check_interpolation, _kind_code, _LatticeCache, _Status,
                       _window, build_table, launch_energies)
from .coarse2fine import (FrameworkConfig, IterationRecord, MetricTrace, decimation_factor, decode_trace,
                          decode_trace_lazy)


@dataclass(frozen=True)
class Box:
    """Inclusive voxel box."""

    min_cell: tuple[int, int, int]
    max_cell: tuple[int, int, int]

    def __post_init__(self):
        lo = tuple(int(v) for v in self.min_cell)
        hi = tuple(int(v) for v in self.max_cell)
        if len(lo) != 3 or len(hi) != 3 or any(a > b for a, b in zip(lo, hi)):
            raise ValueError("box bounds must be 3-vectors with min_cell <= max_cell")
        object.__setattr__(self, "min_cell", lo)
        object.__setattr__(self, "max_cell", hi)

    @property
    def shape(self) -> tuple[int, int, int]:
        return tuple(b - a + 1 for a, b in zip(self.min_cell, self.max_cell))

    @property
    def n_cells(self) -> int:
        w, h, d = self.shape
        return w * h * d

    def bounds(self) -> tuple[int, ...]:
        return (*self.min_cell, *self.max_cell)

    def contains_cell(self, ix: int, iy: int, iz: int) -> bool:
        return all(a <= v <= b for a, v, b in zip(self.min_cell, (ix, iy, iz), self.max_cell))

    def contains_box(self, other: "Box") -> bool:
        return self.contains_cell(*other.min_cell) and self.contains_cell(*other.max_cell)

    def intersection(self, other: "Box") -> "Box | None":
        lo = tuple(max(a, b) for a, b in zip(self.min_cell, other.min_cell))
        hi = tuple(min(a, b) for a, b in zip(self.max_cell, other.max_cell))
        if any(a > b for a, b in zip(lo, hi)):
            return None
        return Box(lo, hi)

    def octants(self) -> "list[Box] | None":
        """8 disjoint children, index = xhigh + 2*yhigh + 4*zhigh; None when a side is 1."""
        if min(self.shape) < 2:
            return None
        halves = []
        for a, (lo, hi) in enumerate(zip(self.min_cell, self.max_cell)):
            mid = lo + (hi - lo + 2) // 2 - 1
            halves.append(((lo, mid), (mid + 1, hi)))
        out = []
        for k in range(8):
            sel = [halves[a][(k >> a) & 1] for a in range(3)]
            out.append(Box(tuple(s[0] for s in sel), tuple(s[1] for s in sel)))
        return out

    def expand(self, fraction: float, clip_to: "Box") -> "Box":
        grow = [math.ceil(fraction * s) for s in self.shape]
        lo = tuple(max(a - g, c) for a, g, c in zip(self.min_cell, grow, clip_to.min_cell))
        hi = tuple(min(b + g, c) for b, g, c in zip(self.max_cell, grow, clip_to.max_cell))
        return Box(lo, hi)

    def to_dict(self) -> dict:
        return {"min_cell": list(self.min_cell), "max_cell": list(self.max_cell)}


def _box(b) -> Box:
    return Box((int(b[0]), int(b[1]), int(b[2])), (int(b[3]), int(b[4]), int(b[5])))


@dataclass(frozen=True)
class VolumeGrid:
    """Uniform voxel grid; voxel (ix, iy, iz) is centred at origin + (i + 0.5) * res."""

    origin: tuple[float, float, float]
    extent: tuple[float, float, float]
    resolution: float
    dims: tuple[int, int, int] = field(init=False)

    def __post_init__(self):
        if not self.resolution > 0:
            raise ValueError("resolution must be > 0")
        o = tuple(float(v) for v in self.origin)
        e = tuple(float(v) for v in self.extent)
        if len(o) != 3 or len(e) != 3 or min(e) <= 0:
            raise ValueError("origin and extent must be 3-vectors with a positive extent")
        res = float(self.resolution)
        object.__setattr__(self, "origin", o)
        object.__setattr__(self, "extent", e)
        object.__setattr__(self, "resolution", res)
        object.__setattr__(self, "dims", tuple(max(1, math.ceil(round(x / res, 9))) for x in e))

    def cell_center(self, ix: int, iy: int, iz: int) -> tuple[float, float, float]:
        r = self.resolution
        return (self.origin[0] + (ix + 0.5) * r, self.origin[1] + (iy + 0.5) * r, self.origin[2] + (iz + 0.5) * r)

    def point_to_cell(self, x: float, y: float, z: float) -> tuple[int, int, int]:
        r = self.resolution
        return tuple(int(math.floor((v - o) / r)) for v, o in zip((x, y, z), self.origin))

    def full_box(self) -> Box:
        nx, ny, nz = self.dims
        return Box((0, 0, 0), (nx - 1, ny - 1, nz - 1))


def hemisphere_mask(grid: VolumeGrid, radius: float, center=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Voxels whose centres lie in the hemisphere |r - c| <= radius, z >= c_z
    (the phantom of configs[4]; the 3-D analogue of breast_mask).  Returned
    read-only, so run_framework_volume can remember its hash per array object
    (a writable mask is re-hashed on every call, ~2 ms at 128^3)."""
    nx, ny, nz = grid.dims
    r = grid.resolution
    px = grid.origin[0] + (np.arange(nx) + 0.5) * r - center[0]
    py = grid.origin[1] + (np.arange(ny) + 0.5) * r - center[1]
    pz = grid.origin[2] + (np.arange(nz) + 0.5) * r - center[2]
    d2 = px[:, None, None] ** 2 + py[None, :, None] ** 2 + pz[None, None, :] ** 2
    mask = (d2 <= radius**2) & (pz[None, None, :] >= 0.0)
    mask.setflags(write=False)
    return mask


class VolumeMap:
    """Dense-backed voxel energy map (the 3-D counterpart of EnergyMap)."""

    def __init__(self, grid: VolumeGrid, values: np.ndarray, valid: np.ndarray, stride: int = 1, roi: Box | None = None,
                 *, checked: bool = False):
        """``checked``: the producing device pass already raised on its
        non-finite flag, so the host scan of every voxel is skipped."""
        self.grid, self.stride, self.roi = grid, stride, roi
        self.values = values
        self.valid = valid
        if not checked and valid.any() and not np.isfinite(values[valid]).all():
            raise ValueError("energy map contains non-finite values")

    @classmethod
    def _from_loader(cls, grid: VolumeGrid, loader, stride: int = 1, roi: Box | None = None):
        """A map whose (values, valid) arrays come from ``loader()`` on first
        use (device-checked finite): the octant framework's latency path."""
        vm = cls.__new__(cls)
        vm.grid, vm.stride, vm.roi = grid, stride, roi
        vm._loader = loader
        return vm

    def __getattr__(self, name):
        # only reached when the attribute is missing: materialise a loader-backed map (once)
        if name in ("values", "valid"):
            with _MATERIALISE:
                d = self.__dict__
                if name not in d and "_loader" in d:
                    d["values"], d["valid"] = d.pop("_loader")()
                if name in d:
                    return d[name]
        raise AttributeError(name)

    def __len__(self) -> int:
        return int(self.valid.sum())

    @property
    def entries(self) -> dict:
        ix, iy, iz = np.nonzero(self.valid)
        vals = self.values[ix, iy, iz].astype(np.float64)
        return dict(zip(zip(ix.tolist(), iy.tolist(), iz.tolist()), vals.tolist()))

    def argmax_cell(self) -> tuple[int, int, int]:
        """Max energy, ties to the lowest (ix, iy, iz)."""
        if not self.valid.any():
            raise ValueError("energy map is empty")
        score = np.where(self.valid, self.values.astype(np.float64), -np.inf)
        return tuple(int(v) for v in np.unravel_index(int(np.argmax(score)), score.shape))

    def argmax_position(self) -> tuple[float, float, float]:
        return self.grid.cell_center(*self.argmax_cell())

    def values_in(self, box: Box) -> np.ndarray:
        (x0, y0, z0), (x1, y1, z1) = box.min_cell, box.max_cell
        v = self.valid[x0 : x1 + 1, y0 : y1 + 1, z0 : z1 + 1]
        return self.values[x0 : x1 + 1, y0 : y1 + 1, z0 : z1 + 1][v].astype(np.float64)


def _volume_pass(scan, grid: VolumeGrid, box: Box, stride: int, mask_t, skip_stride: int, codes: tuple, interp: int,
                 k0: int, w: int, dense: dict, valid: torch.Tensor, status: _Status, count_slot: int,
                 d_region: torch.Tensor | None = None, mode: int = 0) -> None:
    nx, ny, nz = grid.dims
    p_max = math.prod((n + stride - 1) // stride for n in grid.dims)
    dev = dv.device()
    pts = torch.empty((p_max, 3), dtype=torch.float64, device=dev)
    oidx = torch.empty(p_max, dtype=torch.int32, device=dev)
    ws = torch.empty(int(nat.load().mwb_volume_workspace_bytes(nx, ny, nz, stride)), dtype=torch.uint8, device=dev)
    host_box = (ctypes.c_int32 * 6)(*box.bounds())
    count_ptr = status.count_ptr(count_slot)
    nat.call("mwb_enumerate_volume", grid.origin[0], grid.origin[1], grid.origin[2], grid.resolution, nx, ny, nz,
             ctypes.addressof(host_box), nat.ptr(d_region), stride, nat.ptr(mask_t), skip_stride, pts.data_ptr(),
             oidx.data_ptr(), count_ptr, valid.data_ptr(), ws.data_ptr(), dv.stream_handle())
    if w == 0:
        return pts, oidx, None
    table = build_table(scan, pts, p_max, interp, count_ptr)
    launch_energies(scan, pts, p_max, table, interp, k0, w,
                    dense.get(nat.MWB_DAS) if nat.MWB_DAS in codes else None,
                    dense.get(nat.MWB_DMAS) if nat.MWB_DMAS in codes else None,
                    0, oidx, count_ptr, status.key_ptr(0), status.key_ptr(1), status.flags_ptr, mode)
    return pts, oidx, table


# Enumerated voxels and their delay table per scanner geometry, grid, box,
# stride, mask and interpolation (as beamform._LATTICE_CACHE for 2-D grids):
# a stream of volumes from one scanner pays only the energy launch.  A 128^3
# table over 496 pairs is 4.2 GB, so the budget is sized for HBM (180 GB).
_VOLUME_CACHE = _LatticeCache(max_entries=2, max_bytes=12 << 30)


def _upload_mask3(mask, dims) -> torch.Tensor | None:
    if mask is None:
        return None
    m = np.asarray(mask, dtype=bool)
    if m.shape != tuple(dims):
        raise ValueError(f"mask must have the grid's dims {tuple(dims)}, got {m.shape}")
    flat = np.ascontiguousarray(m).view(np.uint8).reshape(-1)
    if not flat.flags.writeable:  # read-only masks (hemisphere_mask): torch wants a writable buffer
        flat = flat.copy()
    return torch.from_numpy(flat).to(dv.device())


def image_volume(ds, kinds, grid: VolumeGrid, box: Box | None = None, stride: int = 1, mask=None,
                 interpolation: str = "linear", *, window=None, mode: str = "smem") -> dict:
    """DAS and/or DMAS voxel maps of ``box`` at ``stride`` in one fused pass."""
    _check_interpolation(interpolation)
    if isinstance(kinds, str) or not hasattr(kinds, "__iter__"):
        kinds = (kinds,)
    codes = tuple(dict.fromkeys(_kind_code(k) for k in kinds))
    if stride < 1:
        raise ValueError("stride must be >= 1")
    box = grid.full_box() if box is None else box
    if not grid.full_box().contains_box(box):
        raise ValueError("box lies outside the grid")
    scan = dv.scan_for(ds)
    k0, w = _window(scan.n_samples, window)
    n = math.prod(grid.dims)
    dev = dv.device()
    interp = nat.INTERP[interpolation]
    kmode = {"smem": 0, "gather": 1}[mode]
    dense = {c: torch.zeros(n, dtype=torch.float32, device=dev) for c in codes}
    status = _Status()
    mh = None if mask is None else hashlib.sha1(np.packbits(np.asarray(mask, dtype=bool))).digest()
    key = (scan.geometry_key(), tuple(grid.origin), float(grid.resolution), tuple(grid.dims), box.bounds(), stride,
           mh, interp) if w else None
    ent = _VOLUME_CACHE.get(key) if key is not None else None
    if ent is not None:
        pts, oidx, table, cnt, valid, n_pts = ent
        launch_energies(scan, pts, pts.shape[0], table, interp, k0, w, dense.get(nat.MWB_DAS),
                        dense.get(nat.MWB_DMAS), 0, oidx, cnt.data_ptr(), status.key_ptr(0), status.key_ptr(1),
                        status.flags_ptr, kmode)
    else:
        valid = torch.zeros(n, dtype=torch.uint8, device=dev)
        made = _volume_pass(scan, grid, box, stride, _upload_mask3(mask, grid.dims), 0, codes, interp, k0, w, dense,
                            valid, status, 0, mode=kmode)
    st, vh, *dh = dv.to_host(status.t, valid.view(*grid.dims), *(dense[c].view(*grid.dims) for c in codes))
    _, counts, flags = status.read(st)
    if flags & 1:
        raise ValueError("energy map contains non-finite values")
    if ent is not None:
        n_eval = n_pts
    else:
        n_eval = int(counts[0])
        if key is not None and made is not None:
            _VOLUME_CACHE.put(key, (*made, torch.tensor([n_eval], dtype=torch.int32, device=dev), valid, n_eval))
    vmask = vh.view(bool)
    out = {}
    for c, h in zip(codes, dh):
        EVAL_COUNTER.add(n_eval)
        out["das" if c == nat.MWB_DAS else "dmas"] = VolumeMap(grid, h, vmask, stride, checked=True)
    return out


@dataclass
class VolumeReport:
    decimation_factor: int
    iterations: int
    final_region: Box
    coarse_points_evaluated: int
    fine_points_evaluated: int
    full_equivalent_points: int
    reduction_ratio: float
    elapsed: dict
    trace: MetricTrace
    argmax_cell: tuple[int, int, int]
    argmax_position: tuple[float, float, float]

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


def select_roi_volume(coarse: VolumeMap, box: Box, cfg: FrameworkConfig = FrameworkConfig()) -> tuple[Box, MetricTrace]:
    """Octant selection on a voxel map (device kernel)."""
    grid = coarse.grid
    nx, ny, nz = grid.dims
    d = max(1, int(coarse.stride))
    ix, iy, iz = np.nonzero(coarse.valid)
    if not coarse.values_in(box).size:
        raise ValueError("coarse map has no entries in the breast region")
    lattice = d if (d > 1 and not ((ix % d).any() or (iy % d).any() or (iz % d).any())) else 1
    dev = dv.device()
    dense_t = torch.from_numpy(np.ascontiguousarray(coarse.values, dtype=np.float32).reshape(-1)).to(dev)
    valid_t = torch.from_numpy(np.ascontiguousarray(coarse.valid).view(np.uint8).reshape(-1)).to(dev)
    region_t = torch.zeros(6, dtype=torch.int32, device=dev)
    trace_t = torch.zeros(nat.TRACE_BYTES, dtype=torch.uint8, device=dev)
    _launch_select3(dense_t, valid_t, grid, lattice, box, cfg, region_t, trace_t)
    final, trace, _ = decode_trace(trace_t.cpu().numpy().tobytes(), region=_box)
    return final, trace


def _launch_select3(dense_t, valid_t, grid, lattice, box, cfg, region_t, trace_t):
    nx, ny, nz = grid.dims
    host_box = (ctypes.c_int32 * 6)(*box.bounds())
    nat.call("mwb_select_roi_volume", dense_t.data_ptr(), valid_t.data_ptr(), nx, ny, nz, lattice,
             ctypes.addressof(host_box), float(cfg.frame_fraction), int(cfg.n_min), region_t.data_ptr(),
             trace_t.data_ptr(), dv.stream_handle())


_MASK_KEYS: dict[int, tuple] = {}


def _mask_key(mask: np.ndarray) -> tuple:
    """(content hash, voxel count) of a phantom mask.  Remembered per array
    object (while it lives) only for READ-ONLY arrays, so a stream of calls
    with one frozen mask hashes it once; a writable mask is hashed on every
    call, because the caller may edit it in place between calls."""
    if mask.flags.writeable:
        return hashlib.sha1(np.packbits(mask)).digest(), int(mask.sum())
    hit = _MASK_KEYS.get(id(mask))
    if hit is not None and hit[0]() is mask:
        return hit[1]
    val = (hashlib.sha1(np.packbits(mask)).digest(), int(mask.sum()))
    try:
        ref = weakref.ref(mask, lambda _r, k=id(mask): _MASK_KEYS.pop(k, None))
        _MASK_KEYS[id(mask)] = (ref, val)
    except TypeError:
        pass
    return val


class _VolumeFrameworkPlan(dv.GraphPlan):
    """The configs[4] octant framework for one scanner geometry, grid, mask and
    configuration, captured as a CUDA graph (coarse voxel lattice, octant
    select, ROI-driven fine pass).  As coarse2fine._FrameworkPlan: buffers live
    with the plan, the graph reads a signal slot every call refills, so a
    stream of volumes of one scanner replays one graph and allocates nothing
    on the device (the fine pass's point list and table are sized for the whole
    grid, since the ROI is only known on the device)."""

    def __init__(self, scan, grid: VolumeGrid, d: int, kcode: int, cfg: FrameworkConfig, interp: int, k0: int,
                 w: int, mask: np.ndarray, full_eq: int):
        self._init_slot(scan)
        self.grid, self.d, self.kcode, self.cfg = grid, d, kcode, cfg
        self.interp, self.k0, self.w = interp, k0, w
        self.full_eq = full_eq
        n = math.prod(grid.dims)
        dev = dv.device()
        self.mask_t = _upload_mask3(mask, grid.dims)
        self.dense = torch.empty(n, dtype=torch.float32, device=dev)  # only valid voxels are read
        self.valid = torch.empty(n, dtype=torch.uint8, device=dev)
        self.region_t = torch.empty(6, dtype=torch.int32, device=dev)
        self.events = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]
        self._ev_handles = None
        self._ms = (ctypes.c_float * 3)()
        self._pin = torch.cuda.is_available()
        self.mask_np = np.ascontiguousarray(mask, dtype=bool)
        # the coarse voxel lattice and its delay table depend on the geometry,
        # grid and mask only: built once here, outside the graph
        self.c_valid = torch.zeros(n, dtype=torch.uint8, device=dev)
        c_status = _Status()
        self.c_pts, self.c_oidx, _ = _volume_pass(self.scan, grid, grid.full_box(), d, self.mask_t, 0, (), interp,
                                                  k0, 0, {}, self.c_valid, c_status, 0)
        self.c_count = torch.empty(1, dtype=torch.int32, device=dev)
        self.c_count.copy_(c_status.t.view(torch.int32)[4:5])  # status count slot 0
        self.c_table = build_table(self.scan, self.c_pts, self.c_pts.shape[0], interp, self.c_count.data_ptr())
        self.n_coarse = int(self.c_count.item())
        self.c_slots = self.c_oidx[: self.n_coarse].clone()
        self.c_slots_host = self.c_slots.cpu().numpy()
        self.c_valid_host = self.c_valid.cpu().numpy().view(bool).reshape(grid.dims)
        # one result block per call, as the 2-D plan's: [status | trace | coarse
        # values, then the final box's voxels (mwb_gather_composite)], a budget
        # of box voxels copied with it, the rest only for a larger box
        self._o_trace = _Status.BYTES
        self._o_vals = (self._o_trace + nat.TRACE_BYTES + 15) // 16 * 16
        self._res_full = self._o_vals + 4 * (self.n_coarse + n)
        self._res_copy = min(self._res_full, self._o_vals + 4 * (self.n_coarse + self.BOX_BUDGET))
        self.res = torch.empty(self._res_full, dtype=torch.uint8, device=dev)
        self.status = _Status(self.res)
        self.trace_t = self.res[self._o_trace: self._o_trace + nat.TRACE_BYTES]
        self.compact = self.res[self._o_vals:].view(torch.float32)

    BOX_BUDGET = 1 << 16  # final-box voxels read back with the result block (256 KB)

    def _enqueue(self) -> None:
        g, d, sc = self.grid, self.d, self.scan
        ev = self.events
        full = g.full_box()
        self.valid.copy_(self.c_valid)
        self.status.t.zero_()
        st = self.status
        ev[0].record()
        launch_energies(sc, self.c_pts, self.c_pts.shape[0], self.c_table, self.interp, self.k0, self.w,
                        self.dense if self.kcode == nat.MWB_DAS else None,
                        self.dense if self.kcode == nat.MWB_DMAS else None, 0, self.c_oidx, self.c_count.data_ptr(),
                        st.key_ptr(0), st.key_ptr(1), st.flags_ptr, 0)
        ev[1].record()
        _launch_select3(self.dense, self.valid, g, d, full, self.cfg, self.region_t, self.trace_t)
        ev[2].record()
        _volume_pass(sc, g, full, 1, self.mask_t, d, (self.kcode,), self.interp, self.k0, self.w,
                     {self.kcode: self.dense}, self.valid, self.status, 1, d_region=self.region_t)
        ev[3].record()
        _, ny, nz = g.dims
        nat.call("mwb_gather_composite", self.dense.data_ptr(), ny, nz, self.c_slots.data_ptr(), self.n_coarse,
                 self.region_t.data_ptr(), self.compact.data_ptr(), self.compact.numel(), dv.stream_handle())

    def launch(self, scan) -> None:
        self.replay(scan)
        self.h_res = torch.empty(self._res_copy, dtype=torch.uint8, pin_memory=self._pin)  # kept by the returned map
        nat.call("mwb_memcpy_async", self.h_res.data_ptr(), self.res.data_ptr(), self._res_copy, dv.stream_handle())

    def _arrays(self, comp: np.ndarray, final: Box) -> tuple[np.ndarray, np.ndarray]:
        """(values, valid) of the composite: coarse voxels from their slots, fine
        voxels = the final box's masked voxels off the coarse lattice."""
        d = self.d
        (x0, y0, z0), (x1, y1, z1) = final.min_cell, final.max_cell
        vals = np.zeros(math.prod(self.grid.dims), dtype=np.float32)
        vals[self.c_slots_host] = comp[: self.n_coarse]
        vals = vals.reshape(self.grid.dims)
        valid = self.c_valid_host.copy()
        ix = np.arange(x0, x1 + 1)[:, None, None] % d == 0
        iy = np.arange(y0, y1 + 1)[None, :, None] % d == 0
        iz = np.arange(z0, z1 + 1)[None, None, :] % d == 0
        fine = self.mask_np[x0: x1 + 1, y0: y1 + 1, z0: z1 + 1] & ~(ix & iy & iz)
        block = comp[self.n_coarse:].reshape(x1 - x0 + 1, y1 - y0 + 1, z1 - z0 + 1)
        vals[x0: x1 + 1, y0: y1 + 1, z0: z1 + 1][fine] = block[fine]
        valid[x0: x1 + 1, y0: y1 + 1, z0: z1 + 1] |= fine
        return vals, valid

    def finish(self) -> tuple[VolumeMap, VolumeReport]:
        dv.sync_stream()
        grid, d = self.grid, self.d
        blk = self.h_res.numpy()
        keys, counts, flags = _Status.decode(blk[: _Status.BYTES].view(np.int64))
        if flags & 1:
            raise ValueError("energy map contains non-finite values")
        final, trace, _ = decode_trace_lazy(blk[self._o_trace: self._o_trace + nat.TRACE_BYTES], region=_box)
        used = self._o_vals + 4 * (self.n_coarse + final.n_cells)
        if used > self._res_copy:  # final box beyond the budget: copy the whole used block again
            self.h_res = torch.empty(used, dtype=torch.uint8, pin_memory=self._pin)
            nat.call("mwb_memcpy_async", self.h_res.data_ptr(), self.res.data_ptr(), used, dv.stream_handle())
            dv.sync_stream()
            blk = self.h_res.numpy()
        comp = blk[self._o_vals: used].view(np.float32)
        composite = VolumeMap._from_loader(grid, functools.partial(self._arrays, comp, final), stride=d, roi=final)
        n_c, n_f = self.n_coarse, int(counts[1])
        EVAL_COUNTER.add(n_c + n_f)
        key = int(keys[0 if self.kcode == nat.MWB_DAS else 1])
        _, ny, nz = grid.dims
        if key:
            slot = 0xFFFFFFFF - (key & 0xFFFFFFFF)
            cell = (slot // (ny * nz), (slot // nz) % ny, slot % nz)
        else:
            cell = composite.argmax_cell()
        if self._ev_handles is None:
            self._ev_handles = (ctypes.c_void_p * 4)(*[e.cuda_event for e in self.events])
        nat.call("mwb_elapsed_ms", self._ev_handles, 4, self._ms)
        t = [self._ms[i] / 1e3 for i in range(3)]
        report = VolumeReport(
            decimation_factor=d, iterations=trace.n_records, final_region=final, coarse_points_evaluated=n_c,
            fine_points_evaluated=n_f, full_equivalent_points=self.full_eq,
            reduction_ratio=self.full_eq / (n_c + n_f),
            elapsed={"coarse": t[0], "select": t[1], "fine": t[2], "total": sum(t)}, trace=trace, argmax_cell=cell,
            argmax_position=grid.cell_center(*cell))
        return composite, report


_VOLUME_PLANS: "OrderedDict[tuple, _VolumeFrameworkPlan]" = OrderedDict()
_VOLUME_PLAN_CAPACITY = 2


def run_framework_volume(ds, kind, grid: VolumeGrid, mode, cfg: FrameworkConfig = FrameworkConfig(), *,
                         mask=None, phantom_radius: float | None = None, interpolation: str = "linear",
                         window=None) -> tuple[VolumeMap, VolumeReport]:
    """Coarse voxel lattice -> device octant selection -> fine pass in the final
    box -> composite (the configs[4] framework with octant splits).

    The phantom mask is ``mask`` if given, else the hemisphere of
    ``phantom_radius`` (default: the largest hemisphere inscribed in the grid).
    Calls with one configuration on volumes of one scanner replay a captured
    CUDA graph (``_VolumeFrameworkPlan``).
    """
    _check_interpolation(interpolation)
    d = decimation_factor(mode, grid.resolution)
    if mask is None:
        if phantom_radius is None:
            phantom_radius = min(grid.extent[0], grid.extent[1]) / 2.0
        mask = hemisphere_mask(grid, phantom_radius)
    if not (isinstance(mask, np.ndarray) and mask.dtype == bool):
        mask = np.asarray(mask, dtype=bool)
    if mask.shape != tuple(grid.dims):
        raise ValueError(f"mask must have the grid's dims {tuple(grid.dims)}, got {mask.shape}")
    mhash, full_eq = _mask_key(mask)
    kcode = _kind_code(kind)
    scan = dv.scan_for(ds)
    k0, w = _window(scan.n_samples, window)
    interp = nat.INTERP[interpolation]
    with dv.PLAN_LOCK:
        key = (scan.geometry_key(), tuple(grid.origin), float(grid.resolution), tuple(grid.dims), d, kcode,
               cfg.frame_fraction, cfg.n_min, interp, k0, w, mhash)
        plan = _VOLUME_PLANS.get(key)
        if plan is None:
            if not mask[::d, ::d, ::d].any():
                raise ValueError("no coarse focal points inside the phantom mask")
            plan = _VolumeFrameworkPlan(scan, grid, d, kcode, cfg, interp, k0, w, mask, full_eq)
            _VOLUME_PLANS[key] = plan
            while len(_VOLUME_PLANS) > _VOLUME_PLAN_CAPACITY:
                _VOLUME_PLANS.popitem(last=False)
        else:
            _VOLUME_PLANS.move_to_end(key)
        plan.launch(scan)
        return plan.finish()


__all__ = [
    "Box",
    "IterationRecord",
    "VolumeGrid",
    "VolumeMap",
    "VolumeReport",
    "hemisphere_mask",
    "image_volume",
    "run_framework_volume",
    "select_roi_volume",
]
