"""The coarse-to-fine framework for a batch of scans (production throughput).

``run_framework`` (coarse2fine.py:301-350) processes one dataset per call.
``FrameworkBatch`` applies the same rules to S scans that share an antenna
geometry and an imaging grid:

1. coarse pass: the stride-D lattice inside the breast mask is enumerated
   and its delay table built once; one energy launch images it for all S
   scans;
2. selection: ``mwb_select_roi_batch`` runs one select_roi CTA per scan
   (coarse2fine.py:169-256 rules, each scan's own trace);
3. fine pass: every scan's ROI cells (stride 1, mask, minus the coarse
   lattice, coarse2fine.py:321-323) are enumerated into one packed list where
   each scan starts on a 256-point tile; a per-tile delay table and one
   energy launch (tile -> scan) evaluate all of them;
4. the per-scan argmax of the composite (coarse + fine) is fused into both
   energy launches.

Values, regions, traces and argmax cells are bit-identical to calling
``run_framework`` once per scan.  One host synchronisation per batch (after
step 2, to size the packed fine list).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _native as nat
from .beamform import EVAL_COUNTER, EnergyMap, _kind, _kind_code, _Status, _window, build_table
from .coarse2fine import FrameworkConfig, MetricTrace, breast_mask, decimation_factor, decode_trace
from .geometry import ArrayGeometry, ImagingGrid, Region, as_grid


@dataclass
class FrameworkBatchResult:
    grid: ImagingGrid
    decimation_factor: int
    final_regions: np.ndarray  # (S, 4) x0, y0, x1, y1
    argmax_cells: np.ndarray  # (S, 2)
    coarse_points_evaluated: int  # per scan
    fine_points_evaluated: np.ndarray  # (S,)
    full_equivalent_points: int
    dense: torch.Tensor  # (S, nx, ny) composite energies on the device (valid cells only)
    elapsed: dict
    _traces: torch.Tensor  # device copy; decoded per scan on demand
    _coarse_valid: np.ndarray
    _mask: np.ndarray

    @property
    def n_scans(self) -> int:
        return int(self.final_regions.shape[0])

    @property
    def reduction_ratios(self) -> np.ndarray:
        return self.full_equivalent_points / (self.coarse_points_evaluated + self.fine_points_evaluated)

    def trace(self, s: int) -> MetricTrace:
        n = nat.TRACE_BYTES
        _, trace, _ = decode_trace(self._traces[s * n : (s + 1) * n].cpu().numpy().tobytes())
        return trace

    def final_region(self, s: int) -> Region:
        x0, y0, x1, y1 = (int(v) for v in self.final_regions[s])
        return Region((x0, y0), (x1, y1))

    def composite(self, s: int) -> EnergyMap:
        """Scan s's composite map (coarse lattice + fine ROI), as run_framework returns it."""
        nx, ny = self.grid.dims
        d = self.decimation_factor
        x0, y0, x1, y1 = (int(v) for v in self.final_regions[s])
        valid = self._coarse_valid.copy()
        roi = np.zeros((nx, ny), dtype=bool)
        roi[x0 : x1 + 1, y0 : y1 + 1] = True
        ix = np.arange(nx)[:, None]
        iy = np.arange(ny)[None, :]
        lattice = (ix % d == 0) & (iy % d == 0)
        valid |= roi & self._mask & ~lattice
        vals = self.dense[s].cpu().numpy()
        return EnergyMap._from_dense(self.grid, vals, valid, stride=d, roi=self.final_region(s), split=d,
                                     checked=True)


class FrameworkBatch:
    def __init__(self, geometry: ArrayGeometry, pairs, n_samples: int, grid: ImagingGrid, mode, kind,
                 cfg: FrameworkConfig = FrameworkConfig(), window=None, interpolation: str = "linear"):
        dev = dv.device()
        grid = as_grid(grid)
        self.grid, self.cfg = grid, cfg
        self.kind = _kind(kind)
        self.kcode = _kind_code(kind)
        self.d = decimation_factor(mode, grid.resolution)
        self.interp = nat.INTERP[interpolation]
        self.n_samples = int(n_samples)
        self.ld = dv.round4(n_samples)
        self.k0, self.w = _window(self.n_samples, window)
        if self.w == 0:
            raise ValueError("the framework needs a non-empty energy window")
        pairs = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
        m = geometry.n_antennas
        self.scan = dv.DeviceScan(
            sig=torch.empty(0, device=dev),
            chan=torch.from_numpy(pairs).to(dev),
            ant=torch.from_numpy(np.array(geometry.antennas, dtype=np.float64)).to(dev),
            inv_scale=1.0 / (float(geometry.propagation_speed) * float(geometry.sample_interval)),
            n_samples=self.n_samples, ld=self.ld, n_ant=m, chan_host=pairs)
        nx, ny = grid.dims
        self.mask_np = breast_mask(grid)
        if not self.mask_np[:: self.d, :: self.d].any():
            raise ValueError("no coarse focal points inside the breast mask")
        self.mask_t = dv.upload_mask(self.mask_np, grid.dims)
        # coarse lattice: enumerated and tabled once, shared by every scan
        d = self.d
        p_max = ((nx + d - 1) // d) * ((ny + d - 1) // d)
        self.c_pts = torch.empty((p_max, 3), dtype=torch.float64, device=dev)
        self.c_idx = torch.empty(p_max, dtype=torch.int32, device=dev)
        self.c_valid = torch.zeros(nx * ny, dtype=torch.uint8, device=dev)
        st = _Status()
        ws = torch.empty(int(nat.load().mwb_lattice_workspace_bytes(nx, ny, d)), dtype=torch.uint8, device=dev)
        nat.call("mwb_enumerate_lattice", grid.origin[0], grid.origin[1], grid.resolution, nx, ny, 0, 0, nx - 1,
                 ny - 1, None, d, self.mask_t.data_ptr(), 0, self.c_pts.data_ptr(), self.c_idx.data_ptr(),
                 st.count_ptr(0), self.c_valid.data_ptr(), ws.data_ptr(), dv.stream_handle())
        _, counts, _ = st.read()
        self.n_coarse = int(counts[0])
        self.c_table = build_table(self.scan, self.c_pts, self.n_coarse, self.interp)
        self.c_valid_host = self.c_valid.view(nx, ny).cpu().numpy().astype(bool)

    @property
    def n_chan(self) -> int:
        return self.scan.n_chan

    def run(self, sig: torch.Tensor) -> FrameworkBatchResult:
        """Run the framework on S device-resident scans (S, C, ld) fp32."""
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
        dense = torch.empty((s_n, nx * ny), dtype=torch.float32, device=dev)
        keys = torch.zeros(s_n, dtype=torch.int64, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        regions = torch.empty((s_n, 6), dtype=torch.int32, device=dev)
        traces = torch.empty(s_n * nat.TRACE_BYTES, dtype=torch.uint8, device=dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        das = self.kcode == nat.MWB_DAS
        sc = self.scan
        ev[0].record()
        # 1. coarse pass for every scan
        nat.call("mwb_energies", sig.data_ptr(), s_n, self.n_chan * self.ld, self.n_chan, self.ld, self.n_samples,
                 sc.chan.data_ptr(), sc.ant.data_ptr(), sc.n_ant, sc.inv_scale, self.c_pts.data_ptr(),
                 self.c_idx.data_ptr(), self.n_coarse, None, self.c_table.data_ptr(), self.interp, self.k0, self.w,
                 dense.data_ptr() if das else None, None if das else dense.data_ptr(), nx * ny,
                 keys.data_ptr() if das else None, None if das else keys.data_ptr(), flags.data_ptr(), 0, stream)
        ev[1].record()
        # 2. one select_roi per scan
        nat.call("mwb_select_roi_batch", dense.data_ptr(), nx * ny, self.c_valid.data_ptr(), nx, ny, self.d, 0, 0,
                 nx - 1, ny - 1, float(self.cfg.frame_fraction), int(self.cfg.n_min), s_n, regions.data_ptr(),
                 traces.data_ptr(), stream)
        ev[2].record()
        # 3. fine pass: packed per-scan ROI cells, one table and one energy launch
        ws = torch.empty(int(lib.mwb_regions_workspace_bytes(s_n)), dtype=torch.uint8, device=dev)
        totals = torch.zeros(2, dtype=torch.int32, device=dev)
        nat.call("mwb_enumerate_regions_count", nx, ny, regions.data_ptr(), s_n, self.mask_t.data_ptr(), self.d,
                 totals.data_ptr(), ws.data_ptr(), stream)
        n_pts, n_tiles = (int(v) for v in totals.cpu().tolist())  # the one host sync: packed list size
        if n_pts > 0:
            f_pts = torch.empty((n_pts, 3), dtype=torch.float64, device=dev)
            f_idx = torch.empty(n_pts, dtype=torch.int32, device=dev)
            tile_info = torch.empty((n_tiles, 2), dtype=torch.int32, device=dev)
            nat.call("mwb_enumerate_regions_write", grid.origin[0], grid.origin[1], grid.resolution, nx, ny,
                     regions.data_ptr(), s_n, self.mask_t.data_ptr(), self.d, f_pts.data_ptr(), f_idx.data_ptr(),
                     tile_info.data_ptr(), ws.data_ptr(), stream)
            f_table = torch.empty(int(lib.mwb_delay_table_bytes(n_pts, self.n_chan)), dtype=torch.uint8, device=dev)
            nat.call("mwb_delay_table_tiles", f_pts.data_ptr(), n_pts, tile_info.data_ptr(), sc.chan.data_ptr(),
                     self.n_chan, sc.ant.data_ptr(), sc.n_ant, sc.inv_scale, self.interp, f_table.data_ptr(), stream)
            nat.call("mwb_energies_tiles", sig.data_ptr(), s_n, self.n_chan * self.ld, self.n_chan, self.ld,
                     self.n_samples, sc.chan.data_ptr(), sc.ant.data_ptr(), sc.n_ant, sc.inv_scale,
                     f_pts.data_ptr(), f_idx.data_ptr(), n_pts, tile_info.data_ptr(), f_table.data_ptr(),
                     self.interp, self.k0, self.w, dense.data_ptr() if das else None,
                     None if das else dense.data_ptr(), nx * ny, keys.data_ptr() if das else None,
                     None if das else keys.data_ptr(), flags.data_ptr(), 0, stream)
        ev[3].record()
        fine_counts = ws.view(torch.int32)[:s_n].cpu().numpy().astype(np.int64)
        if int(flags.item()) & 1:
            raise ValueError("energy map contains non-finite values")
        reg = regions.cpu().numpy()
        k = keys.cpu().numpy().view(np.uint64)
        slot = (0xFFFFFFFF - (k & np.uint64(0xFFFFFFFF))).astype(np.int64)
        cells = np.stack([slot // ny, slot % ny], axis=1)
        EVAL_COUNTER.add(self.n_coarse * s_n + int(fine_counts.sum()))
        elapsed = {"coarse": ev[0].elapsed_time(ev[1]) / 1e3, "select": ev[1].elapsed_time(ev[2]) / 1e3,
                   "fine": ev[2].elapsed_time(ev[3]) / 1e3}
        elapsed["total"] = sum(elapsed.values())
        return FrameworkBatchResult(
            grid=grid, decimation_factor=self.d, final_regions=reg[:, [0, 1, 3, 4]], argmax_cells=cells,
            coarse_points_evaluated=self.n_coarse, fine_points_evaluated=fine_counts,
            full_equivalent_points=int(self.mask_np.sum()), dense=dense.view(s_n, nx, ny), elapsed=elapsed,
            _traces=traces, _coarse_valid=self.c_valid_host, _mask=self.mask_np)
