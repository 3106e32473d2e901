"""Device residency of scans, masks and workspaces.

A scan is uploaded once per (frozen) dataset object: the populated channels
(any nonzero sample) are compacted in the reference's row-major (i, j) channel
order into an fp32 ``[C][ld]`` buffer with a zero tail (ld = N rounded up to
4 samples, so every TMA bulk copy is 16-byte aligned).  All-zero channels are
dropped because they add exactly 0 to DAS and DMAS in the reference
(beamform.py:199-212).  Device buffers are torch tensors; only raw pointers
cross into ``libmwb.so``.
"""

from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass

import numpy as np
import torch


# Captured-graph plans (run_framework, segment, run_framework_volume) own their
# device and pinned buffers; a call holds this lock from the plan lookup to the
# readback so concurrent host threads (e.g. a web service's worker pool) never
# interleave on one plan.
PLAN_LOCK = threading.RLock()


class GraphPlan:
    """Base of the captured-graph plans (image, run_framework, segment,
    run_framework_volume).  A plan owns a signal slot (a copy of the first
    scan's DeviceScan with its own ``sig`` buffer) that its graph reads;
    ``replay(scan)`` refills the slot with ``scan``'s samples (device to
    device), runs ``_enqueue`` eagerly once and captures it on the first call,
    then replays the graph.  Subclasses implement ``_enqueue``."""

    graph = None

    def _init_slot(self, scan: "DeviceScan") -> "DeviceScan":
        import dataclasses

        self.scan = dataclasses.replace(scan, sig=torch.empty_like(scan.sig))
        return self.scan

    def _enqueue(self) -> None:  # pragma: no cover - abstract
        raise NotImplementedError

    _slot_src = None  # the scan whose samples the slot holds (scans are immutable)

    def replay(self, scan: "DeviceScan") -> None:
        if scan is not self._slot_src:
            from . import _native as nat

            nat.call("mwb_memcpy_async", self.scan.sig.data_ptr(), scan.sig.data_ptr(),
                     scan.sig.numel() * scan.sig.element_size(), stream_handle())
            self._slot_src = scan
        if self.graph is None:
            self._enqueue()  # eager run: kernel attributes set, allocator warmed
            torch.cuda.current_stream().synchronize()
            graph = torch.cuda.CUDAGraph()
            # thread-local capture: scan uploads, mask uploads and plan setup
            # that other host threads run outside PLAN_LOCK (pinned allocs,
            # H2D copies, stream syncs) neither invalidate this capture nor
            # are rejected while it is open
            with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                self._enqueue()
            self.graph = graph
        self.graph.replay()


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 imaging path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    """Raw handle of torch's current stream on the current device (the C
    accessor: a Stream object per call costs the latency path ~7 us)."""
    return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())


def sync_stream() -> None:
    """Wait for the current stream through the library (mwb_stream_synchronize)."""
    from . import _native as nat

    nat.call("mwb_stream_synchronize", stream_handle())


def to_host(*tensors: torch.Tensor) -> list[np.ndarray]:
    """Device->host copies of several tensors through pinned staging buffers
    (torch's caching host allocator) with ONE stream sync.  Pageable ``.cpu()``
    copies run at a fraction of the PCIe/C2C rate and sync once per tensor."""
    staged = []
    for t in tensors:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        staged.append(h)
    sync_stream()
    return [h.numpy() for h in staged]


def round4(n: int) -> int:
    return max(4, (int(n) + 3) // 4 * 4)


@dataclass
class DeviceScan:
    sig: torch.Tensor  # (C, ld) float32
    chan: torch.Tensor  # (C, 2) int32
    ant: torch.Tensor  # (M, 3) float64
    inv_scale: float
    n_samples: int
    ld: int
    n_ant: int
    chan_host: np.ndarray  # (C, 2) int32

    ant_host: np.ndarray | None = None  # (M, 3) float64, when known

    @property
    def n_chan(self) -> int:
        return int(self.chan_host.shape[0])

    def geometry_key(self) -> tuple:
        """Everything but the samples: scans with equal keys can share device
        plans (lattices, delay tables, captured graphs)."""
        ants = self.ant_host if self.ant_host is not None else self.ant.cpu().numpy()
        return (np.ascontiguousarray(ants, dtype=np.float64).tobytes(), self.chan_host.tobytes(),
                float(self.inv_scale), int(self.n_samples), int(self.ld), torch.cuda.current_device())


_GEOMS: dict[tuple, tuple[torch.Tensor, torch.Tensor]] = {}


def geometry_tensors(pairs: np.ndarray, antennas: np.ndarray) -> tuple[torch.Tensor, torch.Tensor]:
    """Device (C, 2) int32 channel pairs and (M, 3) float64 antennas, cached per
    geometry so a stream of scans of one scanner uploads them once."""
    key = (pairs.tobytes(), antennas.tobytes(), torch.cuda.current_device())
    hit = _GEOMS.get(key)
    if hit is None:
        dev = device()
        hit = (torch.from_numpy(np.array(pairs, dtype=np.int32)).to(dev),
               torch.from_numpy(np.array(antennas, dtype=np.float64)).to(dev))
        if len(_GEOMS) > 64:
            _GEOMS.clear()
        _GEOMS[key] = hit
    return hit


def upload_rows(rows: np.ndarray, keep: np.ndarray, ld: int) -> torch.Tensor:
    """Device fp32 [len(keep)][ld] (zero tail) of rows[keep] (any float dtype):
    cast once into pinned staging, one asynchronous host->device copy."""
    n = rows.shape[1]
    pinned = torch.cuda.is_available()
    h = torch.empty((keep.size, ld), dtype=torch.float32, pin_memory=pinned)
    hv = h.numpy()
    if ld > n:
        hv[:, n:] = 0.0
    for i, k in enumerate(keep):
        hv[i, :n] = rows[k]
    return h.to(device(), non_blocking=pinned)


def compact_channels(signals: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Populated channels of an (M, M, N) array: (C, N) float32 and (C, 2) pairs.

    A dataset with no populated channel keeps channel (0, 0) (all zeros) so the
    launch shape stays valid; its energies are exactly 0, as in the reference.
    """
    m, _, n = signals.shape
    flat = signals.reshape(m * m, n)
    keep = np.flatnonzero(np.any(flat != 0.0, axis=1)) if n > 0 else np.zeros(0, dtype=np.int64)
    if keep.size == 0:
        keep = np.zeros(1, dtype=np.int64)
    pairs = np.stack([keep // m, keep % m], axis=1).astype(np.int32)
    return flat[keep].astype(np.float32), pairs


_SCANS: dict[int, tuple[weakref.ref, DeviceScan]] = {}


def _upload_record(flat: np.ndarray, ld: int) -> tuple[torch.Tensor, np.ndarray]:
    """Populated rows of an fp64 (rows, n) record -> device fp32 [C][ld] and
    their indices: compacted and converted by mwb_compact_rows_host straight
    into pinned staging (one pass, each row's zero test stopping at its first
    nonzero word), then one asynchronous host->device copy."""
    from . import _native as nat

    rows, n = flat.shape
    pinned = torch.cuda.is_available()
    h = torch.empty((rows, ld), dtype=torch.float32, pin_memory=pinned)
    keep = np.empty(rows, dtype=np.int32)
    count = int(nat.load().mwb_compact_rows_host(flat.ctypes.data, rows, n, ld, h.data_ptr(),
                                                  keep.ctypes.data))
    if count < 1:
        raise RuntimeError(f"mwb_compact_rows_host failed ({count})")
    return h[:count].to(device(), non_blocking=pinned), keep[:count].astype(np.int64)


def _build_scan(ds) -> DeviceScan:
    geom = ds.geometry
    sig = np.asarray(ds.signals)
    m, _, n = sig.shape
    flat = sig.reshape(m * m, n)
    ld = round4(n)
    if sig.dtype == np.float64 and flat.flags.c_contiguous and n > 0:
        dev_sig, keep = _upload_record(flat, ld)
    else:
        keep = np.flatnonzero(np.any(flat != 0.0, axis=1)) if n > 0 else np.zeros(0, dtype=np.int64)
        if keep.size == 0:  # as compact_channels: keep channel (0, 0), all zeros
            keep = np.zeros(1, dtype=np.int64)
        dev_sig = upload_rows(flat, keep, ld)
    pairs = np.stack([keep // m, keep % m], axis=1).astype(np.int32)
    ants = np.ascontiguousarray(np.asarray(geom.antennas, dtype=np.float64))
    chan, ant = geometry_tensors(pairs, ants)
    scale = float(geom.propagation_speed) * float(geom.sample_interval)
    return DeviceScan(
        sig=dev_sig,
        chan=chan,
        ant=ant,
        inv_scale=1.0 / scale,
        n_samples=n,
        ld=ld,
        n_ant=m,
        chan_host=pairs,
        ant_host=ants,
    )


def scan_for(ds) -> DeviceScan:
    """Device copy of ``ds``; cached while ``ds`` lives if its signals are read-only."""
    sig = np.asarray(ds.signals)
    cacheable = not sig.flags.writeable
    key = id(ds)
    if cacheable:
        hit = _SCANS.get(key)
        if hit is not None and hit[0]() is ds:
            return hit[1]
    scan = _build_scan(ds)
    if cacheable:
        try:
            ref = weakref.ref(ds, lambda _r, k=key: _SCANS.pop(k, None))
        except TypeError:
            return scan
        _SCANS[key] = (ref, scan)
    return scan


_MONO: dict[int, tuple[weakref.ref, DeviceScan]] = {}


def mono_scan_for(ds) -> DeviceScan:
    """Device copy of the diagonal (monostatic) channels of ``ds``.

    The reference's monostatic delay is d_i / (2 v dt) (beamform.py:224); the
    energy kernel evaluates (d_tx + d_rx) * inv_scale, so the diagonal channel
    (i, i) with inv_scale = 1 / (4 v dt) gives 2 d_i / (4 v dt), the same delay
    to within one fp64 ulp.  All-zero diagonal channels are dropped (exact).
    """
    sig = np.asarray(ds.signals)
    cacheable = not sig.flags.writeable
    key = id(ds)
    if cacheable:
        hit = _MONO.get(key)
        if hit is not None and hit[0]() is ds:
            return hit[1]
    m, _, n = sig.shape
    idx = np.arange(m)
    diag = sig[idx, idx]  # (M, N)
    keep = np.flatnonzero(np.any(diag != 0.0, axis=1)) if n > 0 else np.zeros(0, dtype=np.int64)
    if keep.size == 0:
        keep = np.zeros(1, dtype=np.int64)
    ld = round4(n)
    host = np.zeros((keep.size, ld), dtype=np.float32)
    host[:, :n] = diag[keep]
    pairs = np.stack([keep, keep], axis=1).astype(np.int32)
    geom = ds.geometry
    dev = device()
    ants = np.ascontiguousarray(np.asarray(geom.antennas, dtype=np.float64))
    chan, ant = geometry_tensors(pairs, ants)
    scan = DeviceScan(
        sig=torch.from_numpy(host).to(dev),
        chan=chan,
        ant=ant,
        ant_host=ants,
        inv_scale=1.0 / (4.0 * float(geom.propagation_speed) * float(geom.sample_interval)),
        n_samples=n,
        ld=ld,
        n_ant=m,
        chan_host=pairs,
    )
    if cacheable:
        try:
            ref = weakref.ref(ds, lambda _r, k=key: _MONO.pop(k, None))
            _MONO[key] = (ref, scan)
        except TypeError:
            pass
    return scan


def upload_mask(mask: np.ndarray | None, dims: tuple[int, int]) -> torch.Tensor | None:
    if mask is None:
        return None
    m = np.asarray(mask, dtype=bool)
    if m.shape != tuple(dims):
        raise ValueError(f"mask must have the grid's dims {tuple(dims)}, got {m.shape}")
    return torch.from_numpy(np.ascontiguousarray(m).view(np.uint8)).to(device())
