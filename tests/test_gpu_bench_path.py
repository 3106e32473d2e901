"""Parity of the exact bench path (BASELINE configs[3]) against the oracle.

bench.py's headline ``e2e`` goes through ``BatchImager(mode="auto").__call__``
— the tensor-core kernel (K1-TC) behind the chunked, ramped H2D / compute /
D2H pipeline — and ``value`` through ``run_device`` on the same imager.  This
module runs that call on 1024 configs[3] scans (256 x 256 px over 12 x 12 cm,
66 pairs, 1024 samples, W = 32) with ``chunk=128`` (the bench's setting: the
ramp [32, 64, 128 x 6, 64, 32] and more chunks than buffer sets) and checks:

* the end-to-end maps and argmax cells are bit-identical to ``run_device``;
* on 8 scans spread over the batch, >= 1000 pixels per scan and kind agree
  with the oracle (reference kernel, beamform.py:169-212, windowed by suffix
  differencing) within BASELINE's 1e-4, normalised by the ORACLE's peak;
* every checked scan's argmax equals the oracle's argmax.

How the argmax and the peak are established without imaging all 65,536
pixels on the CPU: the checked set holds every pixel whose GPU value lies
within 1e-3 of the GPU's peak magnitude of the GPU maximum (and, for the
signed DMAS map, of the GPU minimum).  A pixel outside that set is, on the
GPU, more than 1e-3·peak below the GPU maximum; with the error bound of
1e-4·peak that this test verifies on >= 1000 sampled pixels, its oracle value
is more than 8e-4·peak below the oracle value at the GPU argmax, so neither
the oracle's argmax nor its peak magnitude can lie outside the set.
"""

import numpy as np
import pytest
import torch

from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager, _chunk_ranges

pytestmark = pytest.mark.gpu

S = 1024
CHUNK = 128
TOL = 1e-4
CAND = 1e-3  # candidate band for the argmax / peak (>> TOL)
CHECK_SCANS = (0, 131, 262, 393, 524, 655, 786, 1023)


@pytest.fixture(scope="module")
def bench_path():
    model = synth.ScanModel()
    sig_d, _ = synth.batch_2d_device(model, range(S))
    grid = synth.grid_square(0.12, 256)
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(model.k0, model.window),
                     mode="auto")
    host = sig_d[:, :, : model.n_samples].cpu().pin_memory()
    res = bi(host, kinds=("das", "dmas"), chunk=CHUNK)
    return model, grid, bi, sig_d, host, res


def test_bench_path_uses_tensor_cores_and_ramp(bench_path):
    _, _, bi, _, _, _ = bench_path
    assert bi.uses_tensor_cores
    ranges = _chunk_ranges(S, CHUNK)
    sizes = [b - a for a, b in ranges]
    assert sizes[:2] == [CHUNK // 4, CHUNK // 2] and sizes[-2:] == [CHUNK // 2, CHUNK // 4]
    assert len(ranges) > 4 and sum(sizes) == S


def test_e2e_equals_device_path(bench_path):
    _, grid, bi, sig_d, _, res = bench_path
    n = grid.dims[0] * grid.dims[1]
    for kind in ("das", "dmas"):
        out = torch.empty((S, n), dtype=torch.float32, device="cuda")
        keys = torch.zeros(S, dtype=torch.int64, device="cuda")
        bi.run_device(sig_d, **{f"out_{kind}": out, f"key_{kind}": keys})
        assert torch.equal(res.maps[kind].reshape(S, n), out.cpu()), kind
        assert np.array_equal(res.argmax[kind], bi.decode_keys(keys.cpu().numpy().view(np.uint64))), kind


def _check_cells(dense, rng, kind):
    """Random sample + argmax neighbourhood + the candidate band(s)."""
    nx, ny = dense.shape
    peak = float(np.abs(dense).max())
    cells = {(int(a), int(b)) for a, b in rng.integers(0, (nx, ny), size=(1000, 2))}
    gmax = np.unravel_index(int(np.argmax(dense)), dense.shape)
    for dx in range(-3, 4):
        for dy in range(-3, 4):
            x, y = gmax[0] + dx, gmax[1] + dy
            if 0 <= x < nx and 0 <= y < ny:
                cells.add((x, y))
    band = np.argwhere(dense >= dense.max() - CAND * peak)
    if kind == "dmas":
        band = np.concatenate([band, np.argwhere(dense <= dense.min() + CAND * peak)])
    assert len(band) < 4000, "candidate band too wide for the CPU oracle"
    cells.update((int(a), int(b)) for a, b in band)
    return sorted(cells)


@pytest.mark.parametrize("scan", CHECK_SCANS)
def test_e2e_maps_and_argmax_vs_oracle(bench_path, scan):
    model, grid, _, _, host, res = bench_path
    g = model.geometry()
    full = synth.embed_pairs(12, model.pairs(), host[scan].numpy().astype(np.float64))
    rng = np.random.default_rng(1000 + scan)
    for kind in ("das", "dmas"):
        dense = res.maps[kind][scan].numpy()
        cells = _check_cells(dense, rng, kind)
        assert len(cells) >= 1000
        pts = np.array([grid.cell_center(*c) for c in cells])
        want = orc.windowed_energies(g.antennas, g.propagation_speed, g.sample_interval, full, pts, kind,
                                     model.k0, model.window)
        got = np.array([dense[c] for c in cells], dtype=np.float64)
        ref_peak = float(np.abs(want).max())
        err = float(np.abs(got - want).max()) / ref_peak
        print(f"bench path scan {scan} {kind}: {len(cells)} px, max |gpu - oracle| / oracle peak = {err:.2e}")
        assert err <= TOL, (scan, kind, err)
        # the oracle's argmax over the checked set is the oracle's argmax of
        # the whole map (module docstring); ties -> lowest (ix, iy)
        # (beamform.py:101-104)
        best = max(range(len(cells)), key=lambda i: (want[i], -cells[i][0], -cells[i][1]))
        gpu_cell = tuple(int(v) for v in res.argmax[kind][scan])
        if gpu_cell != cells[best]:
            # excused only as a demonstrated near-tie: the oracle's values at
            # the two cells lie within the tolerance
            gap = abs(want[best] - want[cells.index(gpu_cell)]) / ref_peak
            assert gap <= TOL, (scan, kind, gpu_cell, cells[best], gap)
