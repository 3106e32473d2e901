"""Batched multi-scan imaging (BASELINE configs[3]) — parity of the batched
launch with single-scan image() (bit-identical) and with the oracle, the
end-to-end host path, and per-scan fused argmax."""

import numpy as np
import pytest
import torch

import paper_1709_02549_b200 as mw
from _mwb_helpers import peak_err
from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    model = synth.ScanModel()
    seeds = list(range(40))
    sig, tumours = synth.batch_2d(model, seeds)
    grid = synth.grid_square(0.12, 64)
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(model.k0, model.window))
    return model, sig, tumours, grid, bi


@pytest.mark.parametrize("kind", ["das", "dmas"])
def test_batch_equals_single_scan_image(setup, kind):
    model, sig, _, grid, bi = setup
    sig_d = bi.to_device_layout(sig)
    out = torch.empty((sig.shape[0], grid.dims[0] * grid.dims[1]), dtype=torch.float32, device="cuda")
    keys = torch.zeros(sig.shape[0], dtype=torch.int64, device="cuda")
    bi.run_device(sig_d, **{f"out_{kind}": out, f"key_{kind}": keys})
    o = out.cpu().numpy().reshape(-1, *grid.dims)
    cells = bi.decode_keys(keys.cpu().numpy().view(np.uint64))
    for s in (0, 5, 39):
        ds = mw.BackscatterDataset(model.geometry(), synth.embed_pairs(12, model.pairs(), sig[s].astype(np.float64)))
        em = mw.image(ds, kind, grid, window=(model.k0, model.window))
        dense = np.zeros(grid.dims, dtype=np.float32)
        for (ix, iy), v in em.entries.items():
            dense[ix, iy] = v
        assert np.array_equal(dense, o[s])
        assert tuple(cells[s]) == em.argmax_cell()


@pytest.mark.parametrize("kind", ["das", "dmas"])
def test_batch_vs_oracle(setup, kind):
    model, sig, _, grid, bi = setup
    sig_d = bi.to_device_layout(sig)
    out = torch.empty((sig.shape[0], grid.dims[0] * grid.dims[1]), dtype=torch.float32, device="cuda")
    bi.run_device(sig_d, **{f"out_{kind}": out})
    o = out.cpu().numpy().reshape(-1, *grid.dims)
    g = model.geometry()
    for s in (3, 17):
        full = synth.embed_pairs(12, model.pairs(), sig[s].astype(np.float64))
        cells = [(ix, iy) for ix in range(0, 64, 3) for iy in range(1, 64, 5)]
        pts = np.array([grid.cell_center(*c) for c in cells])
        want = orc.windowed_energies(g.antennas, g.propagation_speed, g.sample_interval, full, pts, kind,
                                     model.k0, model.window)
        got = np.array([o[s][c] for c in cells])
        assert peak_err(got, want) <= 1e-4


def test_end_to_end_host_path_matches_device_path(setup):
    model, sig, _, grid, bi = setup
    host = torch.from_numpy(sig).pin_memory()
    res = bi(host, kinds=("das", "dmas"), chunk=16)
    sig_d = bi.to_device_layout(sig)
    for kind in ("das", "dmas"):
        out = torch.empty((sig.shape[0], grid.dims[0] * grid.dims[1]), dtype=torch.float32, device="cuda")
        keys = torch.zeros(sig.shape[0], dtype=torch.int64, device="cuda")
        bi.run_device(sig_d, **{f"out_{kind}": out, f"key_{kind}": keys})
        assert torch.equal(res.maps[kind].reshape(sig.shape[0], -1), out.cpu())
        assert np.array_equal(res.argmax[kind], bi.decode_keys(keys.cpu().numpy().view(np.uint64)))


def test_detection_rate(setup):
    model, sig, tumours, grid, bi = setup
    res = bi(torch.from_numpy(sig), kinds=("das",), chunk=64)
    hits = [max(abs(a - b) for a, b in zip(res.argmax["das"][s], grid.point_to_cell(*tumours[s]))) <= 2
            for s in range(sig.shape[0])]
    assert np.mean(hits) >= 0.9


def test_masked_batch_grid():
    model = synth.ScanModel(n_samples=512)
    sig, _ = synth.batch_2d(model, range(6))
    grid = synth.grid_square(0.1, 50)
    mask = mw.breast_mask(grid)
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(model.k0, 32), mask=mask)
    assert bi.n_pts == int(mask.sum())
    res = bi(torch.from_numpy(sig), kinds=("dmas",))
    ds = mw.BackscatterDataset(model.geometry(), synth.embed_pairs(12, model.pairs(), sig[2].astype(np.float64)))
    em = mw.image(ds, "dmas", grid, mask=mask, window=(model.k0, 32))
    m = res.maps["dmas"][2].numpy()
    for (ix, iy), v in em.entries.items():
        assert m[ix, iy] == np.float32(v)


def test_fused_launch_equals_single_kind_launches(setup):
    model, sig, _, grid, bi = setup
    sig_d = bi.to_device_layout(sig)
    shape = (sig.shape[0], grid.dims[0] * grid.dims[1])
    both = [torch.empty(shape, dtype=torch.float32, device="cuda") for _ in range(2)]
    keys = [torch.zeros(sig.shape[0], dtype=torch.int64, device="cuda") for _ in range(4)]
    bi.run_device(sig_d, both[0], both[1], keys[0], keys[1])
    das = torch.empty(shape, dtype=torch.float32, device="cuda")
    dmas = torch.empty(shape, dtype=torch.float32, device="cuda")
    bi.run_device(sig_d, out_das=das, key_das=keys[2])
    bi.run_device(sig_d, out_dmas=dmas, key_dmas=keys[3])
    assert torch.equal(both[0], das) and torch.equal(both[1], dmas)
    assert torch.equal(keys[0], keys[2]) and torch.equal(keys[1], keys[3])


def test_gather_mode_bit_identical(setup):
    model, sig, _, grid, bi = setup
    sig_d = bi.to_device_layout(sig[:8])
    shape = (8, grid.dims[0] * grid.dims[1])
    a = [torch.empty(shape, dtype=torch.float32, device="cuda") for _ in range(2)]
    b = [torch.empty(shape, dtype=torch.float32, device="cuda") for _ in range(2)]
    bi.run_device(sig_d, a[0], a[1])
    bi.mode = 1
    try:
        bi.run_device(sig_d, b[0], b[1])
    finally:
        bi.mode = 0
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_images_pair_equals_image():
    model = synth.ScanModel(n_samples=256)
    ds, _ = synth.dataset_2d(model, seed=21)
    grid = synth.grid_square(0.1, 40)
    pair = mw.images(ds, ("das", "dmas"), grid, stride=2, window=(model.k0, 32))
    for kind in ("das", "dmas"):
        assert pair[kind].entries == mw.image(ds, kind, grid, stride=2, window=(model.k0, 32)).entries


def test_end_to_end_ramp_and_buffer_reuse_smem_mode():
    """__call__ with S >= 6 * chunk (the ramped chunk sizes) and more chunks
    than buffer sets, on the CUDA-core kernel: bit-identical to run_device
    (tests/test_gpu_bench_path.py covers the tensor-core mode)."""
    from paper_1709_02549_b200.batch import _chunk_ranges

    model = synth.ScanModel()
    sig, _ = synth.batch_2d(model, list(range(100, 196)))
    grid = synth.grid_square(0.12, 48)
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(model.k0, model.window),
                     mode="smem")
    assert len(_chunk_ranges(96, 16)) > 4 and _chunk_ranges(96, 16)[0] == (0, 4)
    res = bi(torch.from_numpy(sig).pin_memory(), kinds=("das", "dmas"), chunk=16)
    sig_d = bi.to_device_layout(sig)
    n = grid.dims[0] * grid.dims[1]
    for kind in ("das", "dmas"):
        out = torch.empty((96, n), dtype=torch.float32, device="cuda")
        keys = torch.zeros(96, dtype=torch.int64, device="cuda")
        bi.run_device(sig_d, **{f"out_{kind}": out, f"key_{kind}": keys})
        assert torch.equal(res.maps[kind].reshape(96, -1), out.cpu())
        assert np.array_equal(res.argmax[kind], bi.decode_keys(keys.cpu().numpy().view(np.uint64)))


def test_end_to_end_full_record_tensor_cores():
    """__call__ over the full record on the tensor-core path
    (mwb_energies_tc_record): the host pipeline ships the union of the
    chunks' sample ranges and returns exactly what run_device writes."""
    model = synth.ScanModel()
    sig, _ = synth.batch_2d(model, list(range(300, 340)))
    grid = synth.grid_square(0.024, 48)  # 0.5 mm: every tile within the tensor-core path's delay spread
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(0, model.n_samples),
                     mode="auto")
    assert bi.uses_tensor_cores and bi.tc_record
    first, count = bi.input_range()
    assert 0 <= first and first + count <= model.n_samples
    res = bi(torch.from_numpy(sig).pin_memory(), kinds=("das", "dmas"), chunk=16)
    sig_d = bi.to_device_layout(sig)
    n = grid.dims[0] * grid.dims[1]
    outs = {k: torch.zeros((40, n), dtype=torch.float32, device="cuda") for k in ("das", "dmas")}
    keys = {k: torch.zeros(40, dtype=torch.int64, device="cuda") for k in ("das", "dmas")}
    bi.run_device(sig_d, outs["das"], outs["dmas"], keys["das"], keys["dmas"])
    for kind in ("das", "dmas"):
        assert torch.equal(res.maps[kind].reshape(40, -1), outs[kind].cpu())
        assert np.array_equal(res.argmax[kind], bi.decode_keys(keys[kind].cpu().numpy().view(np.uint64)))
