"""Tensor-core energy path (mwb_energies_tc, BatchImager(mode="tc")) against
the fp32 CUDA-core path and the oracle.

The tensor-core path computes the same energies with a different summation
(fp16 hi/lo split products accumulated in TMEM, DMAS self-terms from windowed
Gram entries), so it is compared at tolerance, not bit for bit:
  * vs the fp32 CUDA-core kernel: max |tc - fp32| / max |fp32| <= 3e-5 per scan
    (measured ~1e-5: TMEM accumulation over 3 x 66 MMAs rounds toward zero);
  * vs the oracle (the reference's fp64 algorithm): <= 1e-4 peak-normalised
    (BASELINE's bound), like every other energy map.
"""

import numpy as np
import pytest
import torch

from _mwb_helpers import peak_err
from oracle import mwbeam_oracle as orc
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.batch import BatchImager

pytestmark = pytest.mark.gpu

TOL_FP32 = 3e-5  # measured: see profiles/r01_tc.md
TOL_REF = 1e-4


@pytest.fixture(scope="module")
def setup():
    model = synth.ScanModel()
    seeds = list(range(37))  # not a multiple of the 8-scan group
    sig, tumours = synth.batch_2d(model, seeds)
    grid = synth.grid_square(0.06, 128)  # 0.47 mm pitch, the configs[3] resolution
    win = (model.k0, model.window)
    tc = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, mode="tc")
    ref = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win)
    return model, sig, grid, tc, ref


def run(bi, sig_d, kinds=("das", "dmas")):
    s = sig_d.shape[0]
    n = bi.grid.dims[0] * bi.grid.dims[1]
    outs = {k: torch.full((s, n), np.nan, dtype=torch.float32, device="cuda") for k in kinds}
    keys = {k: torch.zeros(s, dtype=torch.int64, device="cuda") for k in kinds}
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    bi.run_device(sig_d, outs.get("das"), outs.get("dmas"), keys.get("das"), keys.get("dmas"), flags)
    return ({k: v.cpu().numpy() for k, v in outs.items()},
            {k: bi.decode_keys(v.cpu().numpy().view(np.uint64)) for k, v in keys.items()}, int(flags.item()))


def test_tc_is_selected(setup):
    _, _, _, tc, ref = setup
    assert tc.uses_tensor_cores and not ref.uses_tensor_cores


@pytest.mark.parametrize("kinds", [("das", "dmas"), ("das",), ("dmas",)])
def test_tc_matches_fp32_path(setup, kinds):
    _, sig, grid, tc, ref = setup
    sig_d = tc.to_device_layout(sig)
    got, gk, gf = run(tc, sig_d, kinds)
    want, wk, wf = run(ref, sig_d, kinds)
    assert gf == wf == 0
    for k in kinds:
        assert not np.isnan(got[k]).any()
        for s in range(sig.shape[0]):
            assert peak_err(got[k][s], want[k][s]) <= TOL_FP32, (k, s)
        # argmax: identical unless the fp32 map has a near-tie at the top
        for s in range(sig.shape[0]):
            if tuple(gk[k][s]) != tuple(wk[k][s]):
                top = np.sort(want[k][s])[-2:]
                assert (top[1] - top[0]) <= 1e-5 * abs(top[1]), (k, s)


def test_tc_vs_oracle(setup):
    model, sig, grid, tc, _ = setup
    got, _, _ = run(tc, tc.to_device_layout(sig))
    g = model.geometry()
    ny = grid.dims[1]
    cells = [(ix, iy) for ix in range(0, 128, 7) for iy in range(3, 128, 9)]
    pts = np.array([grid.cell_center(*c) for c in cells])
    slots = np.array([ix * ny + iy for ix, iy in cells])
    for s in (0, 36):
        full = synth.embed_pairs(12, model.pairs(), sig[s].astype(np.float64))
        for kind in ("das", "dmas"):
            want = orc.windowed_energies(g.antennas, g.propagation_speed, g.sample_interval, full, pts, kind,
                                         model.k0, model.window)
            assert peak_err(got[kind][s][slots], want) <= TOL_REF


def test_tc_scale_invariance_and_zero_scan(setup):
    """Per-scan power-of-two scaling: scans 10^6 x larger / smaller give the
    same relative maps; an all-zero scan images to exactly zero."""
    _, sig, _, tc, ref = setup
    x = np.array(sig[:8], dtype=np.float32)
    x[1] *= 1e6
    x[2] *= 1e-6
    x[3] = 0.0
    sig_d = tc.to_device_layout(x)
    got, _, _ = run(tc, sig_d)
    want, _, _ = run(ref, sig_d)
    for k in ("das", "dmas"):
        for s in (0, 1, 2):
            assert peak_err(got[k][s], want[k][s]) <= TOL_FP32
        assert (got[k][3] == 0).all()


def test_tc_flags_non_finite(setup):
    _, sig, _, tc, _ = setup
    x = np.array(sig[:3], dtype=np.float32)
    x[1, 5, :] = np.nan  # inside every window of scan 1
    got, _, flags = run(tc, tc.to_device_layout(x))
    assert flags & 1
    assert np.isfinite(got["das"][0]).all() and np.isfinite(got["das"][2]).all()  # other scans unaffected


def test_tc_masked_ragged_grid_padded_tiles():
    """A breast mask on a ragged grid leaves partial lattice tiles; the padded
    layout (table tile = 16 x 16 lattice tile, per-tile counts) keeps them on
    the tensor cores, with cells outside the mask untouched."""
    import paper_1709_02549_b200 as mw

    model = synth.ScanModel()
    sig, _ = synth.batch_2d(model, list(range(11)))
    grid = synth.grid_square(0.05, 107)  # 0.47 mm, 107 = 6 x 16 + 11
    mask = mw.breast_mask(grid)
    win = (model.k0, model.window)
    tc = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, mask=mask, mode="tc")
    ref = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, mask=mask)
    assert tc.uses_tensor_cores and tc.n_valid == ref.n_pts == int(mask.sum()) and tc.n_pts % 256 == 0
    sig_d = tc.to_device_layout(sig)
    got, gk, _ = run(tc, sig_d)
    want, wk, _ = run(ref, sig_d)
    inside = mask.reshape(-1)
    for k in ("das", "dmas"):
        assert np.isnan(got[k][:, ~inside]).all()  # untouched outside the mask
        for s in range(11):
            assert peak_err(got[k][s][inside], want[k][s][inside]) <= TOL_FP32
            assert tuple(gk[k][s]) == tuple(wk[k][s])


def test_tc_eligibility():
    model = synth.ScanModel()
    coarse = synth.grid_square(0.12, 64)  # 1.9 mm pitch: tile spreads exceed 14 samples
    with pytest.raises(ValueError, match="spread"):
        BatchImager(model.geometry(), model.pairs(), model.n_samples, coarse, window=(model.k0, 32), mode="tc")
    auto = BatchImager(model.geometry(), model.pairs(), model.n_samples, coarse, window=(model.k0, 32), mode="auto")
    assert not auto.uses_tensor_cores
    fine = synth.grid_square(0.03, 64)
    with pytest.raises(ValueError, match="window"):
        BatchImager(model.geometry(), model.pairs(), model.n_samples, fine, window=(model.k0, 40), mode="tc")


def test_tc_nearest_interpolation(setup):
    model, sig, grid, _, _ = setup
    win = (model.k0, model.window)
    tc = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, mode="tc",
                     interpolation="nearest")
    ref = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, interpolation="nearest")
    sig_d = tc.to_device_layout(sig[:9])
    got, _, _ = run(tc, sig_d)
    want, _, _ = run(ref, sig_d)
    for k in ("das", "dmas"):
        for s in range(9):
            assert peak_err(got[k][s], want[k][s]) <= TOL_FP32


def test_tc_window_past_record_end():
    """Windows that run past the record read zeros (beamform.py:192-193): the
    producer zero-fills the staged spans beyond ld."""
    model = synth.ScanModel(n_samples=1024)
    sig, _ = synth.batch_2d(model, list(range(8)))
    short = np.ascontiguousarray(sig[:, :, 300:600])  # 300-sample records: late windows overrun
    grid = synth.grid_square(0.06, 96)
    win = (180, 32)  # delays 40..100 samples: windows straddle the 300-sample record end
    tc = BatchImager(model.geometry(), model.pairs(), 300, grid, window=win, mode="tc")
    ref = BatchImager(model.geometry(), model.pairs(), 300, grid, window=win)
    sig_d = tc.to_device_layout(short)
    got, _, _ = run(tc, sig_d)
    want, _, _ = run(ref, sig_d)
    # the cut matters: the same scans with 100 more samples image differently
    longer = np.ascontiguousarray(sig[:, :, 300:700])
    ref_long = BatchImager(model.geometry(), model.pairs(), 400, grid, window=win)
    want_long, _, _ = run(ref_long, ref_long.to_device_layout(longer))
    for k in ("das", "dmas"):
        assert np.abs(want_long[k] - want[k]).max() > 1e-3 * np.abs(want_long[k]).max()
        for s in range(8):
            assert peak_err(got[k][s], want[k][s]) <= TOL_FP32


@pytest.mark.parametrize("n_scans", [1, 3, 9])
def test_tc_window_48(setup, n_scans):
    """W = 48 (configs[4]'s window): 4-scan groups (N = 192) for batches, one
    scan per group (N = 48) below 4 scans."""
    model, sig, grid, _, _ = setup
    win = (model.k0, 48)
    tc = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, mode="tc")
    ref = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win)
    sig_d = tc.to_device_layout(sig[:n_scans])
    got, gk, flags = run(tc, sig_d)
    want, wk, _ = run(ref, sig_d)
    assert flags == 0
    for k in ("das", "dmas"):
        for s in range(n_scans):
            assert peak_err(got[k][s], want[k][s]) <= TOL_FP32
            assert tuple(gk[k][s]) == tuple(wk[k][s])


@pytest.mark.parametrize("n_chan,n_scans", [(1, 1), (5, 17), (24, 16), (25, 3), (49, 33)])
def test_tch_channel_and_scan_counts(setup, n_chan, n_scans):
    """The W = 32 kernel's step plan and staging ring at the edges: one
    channel; fewer channels than ring slots (24); exactly one ring lap; a
    lap plus one (the next item's first channel lands in slot 0 and its
    mirror); 49 channels with two laps per item; scan counts that leave the
    last 8-scan group, or the last group pair, partly empty."""
    model, sig, grid, _, _ = setup
    win = (model.k0, model.window)
    pairs = model.pairs()[:n_chan]
    tc = BatchImager(model.geometry(), pairs, model.n_samples, grid, window=win, mode="tc")
    ref = BatchImager(model.geometry(), pairs, model.n_samples, grid, window=win)
    assert tc.uses_tensor_cores
    sub = np.ascontiguousarray(np.resize(sig, (n_scans,) + sig.shape[1:])[:, :n_chan])
    sig_d = tc.to_device_layout(sub)
    got, gk, flags = run(tc, sig_d)
    want, wk, _ = run(ref, sig_d)
    assert flags == 0
    for k in ("das", "dmas"):
        for s in range(n_scans):
            if n_chan == 1 and k == "dmas":
                # one channel: DMAS is 0 up to the rounding of S^2 - Q
                assert np.abs(got[k][s]).max() <= TOL_FP32 * np.abs(got["das"][s]).max()
                continue
            assert peak_err(got[k][s], want[k][s]) <= TOL_FP32, (k, s)
            top = np.sort(want[k][s])[-2:]
            if top[1] - top[0] > 2 * TOL_FP32 * abs(top[1]):  # few channels: flat maxima tie within rounding
                assert tuple(gk[k][s]) == tuple(wk[k][s]), (k, s)


def test_tch_many_channels_hemisphere():
    """496 channels (configs[4]'s 32-antenna hemisphere) on a 2-D grid at W = 32:
    20 staging-ring laps per item, the mirror slot on every lap, and 2-half
    channels; 17 scans (a partial last group pair)."""
    vm = synth.VolumeModel()
    n_scans = 17
    sig = np.stack([synth.scan_3d(vm, seed)[0] for seed in range(n_scans)]).astype(np.float32)
    grid = synth.grid_square(0.02, 48)
    win = (vm.k0, 32)
    tc = BatchImager(vm.geometry(), vm.pairs(), vm.n_samples, grid, window=win, mode="tc")
    ref = BatchImager(vm.geometry(), vm.pairs(), vm.n_samples, grid, window=win)
    assert tc.uses_tensor_cores and tc.n_chan == 496
    sig_d = tc.to_device_layout(sig)
    got, gk, flags = run(tc, sig_d)
    want, wk, _ = run(ref, sig_d)
    assert flags == 0
    # the fp32 TMEM accumulation rounds toward zero once per MMA, so the
    # tensor-core maps carry a small negative bias that grows with the number
    # of accumulated steps: ~7e-6 of the peak at 66 channels, ~3e-5 at 496
    # (measured); still inside BASELINE's 1e-4
    for k in ("das", "dmas"):
        for s in range(n_scans):
            assert peak_err(got[k][s], want[k][s]) <= 6e-5, (k, s)


@pytest.mark.parametrize("window", ["full", 64])
def test_tc_record_windows(setup, window):
    """Windows of several 32-sample chunks on the tensor cores
    (mwb_energies_tc_record): the reference's default full record
    (beamform.py:211-212) and a 2-chunk window, against the fp32 CUDA-core
    kernel over the same window; cells outside the mask stay untouched."""
    model, sig, grid, _, _ = setup
    win = (0, model.n_samples) if window == "full" else (model.k0, 64)
    nx, ny = grid.dims
    yy, xx = np.meshgrid(np.arange(ny), np.arange(nx))
    mask = (xx - nx / 2) ** 2 + (yy - ny / 2) ** 2 <= (0.45 * nx) ** 2
    tc = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, mask=mask, mode="auto")
    ref = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=win, mask=mask)
    assert tc.uses_tensor_cores and tc.tc_record and not ref.uses_tensor_cores
    n = 9
    sig_d = tc.to_device_layout(sig[:n])
    got, gk, flags = run(tc, sig_d)
    want, wk, _ = run(ref, sig_d)
    assert flags == 0
    inside = mask.reshape(-1)
    # each chunk carries the TMEM accumulation bias of its S^2; over the full
    # record the noise energy of 32 chunks makes S^2 and Q large against the
    # DMAS peak, so the DMAS error relative to that peak grows (3.2e-5
    # measured), inside BASELINE's 1e-4
    tol = TOL_REF if window == "full" else TOL_FP32
    for k in ("das", "dmas"):
        assert np.isnan(got[k][:, ~inside]).all()  # untouched
        for s in range(n):
            assert peak_err(got[k][s][inside], want[k][s][inside]) <= tol, (k, s)
            top = np.sort(want[k][s][inside])[-2:]
            if top[1] - top[0] > 2 * TOL_FP32 * abs(top[1]):
                assert tuple(gk[k][s]) == tuple(wk[k][s]), (k, s)


@pytest.mark.parametrize("seed", range(8))
def test_tch_fuzz_geometries_vs_oracle(seed):
    """Seeded random set-ups around configs[3]: ring radius, permittivity
    (sample scale), antenna count, window start, off-centre rectangular grids
    with ragged dims and pitches up to the tensor-core limit, scan counts that
    are no multiple of 8 or 16.  Whatever kernel mode="auto" picks, sampled
    pixels agree with the oracle (reference fp64 algorithm, beamform.py:169-212)
    within BASELINE's 1e-4 of the oracle's peak; when it picks the tensor
    cores, the whole maps also agree with the fp32 CUDA-core kernel."""
    from paper_1709_02549_b200.geometry import ImagingGrid

    rng = np.random.default_rng(1000 + seed)
    model = synth.ScanModel(n_ant=int(rng.integers(4, 13)), ring_radius=float(rng.uniform(0.06, 0.09)),
                            eps_r=float(rng.uniform(6.0, 12.0)), t_c=float(rng.uniform(400e-12, 900e-12)))
    n_scans = int(rng.integers(1, 21))
    sig, _ = synth.batch_2d(model, [int(s) for s in rng.integers(0, 10_000, n_scans)], phantom_radius=(0.02, 0.03))
    res = float(rng.uniform(0.25e-3, 0.6e-3))
    nx, ny = (int(v) for v in rng.integers(20, 90, 2))
    origin = (float(rng.uniform(-0.03, 0.0)), float(rng.uniform(-0.03, 0.0)))
    grid = ImagingGrid(origin, (nx * res, ny * res), res)
    assert grid.dims == (nx, ny)
    win = (max(0, model.k0 + int(rng.integers(-6, 7))), 32)
    g, pairs = model.geometry(), model.pairs()
    auto = BatchImager(g, pairs, model.n_samples, grid, window=win, mode="auto")
    ref = BatchImager(g, pairs, model.n_samples, grid, window=win)
    sig_d = auto.to_device_layout(sig)
    got, gk, flags = run(auto, sig_d)
    want, wk, _ = run(ref, sig_d)
    assert flags == 0
    worst = {"fp32": 0.0, "oracle": 0.0}
    if auto.uses_tensor_cores:
        for k in ("das", "dmas"):
            for s in range(n_scans):
                worst["fp32"] = max(worst["fp32"], peak_err(got[k][s], want[k][s]))
                assert peak_err(got[k][s], want[k][s]) <= TOL_FP32, (k, s)
    cells = [(int(ix), int(iy)) for ix, iy in zip(rng.integers(0, nx, 60), rng.integers(0, ny, 60))]
    for s in sorted({0, n_scans - 1}):
        check = cells + [tuple(int(v) for v in wk[k][s]) for k in ("das", "dmas")]
        pts = np.array([grid.cell_center(*c) for c in check])
        slots = np.array([ix * ny + iy for ix, iy in check])
        full = synth.embed_pairs(model.n_ant, pairs, sig[s].astype(np.float64))
        for kind in ("das", "dmas"):
            o = orc.windowed_energies(g.antennas, g.propagation_speed, g.sample_interval, full, pts, kind, *win)
            peak = max(np.abs(o).max(), np.abs(want[kind][s]).max())
            worst["oracle"] = max(worst["oracle"], np.abs(got[kind][s][slots] - o).max() / peak)
            assert np.abs(got[kind][s][slots] - o).max() <= TOL_REF * peak
    print(f"fuzz {seed}: M={model.n_ant} C={len(pairs)} S={n_scans} grid={nx}x{ny} res={res * 1e3:.3f} mm "
          f"tc={auto.uses_tensor_cores} vs fp32 {worst['fp32']:.2e} vs oracle {worst['oracle']:.2e}")
