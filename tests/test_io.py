"""Wire formats either side of the path (reference io.py) — byte-compatibility
with files written by the real reference (tests/golden/small.mwb,
export_small.*), typed errors, and the device staging of a loaded container."""

import json

import numpy as np
import pytest

import paper_1709_02549_b200 as mw
from _mwb_helpers import GOLDEN
from paper_1709_02549_b200 import io as mio


def test_container_round_trip_is_byte_identical(tmp_path):
    ds = mio.load_dataset(GOLDEN / "small.mwb")
    assert ds.signals.shape == (4, 4, 48) and ds.t0 == 1.5e-10
    assert ds.geometry.propagation_speed == 1.2e8 and ds.geometry.sample_interval == 2e-11
    out = tmp_path / "again.mwb"
    mio.save_dataset(ds, out)
    assert out.read_bytes() == (GOLDEN / "small.mwb").read_bytes()
    assert mio.dataset_file_size(4, 48) == len(out.read_bytes())


def test_container_errors(tmp_path):
    raw = (GOLDEN / "small.mwb").read_bytes()
    bad = tmp_path / "bad.mwb"
    bad.write_bytes(b"NOTMWB\x00\x00" + raw[8:])
    with pytest.raises(mio.DatasetFormatError, match="magic"):
        mio.load_dataset(bad)
    bad.write_bytes(raw[:8] + (2).to_bytes(4, "little") + raw[12:])
    with pytest.raises(mio.DatasetVersionError):
        mio.load_dataset(bad)
    bad.write_bytes(raw[:-10])
    with pytest.raises(mio.DatasetTruncatedError):
        mio.load_dataset(bad)
    bad.write_bytes(raw[:20])
    with pytest.raises(mio.DatasetTruncatedError):
        mio.load_dataset(bad)


@pytest.mark.gpu
def test_export_is_byte_identical_to_the_reference(tmp_path):
    side = json.loads((GOLDEN / "export_small.json").read_text())
    g = side["grid"]
    grid = mw.ImagingGrid(tuple(g["origin"]), tuple(g["extent"]), g["resolution"])
    roi = mw.Region.from_dict(side["roi"]) if side["roi"] else None
    emap = mio.import_energy_map_csv(GOLDEN / "export_small.csv", grid, side["stride"], roi)
    paths = mio.export_energy_map(emap, tmp_path / "mine")
    for ext in ("csv", "pgm", "json"):
        assert open(paths[ext], "rb").read() == (GOLDEN / f"export_small.{ext}").read_bytes(), ext


def test_csv_import_round_trip_is_exact(tmp_path):
    rng = np.random.default_rng(5)
    grid = mw.ImagingGrid((0, 0), (0.02, 0.01), 0.001)
    entries = {(int(a), int(b)): float(v) for a, b, v in zip(rng.integers(0, 20, 40), rng.integers(0, 10, 40),
                                                              rng.normal(size=40) * 1e-7)}
    path = tmp_path / "m.csv"
    path.write_text("".join(f"{a},{b},{v!r}\n" for (a, b), v in entries.items()))
    back = mio.import_energy_map_csv(path, grid, 2)
    assert back.entries == entries and back.stride == 2


def test_header_layout_matches_the_reference_struct():
    import struct

    h = np.zeros((), dtype=mio.HEADER)
    h["magic"], h["version"], h["m"], h["n"], h["dt"], h["t0"], h["v"] = mio.MAGIC, 1, 12, 1024, 2e-11, 1e-10, 1e8
    assert h.tobytes() == struct.pack("<8sIIIddd", mio.MAGIC, 1, 12, 1024, 2e-11, 1e-10, 1e8)


def _reference_export_bytes(entries, dims, stride):
    """numpy restatement of the reference's CSV and PGM bodies
    (io.py:114-136 over EnergyMap.dense, beamform.py:116-128)."""
    rows = sorted(entries.items(), key=lambda kv: (kv[0][1], kv[0][0]))
    csv = "".join(f"{ix},{iy},{float(v)!r}\n" for (ix, iy), v in rows).encode()
    nx, ny = dims
    dense = np.full((nx, ny), np.nan)
    if stride > 1:
        for (ix, iy), v in entries.items():
            if ix % stride == 0 and iy % stride == 0:
                dense[ix: min(ix + stride, nx), iy: min(iy + stride, ny)] = v
    for (ix, iy), v in entries.items():
        dense[ix, iy] = v
    vals = np.fromiter(entries.values(), dtype=np.float64)
    vmin, vmax = float(vals.min()), float(vals.max())
    if vmax > vmin:
        norm = (dense - vmin) / (vmax - vmin)
        raster = np.rint(255.0 * np.where(np.isnan(norm), 0.0, np.clip(norm, 0.0, 1.0))).astype(np.uint8)
    else:
        raster = np.zeros((nx, ny), dtype=np.uint8)
    return csv, f"P5\n{nx} {ny}\n255\n".encode() + raster.T.tobytes(), vmin, vmax


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["framework_composite", "dict_stride3", "constant", "signed_dmas"])
def test_device_render_matches_reference_exporter(tmp_path, case):
    from paper_1709_02549_b200 import synth

    model = synth.ScanModel(n_samples=512)
    ds, _ = synth.dataset_2d(model, seed=6)
    grid = synth.grid_square(0.1, 70)
    rng = np.random.default_rng(9)
    if case == "framework_composite":
        emap, _ = mw.run_framework(ds, "das", grid, mw.Manual(4), window=(model.k0, 32))  # dense-backed, stride 4
    elif case == "dict_stride3":
        cells = {(3 * a, 3 * b) for a, b in rng.integers(0, 23, (300, 2))} | {tuple(c) for c in rng.integers(0, 70, (50, 2))}
        emap = mw.EnergyMap(grid, {c: float(rng.normal()) for c in sorted(cells)}, 3)
    elif case == "constant":
        emap = mw.EnergyMap(grid, {(i, j): 2.5 for i in range(0, 70, 7) for j in range(5)}, 1)
    else:
        emap = mw.image(ds, "dmas", grid, window=(model.k0, 32), mask=mw.breast_mask(grid))
    paths = mio.export_energy_map(emap, tmp_path / case)
    csv, pgm, vmin, vmax = _reference_export_bytes(emap.entries, grid.dims, emap.stride)
    assert open(paths["csv"], "rb").read() == csv
    assert open(paths["pgm"], "rb").read() == pgm
    side = json.loads(open(paths["json"]).read())
    assert side["vmin"] == vmin and side["vmax"] == vmax and side["entries"] == len(emap.entries)


@pytest.mark.gpu
def test_render_rasters_batch_matches_single_exports(tmp_path):
    """render_rasters over a BatchImager step's maps on the device: each raster
    equals the PGM body the exporter writes for that map alone."""
    import torch

    from paper_1709_02549_b200 import synth
    from paper_1709_02549_b200.batch import BatchImager

    model = synth.ScanModel()
    sig, _ = synth.batch_2d_device(model, range(6))
    grid = synth.grid_square(0.12, 64)
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(model.k0, model.window))
    out = torch.empty((6, 64 * 64), dtype=torch.float32, device="cuda")
    bi.run_device(sig, out_dmas=out)
    valid = torch.ones((6, 64, 64), dtype=torch.bool, device="cuda")
    raster, vrange = mio.render_rasters(out.view(6, 64, 64), valid)
    host = out.view(6, 64, 64).cpu().numpy()
    for s in range(6):
        entries = {(ix, iy): float(host[s, ix, iy]) for ix in range(64) for iy in range(64)}
        _, pgm, vmin, vmax = _reference_export_bytes(entries, (64, 64), 1)
        assert mio._pgm_bytes(raster[s].cpu().numpy()) == pgm
        assert vrange[s].tolist() == [vmin, vmax]


def test_export_rejects_empty_map(tmp_path):
    grid = mw.ImagingGrid((0, 0), (0.01, 0.01), 0.001)
    with pytest.raises(ValueError):
        mio.export_energy_map(mw.EnergyMap(grid, {}), tmp_path / "x")


@pytest.mark.gpu
def test_device_staged_load_matches_host_path(tmp_path):
    import torch

    from paper_1709_02549_b200 import synth

    model = synth.ScanModel(n_samples=512)
    ds, _ = synth.dataset_2d(model, seed=4)
    path = tmp_path / "scan.mwb"
    mio.save_dataset(ds, path)
    a = mio.load_dataset(path, device=True)
    b = mio.load_dataset(path)
    grid = synth.grid_square(0.1, 60)
    for kind in ("das", "dmas"):
        assert mw.image(a, kind, grid, window=(model.k0, 32)).entries == \
            mw.image(b, kind, grid, window=(model.k0, 32)).entries
    comp, _ = mw.run_framework(a, "das", grid, mw.Manual(3))
    # the staged scan equals the host compaction (_device.scan_for) bit for bit
    from paper_1709_02549_b200 import _device as dv

    sa, sb = dv.scan_for(a), dv.scan_for(b)
    assert np.array_equal(sa.chan_host, sb.chan_host) and torch.equal(sa.sig, sb.sig)
    paths = mio.export_energy_map(comp, tmp_path / "fw")
    back = mio.import_energy_map_csv(paths["csv"], grid, 3, comp.roi)
    assert back.entries == comp.entries
