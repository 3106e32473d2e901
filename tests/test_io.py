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


def test_export_is_byte_identical_to_the_reference(tmp_path):
    side = json.loads((GOLDEN / "export_small.json").read_text())
    g = side["grid"]
    grid = mw.ImagingGrid(tuple(g["origin"]), tuple(g["extent"]), g["resolution"])
    roi = mw.Region.from_dict(side["roi"]) if side["roi"] else None
    emap = mio.import_energy_map_csv(GOLDEN / "export_small.csv", grid, side["stride"], roi)
    paths = mio.export_energy_map(emap, tmp_path / "mine")
    for ext in ("csv", "pgm", "json"):
        assert open(paths[ext], "rb").read() == (GOLDEN / f"export_small.{ext}").read_bytes(), ext


def test_export_rejects_empty_map(tmp_path):
    grid = mw.ImagingGrid((0, 0), (0.01, 0.01), 0.001)
    with pytest.raises(ValueError):
        mio.export_energy_map(mw.EnergyMap(grid, {}), tmp_path / "x")


@pytest.mark.gpu
def test_device_staged_load_matches_host_path(tmp_path):
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
    paths = mio.export_energy_map(comp, tmp_path / "fw")
    back = mio.import_energy_map_csv(paths["csv"], grid, 3, comp.roi)
    assert back.entries == comp.entries
