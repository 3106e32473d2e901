"""The C-ABI library loads and exports every symbol include/mwb.h declares
(CPU-only: no compute call needs a GPU; argument validation runs before any
CUDA call, so error paths are testable here)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1709_02549_b200 import _build, _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "mwb.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mwb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _native.load()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 8
    for name in names:
        assert hasattr(lib, name), name


def test_binding_covers_header():
    assert set(declared_functions()) == set(_native.EXPORTED)


def test_integration_lists_every_export():
    """INTEGRATION.md names every entry point a maintainer could bind."""
    doc = (HEADER.parents[1] / "INTEGRATION.md").read_text()
    missing = [n for n in declared_functions() if not re.search(rf"\b{n}\b", doc)]
    assert not missing, missing


def test_trace_layout_matches_c(lib):
    assert lib.mwb_trace_bytes() == _native.TRACE_BYTES
    assert ctypes.sizeof(_native.IterRecord) == 496


def test_version(lib):
    assert lib.mwb_version() >= 1


def energies_args(**kw):
    """Positional argument list of mwb_energies (include/mwb.h) with overrides."""
    names = ["sig", "n_scans", "scan_stride", "n_chan", "ld", "n_samples", "chan", "ant", "n_ant", "inv_scale",
             "pts", "out_idx", "n_pts", "d_count", "table", "interp", "k0", "window", "out_das", "out_dmas",
             "out_stride", "key_das", "key_dmas", "flags", "mode", "stream"]
    base = dict(sig=None, n_scans=1, scan_stride=0, n_chan=1, ld=4, n_samples=4, chan=None, ant=None, n_ant=2,
                inv_scale=1.0, pts=None, out_idx=None, n_pts=1, d_count=None, table=None, interp=0, k0=0, window=4,
                out_das=None, out_dmas=None, out_stride=0, key_das=None, key_dmas=None, flags=None, mode=0,
                stream=None)
    base.update(kw)
    assert len(names) == len(_native._SIGNATURES["mwb_energies"][0])
    return [base[n] for n in names]


def test_argument_errors_set_last_error(lib):
    assert lib.mwb_energies(*energies_args(n_pts=-1)) == -1
    assert b"negative" in lib.mwb_last_error()
    assert lib.mwb_energies(*energies_args()) == -1
    assert b"no output" in lib.mwb_last_error()
    assert lib.mwb_energies(*energies_args(out_das=16, interp=5)) == -1
    assert b"interpolation" in lib.mwb_last_error()
    assert lib.mwb_energies(*energies_args(out_das=16, ld=6)) == -1
    assert b"multiples of 4" in lib.mwb_last_error()
    assert lib.mwb_energies(*energies_args(out_das=16, n_ant=99)) == -3
    assert lib.mwb_delay_table(None, 10, None, None, 0, None, 2, 1.0, 0, None, None) == -1
    assert lib.mwb_delay_table_bytes(1000, 66) >= 1000 * 66 * 4
    assert lib.mwb_delay_table_bytes(-1, 66) == -1
    rc = lib.mwb_select_roi(None, None, 10, 10, 1, 0, 0, 10, 9, 0.25, 4, None, None, None)
    assert rc == -1 and b"outside" in lib.mwb_last_error()
    rc = lib.mwb_select_roi(None, None, 10, 10, 1, 0, 0, 9, 9, 1.5, 4, None, None, None)
    assert rc == -1 and b"frame_fraction" in lib.mwb_last_error()
    rc = lib.mwb_enumerate_lattice(0.0, 0.0, 1.0, 10, 10, 0, 0, 9, 9, None, 0, None, 0, None, None, None, None,
                                   None, None)
    assert rc == -1
    assert lib.mwb_lattice_workspace_bytes(0, 5, 1) == -1
    assert lib.mwb_lattice_workspace_bytes(100, 100, 1) > 0
    assert lib.mwb_image_lattice_workspace_bytes(100, 100, 0, 66) == -1
    assert lib.mwb_image_lattice_workspace_bytes(100, 100, 2, 66) >= 50 * 50 * (24 + 4 + 66 * 4)
    rc = lib.mwb_image_lattice(None, 66, 1024, 1024, None, None, 12, 1.0, 0, 0, 32, 0.0, 0.0, 1e-3, 100, 100,
                               0, 0, 99, 99, 1, None, 0, None, None, None, None, None, None, None, None, None)
    assert rc == -1 and b"no output" in lib.mwb_last_error()


def test_native_check_raises_with_message(lib):
    lib.mwb_argmax_dense(None, None, -1, None, None)
    with pytest.raises(RuntimeError, match="bad arguments"):
        _native.check(-1, "mwb_argmax_dense")


def test_sass_is_sm100a():
    """The built library carries sm_100a SASS with FFMA2 and TMA bulk copies."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    _build.build()
    out = subprocess.run([tool, "-sass", str(_build.LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "FFMA2" in out
    assert "UBLKCP" in out


def tc_args(**kw):
    """Positional argument list of mwb_energies_tc (include/mwb.h) with overrides;
    fake non-null pointers pass the null checks (nothing is dereferenced before
    the argument errors tested here)."""
    names = ["sig", "n_scans", "scan_stride", "n_chan", "ld", "n_samples", "chan", "ant", "n_ant", "inv_scale",
             "pts", "out_idx", "n_pts", "d_count", "tile_info", "table", "interp", "k0", "window", "out_das",
             "out_dmas", "out_stride", "key_das", "key_dmas", "flags", "j_lo", "j_count", "workspace", "stream"]
    base = dict(sig=256, n_scans=8, scan_stride=4096, n_chan=66, ld=1024, n_samples=1024, chan=256, ant=256,
                n_ant=12, inv_scale=500.0, pts=256, out_idx=None, n_pts=256, d_count=None, tile_info=None,
                table=256, interp=0, k0=8, window=32, out_das=256, out_dmas=None, out_stride=0, key_das=None,
                key_dmas=None, flags=None, j_lo=10, j_count=64, workspace=256, stream=None)
    base.update(kw)
    assert len(names) == len(_native._SIGNATURES["mwb_energies_tc"][0])
    return [base[n] for n in names]


def test_tensor_core_entry_argument_errors(lib):
    assert lib.mwb_energies_tc(*tc_args(window=40)) == -1
    assert b"window must be 32 or 48" in lib.mwb_last_error()
    assert lib.mwb_energies_tc(*tc_args(workspace=None)) == -1
    assert b"workspace" in lib.mwb_last_error()
    assert lib.mwb_energies_tc(*tc_args(j_count=8)) == -1
    assert b"window-offset range" in lib.mwb_last_error()
    assert lib.mwb_energies_tc(*tc_args(out_das=None)) == -1
    assert b"no output" in lib.mwb_last_error()
    assert lib.mwb_energies_tc(*tc_args(n_pts=0)) == 0  # nothing to do
    assert lib.mwb_energies_tc_workspace_bytes(8, 66, 8, 256) == -1
    assert lib.mwb_energies_tc_workspace_bytes(8, 66, 64, -1) == -1
    small = lib.mwb_energies_tc_workspace_bytes(8, 66, 64, 256)
    assert small >= 2 * 16 * 2 * 66 * 64 + 8 * 66 * 4
    assert lib.mwb_energies_tc_workspace_bytes(4096, 66, 152, 65536) > 4096 * 66 * 152 * 8 + 256 * 8 * 66 * 4
    steps = ctypes.c_int64()
    assert lib.mwb_tc_plan_steps(None, 8, 66, 64, 256, 32, ctypes.byref(steps)) == -1
    assert lib.mwb_tc_plan_steps(ctypes.c_void_p(16), 8, 66, 64, 256, 48, ctypes.byref(steps)) == -1
    assert b"window 32" in lib.mwb_last_error()
    assert lib.mwb_table_max_span(None, 10, 66, None, None) == -1
    assert lib.mwb_table_lo_range(None, 10, 66, None, None, None) == -1
    assert lib.mwb_lattice_tile_count(256, 256, 1) == 256
    assert lib.mwb_lattice_tile_count(100, 100, 1) == 49
    assert lib.mwb_enumerate_lattice_padded(0.0, 0.0, 1.0, 10, 10, 0, 0, 10, 9, 1, None, 0, None, None, None, None,
                                            None, None, None) == -1
    assert b"outside" in lib.mwb_last_error()


def _tree_counts(region, stop, max_iters):
    """Python restatement of the region tree (Region.quadrants split,
    geometry.py:225-242; a region is split while its larger side exceeds the
    stop size and both sides are >= 2, for at most max_iters levels)."""
    search = term = 0
    fine_tps = 0
    todo = [(region, 0)]
    while todo:
        (x0, y0, x1, y1), depth = todo.pop()
        w, h = x1 - x0 + 1, y1 - y0 + 1
        if max(w, h) <= stop or w < 2 or h < 2 or depth >= max_iters:
            term += 1
            fine_tps = max(fine_tps, -(-(w * h) // 256))
            continue
        search += 1
        mx, my = x0 + (w + 1) // 2 - 1, y0 + (h + 1) // 2 - 1
        for qx0, qx1 in ((x0, mx), (mx + 1, x1)):
            for qy0, qy1 in ((y0, my), (my + 1, y1)):
                todo.append(((qx0, qy0, qx1, qy1), depth + 1))
    return search, term, fine_tps


@pytest.mark.parametrize("region,stop,iters", [((0, 0, 403, 403), 40, 4), ((3, 11, 190, 170), 8, 5),
                                               ((0, 0, 39, 39), 40, 0), ((0, 0, 480, 100), 40, 4)])
def test_segment_plan_info_matches_tree(lib, region, stop, iters):
    """The host-side region tree behind mwb_segment_plan_* (no GPU needed)."""
    info = (ctypes.c_int64 * 4)()
    x0, y0, x1, y1 = region
    assert lib.mwb_segment_plan_info(x1 + 1, y1 + 1, x0, y0, x1, y1, 16, stop, iters, 66, info) == 0
    search, term, fine_tps = _tree_counts(region, stop, iters)
    assert (info[1], info[2], info[3]) == (search, term, fine_tps)
    assert info[0] > 0


def test_segment_plan_info_rejects_huge_trees_and_bad_args(lib):
    info = (ctypes.c_int64 * 4)()
    assert lib.mwb_segment_plan_info(4096, 4096, 0, 0, 4095, 4095, 16, 1, 12, 66, info) != 0  # > 16384 regions
    assert b"too many regions" in lib.mwb_last_error()
    assert lib.mwb_segment_plan_info(100, 100, 0, 0, 100, 99, 16, 8, 4, 66, info) != 0  # region outside the grid
    assert lib.mwb_segment_plan_info(100, 100, 0, 0, 99, 99, 0, 8, 4, 66, info) != 0  # n_sub
    assert lib.mwb_segment_run_workspace_bytes(0, 16, 3, 32) == -1


def test_round2_entry_points_validate_arguments(lib):
    """The round-2 entry points reject bad arguments before any CUDA call."""
    import ctypes

    rc = lib.mwb_energies_region(None, 66, 1024, 1024, None, None, 12, 1.0, None, None, 256, None, None, 0, 0, 32,
                                 None, None, None, None, None, None, 10, 3, None, None, 0, None, 0, None)
    assert rc == -1 and b"mwb_energies_region" in lib.mwb_last_error()
    assert lib.mwb_render_pgm(None, 16, None, 1, 4, 4, 16, 1, None, None, None) == -1
    assert b"value_bits" in lib.mwb_last_error()
    assert lib.mwb_render_pgm(None, 32, None, 1, 4, 4, 8, 1, None, None, None) == -1  # map_stride < nx*ny
    assert lib.mwb_compact_payload(None, 0, 10, 12, None, None, None, None, None) == -1
    assert lib.mwb_compact_payload(None, 4, 10, 8, None, None, None, None, None) == -1  # ld < n
    assert lib.mwb_gather_composite(None, 10, 1, None, 0, None, None, 0, None) == -1
    assert lib.mwb_memcpy2d_async(None, 4, None, 16, 8, 1, None) == -1  # dpitch < width
    assert lib.mwb_memcpy_async(None, None, 0, None) == 0  # nothing to copy
    assert lib.mwb_elapsed_ms(None, 1, None) == -1
    out = (ctypes.c_int32 * 2)()
    assert lib.mwb_tc_sample_range(477, 10, 150, 1024, out) == 0
    first, count = out[0], out[1]
    assert first == 487 and 150 + 32 <= count <= 1024 - first  # covers every window offset plus W
    assert lib.mwb_tc_sample_range(1000, 10, 150, 1024, out) == 0 and out[0] + out[1] == 1024  # clipped to ld
    assert lib.mwb_tc_sample_range(0, 0, 8, 1024, out) == -1  # fewer than 16 offsets


def test_compact_rows_host_matches_numpy():
    """mwb_compact_rows_host (a host function: no GPU needed) keeps exactly the
    rows numpy's flat != 0.0 keeps (-0.0 is zero, NaN is not), converts them to
    fp32 with a zero tail, and keeps row 0 for an all-zero record."""
    import numpy as np

    from paper_1709_02549_b200 import _native as nat

    lib = nat.load()
    rng = np.random.default_rng(7)
    for rows, n, ld in ((144, 2048, 2048), (9, 13, 16), (5, 1, 4)):
        rec = rng.standard_normal((rows, n))
        rec[rng.random(rows) < 0.5] = 0.0
        rec[1] = -0.0
        if rows > 3:
            rec[3] = 0.0
            rec[3, n // 2] = np.nan
        dst = np.full((rows, ld), 7.0, dtype=np.float32)
        keep = np.zeros(rows, dtype=np.int32)
        cnt = lib.mwb_compact_rows_host(rec.ctypes.data, rows, n, ld, dst.ctypes.data, keep.ctypes.data)
        want = np.flatnonzero(np.any(rec != 0.0, axis=1))
        assert cnt == max(1, want.size)
        assert np.array_equal(keep[:cnt], want)
        assert np.array_equal(dst[:cnt, :n], rec[want].astype(np.float32), equal_nan=True)
        assert not dst[:cnt, n:].any()
    zero = np.zeros((4, 8))
    dst = np.ones((4, 8), dtype=np.float32)
    keep = np.full(4, -1, dtype=np.int32)
    assert lib.mwb_compact_rows_host(zero.ctypes.data, 4, 8, 8, dst.ctypes.data, keep.ctypes.data) == 1
    assert keep[0] == 0 and not dst[0].any()
    assert lib.mwb_compact_rows_host(None, 4, 8, 8, dst.ctypes.data, keep.ctypes.data) < 0
