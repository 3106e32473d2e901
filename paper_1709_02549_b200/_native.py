"""ctypes binding of ``libmwb.so`` (the C ABI in include/mwb.h).

There is no CPU fallback: if the library is missing or a call fails, a
``RuntimeError`` carrying ``mwb_last_error()`` is raised.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from ._build import LIB

MWB_DAS = 0
MWB_DMAS = 1
INTERP = {"linear": 0, "nearest": 1}
MAX_ITERS = 64

TERMINATION = {
    0: "",
    1: "degenerate",
    2: "region-floor",
    3: "n-min",
    4: "distance-metrics",
    -1: "empty",
    -2: "overflow",
}


MAX_CHILDREN = 8


class IterRecord(C.Structure):
    _fields_ = [
        ("iteration", C.c_int32),
        ("n_children", C.c_int32),
        ("counts", C.c_int32 * MAX_CHILDREN),
        ("selected", C.c_int32),
        ("satisfied", C.c_int32),
        ("has_stats", C.c_int32 * MAX_CHILDREN),
        ("clamped", C.c_int32 * MAX_CHILDREN),
        ("selected_region", C.c_int32 * 6),
        ("expanded_region", C.c_int32 * 6),
        ("scores", C.c_double * MAX_CHILDREN),
        ("mu", C.c_double * MAX_CHILDREN),
        ("var", C.c_double * MAX_CHILDREN),
        ("delta_raw", C.c_double * MAX_CHILDREN),
        ("delta", C.c_double * MAX_CHILDREN),
        ("w", C.c_double),
        ("b", C.c_double),
    ]


class Trace(C.Structure):
    _fields_ = [
        ("termination", C.c_int32),
        ("n_records", C.c_int32),
        ("final_region", C.c_int32 * 6),
        ("records", IterRecord * MAX_ITERS),
    ]


SEG_MAX_ITERS = 32


class SegRecord(C.Structure):
    _fields_ = [
        ("iteration", C.c_int32),
        ("selected", C.c_int32),
        ("parent", C.c_int32 * 6),
        ("selected_region", C.c_int32 * 6),
        ("shift", C.c_double),
        ("score", C.c_double * 4),
        ("emax", C.c_double * 4),
        ("emean", C.c_double * 4),
    ]


class SegTrace(C.Structure):
    _fields_ = [
        ("n_records", C.c_int32),
        ("stopped", C.c_int32),
        ("final_region", C.c_int32 * 6),
        ("records", SegRecord * SEG_MAX_ITERS),
    ]


TRACE_BYTES = C.sizeof(Trace)
SEG_TRACE_BYTES = C.sizeof(SegTrace)

_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.c_double

_SIGNATURES = {
    "mwb_last_error": ([], C.c_char_p),
    "mwb_version": ([], _I),
    "mwb_trace_bytes": ([], _I64),
    "mwb_delay_table_bytes": ([_I, _I], _I64),
    "mwb_delay_table": ([_P, _I, _P, _P, _I, _P, _I, _D, _I, _P, _P], _I),
    "mwb_energies": (
        [_P, _I, _I64, _I, _I, _I, _P, _P, _I, _D, _P, _P, _I, _P, _P, _I, _I, _I, _P, _P, _I64, _P, _P, _P, _I,
         _P],
        _I,
    ),
    "mwb_energies_split_bytes": ([_I, _I, _I], _I64),
    "mwb_energies_split": (
        [_P, _I, _I64, _I, _I, _I, _P, _P, _I, _D, _P, _P, _I, _P, _P, _I, _I, _I, _P, _P, _I64, _P, _P, _P, _I,
         _P, _I64, _P],
        _I,
    ),
    "mwb_energies_tc_workspace_bytes": ([_I, _I, _I, _I], _I64),
    "mwb_table_max_span": ([_P, _I, _I, _P, _P], _I),
    "mwb_table_lo_range": ([_P, _I, _I, _P, _P, _P], _I),
    "mwb_energies_tc": (
        [_P, _I, _I64, _I, _I, _I, _P, _P, _I, _D, _P, _P, _I, _P, _P, _P, _I, _I, _I, _P, _P, _I64, _P, _P, _P,
         _I, _I, _P, _P],
        _I,
    ),
    "mwb_energies_tc_record_workspace_bytes": ([_I, _I, _I, _I, _I], _I64),
    "mwb_energies_tc_record": (
        [_P, _I, _I64, _I, _I, _I, _P, _P, _I, _D, _P, _P, _I, _P, _P, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P,
         _I, _I, _P, _P],
        _I,
    ),
    "mwb_compact_rows_host": ([_P, _I, _I, _I, _P, _P], _I),
    "mwb_lattice_tile_count": ([_I, _I, _I], _I64),
    "mwb_enumerate_lattice_padded": (
        [_D, _D, _D, _I, _I, _I, _I, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P, _P, _P],
        _I,
    ),
    "mwb_delay_table_tiles": ([_P, _I, _P, _P, _I, _P, _I, _D, _I, _P, _P], _I),
    "mwb_energies_tiles": (
        [_P, _I, _I64, _I, _I, _I, _P, _P, _I, _D, _P, _P, _I, _P, _P, _I, _I, _I, _P, _P, _I64, _P, _P, _P, _I,
         _P],
        _I,
    ),
    "mwb_regions_workspace_bytes": ([_I], _I64),
    "mwb_enumerate_regions_count": ([_I, _I, _P, _I, _P, _I, _P, _P, _P], _I),
    "mwb_enumerate_regions_write": ([_D, _D, _D, _I, _I, _P, _I, _P, _I, _P, _P, _P, _P, _P], _I),
    "mwb_select_roi_batch": ([_P, _I64, _P, _I, _I, _I, _I, _I, _I, _I, _D, _I, _I, _P, _P, _P], _I),
    "mwb_lattice_workspace_bytes": ([_I, _I, _I], _I64),
    "mwb_volume_workspace_bytes": ([_I, _I, _I, _I], _I64),
    "mwb_enumerate_volume": (
        [_D, _D, _D, _D, _I, _I, _I, _P, _P, _I, _P, _I, _P, _P, _P, _P, _P, _P],
        _I,
    ),
    "mwb_select_roi_volume": ([_P, _P, _I, _I, _I, _I, _P, _D, _I, _P, _P, _P], _I),
    "mwb_enumerate_lattice": (
        [_D, _D, _D, _I, _I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _P, _P, _P, _P, _P],
        _I,
    ),
    "mwb_select_roi": ([_P, _P, _I, _I, _I, _I, _I, _I, _I, _D, _I, _P, _P, _P], _I),
    "mwb_argmax_dense": ([_P, _P, _I, _P, _P], _I),
    "mwb_image_lattice_workspace_bytes": ([_I, _I, _I, _I], _I64),
    "mwb_image_lattice": (
        [_P, _I, _I, _I, _P, _P, _I, _D, _I, _I, _I, _D, _D, _D, _I, _I, _I, _I, _I, _I, _I, _P, _I,
         _P, _P, _P, _P, _P, _P, _P, _P, _P],
        _I,
    ),
    "mwb_segment_workspace_bytes": ([_I, _I], _I64),
    "mwb_simulate": (
        [_P, _I, _I, _I, _I, _P, _P, _I, _P, _I, _D, _D, _D, _I, _D, _D, _D, _P, _I, C.c_uint64, _P, _P],
        _I,
    ),
    "mwb_segment": (
        [_P, _I, _I, _I, _P, _P, _I, _D, _I, _I, _I, _I, _D, _D, _D, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P,
         _P, _P],
        _I,
    ),
    "mwb_segment_batch_workspace_bytes": ([_I, _I, _I], _I64),
    "mwb_segment_batch": (
        [_P, _I, _I64, _I, _I, _I, _P, _P, _I, _D, _I, _I, _I, _I, _D, _D, _D, _I, _I, _I, _I, _I, _I, _I, _I, _I,
         _P, _P, _P, _P, _P],
        _I,
    ),
    "mwb_segment_plan_info": ([_I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P], _I),
    "mwb_segment_plan_prepare": (
        [_P, _I, _P, _I, _D, _I, _D, _D, _D, _I, _I, _I, _I, _I, _I, _P, _I, _I, _I, _P, _P],
        _I,
    ),
    "mwb_segment_run_workspace_bytes": ([_I, _I, _I, _I], _I64),
    "mwb_segment_run": (
        [_P, _P, _I, _I64, _I, _I, _I, _P, _P, _I, _D, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P,
         _P, _P, _I64, _P, _P, _P, _P, _P],
        _I,
    ),
    "mwb_energies_region": (
        [_P, _I, _I, _I, _P, _P, _I, _D, _P, _P, _I, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P,
         _I, _P, _I64, _P],
        _I,
    ),
    "mwb_gather_composite": ([_P, _I, _I, _P, _I, _P, _P, _I64, _P], _I),
    "mwb_memcpy_async": ([_P, _P, _I64, _P], _I),
    "mwb_memcpy2d_async": ([_P, _I64, _P, _I64, _I64, _I64, _P], _I),
    "mwb_stream_synchronize": ([_P], _I),
    "mwb_tc_plan_steps": ([_P, _I, _I, _I, _I, _I, _P], _I),
    "mwb_tc_sample_range": ([_I, _I, _I, _I, _P], _I),
    "mwb_elapsed_ms": ([_P, _I, _P], _I),
    "mwb_compact_payload": ([_P, _I, _I, _I, _P, _P, _P, _P, _P], _I),
    "mwb_render_pgm": ([_P, _I, _P, _I, _I, _I, _I64, _I, _P, _P, _P], _I),
    "mwb_microbench": ([_I, C.POINTER(C.c_double), C.POINTER(C.c_float), _P], _I),
}

EXPORTED = tuple(_SIGNATURES)

_lib: C.CDLL | None = None


def load(path: Path | str | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raise if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    if path is None and os.environ.get("MWB_LIB"):  # experiments: an alternative build
        path = os.environ["MWB_LIB"]
    p = Path(path) if path is not None else LIB
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the GPU path has no CPU fallback)"
        )
    lib = C.CDLL(str(p))
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None or os.environ.get("MWB_LIB") == str(path):
        _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load().mwb_last_error()
        raise RuntimeError(f"{what} failed ({status}): {msg.decode() if msg else ''}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
