"""bench.py's CPU side on the CPU box: the reference arm's timing routine runs
the staged, unmodified reference (baseline/_ref) and reports what it used."""

import importlib.util
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", REPO / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_cpu_reference_rate_times_the_real_reference(bench):
    staged = (REPO / "baseline" / "_ref" / "mwbeam" / "__init__.py").exists()
    r = bench.cpu_reference_rate(0.3, 1, seed=2)
    assert r["kind"] == ("reference" if staged else "port")
    assert r["value"] > 0 and r["cores"] == 1 and 0.5 <= r["busy_cores"] <= 1.5
    assert "suffix-difference" in r["sample"] and r["unit"] == bench.UNIT


def test_thread_candidates_include_one_and_all(bench):
    c = bench.thread_candidates()
    assert c[0] == 1 and c[-1] == bench.host_threads() and c == sorted(set(c))
