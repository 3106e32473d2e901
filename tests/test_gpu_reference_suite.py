"""The reference's OWN tests, run unmodified against the drop-in on the B200.

baseline/stage.py stages /root/reference/pkg (installed ``mwbeam`` + its
``tests/``) into the git-ignored baseline/_ref, which travels to the GPU box.
Each module runs in a subprocess with tests/refsuite_plugin.py, which calls
``paper_1709_02549_b200.install.install("mwbeam")`` before collection, so
every import-time binding of image / das_energy / dmas_energy /
_multistatic_energies / select_roi / run_framework / consistency_check /
EVAL_COUNTER in the reference (and in its tests) is the GPU path.  The
reference's own objects (BackscatterDataset, ImagingGrid, Region, EnergyMap,
FrameworkConfig, Automatic/Manual, BeamformerKind) flow through it, and the
maps it returns go through the reference's export_energy_map / service /
CLI unchanged.

Cases restated at fp32 tolerance are listed with their reason in
refsuite_plugin.RESTATED.
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
REF = REPO / "baseline" / "_ref"
SUITE = REF / "suite"

MODULES = ["test_beamform.py", "test_coarse2fine.py", "test_acceptance.py", "test_io.py", "test_service.py",
           "test_cli.py", "test_geometry.py", "test_simulate.py"]


def _run(module, tmp_path):
    if not (SUITE / "tests" / module).exists():
        pytest.fail("baseline/_ref is not staged (run `python baseline/stage.py` or build())")
    patched = tmp_path / "patched.txt"
    env = {**os.environ, "PYTHONPATH": os.pathsep.join([str(REF), str(REPO), str(REPO / "tests")]),
           "PYTHONDONTWRITEBYTECODE": "1", "MWB_REFSUITE_PATCHED": str(patched)}
    cmd = [sys.executable, "-m", "pytest", f"tests/{module}", "-p", "refsuite_plugin", "-p", "no:cacheprovider",
           "-q", "-rA", "--tb=short"]
    res = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=1800)
    out = res.stdout + res.stderr
    print(out[-6000:])
    logdir = os.environ.get("MWB_REFSUITE_LOGDIR")
    if logdir:
        Path(logdir).mkdir(parents=True, exist_ok=True)
        (Path(logdir) / f"{module}.log").write_text(out)
    m = re.search(r"(\d+) passed", out)
    passed = int(m.group(1)) if m else 0
    failed = re.search(r"(\d+) failed", out)
    errors = re.search(r"(\d+) error", out)
    return res.returncode, passed, failed, errors, patched.read_text().split() if patched.exists() else []


@pytest.mark.parametrize("module", MODULES)
def test_reference_module_passes_with_dropin(module, tmp_path):
    rc, passed, failed, errors, patched = _run(module, tmp_path)
    assert "mwbeam.coarse2fine.image" in patched and "mwbeam.beamform.image" in patched
    assert rc == 0 and passed > 0 and not failed and not errors, (module, rc, passed)
