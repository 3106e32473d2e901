"""Stage the UNMODIFIED reference package into ``baseline/_ref`` (git-ignored,
travels to the GPU box with the gpurun snapshot).

Two things land there, both read-only copies of ``/root/reference/pkg``:

* ``baseline/_ref/mwbeam`` — the reference installed with pip (``--no-deps``:
  its runtime dependencies numpy / click / fastapi / pydantic / uvicorn /
  httpx are already in the image; ``--no-index`` resolution of them fails
  only because they are not wheels in /opt/wheelhouse).  pip builds from a
  scratch copy under /tmp because setuptools writes egg-info next to the
  sources and /root/reference is read-only.  bench.py's CPU baseline and
  ``--impl reference`` time this package's own ``image()``.
* ``baseline/_ref/suite/tests`` — the reference's own test modules plus an
  empty ``__init__.py`` (test_acceptance.py:31 imports ``tests.test_beamform``),
  run on the GPU box with the drop-in installed by
  ``tests/test_gpu_reference_suite.py``.

Nothing here is product code; build() calls ``stage()`` when /root/reference
exists (the build container) and the GPU box uses the staged copy.
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_PKG = Path("/root/reference/pkg")
TARGET = HERE / "_ref"


def staged() -> bool:
    return (TARGET / "mwbeam" / "__init__.py").exists() and (TARGET / "suite" / "tests").is_dir()


def stage(force: bool = False) -> Path:
    if staged() and not force:
        return TARGET
    if not REF_PKG.exists():
        raise FileNotFoundError(f"{REF_PKG} not present: cannot stage the reference")
    if TARGET.exists():
        shutil.rmtree(TARGET)
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_PKG, src)
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
                        "--find-links", "/opt/wheelhouse", "--target", str(TARGET), str(src), "-q"],
                       check=True, cwd=tmp)
    suite = TARGET / "suite" / "tests"
    shutil.copytree(REF_PKG / "tests", suite)
    (suite / "__init__.py").write_text("")
    return TARGET


if __name__ == "__main__":
    print(stage(force="--force" in sys.argv))
