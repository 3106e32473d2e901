"""The drop-in installer rebinds every import-time binding of the hot-path
names in the reference package.  Runs wherever the reference
is importable: the staged copy in baseline/_ref (here and on the GPU box) or
/root/reference."""

import sys
from pathlib import Path

import pytest

# the unmodified reference: staged by baseline/stage.py (travels to the GPU
# box), else the read-only source tree of the build container
STAGED = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
REF = STAGED if (STAGED / "mwbeam" / "__init__.py").exists() else Path("/root/reference/pkg/src")


@pytest.fixture
def mwbeam():
    if not REF.exists():
        pytest.skip("reference package not present on this machine")
    sys.path.insert(0, str(REF))
    try:
        import mwbeam
        import mwbeam.bench
        import mwbeam.coarse2fine
    finally:
        sys.path.remove(str(REF))
    return mwbeam


def test_install_rebinds_and_restores(mwbeam):
    import paper_1709_02549_b200 as mw
    from paper_1709_02549_b200.install import install

    orig = mwbeam.coarse2fine.image
    with install() as inst:
        assert mwbeam.image is mw.image
        assert mwbeam.beamform.image is mw.image
        assert mwbeam.coarse2fine.image is mw.image  # bound at import (coarse2fine.py:19)
        assert mwbeam.coarse2fine.run_framework is mw.run_framework
        assert mwbeam.bench.run_framework is mw.run_framework  # bench.py:15-22
        assert mwbeam.beamform.das_energy is mw.das_energy
        assert "mwbeam.coarse2fine.select_roi" in inst.patched
    assert mwbeam.coarse2fine.image is orig


def test_gpu_types_accept_reference_objects(mwbeam):
    """Host-side pieces of the drop-in work on the reference's own types."""
    import numpy as np

    import paper_1709_02549_b200 as mw

    grid = mwbeam.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 0.002)
    np.testing.assert_array_equal(mw.breast_mask(grid), mwbeam.breast_mask(grid))
    assert mw.decimation_factor(mwbeam.Manual(3), 0.002) == 3
    assert mw.decimation_factor(mwbeam.Automatic(0.01), 0.002) == 3
    from paper_1709_02549_b200.beamform import _kind

    assert _kind(mwbeam.BeamformerKind.DMAS) is mw.BeamformerKind.DMAS
