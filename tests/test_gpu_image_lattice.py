"""mwb_image_lattice, the one-call C entry point a non-Python binding uses
(include/mwb.h), against the Python image path (beamform.images): identical
maps, validity, counts and argmax keys, bit for bit, for full grids, strided
masked lattices with a skip stride, sub-regions and both kinds at once."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1709_02549_b200 as mw
from paper_1709_02549_b200 import _device as dv
from paper_1709_02549_b200 import _native as nat
from paper_1709_02549_b200 import synth

pytestmark = pytest.mark.gpu


def c_image(ds, grid, region, stride, mask, skip, window):
    scan = dv.scan_for(ds)
    nx, ny = grid.dims
    dev = torch.device("cuda")
    das = torch.zeros(nx * ny, dtype=torch.float32, device=dev)
    dmas = torch.zeros(nx * ny, dtype=torch.float32, device=dev)
    valid = torch.zeros(nx * ny, dtype=torch.uint8, device=dev)
    small = torch.zeros(4, dtype=torch.int64, device=dev)  # key_das, key_dmas, count | flags
    ws = torch.empty(int(nat.load().mwb_image_lattice_workspace_bytes(nx, ny, stride, scan.n_chan)),
                     dtype=torch.uint8, device=dev)
    m = None if mask is None else torch.from_numpy(np.ascontiguousarray(mask).view(np.uint8).reshape(-1)).to(dev)
    (x0, y0), (x1, y1) = region.min_cell, region.max_cell
    b = small.data_ptr()
    nat.call("mwb_image_lattice", scan.sig.data_ptr(), scan.n_chan, scan.ld, scan.n_samples, scan.chan.data_ptr(),
             scan.ant.data_ptr(), scan.n_ant, scan.inv_scale, 0, window[0], window[1], grid.origin[0],
             grid.origin[1], grid.resolution, nx, ny, x0, y0, x1, y1, stride, nat.ptr(m), skip, das.data_ptr(),
             dmas.data_ptr(), valid.data_ptr(), b + 16, b, b + 8, b + 20, ws.data_ptr(), dv.stream_handle())
    h = small.cpu().numpy()
    return (das.view(nx, ny).cpu().numpy(), dmas.view(nx, ny).cpu().numpy(), valid.view(nx, ny).cpu().numpy() > 0,
            int(h[2] & 0xFFFFFFFF), h[:2].view(np.uint64))


@pytest.mark.parametrize("case", ["full", "strided-masked-skip", "subregion"])
def test_matches_python_image(case):
    model = synth.ScanModel()
    ds, _ = synth.dataset_2d(model, seed=3)
    grid = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
    region, stride, mask, skip = grid.full_region(), 1, None, 0
    if case == "strided-masked-skip":
        stride, mask, skip = 3, mw.breast_mask(grid), 6
    elif case == "subregion":
        region = mw.Region((17, 5), (80, 61))
    window = (model.k0, model.window)
    das, dmas, valid, count, keys = c_image(ds, grid, region, stride, mask, skip, window)
    skip_mask = None
    if skip:
        ix, iy = np.meshgrid(np.arange(grid.dims[0]), np.arange(grid.dims[1]), indexing="ij")
        skip_mask = (ix % skip == 0) & (iy % skip == 0)
    before = mw.EVAL_COUNTER.value
    want = mw.images(ds, ("das", "dmas"), grid, region=region, stride=stride, mask=mask,
                     skip=None if skip_mask is None else {(int(a), int(b)) for a, b in zip(*np.nonzero(skip_mask))},
                     window=window)
    n_py = (mw.EVAL_COUNTER.value - before) // 2
    assert count == n_py == int(valid.sum())
    for name, got in (("das", das), ("dmas", dmas)):
        ref = np.zeros(grid.dims)
        ref_valid = np.zeros(grid.dims, dtype=bool)
        for (ix, iy), v in want[name].entries.items():  # evaluated cells only (dense() holds strided values)
            ref[ix, iy], ref_valid[ix, iy] = v, True
        assert np.array_equal(valid, ref_valid)
        assert np.array_equal(got[valid], ref[valid].astype(np.float32))
    cells = [np.unravel_index(int(0xFFFFFFFF - (int(k) & 0xFFFFFFFF)), grid.dims) for k in keys]
    assert tuple(int(v) for v in cells[0]) == want["das"].argmax_cell()
    assert tuple(int(v) for v in cells[1]) == want["dmas"].argmax_cell()
