"""Window-split launches (mwb_energies_split): a small launch over a long
window (the reference's full record) spreads its 32-sample chunks over more
CTAs and sums each point's chunk partials in chunk order in a second kernel.
Every energy, argmax key and flag must be bit-identical to mwb_energies."""

import numpy as np
import pytest
import torch

from paper_1709_02549_b200 import _device as dv
from paper_1709_02549_b200 import _native as nat
from paper_1709_02549_b200 import synth
from paper_1709_02549_b200.beamform import build_table

pytestmark = pytest.mark.gpu


def _launch(name, scan, sig, n_scans, pts, n, table, k0, w, both, ws=None, d_count=None):
    dev = pts.device
    das = torch.full((n_scans, n), np.nan, dtype=torch.float32, device=dev) if both[0] else None
    dmas = torch.full((n_scans, n), np.nan, dtype=torch.float32, device=dev) if both[1] else None
    keys = torch.zeros((2, n_scans), dtype=torch.int64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    args = [sig.data_ptr(), n_scans, scan.n_chan * scan.ld, scan.n_chan, scan.ld, scan.n_samples, scan.chan.data_ptr(),
            scan.ant.data_ptr(), scan.n_ant, scan.inv_scale, pts.data_ptr(), None, n, d_count, table.data_ptr(), 0,
            k0, w, nat.ptr(das), nat.ptr(dmas), n, keys[0].data_ptr(), keys[1].data_ptr(), flags.data_ptr(), 0]
    if name == "mwb_energies_split":
        args += [nat.ptr(ws), ws.numel() if ws is not None else 0]
    nat.call(name, *args, dv.stream_handle())
    torch.cuda.synchronize()
    return [t.cpu().numpy() if t is not None else None for t in (das, dmas)], keys.cpu().numpy(), int(flags.item())


@pytest.mark.parametrize("n_pts,n_scans,w,both", [(1, 1, 1024, (1, 1)), (300, 1, 1024, (1, 0)),
                                                  (700, 3, 512, (0, 1)), (5000, 2, 256, (1, 1)),
                                                  (257, 1, 100, (1, 1)), (64, 1, 96 * 3, (1, 1))])
def test_split_is_bit_identical(n_pts, n_scans, w, both):
    model = synth.ScanModel()
    sig_h, _ = synth.batch_2d(model, range(n_scans))
    sig = torch.from_numpy(np.ascontiguousarray(sig_h)).cuda()
    scan = dv.DeviceScan(sig=sig, chan=torch.from_numpy(model.pairs()).cuda(),
                         ant=torch.from_numpy(np.array(model.geometry().antennas)).cuda(),
                         inv_scale=1.0 / (model.v * model.dt), n_samples=model.n_samples, ld=model.n_samples,
                         n_ant=model.n_ant, chan_host=model.pairs())
    rng = np.random.default_rng(n_pts)
    p = np.zeros((n_pts, 3))
    p[:, :2] = rng.uniform(-0.05, 0.05, size=(n_pts, 2))
    pts = torch.from_numpy(p).cuda()
    table = build_table(scan, pts, n_pts, 0)
    k0 = 0 if w >= model.n_samples else 7
    ws = torch.empty(int(nat.load().mwb_energies_split_bytes(n_pts, n_scans, w)), dtype=torch.uint8, device="cuda")
    a = _launch("mwb_energies", scan, sig, n_scans, pts, n_pts, table, k0, w, both)
    b = _launch("mwb_energies_split", scan, sig, n_scans, pts, n_pts, table, k0, w, both, ws)
    for x, y in zip(a[0], b[0]):
        if x is not None:
            assert np.array_equal(x, y)
    assert np.array_equal(a[1], b[1]) and a[2] == b[2] == 0
    # too small a workspace: exactly the unsplit launch
    c = _launch("mwb_energies_split", scan, sig, n_scans, pts, n_pts, table, k0, w, both, ws[:8])
    for x, y in zip(a[0], c[0]):
        if x is not None:
            assert np.array_equal(x, y)


def test_split_device_count_and_nonfinite_flag():
    model = synth.ScanModel(n_samples=512)
    sig_h, _ = synth.batch_2d(model, [4])
    sig_h[0, 3, 100] = np.nan
    sig = torch.from_numpy(np.ascontiguousarray(sig_h)).cuda()
    scan = dv.DeviceScan(sig=sig, chan=torch.from_numpy(model.pairs()).cuda(),
                         ant=torch.from_numpy(np.array(model.geometry().antennas)).cuda(),
                         inv_scale=1.0 / (model.v * model.dt), n_samples=512, ld=512, n_ant=model.n_ant,
                         chan_host=model.pairs())
    p = np.zeros((1000, 3))
    p[:, :2] = np.random.default_rng(1).uniform(-0.05, 0.05, size=(1000, 2))
    pts = torch.from_numpy(p).cuda()
    cnt = torch.tensor([613], dtype=torch.int32, device="cuda")
    table = build_table(scan, pts, 1000, 0, cnt.data_ptr())
    ws = torch.empty(int(nat.load().mwb_energies_split_bytes(1000, 1, 512)), dtype=torch.uint8, device="cuda")
    a = _launch("mwb_energies", scan, sig, 1, pts, 1000, table, 0, 512, (1, 1), d_count=cnt.data_ptr())
    b = _launch("mwb_energies_split", scan, sig, 1, pts, 1000, table, 0, 512, (1, 1), ws, d_count=cnt.data_ptr())
    for x, y in zip(a[0], b[0]):
        assert np.array_equal(x[:, :613], y[:, :613], equal_nan=True)
        assert np.isnan(y[:, 613:]).all()  # beyond the device count: untouched
    assert np.array_equal(a[1], b[1]) and a[2] == b[2] == 1
