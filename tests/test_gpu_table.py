"""Delay-table words (mwb_delay_table) against a numpy restatement of the
reference's delay split (beamform.py:186-190): per (point, channel) the word
is ((i0 - lo_c) << 23) | trunc((n - floor n) * 2^23) with
n = (d_tx + d_rx) * inv_scale in fp64, bit for bit, and every i0 lies inside
its tile's [lo_c, hi_c] span.  Tiles whose span exceeds 9 bits are flagged
wide and carry no words."""

import numpy as np
import pytest
import torch

from paper_1709_02549_b200 import _native as nat

pytestmark = pytest.mark.gpu

TILE, SPAN_MAX = 256, 511


def layout(tiles, c):
    """Byte offsets of the words, spans and wide flags (table_layout in csrc/mwb_common.cuh)."""
    span = (4 * tiles * c * TILE + 15) // 16 * 16
    wide = (span + 8 * tiles * c + 15) // 16 * 16
    return 0, span, wide


def reference_split(pts, ant, chan, inv_scale, interp):
    d = np.sqrt(((pts[:, None, 0] - ant[None, :, 0]) ** 2 + (pts[:, None, 1] - ant[None, :, 1]) ** 2)
                + (pts[:, None, 2] - ant[None, :, 2]) ** 2)
    n = (d[:, chan[:, 0]] + d[:, chan[:, 1]]) * inv_scale
    if interp == nat.INTERP["nearest"]:
        n = np.rint(n)
    n = np.clip(n, 0.0, 2.0**30)
    fl = np.floor(n)
    return fl.astype(np.int64), np.trunc((n - fl) * 2.0**23).astype(np.int64)


def run_table(pts, ant, chan, inv_scale, interp):
    dev = torch.device("cuda")
    p_t = torch.from_numpy(pts).to(dev)
    a_t = torch.from_numpy(ant).to(dev)
    c_t = torch.from_numpy(chan.astype(np.int32)).to(dev)
    nbytes = int(nat.load().mwb_delay_table_bytes(len(pts), len(chan)))
    table = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    nat.call("mwb_delay_table", p_t.data_ptr(), len(pts), None, c_t.data_ptr(), len(chan), a_t.data_ptr(), len(ant),
             inv_scale, interp, table.data_ptr(), torch.cuda.current_stream().cuda_stream)
    h = table.cpu().numpy()
    tiles = (len(pts) + TILE - 1) // TILE
    ow, osp, owd = layout(tiles, len(chan))
    words = h[ow : ow + 4 * tiles * len(chan) * TILE].view(np.uint32).reshape(tiles, len(chan), TILE)
    span = h[osp : osp + 8 * tiles * len(chan)].view(np.int32).reshape(tiles, len(chan), 2)
    wide = h[owd : owd + 4 * tiles].view(np.int32)
    return words, span, wide


@pytest.mark.parametrize("interp", ["linear", "nearest"])
def test_table_words_bit_exact(interp):
    rng = np.random.default_rng(5)
    m = 10
    th = rng.uniform(0, 2 * np.pi, m)
    ant = np.stack([0.07 * np.cos(th), 0.07 * np.sin(th), rng.uniform(-0.01, 0.01, m)], 1)
    i, j = np.triu_indices(m)
    chan = np.stack([i, j], 1)
    inv_scale = 1.0 / (1e8 * 2e-11)
    pts = rng.uniform(-0.02, 0.02, (1000, 3))
    pts[512:768] *= 50.0  # one tile spread over 2 m: wide
    code = nat.INTERP[interp]
    words, span, wide = run_table(pts, ant, chan, inv_scale, code)
    i0, fq = reference_split(pts, ant, chan, inv_scale, code)
    assert list(wide) == [0, 0, 1, 0]
    for t in range(words.shape[0]):
        if wide[t]:
            continue
        sl = slice(t * TILE, min((t + 1) * TILE, len(pts)))
        ti0, tfq = i0[sl].T, fq[sl].T  # [C][pts]
        lo, hi = span[t, :, 0:1], span[t, :, 1:2]
        assert (ti0 >= lo).all() and (ti0 <= hi).all() and ((hi - lo) <= SPAN_MAX).all()
        want = ((ti0 - lo) << 23) | tfq
        assert np.array_equal(words[t, :, : ti0.shape[1]].astype(np.int64), want)


def test_table_exact_integer_and_boundary_delays():
    # Pythagorean distances with inv_scale 1 give integral delays (fq = 0); a
    # tiny offset below/above an integer exercises the floor boundary.
    ant = np.array([[0.0, 0.0, 0.0], [6.0, 0.0, 0.0]])
    chan = np.array([[0, 0], [0, 1], [1, 1]])
    base = np.array([[3.0, 4.0, 0.0], [3.0, -4.0, 0.0], [3.0, 4.0, 12.0], [0.0, 0.0, 0.0]])
    eps = np.array([0.0, 1e-12, -1e-12, 2.0**-40])
    pts = np.concatenate([base + e for e in eps])
    words, span, wide = run_table(pts, ant, chan, 1.0, nat.INTERP["linear"])
    i0, fq = reference_split(pts, ant, chan, 1.0, nat.INTERP["linear"])
    assert wide[0] == 0
    lo = span[0, :, 0:1]
    want = ((i0.T - lo) << 23) | fq.T
    assert np.array_equal(words[0, :, : len(pts)].astype(np.int64), want)
    assert (fq[: len(base)] == 0).all()  # exact integers
