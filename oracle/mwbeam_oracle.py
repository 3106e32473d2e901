"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference algorithm for the imaging hot path of
`mwbeam` (/root/reference/pkg/src/mwbeam).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
this module, and only as the checker / the timed CPU baseline.  The GPU path
in ``paper_1709_02549_b200`` never calls it.

Parity pin: every function is checked against golden vectors produced by the
real reference package (``tests/golden/make_golden.py`` imports
/root/reference/pkg/src in the build container; the fixtures travel, the
reference does not) and against the reference's own known-answer tests
(tests/test_oracle_pins.py), both on the CPU.

Citations are to /root/reference/pkg/src/mwbeam/<file>:<line>.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

BATCH = 64  # beamform.py:37-38

SPEED_OF_LIGHT = 2.99792458e8


# ---------------------------------------------------------------------------
# energy kernel — beamform.py:169-212
# ---------------------------------------------------------------------------
def multistatic_energies(antennas, v, dt, signals, points, kind: str, interpolation: str = "linear"):
    """Energies of a (P, 2) batch of z=0 focal points, full-record sum.

    beamform.py:182-190 delays, 192-194 zero padding, 199-209 the per-channel
    interpolate + accumulate loop, 210-212 the DAS / DMAS epilogue.
    """
    ants = np.asarray(antennas, dtype=np.float64)
    sig = np.asarray(signals, dtype=np.float64)
    m, _, nsamp = sig.shape
    c = m * m
    scale = v * dt
    pts = np.asarray(points, dtype=np.float64)
    dx = pts[:, 0, None] - ants[None, :, 0]
    dy = pts[:, 1, None] - ants[None, :, 1]
    dz = ants[None, :, 2]
    d = np.sqrt(dx * dx + dy * dy + dz * dz)
    shifts = ((d[:, :, None] + d[:, None, :]) / scale).reshape(len(pts), c)
    if interpolation == "nearest":
        shifts = np.rint(shifts)
    i0 = np.floor(shifts).astype(np.int64)
    frac = shifts - i0
    ypad = np.zeros((c, nsamp + int(i0.max()) + 2))
    ypad[:, :nsamp] = sig.reshape(c, nsamp)
    win = sliding_window_view(ypad, nsamp + 1, axis=1)
    s = np.zeros((len(pts), nsamp))
    q = np.zeros((len(pts), nsamp)) if kind == "dmas" else None
    for ch in range(c):
        w = win[ch, i0[:, ch]]
        f1 = frac[:, ch, None]
        f0 = 1.0 - f1
        if q is None:
            s += f0 * w[:, :nsamp]
            s += f1 * w[:, 1:]
        else:
            a = f0 * w[:, :nsamp] + f1 * w[:, 1:]
            s += a
            q += a * a
    if q is None:
        return (s * s).sum(axis=1)
    return 0.5 * ((s * s) - q).sum(axis=1)


def windowed_energies(antennas, v, dt, signals, points, kind: str, k0: int, w: int, interpolation="linear"):
    """Energy over aligned samples [k0, k0+W) via the reference kernel only.

    Suffix differencing (SURVEY.md §8c adapter 2): with the record truncated
    at b >= k0+W+max_delay+2, E[k0,k0+W) = E(sig[..., k0:b]) - E(sig[..., k0+W:b]).
    Both terms are full-record reference sums, so only the reference
    arithmetic computes the values.  Exact in real arithmetic: shifting the
    record start by k0 shifts every aligned sample index by k0.
    """
    sig = np.asarray(signals, dtype=np.float64)
    n = sig.shape[2]
    ants = np.asarray(antennas, dtype=np.float64)
    pts = np.asarray(points, dtype=np.float64)
    dx = pts[:, 0, None] - ants[None, :, 0]
    dy = pts[:, 1, None] - ants[None, :, 1]
    d = np.sqrt(dx * dx + dy * dy + ants[None, :, 2] ** 2)
    maxdel = int(np.ceil(2 * d.max() / (v * dt))) + 2
    b = min(n, k0 + w + maxdel + 2)
    if k0 >= b:
        return np.zeros(len(pts))
    head = np.zeros(sig.shape[:2] + (max(b - k0, 1),))
    head[..., : b - k0] = sig[..., k0:b]
    e_all = multistatic_energies(ants, v, dt, head, pts, kind, interpolation)
    if k0 + w >= b:
        return e_all
    tail = np.zeros(sig.shape[:2] + (b - k0 - w,))
    tail[...] = sig[..., k0 + w : b]
    return e_all - multistatic_energies(ants, v, dt, tail, pts, kind, interpolation)


def windowed_energies_direct(antennas, v, dt, signals, points, kind, k0, w, interpolation="linear"):
    """Direct restatement of the windowed energy (independent check of the adapter)."""
    sig = np.asarray(signals, dtype=np.float64)
    m, _, n = sig.shape
    ants = np.asarray(antennas, dtype=np.float64)
    pts = np.asarray(points, dtype=np.float64)
    out = np.zeros(len(pts))
    ks = np.arange(k0, k0 + w)
    for p, (x, y) in enumerate(pts[:, :2]):
        d = np.sqrt((x - ants[:, 0]) ** 2 + (y - ants[:, 1]) ** 2 + ants[:, 2] ** 2)
        s = np.zeros(w)
        q = np.zeros(w)
        for i in range(m):
            for j in range(m):
                sh = (d[i] + d[j]) / (v * dt)
                if interpolation == "nearest":
                    sh = float(np.rint(sh))
                i0 = int(np.floor(sh))
                f = sh - i0
                ypad = np.concatenate([sig[i, j], np.zeros(k0 + w + i0 + 2)])
                a = (1 - f) * ypad[ks + i0] + f * ypad[ks + i0 + 1]
                s += a
                q += a * a
        out[p] = (s * s).sum() if kind == "das" else 0.5 * ((s * s) - q).sum()
    return out


# ---------------------------------------------------------------------------
# lattice + image driver — beamform.py:268-342
# ---------------------------------------------------------------------------
def region_cells(dims, region, stride, mask=None):
    """beamform.py:268-280: stride multiples, ix-major, optional mask."""
    (x0, y0), (x1, y1) = region
    xs = np.arange(((x0 + stride - 1) // stride) * stride, x1 + 1, stride)
    ys = np.arange(((y0 + stride - 1) // stride) * stride, y1 + 1, stride)
    ix, iy = np.meshgrid(xs, ys, indexing="ij")
    ix, iy = ix.ravel(), iy.ravel()
    if mask is not None:
        keep = np.asarray(mask)[ix, iy]
        ix, iy = ix[keep], iy[keep]
    return ix, iy


def image(antennas, v, dt, signals, kind, origin, res, dims, region=None, stride=1, mask=None, skip=None,
          interpolation="linear", window=None, threads=None):
    """beamform.py:283-342 -> dict {(ix, iy): energy} in evaluation order."""
    if region is None:
        region = ((0, 0), (dims[0] - 1, dims[1] - 1))
    ix, iy = region_cells(dims, region, stride, mask)
    if skip:
        keep = np.fromiter(((int(a), int(b)) not in skip for a, b in zip(ix, iy)), dtype=bool, count=len(ix))
        ix, iy = ix[keep], iy[keep]
    if len(ix) == 0:
        return {}
    px = origin[0] + (ix + 0.5) * res
    py = origin[1] + (iy + 0.5) * res
    pts = np.stack([px, py], axis=1)
    batches = [slice(b, min(b + BATCH, len(pts))) for b in range(0, len(pts), BATCH)]
    res_list = [None] * len(batches)

    def work(k):
        if window is None:
            res_list[k] = multistatic_energies(antennas, v, dt, signals, pts[batches[k]], kind, interpolation)
        else:
            res_list[k] = windowed_energies(antennas, v, dt, signals, pts[batches[k]], kind, window[0], window[1],
                                            interpolation)

    threads = threads or 1
    if threads > 1 and len(batches) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(work, range(len(batches))))
    else:
        for k in range(len(batches)):
            work(k)
    e = np.concatenate(res_list)
    return {(a, b): float(x) for a, b, x in zip(ix.tolist(), iy.tolist(), e.tolist())}


def argmax_cell(entries):
    """beamform.py:101-104."""
    return max(entries, key=lambda k: (entries[k], (-k[0], -k[1])))


# ---------------------------------------------------------------------------
# geometry helpers — geometry.py:149-150, 225-257
# ---------------------------------------------------------------------------
def grid_dims(extent, res):
    return (max(1, math.ceil(round(extent[0] / res, 9))), max(1, math.ceil(round(extent[1] / res, 9))))


def quadrants(region):
    (x0, y0), (x1, y1) = region
    w, h = x1 - x0 + 1, y1 - y0 + 1
    if w < 2 or h < 2:
        return None
    xm = x0 + (w + 1) // 2 - 1
    ym = y0 + (h + 1) // 2 - 1
    return [((x0, y0), (xm, ym)), ((xm + 1, y0), (x1, ym)), ((x0, ym + 1), (xm, y1)), ((xm + 1, ym + 1), (x1, y1))]


def expand(region, f, clip):
    (x0, y0), (x1, y1) = region
    px = math.ceil(f * (x1 - x0 + 1))
    py = math.ceil(f * (y1 - y0 + 1))
    (cx0, cy0), (cx1, cy1) = clip
    return ((max(x0 - px, cx0), max(y0 - py, cy0)), (min(x1 + px, cx1), min(y1 + py, cy1)))


def values_in(entries, region):
    (x0, y0), (x1, y1) = region
    return np.array([v for (ix, iy), v in entries.items() if x0 <= ix <= x1 and y0 <= iy <= y1])


# ---------------------------------------------------------------------------
# framework — coarse2fine.py:49-109, 169-268, 301-350
# ---------------------------------------------------------------------------
def auto_decimation_factor(min_tumor_diameter, resolution):
    return max(1, math.floor((min_tumor_diameter / math.sqrt(2.0)) / resolution))


def metric_parts(vals, sigma_prev_sq):
    mu = float(vals.mean())
    var = float(vals.var())
    if var == 0.0:
        return mu, {"mu": mu, "var": var, "delta_raw": 0.0, "delta": 0.0, "clamped": False}
    delta_raw = (var - sigma_prev_sq) / var
    delta = min(max(delta_raw, 0.0), 1.0)
    return (1.0 - delta) * mu + delta * var, {"mu": mu, "var": var, "delta_raw": delta_raw, "delta": delta,
                                              "clamped": delta != delta_raw}


def class_distances(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    ma, mb = a.mean(), b.mean()
    w = float(((a - ma) ** 2).sum() + ((b - mb) ** 2).sum())
    g = np.concatenate([a, b]).mean()
    return w, float(a.size * (ma - g) ** 2 + b.size * (mb - g) ** 2)


def select_roi(entries, breast_region, frame_fraction=0.25, n_min=4):
    """coarse2fine.py:169-256 -> (final_region, trace dict)."""
    trace = {"records": [], "termination": "", "warning": None}
    vals = values_in(entries, breast_region)
    if vals.size == 0:
        raise ValueError("coarse map has no entries in the breast region")
    if vals.max() == vals.min():
        trace["termination"] = "degenerate"
        trace["warning"] = "energy map has no discriminating signal"
        return breast_region, trace
    sel, sel_vals = breast_region, vals
    sigma_prev_sq = float(vals.var())
    prev_w = prev_b = None
    it = 0
    while True:
        quads = quadrants(sel)
        if quads is None:
            trace["termination"] = "region-floor"
            return sel, trace
        scores, stats, counts = [], [], []
        for q in quads:
            v = values_in(entries, q)
            counts.append(int(v.size))
            if v.size == 0:
                scores.append(-np.inf)
                stats.append(None)
            elif it == 0:
                scores.append(float(v.var()))
                stats.append({"mu": float(v.mean()), "var": float(v.var())})
            else:
                val, parts = metric_parts(v, sigma_prev_sq)
                scores.append(val)
                stats.append(parts)
        selected = int(np.argmax(scores))
        if counts[selected] < n_min:
            trace["termination"] = "n-min"
            return sel, trace
        it += 1
        expanded = expand(quads[selected], frame_fraction, sel)
        new_vals = values_in(entries, expanded)
        w, b = class_distances(sel_vals, new_vals)
        satisfied = prev_w is None or (b > prev_b or w < prev_w)
        trace["records"].append({"iteration": it, "quadrant_counts": counts, "scores": [float(s) for s in scores],
                                 "stats": stats, "selected": selected, "selected_region": quads[selected],
                                 "expanded_region": expanded, "W": w, "B": b, "satisfied": satisfied})
        if not satisfied:
            trace["termination"] = "distance-metrics"
            return sel, trace
        sigma_prev_sq = float(new_vals.var())
        sel, sel_vals = expanded, new_vals
        prev_w, prev_b = w, b


def breast_mask(origin, res, dims):
    """coarse2fine.py:259-268."""
    nx, ny = dims
    cx = origin[0] + nx * res / 2.0
    cy = origin[1] + ny * res / 2.0
    radius = min(nx, ny) * res / 2.0
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    px = origin[0] + (ix + 0.5) * res
    py = origin[1] + (iy + 0.5) * res
    return (px - cx) ** 2 + (py - cy) ** 2 <= radius**2


def run_framework(antennas, v, dt, signals, kind, origin, res, dims, d, frame_fraction=0.25, n_min=4,
                  window=None, threads=None):
    """coarse2fine.py:301-350 -> (composite entries, report dict)."""
    full = ((0, 0), (dims[0] - 1, dims[1] - 1))
    mask = breast_mask(origin, res, dims)
    coarse = image(antennas, v, dt, signals, kind, origin, res, dims, full, d, mask, window=window, threads=threads)
    if not coarse:
        raise ValueError("no coarse focal points inside the breast mask")
    final, trace = select_roi(coarse, full, frame_fraction, n_min)
    fine = image(antennas, v, dt, signals, kind, origin, res, dims, final, 1, mask, skip=set(coarse), window=window,
                 threads=threads)
    comp = dict(coarse)
    comp.update(fine)
    full_eq = int(mask.sum())
    return comp, {
        "decimation_factor": d,
        "iterations": len(trace["records"]),
        "final_region": final,
        "coarse_points_evaluated": len(coarse),
        "fine_points_evaluated": len(fine),
        "full_equivalent_points": full_eq,
        "reduction_ratio": full_eq / (len(coarse) + len(fine)),
        "trace": trace,
        "argmax_cell": argmax_cell(comp),
    }


# ---------------------------------------------------------------------------
# reference simulator (input producer for the reference-style test cases) —
# simulate.py:53-73, 111-162 and presets.py:58-67
# ---------------------------------------------------------------------------
def gaussian_modulated_pulse(t, fc=4e9, width=100e-12, duration=600e-12):
    u = np.asarray(t, dtype=np.float64) - duration / 2.0
    return np.exp(-(u**2) / (2.0 * width**2)) * np.cos(2.0 * np.pi * fc * u)


def ring_antennas(n, radius, center=(0.0, 0.0)):
    ang = 2.0 * np.pi * np.arange(n) / n
    return np.stack([center[0] + radius * np.cos(ang), center[1] + radius * np.sin(ang), np.zeros(n)], axis=1)


def simulate(antennas, v, dt, n_samples, scatterers, noise_std=0.0, seed=0, t0=0.0):
    """simulate.py:111-162 (record-length check included)."""
    ants = np.asarray(antennas, dtype=np.float64)
    m = ants.shape[0]
    t = t0 + dt * np.arange(n_samples)
    signals = np.zeros((m, m, n_samples))
    for (sx, sy), contrast in scatterers:
        d = np.sqrt((ants[:, 0] - sx) ** 2 + (ants[:, 1] - sy) ** 2 + ants[:, 2] ** 2)
        tau = (d[:, None] + d[None, :]) / v
        if float(tau.max()) + 600e-12 > t0 + (n_samples - 1) * dt:
            raise ValueError("record window too short")
        amp = contrast / np.maximum(d[:, None] * d[None, :], 1e-9)
        signals += amp[:, :, None] * gaussian_modulated_pulse(t[None, None, :] - tau[:, :, None])
    if noise_std > 0:
        signals = signals + np.random.default_rng(seed).normal(0.0, noise_std, signals.shape)
    return signals


def grid_for_antennas(antennas, resolution):
    """presets.py:58-67 -> (origin, extent, resolution)."""
    xy = np.asarray(antennas)[:, :2]
    cx, cy = xy.mean(axis=0)
    radius = float(((xy[:, 0] - cx) ** 2 + (xy[:, 1] - cy) ** 2).max() ** 0.5)
    return (cx - radius, cy - radius), (2.0 * radius, 2.0 * radius), resolution


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# 3-D voxels (BASELINE configs[4]).  Energies come from the reference kernel
# through the exact z-shift adapter (SURVEY.md §8c adapter 3): voxel (x, y, z)
# = point (x, y) with every antenna shifted by -z (beamform.py:182-185 uses
# dz = antenna z with points at z = 0).  The octant control flow has no
# reference counterpart; it restates select_roi (coarse2fine.py:169-256) with
# 8 children per box (index = xhigh + 2*yhigh + 4*zhigh).
# ---------------------------------------------------------------------------
def volume_energies(antennas, v, dt, signals, points3, kind, k0=None, w=None, interpolation="linear"):
    ants = np.asarray(antennas, dtype=np.float64)
    pts = np.asarray(points3, dtype=np.float64)
    out = np.zeros(len(pts))
    for z in np.unique(pts[:, 2]):
        sel = pts[:, 2] == z
        shifted = ants - np.array([0.0, 0.0, z])
        if w is None:
            out[sel] = multistatic_energies(shifted, v, dt, signals, pts[sel, :2], kind, interpolation)
        else:
            out[sel] = windowed_energies(shifted, v, dt, signals, pts[sel, :2], kind, k0, w, interpolation)
    return out


def octants(box):
    lo, hi = box
    if min(h - l + 1 for l, h in zip(lo, hi)) < 2:
        return None
    mids = [l + (h - l + 2) // 2 - 1 for l, h in zip(lo, hi)]
    out = []
    for k in range(8):
        a = []
        b = []
        for ax in range(3):
            if (k >> ax) & 1:
                a.append(mids[ax] + 1)
                b.append(hi[ax])
            else:
                a.append(lo[ax])
                b.append(mids[ax])
        out.append((tuple(a), tuple(b)))
    return out


def expand3(box, f, clip):
    lo, hi = box
    g = [math.ceil(f * (h - l + 1)) for l, h in zip(lo, hi)]
    return (tuple(max(l - gg, c) for l, gg, c in zip(lo, g, clip[0])),
            tuple(min(h + gg, c) for h, gg, c in zip(hi, g, clip[1])))


def values_in3(entries, box):
    lo, hi = box
    return np.array([v for c, v in entries.items() if all(a <= x <= b for a, x, b in zip(lo, c, hi))])


def select_roi_3d(entries, box, frame_fraction=0.25, n_min=4):
    """select_roi (coarse2fine.py:169-256) with octants."""
    trace = {"records": [], "termination": "", "warning": None}
    vals = values_in3(entries, box)
    if vals.size == 0:
        raise ValueError("coarse map has no entries in the breast region")
    if vals.max() == vals.min():
        trace["termination"] = "degenerate"
        return box, trace
    sel, sel_vals = box, vals
    sigma_prev_sq = float(vals.var())
    prev_w = prev_b = None
    it = 0
    while True:
        kids = octants(sel)
        if kids is None:
            trace["termination"] = "region-floor"
            return sel, trace
        scores, counts = [], []
        for q in kids:
            v = values_in3(entries, q)
            counts.append(int(v.size))
            if v.size == 0:
                scores.append(-np.inf)
            elif it == 0:
                scores.append(float(v.var()))
            else:
                scores.append(metric_parts(v, sigma_prev_sq)[0])
        selected = int(np.argmax(scores))
        if counts[selected] < n_min:
            trace["termination"] = "n-min"
            return sel, trace
        it += 1
        expanded = expand3(kids[selected], frame_fraction, sel)
        new_vals = values_in3(entries, expanded)
        w, b = class_distances(sel_vals, new_vals)
        satisfied = prev_w is None or (b > prev_b or w < prev_w)
        trace["records"].append({"selected": selected, "scores": scores, "quadrant_counts": counts, "W": w, "B": b,
                                 "selected_region": kids[selected], "expanded_region": expanded,
                                 "satisfied": satisfied})
        if not satisfied:
            trace["termination"] = "distance-metrics"
            return sel, trace
        sigma_prev_sq = float(new_vals.var())
        sel, sel_vals = expanded, new_vals
        prev_w, prev_b = w, b


def hemisphere_mask(origin, res, dims, radius):
    nx, ny, nz = dims
    px = origin[0] + (np.arange(nx) + 0.5) * res
    py = origin[1] + (np.arange(ny) + 0.5) * res
    pz = origin[2] + (np.arange(nz) + 0.5) * res
    d2 = px[:, None, None] ** 2 + py[None, :, None] ** 2 + pz[None, None, :] ** 2
    return (d2 <= radius**2) & (pz[None, None, :] >= 0.0)


def run_framework_3d(antennas, v, dt, signals, kind, origin, res, dims, d, radius, frame_fraction=0.25, n_min=4,
                     window=None):
    """run_framework (coarse2fine.py:301-350) on voxels with octant selection."""
    mask = hemisphere_mask(origin, res, dims, radius)
    full = ((0, 0, 0), tuple(n - 1 for n in dims))

    def evaluate(cells):
        if not cells:
            return {}
        pts = np.array([[origin[a] + (c[a] + 0.5) * res for a in range(3)] for c in cells])
        k0, w = window if window is not None else (None, None)
        e = volume_energies(antennas, v, dt, signals, pts, kind, k0, w)
        return dict(zip(cells, e.tolist()))

    coarse_cells = [(ix, iy, iz) for ix in range(0, dims[0], d) for iy in range(0, dims[1], d)
                    for iz in range(0, dims[2], d) if mask[ix, iy, iz]]
    coarse = evaluate(coarse_cells)
    final, trace = select_roi_3d(coarse, full, frame_fraction, n_min)
    (x0, y0, z0), (x1, y1, z1) = final
    fine_cells = [(ix, iy, iz) for ix in range(x0, x1 + 1) for iy in range(y0, y1 + 1) for iz in range(z0, z1 + 1)
                  if mask[ix, iy, iz] and (ix, iy, iz) not in coarse]
    fine = evaluate(fine_cells)
    comp = dict(coarse)
    comp.update(fine)
    best = max(comp, key=lambda k: (comp[k], tuple(-x for x in k)))
    return comp, {"final_region": final, "trace": trace, "argmax_cell": best, "coarse": len(coarse),
                  "fine": len(fine)}


# ---------------------------------------------------------------------------
# BASELINE configs[2] segmentation variant: reference
# energies on per-quadrant n_sub x n_sub sub-grids + a restated control loop
# (quadrant split = Region.quadrants, geometry.py:225-242; max/mean score,
# DMAS shifted by the iteration minimum; argmax with first-index ties; stop
# when the kept segment's larger side <= stop_cells).
# ---------------------------------------------------------------------------
def segment_baseline(antennas, v, dt, signals, kind, origin, res, dims, n_sub=16, stop_cells=40, window=None,
                     region=None, mask=None):
    def energies(pts):
        if window is None:
            return multistatic_energies(antennas, v, dt, signals, pts, kind)
        return windowed_energies(antennas, v, dt, signals, pts, kind, window[0], window[1])

    sel = region if region is not None else ((0, 0), (dims[0] - 1, dims[1] - 1))
    records = []
    lowres = None
    while True:
        (x0, y0), (x1, y1) = sel
        w, h = x1 - x0 + 1, y1 - y0 + 1
        if max(w, h) <= stop_cells or w < 2 or h < 2:
            break
        quads = quadrants(sel)
        pts = []
        for (qx0, qy0), (qx1, qy1) in quads:
            wx, wy = (qx1 - qx0 + 1) * res, (qy1 - qy0 + 1) * res
            cx, cy = origin[0] + qx0 * res, origin[1] + qy0 * res
            for i in range(n_sub):
                for j in range(n_sub):
                    pts.append((cx + (i + 0.5) * (wx / n_sub), cy + (j + 0.5) * (wy / n_sub)))
        e = energies(np.array(pts)).reshape(4, n_sub, n_sub)
        if lowres is None:
            lowres = np.zeros((2 * n_sub, 2 * n_sub))
            for k in range(4):
                lowres[(k & 1) * n_sub:(k & 1) * n_sub + n_sub, (k >> 1) * n_sub:(k >> 1) * n_sub + n_sub] = e[k]
        shift = float(e.min()) if kind == "dmas" else 0.0
        scores = []
        for k in range(4):
            ek = e[k] - shift
            mean = float(ek.mean())
            scores.append(float(ek.max()) / mean if mean > 0 else 0.0)
        selected = int(np.argmax(scores))
        records.append({"selected": selected, "scores": scores, "parent": sel, "selected_region": quads[selected]})
        sel = quads[selected]
    (x0, y0), (x1, y1) = sel
    cells = [(ix, iy) for ix in range(x0, x1 + 1) for iy in range(y0, y1 + 1) if mask is None or mask[ix, iy]]
    fine = {}
    if cells:
        pts = np.array([(origin[0] + (ix + 0.5) * res, origin[1] + (iy + 0.5) * res) for ix, iy in cells])
        fine = dict(zip(cells, energies(pts).tolist()))
    best = argmax_cell(fine) if fine else None
    return {"final_region": sel, "records": records, "fine": fine, "argmax_cell": best, "lowres": lowres}


# ---------------------------------------------------------------------------
# monostatic DAS — beamform.py:215-239 (Eq. (1) delay d / (2 v dt), diagonal
# channels only)
# ---------------------------------------------------------------------------
def monostatic_energies(antennas, v, dt, signals, points):
    ants = np.asarray(antennas, dtype=np.float64)
    sig = np.asarray(signals, dtype=np.float64)
    m, _, nsamp = sig.shape
    pts = np.asarray(points, dtype=np.float64)
    dx = pts[:, 0, None] - ants[None, :, 0]
    dy = pts[:, 1, None] - ants[None, :, 1]
    dz = ants[None, :, 2]
    d = np.sqrt(dx * dx + dy * dy + dz * dz)
    shifts = d / (2.0 * v * dt)
    i0 = np.floor(shifts).astype(np.int64)
    frac = shifts - i0
    diag = sig[np.arange(m), np.arange(m)]
    ypad = np.zeros((m, nsamp + int(i0.max()) + 2))
    ypad[:, :nsamp] = diag
    win = sliding_window_view(ypad, nsamp + 1, axis=1)
    s = np.zeros((len(pts), nsamp))
    for ch in range(m):
        w = win[ch, i0[:, ch]]
        f1 = frac[:, ch, None]
        s += (1.0 - f1) * w[:, :nsamp]
        s += f1 * w[:, 1:]
    return (s * s).sum(axis=1)
