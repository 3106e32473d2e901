"""Benchmark of the B200 DAS/DMAS imaging path (one JSON line on rank 0).

Workload (BASELINE.json configs[3], the batched-throughput configuration):
4096 independent seeded scans per GPU, 12 antennas / 66 Tx-Rx pairs, 1024
fp32 samples, each imaged with DAS and with DMAS on a 256 x 256 grid over
12 x 12 cm with a 32-sample energy window.  One step = DAS + DMAS over all
scans of the rank.  ``value`` is pixel-pair evaluations per second over the
whole job (inputs resident in HBM); ``e2e`` is the same metric through the
public host API (pinned host scans in, host energy maps out, H2D/D2H inside
the timed region).  Multi-GPU: scans are sharded across ranks (weak scaling,
no data-path collective); the step time is the max over ranks.

``--impl reference`` times the reference's own CPU implementation (the
unmodified ``mwbeam`` staged in baseline/_ref, its ``image()`` with every host
core) on a bounded sample of the same workload; the ``cpu_baseline`` leg of
our arm runs the same routine (plus a threads=1 figure).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

METRIC = "DAS+DMAS pixel-pair evals/s (66 Tx-Rx pairs, 32-sample window)"
UNIT = "pixel-pair evals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scans", type=int, default=4096)
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--chunk", type=int, default=128)
    ap.add_argument("--mode", choices=["smem", "gather", "tc", "auto"], default="auto",
                    help="auto: tensor-core path when the table qualifies (configs[3] does), else smem")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def config_block(args, world):
    return {
        "workload": f"BASELINE configs[3] batched: {args.scans} scans/GPU x {args.grid}x{args.grid} px x (DAS + DMAS)",
        "scans_per_gpu": args.scans,
        "grid": [args.grid, args.grid],
        "extent_m": 0.12,
        "antennas": 12,
        "pairs": 66,
        "samples": 1024,
        "window": 32,
        "l2": "inputs (1.1 GB per GPU) larger than the 126 MB L2; no flush needed",
        "parallelism": f"scans sharded over {world} rank(s), no data-path collective",
    }


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class Clocks:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None
        self.t_on = self.t_off = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.file, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)

    def mark_on(self):
        self.t_on = time.time()

    def mark_off(self):
        self.t_off = time.time()

    def stop(self) -> dict:
        time.sleep(0.25)
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
        self.file.flush()
        rows = []
        for line in Path(self.file.name).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[4:]))
            except ValueError:
                continue
        os.unlink(self.file.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        # samples during the timed region: the middle of the run (the clock
        # sampler runs only while the timed loop executes, plus 0.3 s before)
        busy = [r for r in rows if r[0] > 0.5 * max(x[0] for x in rows)] or rows
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, flags in busy:
            for n, f in zip(names[1:], flags[1:]):
                if f.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(r[0] for r in busy), "sm_max_mhz": max(r[1] for r in rows),
                "samples": len(busy), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU reference: the real reference package (baseline/_ref, staged by
# baseline/stage.py), its own image() on the box's host cores
# ---------------------------------------------------------------------------
def _reference_package():
    """The unmodified ``mwbeam`` staged in baseline/_ref (None if not staged)."""
    ref = REPO / "baseline" / "_ref"
    if not (ref / "mwbeam" / "__init__.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import importlib
    import types

    # submodules by import path: the package namespace re-exports a function
    # named ``simulate`` over the module of that name
    return types.SimpleNamespace(**{m: importlib.import_module(f"mwbeam.{m}")
                                    for m in ("beamform", "geometry", "simulate")})


def cpu_reference_rate(seconds: float, threads: int, seed: int = 0) -> dict:
    """Pixel-pair evals/s of the reference's own ``image()`` (beamform.py:283-342)
    on host cores, DAS and DMAS alternating, on one configs[3] scan.

    The reference sums the full record (beamform.py:211-212); the configs[3]
    energy is over the window [k0, k0+W).  The reference computes it through
    the suffix-difference adapter (SURVEY.md §8c adapter 2): two calls of its
    own image() on the record truncated at b >= k0+W+max_delay+2,
    E = image(sig[..., k0:b]) - image(sig[..., k0+W:b]).  Each block is a
    region of whole grid rows holding >= 2 x threads x 64 cells, so the
    reference's ThreadPoolExecutor (beamform.py:331-336) has >= 2 batches of
    64 points for every worker.  ``busy_cores`` = process CPU time / wall
    time over the timed blocks (how many cores actually worked).
    Falls back to the numpy oracle port (``kind: port``) when the reference
    is not staged.
    """
    from paper_1709_02549_b200 import synth

    mb = _reference_package()
    model = synth.ScanModel()
    sig, _ = synth.batch_2d(model, [seed])
    full = synth.embed_pairs(12, model.pairs(), sig[0].astype(np.float64))
    g = model.geometry()
    ants = np.asarray(g.antennas, dtype=np.float64)
    n_side, side = 256, 0.12
    res = side / n_side
    # farthest cell centre from any antenna bounds every delay
    corner = np.array([[-side / 2, -side / 2], [side / 2, -side / 2], [-side / 2, side / 2], [side / 2, side / 2]])
    dmax = np.sqrt(((corner[:, None, :] - ants[None, :, :2]) ** 2).sum(-1) + ants[None, :, 2] ** 2).max()
    b = min(model.n_samples, model.k0 + model.window + int(np.ceil(2 * dmax / (g.propagation_speed *
                                                                                 g.sample_interval))) + 4)
    k0, w = model.k0, model.window
    rows = max(1, -(-2 * threads * 64 // n_side))
    kind_names = ("das", "dmas")
    if mb is not None:
        geom = mb.geometry.ArrayGeometry(ants, g.propagation_speed, g.sample_interval)
        head = mb.simulate.BackscatterDataset(geom, np.ascontiguousarray(full[..., k0:b]))
        tail = mb.simulate.BackscatterDataset(geom, np.ascontiguousarray(full[..., k0 + w:b]))
        grid = mb.geometry.ImagingGrid((-side / 2, -side / 2), (side, side), res)
        kinds = (mb.beamform.BeamformerKind.DAS, mb.beamform.BeamformerKind.DMAS)

        def block(i):
            x0 = (i * rows) % n_side
            reg = mb.geometry.Region((x0, 0), (min(n_side - 1, x0 + rows - 1), n_side - 1))
            e = mb.beamform.image(head, kinds[i % 2], grid, region=reg, threads=threads)
            t = mb.beamform.image(tail, kinds[i % 2], grid, region=reg, threads=threads)
            return [e.entries[c] - t.entries[c] for c in e.entries]
        kind = "reference"
        what = "mwbeam.beamform.image (baseline/_ref, unmodified)"
    else:
        from oracle import mwbeam_oracle as orc

        def block(i):
            x0 = (i * rows) % n_side
            cells = [(x, y) for x in range(x0, min(n_side, x0 + rows)) for y in range(n_side)]
            pts = np.array([((x + 0.5) * res - side / 2, (y + 0.5) * res - side / 2) for x, y in cells])
            batches = [pts[j:j + orc.BATCH] for j in range(0, len(pts), orc.BATCH)]
            from concurrent.futures import ThreadPoolExecutor

            with ThreadPoolExecutor(max_workers=threads) as pool:
                return list(pool.map(lambda bt: orc.windowed_energies(ants, g.propagation_speed, g.sample_interval,
                                                                        full, bt, kind_names[i % 2], k0, w), batches))
        kind = "port"
        what = "numpy oracle port (baseline/_ref not staged)"
    block(0)  # warm-up (imports, first allocations)
    done_px = 0
    i = 0
    c0, t0 = time.process_time(), time.perf_counter()
    while True:
        block(i)
        done_px += rows * n_side
        i += 1
        el = time.perf_counter() - t0
        if el >= seconds and i % 2 == 0:
            break
    cpu = time.process_time() - c0
    return {"value": done_px * 66 / el, "unit": UNIT, "cores": threads, "busy_cores": round(cpu / el, 2),
            "kind": kind,
            "sample": f"{what}: {done_px} px of one configs[3] scan in {i} blocks of {rows} x {n_side} cells "
                      f"(DAS, DMAS alternating), threads={threads}, {el:.1f} s; windowed energy = two reference "
                      f"image() calls on the record truncated at {b} samples (suffix-difference adapter)",
            "cpu_model": _cpu_model()}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def thread_candidates() -> list[int]:
    n = host_threads()
    return sorted({1, 2, 4, n} & set(range(1, n + 1)))


def cpu_baseline_block(seconds: float) -> dict:
    """The reference's CPU rate at its best thread count on this host.

    The reference parallelises only through a ThreadPoolExecutor over 64-point
    numpy batches (beamform.py:325-336), which the GIL serialises in part, so
    more threads is not always faster.  Every candidate count (1, 2, 4, all
    host threads) is timed on the same routine; the fastest is the reported
    baseline, and the per-count rates (threads=1 and threads=all included, as
    BASELINE.md §3 asks) are listed beside it with the cores each kept busy.
    """
    cands = thread_candidates()
    runs = {t: cpu_reference_rate(seconds / len(cands), t) for t in cands}
    best = max(runs, key=lambda t: runs[t]["value"])
    out = dict(runs[best])
    out["by_threads"] = {str(t): {"value": r["value"], "busy_cores": r["busy_cores"]} for t, r in runs.items()}
    out["threads1_value"] = runs[1]["value"]
    out["threads_all_value"] = runs[cands[-1]]["value"]
    out["host_threads"] = host_threads()
    return out


def _cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the reference's own CPU image() through
    cpu_reference_rate — the routine of our arm's cpu_baseline leg — at the
    thread count that runs it fastest on this host (the warm-up steps try
    1, 2, 4 and all host threads; every timed step uses the best), one bounded
    sample per step; rank 0 only."""
    rank, _, world = env_rank()
    if rank != 0:
        return
    per_step = max(1.0, min(6.0, 90.0 / max(1, args.steps + args.warmup)))
    cands = thread_candidates()
    trial = {}
    for i, t in enumerate(cands * max(1, -(-args.warmup // len(cands)))):
        trial.setdefault(t, []).append(cpu_reference_rate(per_step, t, seed=i)["value"])
    threads = max(trial, key=lambda t: statistics.median(trial[t]))
    vals = [cpu_reference_rate(per_step, threads, seed=args.warmup + i) for i in range(args.steps)]
    v = statistics.median(x["value"] for x in vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[3] signal model)",
        "config": config_block(args, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads,
                         "busy_cores": statistics.median(x["busy_cores"] for x in vals), "kind": vals[0]["kind"],
                         "sample": f"per step: {vals[0]['sample']}", "cpu_model": vals[0]["cpu_model"],
                         "warmup_rates_by_threads": {str(t): statistics.median(r) for t, r in trial.items()},
                         "host_threads": host_threads()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def smem_peak_gbs(lib) -> float:
    work, ms = ctypes.c_double(), ctypes.c_float()
    best = 0.0
    for _ in range(3):
        rc = lib.mwb_microbench(0, ctypes.byref(work), ctypes.byref(ms), None)
        if rc != 0:
            raise RuntimeError("microbench failed")
        best = max(best, work.value / (ms.value * 1e-3) / 1e9)
    return best


def fp32_peak_tflops(lib) -> float:
    work, ms = ctypes.c_double(), ctypes.c_float()
    best = 0.0
    for which in (1, 2):
        lib.mwb_microbench(which, ctypes.byref(work), ctypes.byref(ms), None)
        best = max(best, work.value / (ms.value * 1e-3) / 1e12)
    return best


def other_configs() -> dict:
    """Latency of the public API on the other BASELINE configurations (device
    time from CUDA events around whole calls, median of a few repeats)."""
    import torch

    import paper_1709_02549_b200 as mw
    from paper_1709_02549_b200 import synth
    from paper_1709_02549_b200.segment import segment
    from paper_1709_02549_b200.volume import VolumeGrid, hemisphere_mask, image_volume, run_framework_volume

    def med_ms(fn, reps=7):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    out = {}
    m0 = synth.ScanModel()
    ds, _ = synth.dataset_2d(m0, seed=0)
    win = (m0.k0, m0.window)
    g0 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 1e-3)
    g1 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 5e-4)
    t = med_ms(lambda: mw.image(ds, "das", g0, window=win))
    out["cfg0_das_100x100_image"] = {"ms": t, "pixel_pair_evals_per_s": 1e4 * 66 / (t * 1e-3)}
    # the reference's own semantics: energy over the full 1024-sample record (window=None)
    t = med_ms(lambda: mw.image(ds, "das", g0))
    out["cfg0_das_100x100_image_full_record"] = {"ms": t, "pixel_pair_evals_per_s": 1e4 * 66 / (t * 1e-3),
                                                 "pixel_pair_samples_per_s": 1e4 * 66 * 1024 / (t * 1e-3)}
    t = med_ms(lambda: mw.image(ds, "dmas", g1, window=win))
    out["cfg1_dmas_200x200_image"] = {"ms": t, "pixel_pair_evals_per_s": 4e4 * 66 / (t * 1e-3), "images_per_s": 1e3 / t}
    # the same configuration for a stream of scans: one launch per 1024 scans
    from paper_1709_02549_b200.batch import BatchImager

    sig1, _ = synth.batch_2d_device(m0, range(1024), phantom_radius=0.05, snr_db=20.0)
    bi1 = BatchImager(m0.geometry(), m0.pairs(), m0.n_samples, g1, window=win, mode="auto")
    o1 = torch.empty((1024, 200 * 200), dtype=torch.float32, device="cuda")
    t = med_ms(lambda: bi1.run_device(sig1, out_dmas=o1), reps=5)
    out["cfg1_dmas_200x200_batched_1024_scans"] = {"ms": t, "images_per_s": 1024 / (t * 1e-3),
                                                   "pixel_pair_evals_per_s": 1024 * 4e4 * 66 / (t * 1e-3),
                                                   "tensor_cores": bi1.uses_tensor_cores}
    del sig1, o1
    # configs[3] with the reference's own semantics: energy over the full
    # 1024-sample record (beamform.py:211-212); 256 of the 4096 scans, on the
    # CUDA-core K1 and on the tensor cores (32 chunks of 32 samples,
    # mwb_energies_tc_record)
    sig3, _ = synth.batch_2d_device(m0, range(256))
    g3 = synth.grid_square(0.12, 256)
    bi3 = BatchImager(m0.geometry(), m0.pairs(), m0.n_samples, g3, window=None, mode="smem")
    o3 = {k: torch.empty((256, 256 * 256), dtype=torch.float32, device="cuda") for k in ("das", "dmas")}
    t = med_ms(lambda: bi3.run_device(sig3, o3["das"], o3["dmas"]), reps=3)
    pe = 2.0 * 256 * 65536 * 66
    out["cfg3_full_record_256_scans"] = {"ms": t, "pixel_pair_evals_per_s": pe / (t * 1e-3),
                                         "pixel_pair_samples_per_s": 256 * 65536 * 66 * 1024 / (t * 1e-3),
                                         "note": "DAS + DMAS fused (one pass), window = full 1024-sample record, "
                                                 "energy_kernel<BOTH>; pixel_pair_samples counted once per pair"}
    del bi3
    bi3t = BatchImager(m0.geometry(), m0.pairs(), m0.n_samples, g3, window=None, mode="auto")
    if bi3t.uses_tensor_cores:
        t = med_ms(lambda: bi3t.run_device(sig3, o3["das"], o3["dmas"]), reps=3)
        out["cfg3_full_record_256_scans_tc"] = {
            "ms": t, "pixel_pair_evals_per_s": pe / (t * 1e-3),
            "pixel_pair_samples_per_s": 256 * 65536 * 66 * 1024 / (t * 1e-3),
            "note": "the same on the tensor cores: 32 fused W = 32 K1-TCH passes (one per 32-sample chunk), "
                    "chunk energies summed in fp64 (mwb_energies_tc_record)"}
    del sig3, o3, bi3t
    m2 = synth.ScanModel(n_samples=2048)
    ds2, _ = synth.dataset_2d(m2, seed=1000, phantom_radius=0.05)
    g2 = mw.ImagingGrid((-0.05, -0.05), (0.1, 0.1), 2.5e-4)
    d = g2.dims[0] // 32
    mask2 = mw.breast_mask(g2)  # computed once, as a scanner would
    for kind in ("das", "dmas"):
        out[f"cfg2_run_framework_{kind}"] = {"ms": med_ms(lambda: mw.run_framework(ds2, kind, g2, mw.Manual(d),
                                                                                    window=(m2.k0, 32)), reps=21)}
        out[f"cfg2_segment_{kind}"] = {"ms": med_ms(lambda: segment(ds2, kind, g2, 16, 0.01, window=(m2.k0, 32)),
                                                    reps=21)}
        out[f"cfg2_full_image_{kind}"] = {"ms": med_ms(lambda: mw.image(ds2, kind, g2, mask=mask2,
                                                                           window=(m2.k0, 32)), reps=21)}
    # the reference's acceptance criterion 2 (test_acceptance.py:86-111) on this
    # scan: median wall time of the full masked DMAS image over the framework
    # report's elapsed total, and wall over wall
    full_w, fw_w, fw_el = [], [], []
    for _ in range(21):
        t0 = time.perf_counter()
        mw.image(ds2, "dmas", g2, mask=mask2, window=(m2.k0, 32))
        full_w.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        _, rep2 = mw.run_framework(ds2, "dmas", g2, mw.Manual(d), window=(m2.k0, 32))
        fw_w.append(time.perf_counter() - t0)
        fw_el.append(rep2.elapsed["total"])
    out["cfg2_criterion2_dmas"] = {
        "full_image_wall_ms": statistics.median(full_w) * 1e3, "framework_wall_ms": statistics.median(fw_w) * 1e3,
        "framework_elapsed_total_ms": statistics.median(fw_el) * 1e3,
        "ratio_reference_formula": statistics.median(full_w) / statistics.median(fw_el),
        "ratio_wall": statistics.median(full_w) / statistics.median(fw_w),
        "point_reduction": rep2.reduction_ratio}
    # a stream of distinct scans through the drop-in API: every call uploads a new dataset
    stream1 = [synth.dataset_2d(m0, seed=500 + i)[0] for i in range(8)]
    stream2 = [synth.dataset_2d(m2, seed=1500 + i, phantom_radius=0.05)[0] for i in range(8)]
    it1, it2 = iter(stream1), iter(stream2)
    out["cfg1_dmas_200x200_image_new_dataset_each_call"] = {
        "ms": med_ms(lambda: mw.image(next(it1), "dmas", g1, window=win))}
    out["cfg2_run_framework_das_new_dataset_each_call"] = {
        "ms": med_ms(lambda: mw.run_framework(next(it2), "das", g2, mw.Manual(d), window=(m2.k0, 32)))}
    del stream1, stream2
    # the configs[2] framework for a batch of 4096 scans (FrameworkBatch)
    from paper_1709_02549_b200.fwbatch import FrameworkBatch

    sig2, _ = synth.batch_2d_device(m2, range(4096), phantom_radius=(0.04, 0.05))
    for kind in ("das", "dmas"):
        fb = FrameworkBatch(m2.geometry(), m2.pairs(), m2.n_samples, g2, mw.Manual(d), kind, window=(m2.k0, 32))
        t = med_ms(lambda: fb.run(sig2), reps=5)
        out[f"cfg2_framework_batch_4096_{kind}"] = {"ms": t, "segmented_images_per_s": 4096 / (t * 1e-3)}
        del fb
    # the BASELINE segmentation rule for the same 4096 scans (SegmentBatch)
    from paper_1709_02549_b200.segment import SegmentBatch

    for kind in ("das", "dmas"):
        sb = SegmentBatch(m2.geometry(), m2.pairs(), m2.n_samples, g2, kind, 16, 0.01, window=(m2.k0, 32))
        t = med_ms(lambda: sb.run(sig2), reps=5)
        out[f"cfg2_segment_batch_4096_{kind}"] = {"ms": t, "segmented_images_per_s": 4096 / (t * 1e-3)}
        del sb
    del sig2
    vm = synth.VolumeModel()
    sig, _ = synth.scan_3d(vm, seed=9)
    ds4 = mw.BackscatterDataset(vm.geometry(), synth.embed_pairs(vm.n_ant, vm.pairs(), sig))
    g4 = VolumeGrid((-0.06, -0.06, 0.0), (0.12, 0.12, 0.12), 0.12 / 128)
    from paper_1709_02549_b200 import volume as vmod

    def cold():
        vmod._VOLUME_CACHE.clear()
        image_volume(ds4, "dmas", g4, window=(vm.k0, vm.window))

    t = med_ms(cold, reps=3)
    out["cfg4_dmas_128cubed_volume"] = {"ms": t, "voxel_pair_evals_per_s": 128**3 * 496 / (t * 1e-3),
                                        "note": "first call for the geometry: enumeration + delay table + energies"}
    t = med_ms(lambda: image_volume(ds4, "dmas", g4, window=(vm.k0, vm.window)), reps=3)
    out["cfg4_dmas_128cubed_volume_repeat"] = {"ms": t, "voxel_pair_evals_per_s": 128**3 * 496 / (t * 1e-3),
                                               "note": "same scanner geometry: cached voxels and delay table"}
    vmod._VOLUME_CACHE.clear()
    mask = hemisphere_mask(g4, vm.phantom_radius)
    out["cfg4_octant_framework"] = {"ms": med_ms(lambda: run_framework_volume(
        ds4, "dmas", g4, mw.Automatic(0.01), mask=mask, window=(vm.k0, vm.window)), reps=3)}
    return out


def load_traffic():
    p = REPO / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return None
    return None


def smem_roofline(pps_launch, avg, smem_gbs, fp32_tf, traffic):
    """CUDA-core kernel: one fp32 sample per point-pair-sample serves both kinds
    (4 B of LDS), 4 FP32-pipe ops per point-pair-sample."""
    achieved = pps_launch * 4.0 / (avg * 1e-3) / 1e9
    fp32_frac = pps_launch * 4.0 / (avg * 1e-3) / (fp32_tf * 1e12 / 2.0)
    return {
        "bound": "smem",
        "kernel": "energy_kernel<BOTH> (fused DAS+DMAS)",
        "achieved": achieved,
        "peak": smem_gbs,
        "unit": "GB/s",
        "frac": achieved / smem_gbs,
        "traffic": traffic.get("energy_kernel_both") if isinstance(traffic, dict) else None,
        "algorithmic_bytes_per_launch": pps_launch * 4.0,
        "per_unit": "4 B of shared memory per point-pair-sample (one fresh fp32 sample serves DAS and DMAS; "
                    "the interpolation neighbour is reused in a register)",
        "peak_source": "LDS.32 bandwidth microbenchmark run live in this process (mwb_microbench 0)",
        "launch_ms": avg,
        "fp32_pipe_frac": fp32_frac,
        "fp32_ops_per_unit": 4,
        "fp32_peak_tflops": fp32_tf,
        "co_bound": "smem (1 LDS.32/pps) and FP32 pipe (FMUL+FFMA+FADD+FFMA per pps) peak at the same 32 pps/clk/SM",
    }


def pcie_floor(host_in, out_h, outs) -> float:
    """Seconds for one step's PCIe traffic with no compute: H2D of the step's
    input bytes (host_in, pinned) on one stream, D2H of the DAS and DMAS maps
    (outs -> out_h) on another, both in flight together; min of 3."""
    import torch

    dst = torch.empty(host_in.shape, dtype=host_in.dtype, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = float("inf")
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            dst.copy_(host_in, non_blocking=True)
        with torch.cuda.stream(s2):
            for k in ("das", "dmas"):
                out_h[k].copy_(outs[k], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    del dst
    return best


def tensor_peak():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (burst, cuBLAS)"
        except (ValueError, KeyError):
            pass
    return 1590.0, "fallback 1.59 PFLOP/s of B200_PROFILING.md (MEASURED_PEAKS.json absent)"


def tc_roofline(S, plan_steps, avg, traffic):
    """Tensor-core kernel (W = 32, energy_tch_kernel): per MMA step of a
    (128-point M-block, pair of 8-scan groups) item, six tcgen05.mma
    M128 x N256 x K16 f16 (two scan groups x the hi*hi, hi*lo, lo*hi split) =
    6 * 2 * 128 * 256 * 16 FLOP.  A step holds two 8-tap K halves, i.e. one
    channel whose points span <= 7 sample offsets, or half of a wider one;
    ``plan_steps`` counts the steps of all M-blocks for one pair of groups."""
    pairs = (S + 15) // 16
    flop_unit = 6 * 2 * 128 * 256 * 16
    flops = float(plan_steps) * pairs * flop_unit
    achieved = flops / (avg * 1e-3) / 1e12
    peak, source = tensor_peak()
    return {
        "bound": "tensor",
        "kernel": "energy_tch_kernel<BOTH> (tcgen05 fp16 hi/lo split, Hankel operand read in place from the "
                  "TMA-staged planes, 8-tap K packing; TMEM accumulation; DAS+DMAS fused)",
        "achieved": achieved,
        "peak": peak,
        "unit": "TFLOP/s",
        "frac": achieved / peak,
        "traffic": traffic.get("energy_tch_kernel_both") if isinstance(traffic, dict) else None,
        "algorithmic_flops_per_launch": flops,
        "mma_steps_per_pair": plan_steps,
        "per_unit": "6 x 2 x 128 x 256 x 16 FLOP per MMA step of a (128-point M-block, 16-scan pair) item; "
                    "steps = 8-tap K halves / 2 (one half per channel whose points span <= 7 offsets, else two)",
        "peak_source": source,
        "launch_ms": avg,
        "note": "launch_ms brackets the whole mwb_energies_tc call: the windowed-Gram / per-scan |y| max pre-pass, "
                "the 8-scan interleaved fp16-plane pre-pass, the per-tile step plan and the tensor-core kernel; "
                "FLOPs count only the kernel's MMAs",
    }


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1709_02549_b200 import _native as nat
    from paper_1709_02549_b200 import shard, synth
    from paper_1709_02549_b200.batch import BatchImager

    rank, local, world = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    lib = nat.load()

    model = synth.ScanModel()
    S = args.scans
    t_gen = time.perf_counter()
    # scans are synthesised on the device (mwb_simulate): same tumour/SNR draws
    # as the host generator, Philox noise; 4096 scans in ~60 ms
    sig_d, _ = synth.batch_2d_device(model, shard.scan_block(rank, world, S), noise_seed=rank)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    grid = synth.grid_square(0.12, args.grid)
    bi = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(model.k0, model.window),
                     mode=args.mode)
    P, C, W = bi.n_valid, bi.n_chan, model.window  # evaluated cells (the padded TC layout has more slots)
    nxny = grid.dims[0] * grid.dims[1]
    outs = {k: torch.empty((S, nxny), dtype=torch.float32, device=dev) for k in ("das", "dmas")}  # 2.1 GB
    keys = {k: torch.zeros(S, dtype=torch.int64, device=dev) for k in ("das", "dmas")}

    smem_gbs = smem_peak_gbs(lib)
    fp32_tf = fp32_peak_tflops(lib)

    def step(ev=None):
        # one fused launch: DAS and DMAS share the per-sample channel sum
        if ev is not None:
            ev[0].record()
        bi.run_device(sig_d, outs["das"], outs["dmas"], keys["das"], keys["dmas"])
        if ev is not None:
            ev[1].record()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks.mark_on()
    e0.record()
    for i in range(args.steps):
        step(evs[i])
    e1.record()
    torch.cuda.synchronize()
    clocks.mark_off()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = e0.elapsed_time(e1)
    launch_ms = [a.elapsed_time(b) for a, b in evs]
    elapsed_ms = shard.max_over_ranks(elapsed_ms, dev)  # device time, max over ranks
    ms_step = elapsed_ms / args.steps
    pair_evals = 2.0 * S * P * C * world
    value = pair_evals / (ms_step * 1e-3)
    images_s = 2.0 * S * world / (ms_step * 1e-3)

    avg = statistics.mean(launch_ms)
    pps_launch = float(S) * P * C * W
    traffic = load_traffic()
    if bi.uses_tensor_cores:
        roofline = tc_roofline(S, bi.tc_plan_steps(), avg, traffic)
        # useful work against the CUDA-core formulation's co-roofline (32 pps/clk/SM)
        pps_s = pps_launch / (avg * 1e-3)
        core_peak = smem_gbs * 1e9 / 4.0
        roofline["useful_pps_per_s"] = pps_s
        roofline["vs_cuda_core_roofline"] = pps_s / core_peak
        roofline["cuda_core_roofline_pps_per_s"] = core_peak
    else:
        roofline = smem_roofline(pps_launch, avg, smem_gbs, fp32_tf, traffic)


    # the CUDA-core kernel (north_star's design: shared-memory staging, FP32
    # pipe) on the same workload, timed in the same run, with its roofline
    core = None
    if bi.uses_tensor_cores and not args.no_configs:
        bk = BatchImager(model.geometry(), model.pairs(), model.n_samples, grid, window=(model.k0, model.window),
                         mode="smem")
        for _ in range(2):
            bk.run_device(sig_d, outs["das"], outs["dmas"], keys["das"], keys["dmas"])
        torch.cuda.synchronize()
        k_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        for a, b in k_ev:
            a.record()
            bk.run_device(sig_d, outs["das"], outs["dmas"], keys["das"], keys["dmas"])
            b.record()
        torch.cuda.synchronize()
        k_ms = statistics.mean(a.elapsed_time(b) for a, b in k_ev)
        core = {"kernel": "energy_kernel<BOTH> (CUDA cores, mode smem)", "ms_per_step": k_ms,
                "value": 2.0 * S * P * C / (k_ms * 1e-3), "unit": UNIT,
                "roofline": smem_roofline(pps_launch, k_ms, smem_gbs, fp32_tf, traffic)}
        # DAS alone (no per-sample DMAS self-term: 3 FP32 ops per pps, so the
        # smem side binds): the kernel's roofline fraction without the q FFMA
        d_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        for a, b in d_ev:
            a.record()
            bk.run_device(sig_d, out_das=outs["das"], key_das=keys["das"])
            b.record()
        torch.cuda.synchronize()
        d_ms = statistics.mean(a.elapsed_time(b) for a, b in d_ev)
        core["das_only"] = {"kernel": "energy_kernel<DAS>", "ms_per_step": d_ms,
                            "pixel_pair_evals_per_s": S * P * C / (d_ms * 1e-3),
                            "smem_frac": pps_launch * 4.0 / (d_ms * 1e-3) / 1e9 / smem_gbs}
        del bk

    # end to end through the public host API
    e2e = None
    if not args.no_e2e:
        host = sig_d[:, :, : model.n_samples].cpu().pin_memory()  # the e2e input lives in pinned host memory
        out_h = {k: torch.empty((S, nxny), dtype=torch.float32, pin_memory=True) for k in ("das", "dmas")}
        bi(host, kinds=("das", "dmas"), chunk=args.chunk, out=out_h)  # warm-up
        h2d = bi.h2d_bytes(S)  # __call__ ships only the sample range the kernels read
        floor_s = pcie_floor(host.view(-1)[: h2d // 4], out_h, outs)
        times = []
        for _ in range(max(1, min(args.steps, 5))):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bi(host, kinds=("das", "dmas"), chunk=args.chunk, out=out_h)
            times.append(time.perf_counter() - t0)
        e2e_s = shard.max_over_ranks(statistics.median(times), dev)
        from paper_1709_02549_b200.batch import _chunk_ranges

        chunks = len(_chunk_ranges(S, min(args.chunk, S))) * bi.kernels_per_call
        first, count = bi.input_range()
        e2e = {"value": pair_evals / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "h2d_what": f"samples [{first}, {first + count}) of every channel row (the range the tensor-core "
                           f"kernels read; whole rows are {int(host.numel() * 4)} B per step)",
               "d2h_bytes_per_step": int(2 * S * nxny * 4 + 2 * S * 8), "seconds_per_step": e2e_s,
               "api": "paper_1709_02549_b200.batch.BatchImager.__call__ (pinned host in, host maps out)",
               "gpu_launches_per_step": chunks,
               "pcie_floor_s": floor_s, "pcie_frac": floor_s / e2e_s,
               "pcie_floor_how": "the same step's bytes as two plain copies on two streams, measured in this run: "
                                 "H2D of the step's input bytes into device memory concurrent with D2H of both "
                                 "device maps into the pinned outputs (min of 3)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_block(args.cpu_seconds)
    others = other_configs() if (rank == 0 and world == 1 and not args.no_configs) else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            # arithmetic of the measured kernel: tcgen05 kind::f16 with fp16 hi/lo-split operands (3 products)
            # accumulating in fp32 TMEM, or fp32 FFMA on the CUDA-core path
            "dtype": "f16x3-split/f32-acc" if bi.uses_tensor_cores else "f32",
            "data": "synthetic: seeded differentiated-Gaussian scans (BASELINE configs[3] signal model) synthesised "
                    "on the device by mwb_simulate, no dataset",
            "config": config_block(args, world),
            "images_per_s": images_s,
            "pixel_pair_samples_per_s": value * W,
            "roofline": roofline,
            "cuda_core_path": core,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "other_configs": others,
            "gpu_launches": args.steps * bi.kernels_per_call,  # W = 32 TC: gram, planes, plan, A operands, energy
            "tensor_cores": bi.uses_tensor_cores,
            "clocks": clk,
            "kernel_mode": args.mode,
            "host_generate_s": t_gen,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
