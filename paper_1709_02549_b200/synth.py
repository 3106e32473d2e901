"""Seeded synthetic multistatic scans for the BASELINE.json configurations.

No public dataset is involved: BASELINE.json defines the workloads by their
signal model, which this generator implements.

* Antennas: ``n_ant`` evenly on a ring of radius 7 cm (2-D configs) or on a
  hemisphere of radius 8 cm (3-D config, Fibonacci placement, z >= 0).
* Tissue: relative permittivity 9, so v = c/3; sampling 50 GS/s (dt = 20 ps).
* Pulse: differentiated Gaussian p(u) = -(u/tau) e^{1/2} e^{-u^2/(2 tau^2)},
  tau = 60 ps, peak amplitude 1, centred at t_c = 480 ps.
* Channel (i, j), i < j (the 66 / 496 unordered pairs; the diagonal and the
  lower triangle stay zero): Y_ij[k] = sum_s p(k dt - (d_i + d_j)/v - t_c) / (d_i d_j)
  over the point scatterers s.
* Noise: white Gaussian, sigma = max|clean| / 10^(SNR/20) per scan.
* Energy window: W samples starting at k0 = round(t_c/dt) - W/2, i.e. centred
  on the aligned pulse.

Everything is numpy with ``default_rng(seed)``, so a scan is reproducible
from its seed on any host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .dataset import BackscatterDataset
from .geometry import SPEED_OF_LIGHT, ArrayGeometry, ImagingGrid, ring_array


@dataclass(frozen=True)
class ScanModel:
    n_ant: int = 12
    ring_radius: float = 0.07
    eps_r: float = 9.0
    dt: float = 20e-12
    n_samples: int = 1024
    tau: float = 60e-12
    t_c: float = 480e-12
    window: int = 32

    @property
    def v(self) -> float:
        return SPEED_OF_LIGHT / math.sqrt(self.eps_r)

    @property
    def k0(self) -> int:
        return int(round(self.t_c / self.dt)) - self.window // 2

    def geometry(self) -> ArrayGeometry:
        return ring_array(self.n_ant, self.ring_radius, propagation_speed=self.v, sample_interval=self.dt)

    def pairs(self) -> np.ndarray:
        i, j = np.triu_indices(self.n_ant, k=1)
        return np.stack([i, j], axis=1).astype(np.int32)


def diff_gaussian(u: np.ndarray, tau: float) -> np.ndarray:
    x = u / tau
    return -x * np.exp(0.5 - 0.5 * x * x)


PULSE_SUPPORT = 12.0  # the pulse is evaluated within +-12 tau (|p| < 1e-29 beyond)


def clean_pairs(model: ScanModel, antennas: np.ndarray, scatterers, pairs: np.ndarray) -> np.ndarray:
    """(C, N) noiseless pair signals for point scatterers [((x, y, z), amplitude)]."""
    n = model.n_samples
    out = np.zeros((pairs.shape[0], n))
    half = int(math.ceil(PULSE_SUPPORT * model.tau / model.dt)) + 1
    offs = np.arange(-half, half + 1)
    rows = np.arange(pairs.shape[0])[:, None]
    for pos, amp in scatterers:
        p = np.asarray(pos, dtype=np.float64)
        if p.shape == (2,):
            p = np.array([p[0], p[1], 0.0])
        d = np.linalg.norm(antennas - p[None, :], axis=1)
        di, dj = d[pairs[:, 0]], d[pairs[:, 1]]
        delay = (di + dj) / model.v + model.t_c
        k = np.rint(delay / model.dt).astype(np.int64)[:, None] + offs[None, :]
        ok = (k >= 0) & (k < n)
        kc = np.clip(k, 0, n - 1)
        vals = amp * diff_gaussian(model.dt * kc - delay[:, None], model.tau) / (di * dj)[:, None]
        out[np.broadcast_to(rows, k.shape)[ok], kc[ok]] += vals[ok]
    return out


def add_noise(clean: np.ndarray, snr_db: float, rng: np.random.Generator) -> np.ndarray:
    peak = float(np.abs(clean).max())
    sigma = peak / (10.0 ** (snr_db / 20.0)) if peak > 0 else 0.0
    return clean + sigma * rng.standard_normal(clean.shape)


def uniform_in_disc(rng: np.random.Generator, radius: float) -> tuple[float, float]:
    r = radius * math.sqrt(rng.uniform())
    th = 2.0 * math.pi * rng.uniform()
    return (r * math.cos(th), r * math.sin(th))


def embed_pairs(m: int, pairs: np.ndarray, sig: np.ndarray) -> np.ndarray:
    full = np.zeros((m, m, sig.shape[-1]))
    full[pairs[:, 0], pairs[:, 1]] = sig
    return full


def scan_2d(model: ScanModel, seed: int, phantom_radius=0.05, snr_db=20.0):
    """One 2-D scan: (C, N) float64 pair signals and the tumour (x, y).

    ``phantom_radius`` / ``snr_db`` may be (lo, hi) ranges drawn per scan.
    """
    rng = np.random.default_rng(seed)
    radius = rng.uniform(*phantom_radius) if isinstance(phantom_radius, tuple) else phantom_radius
    snr = rng.uniform(*snr_db) if isinstance(snr_db, tuple) else snr_db
    tumour = uniform_in_disc(rng, radius)
    geom = model.geometry()
    pairs = model.pairs()
    clean = clean_pairs(model, geom.antennas, [(tumour, 1.0)], pairs)
    return add_noise(clean, snr, rng), tumour


def dataset_2d(model: ScanModel, seed: int, phantom_radius=0.05, snr_db=20.0) -> tuple[BackscatterDataset, tuple]:
    sig, tumour = scan_2d(model, seed, phantom_radius, snr_db)
    geom = model.geometry()
    return BackscatterDataset(geom, embed_pairs(model.n_ant, model.pairs(), sig)), tumour


def batch_2d(model: ScanModel, seeds, phantom_radius=(0.04, 0.06), snr_db=(10.0, 30.0)):
    """(S, C, N) float32 pair signals for a list of seeds plus (S, 2) tumour positions."""
    from concurrent.futures import ThreadPoolExecutor

    seeds = list(seeds)
    out = np.empty((len(seeds), model.n_ant * (model.n_ant - 1) // 2, model.n_samples), dtype=np.float32)
    tumours = np.empty((len(seeds), 2))

    def one(k: int) -> None:
        sig, tumour = scan_2d(model, seeds[k], phantom_radius, snr_db)
        out[k] = sig
        tumours[k] = tumour

    with ThreadPoolExecutor(max_workers=min(16, max(1, len(seeds)))) as pool:
        list(pool.map(one, range(len(seeds))))
    return out, tumours


def scan_params_2d(model: ScanModel, seeds, phantom_radius=(0.04, 0.06), snr_db=(10.0, 30.0)):
    """Per-scan (tumour x, y, SNR) drawn exactly as scan_2d draws them."""
    out = np.empty((len(seeds), 3))
    for k, seed in enumerate(seeds):
        rng = np.random.default_rng(seed)
        radius = rng.uniform(*phantom_radius) if isinstance(phantom_radius, tuple) else phantom_radius
        snr = rng.uniform(*snr_db) if isinstance(snr_db, tuple) else snr_db
        out[k, :2] = uniform_in_disc(rng, radius)
        out[k, 2] = snr
    return out


def batch_2d_device(model: ScanModel, seeds, phantom_radius=(0.04, 0.06), snr_db=(10.0, 30.0), noise_seed: int = 0,
                    noise: bool = True):
    """Device-side twin of batch_2d: (S, C, ld) fp32 CUDA tensor + (S, 2) tumours.

    Tumour positions and SNRs are the host generator's (same seeds, same draws);
    the clean pulses are evaluated on the GPU in fp64 with the same support;
    the noise is the device's Philox stream (statistically equivalent, not
    numpy's PCG64 sequence).  Produces the layout BatchImager.run_device takes.
    """
    import torch

    from . import _device as dv
    from . import _native as nat

    seeds = list(seeds)
    params = scan_params_2d(model, seeds, phantom_radius, snr_db)
    dev = dv.device()
    pairs = model.pairs()
    ld = dv.round4(model.n_samples)
    out = torch.empty((len(seeds), pairs.shape[0], ld), dtype=torch.float32, device=dev)
    scat = np.zeros((len(seeds), 1, 4))
    scat[:, 0, :2] = params[:, :2]
    scat[:, 0, 3] = 1.0
    scat_t = torch.from_numpy(scat).to(dev)
    snr_t = torch.from_numpy(np.ascontiguousarray(params[:, 2])).to(dev)
    peak = torch.empty(max(1, len(seeds)), dtype=torch.int32, device=dev)
    chan = torch.from_numpy(pairs).to(dev)
    ant = torch.from_numpy(np.array(model.geometry().antennas)).to(dev)
    nat.call("mwb_simulate", out.data_ptr(), len(seeds), pairs.shape[0], model.n_samples, ld, chan.data_ptr(),
             ant.data_ptr(), model.n_ant, scat_t.data_ptr(), 1, model.v, model.dt, 0.0, 1, model.tau, model.t_c, 0.0,
             snr_t.data_ptr(), 2 if noise else 0, noise_seed, peak.data_ptr(), dv.stream_handle())
    return out, params[:, :2].copy()


def grid_square(side: float, n: int) -> ImagingGrid:
    """n x n grid covering [-side/2, side/2]^2."""
    return ImagingGrid((-side / 2, -side / 2), (side, side), side / n)


# ---------------------------------------------------------------------------
# 3-D stress configuration (BASELINE configs[4])
# ---------------------------------------------------------------------------
def hemisphere_antennas(n: int, radius: float) -> np.ndarray:
    """Fibonacci points on the upper hemisphere (z >= 0) of ``radius``."""
    k = np.arange(n) + 0.5
    z = 1.0 - k / n  # cos(polar) uniform in (0, 1]
    r = np.sqrt(1.0 - z * z)
    phi = math.pi * (3.0 - math.sqrt(5.0)) * np.arange(n)
    return radius * np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


@dataclass(frozen=True)
class VolumeModel(ScanModel):
    n_ant: int = 32
    hemi_radius: float = 0.08
    n_samples: int = 2048
    window: int = 48
    phantom_radius: float = 0.06

    def geometry(self) -> ArrayGeometry:
        return ArrayGeometry(hemisphere_antennas(self.n_ant, self.hemi_radius), self.v, self.dt)


def scan_3d(model: VolumeModel, seed: int, snr_db=20.0):
    """(C, N) pair signals with 1-3 point tumours inside the hemispherical phantom."""
    rng = np.random.default_rng(seed)
    n_t = int(rng.integers(1, 4))
    tumours = []
    while len(tumours) < n_t:
        p = rng.uniform(-model.phantom_radius, model.phantom_radius, 3)
        p[2] = abs(p[2])
        if np.linalg.norm(p) < 0.8 * model.phantom_radius:
            tumours.append(p)
    geom = model.geometry()
    clean = clean_pairs(model, geom.antennas, [(t, 1.0) for t in tumours], model.pairs())
    return add_noise(clean, snr_db, rng), np.array(tumours)
