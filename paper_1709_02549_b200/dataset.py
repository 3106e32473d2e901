"""Input container of the imaging path.

``BackscatterDataset`` mirrors the reference's frozen container
(/root/reference/pkg/src/mwbeam/simulate.py:76-108): ``signals[i, j, k]`` is
sample k of transmitter i / receiver j, shape (M, M, N) float64, made
read-only on construction.  Because it is frozen, the GPU path may cache the
fp32 compaction of its populated channels on the device (see ``_device``).
Any object with the same attributes (e.g. the reference's own dataset class)
is accepted by the imaging functions.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import ArrayGeometry


@dataclass(frozen=True, eq=False)
class BackscatterDataset:
    geometry: ArrayGeometry
    signals: np.ndarray
    t0: float = 0.0

    def __post_init__(self):
        sig = np.array(self.signals, dtype=np.float64, copy=True)
        m = self.geometry.n_antennas
        if sig.ndim != 3 or sig.shape[:2] != (m, m):
            raise ValueError("signals must have shape (M, M, N)")
        sig.setflags(write=False)
        object.__setattr__(self, "signals", sig)

    @property
    def n_antennas(self) -> int:
        return int(self.signals.shape[0])

    @property
    def n_samples(self) -> int:
        return int(self.signals.shape[2])

    def is_monostatic(self) -> bool:
        """True when every off-diagonal channel is identically zero."""
        off = self.signals.copy()
        idx = np.arange(self.n_antennas)
        off[idx, idx] = 0.0
        return not off.any()
