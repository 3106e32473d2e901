"""Drop-in installer: rebind the hot-path names of an importable ``mwbeam``.

SURVEY.md §8(b): several reference modules bind the hot-path names at import
time (``from .beamform import image`` in coarse2fine.py:19, bench.py:14,
service/app.py:17; ``run_framework`` in bench.py:15-22 and service/app.py:19-24;
the package namespace, __init__.py:3-43).  Patching only
``_multistatic_energies`` would be functionally correct but launch-bound
(one launch per 64 points, beamform.py:325), so every binding of ``image``,
``das_energy``, ``dmas_energy``, ``point_energy``, ``select_roi``,
``run_framework`` and ``consistency_check`` is replaced, together with the
kernel entry ``_multistatic_energies`` and the ``EVAL_COUNTER`` object the
GPU ``image()`` adds to.

The GPU functions duck-type the reference's argument objects (grids, regions,
datasets, kinds, modes, configs) and return this package's result types,
which expose the same attributes and ``to_dict`` keys.
"""

from __future__ import annotations

import importlib

from . import beamform as bf
from . import coarse2fine as c2f

REPLACEMENTS = {
    "image": bf.image,
    "_multistatic_energies": bf._multistatic_energies,
    "EVAL_COUNTER": bf.EVAL_COUNTER,  # the counter the GPU image() adds to (beamform.py:74-75, 339)
    "das_energy": bf.das_energy,
    "dmas_energy": bf.dmas_energy,
    "point_energy": bf.point_energy,
    "das_energy_monostatic": bf.das_energy_monostatic,
    "select_roi": c2f.select_roi,
    "run_framework": c2f.run_framework,
    "consistency_check": c2f.consistency_check,
}

MODULES = ("", ".beamform", ".coarse2fine", ".bench", ".service.app")


class Installation:
    def __init__(self, saved: list):
        self.saved = saved

    @property
    def patched(self) -> list[str]:
        return [f"{m.__name__}.{name}" for m, name, _ in self.saved]

    def uninstall(self) -> None:
        for module, name, old in reversed(self.saved):
            setattr(module, name, old)
        self.saved = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.uninstall()


def install(package: str = "mwbeam") -> Installation:
    """Rebind every hot-path name in ``package`` and its submodules that bind
    them; returns a handle whose ``uninstall()`` restores the originals."""
    saved = []
    for suffix in MODULES:
        try:
            mod = importlib.import_module(package + suffix)
        except ImportError:
            continue  # optional submodules (service needs fastapi)
        for name, fn in REPLACEMENTS.items():
            if hasattr(mod, name):
                saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, fn)
    if not saved:
        raise ImportError(f"{package} is not importable: nothing to install into")
    return Installation(saved)
