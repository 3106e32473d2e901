"""Shared-memory load-width / broadcast probe (development aid)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_02549_b200 import _native as nat
lib = nat.load()
names = ["consecutive", "all-same", "lane/2", "lane/4", "lane/8", "3*lane/8"]
for wsel, wname in ((100, "LDS.32"), (110, "LDS.64"), (120, "LDS.128")):
    for p, pn in enumerate(names):
        work, ms = ctypes.c_double(), ctypes.c_float()
        nat.check(lib.mwb_microbench(wsel + p, ctypes.byref(work), ctypes.byref(ms), None), "mb")
        print(f"{wname:8s} {pn:12s} {work.value / (ms.value * 1e-3) / 1e12:7.2f} TB/s to registers")
for w, n in ((0, "LDS.32 baseline"), (1, "FFMA2"), (2, "FFMA")):
    work, ms = ctypes.c_double(), ctypes.c_float()
    nat.check(lib.mwb_microbench(w, ctypes.byref(work), ctypes.byref(ms), None), "mb")
    print(n, work.value / (ms.value * 1e-3) / 1e12)
