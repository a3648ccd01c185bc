"""FP64 pipe probes (fe_fp64_peak): 0 DFMA, 1 DMMA, 2 half-and-half (shared
datapath?), 100 + w: DFMA with w warps per SM (16 independent chains each)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12220_b200 import feinsum as fe  # noqa: E402

for w in [0, 1, 2, 104, 108, 112, 116, 124, 132]:
    v = ctypes.c_double()
    fe.lib().fe_fp64_peak(w, ctypes.byref(v))
    print(w, round(v.value, 2))
