"""Integer-pipe roofline probe, standalone (for ncu): k_peak_modmul in both forms.

    python scripts/peak_probe.py
    ncu --set full -k regex:k_peak_modmul python scripts/peak_probe.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import rotation_params  # noqa: E402
from paper_2102_03494_b200.rlwe import Evaluator  # noqa: E402

ev = Evaluator(rotation_params())
for kind, name in ((0, "shoup_exact"), (1, "shoup_approx")):
    v = ctypes.c_double()
    ev.lib.call("fhe_peak_modmul_kind", ev.ctx, 20000, kind, ctypes.byref(v))
    print(f"{name}: {v.value / 1e9:.1f} Gmodmul/s")
