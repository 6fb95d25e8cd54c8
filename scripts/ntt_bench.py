"""NTT core variant benchmark (n = 2^14, 1024 rows): time per row and modmul rate."""
import ctypes, json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03494_b200.params import make_params
from paper_2102_03494_b200.rlwe import Evaluator

P = make_params(8192, [65537], levels=2, q_bits=int(os.environ.get('QBITS', 59)), p_bits=int(os.environ.get('QBITS', 59)) + 1, aux=False)
ev = Evaluator(P)
peak = ctypes.c_double()
ev.lib.call("fhe_peak_modmul", ev.ctx, 20000, ctypes.byref(peak))
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
out = {"peak_gmodmul": peak.value / 1e9, "rows": rows}
WS = os.environ.get("WS")
plan = tuple((inv, tuple(int(w) for w in WS.split(","))) for inv in (0, 1)) if WS else ((0, (4, 5, 100)), (1, (4, 5, 100)))
for inv, Ws in plan:
    for W in Ws:
        ms, bad = ctypes.c_float(), ctypes.c_uint32()
        ev.lib.call("fhe_bench_ntt", ev.ctx, W, inv, rows, 20, ctypes.byref(ms), ctypes.byref(bad))
        mm = rows * 8192 * 14 / (ms.value * 1e-3)
        out[f"{'inv' if inv else 'fwd'}_W{W}"] = {"ms": ms.value, "us_per_row": 1e3 * ms.value / rows,
                                                  "gmodmul": mm / 1e9, "frac": mm / peak.value,
                                                  "gbs": rows * 8192 * 16 * 2 / (ms.value * 1e-3) / 1e9,
                                                  "mismatch_rows": bad.value}
print(json.dumps(out, indent=1))
