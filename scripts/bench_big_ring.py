"""Key-switched rotation throughput at the configs[3] parameters (ring 2^16, L = 8,
T = 6): same-key batches, per-ciphertext keys, and a per-kernel breakdown."""
import ctypes, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import bench  # noqa: E402
from paper_2102_03494_b200.rlwe import Evaluator  # noqa: E402
from paper_2102_03494_b200.abi import cuda_library  # noqa: E402

net, plan, ws, xs, rp, ref = bench.cfg3_setup(2, seed=bench.CFG1["seed"])
lib = cuda_library()
ev = Evaluator(rp, lib)
R = int(os.environ.get("ROWS", "8"))
rng = np.random.default_rng(0)
s = np.stack([rng.integers(0, ti, size=(R, rp.n), dtype=np.uint64) for ti in rp.t]).astype(np.uint64)
ct = ev.encrypt(s)
phys = R * len(rp.t)
out = {"n": rp.n, "L": rp.L, "T": len(rp.t), "phys_cts": phys}
ev.rotate(ct, 3)
ev.sync()
t0 = time.perf_counter()
for it in range(5):
    ev.rotate(ct, 3)
ev.sync()
out["same_key_rot_per_s"] = 5 * phys / (time.perf_counter() - t0)
steps = [int(k) for k in rng.choice(np.arange(1, rp.n // 2), size=R, replace=False)]
cts1 = [ev.encrypt(s[:, :1]) for _ in range(R)]
ev.sync()
t0 = time.perf_counter()
ev.rotate_multi(cts1, steps)
ev.sync()
out["fresh_keys_rot_per_s"] = R * len(rp.t) / (time.perf_counter() - t0)
t0 = time.perf_counter()
ev.rotate_multi(cts1, steps)
ev.sync()
out["cached_keys_rot_per_s"] = R * len(rp.t) / (time.perf_counter() - t0)
lib.call("fhe_prof_enable", ev.ctx, 1)
ev.rotate(ct, 3)
ev.rotate_multi(cts1, [k + 1 for k in steps])
buf = ctypes.create_string_buffer(1 << 16)
lib.call("fhe_prof_report", ev.ctx, buf, len(buf))
lib.call("fhe_prof_enable", ev.ctx, 0)
out["prof"] = {k: {"calls": c, "ms": round(m, 3)} for k, (c, m) in bench.parse_prof(buf.value.decode()).items()}
print(json.dumps(out, indent=1))
