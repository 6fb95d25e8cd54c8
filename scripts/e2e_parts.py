"""Where the configs[1] end-to-end step spends its time (1024 ciphertexts)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import bench  # noqa: E402
from paper_2102_03494_b200.abi import cuda_library  # noqa: E402
from paper_2102_03494_b200.rlwe import Evaluator  # noqa: E402

P = bench.rotation_params()
ev = Evaluator(P, cuda_library())
B, n = 1024, P.n
rng = np.random.default_rng(0)
slots = np.mod(rng.integers(-1, 2, size=(1, B, n)), P.t[0]).astype(np.uint64)
pin_in = torch.from_numpy(slots.view(np.int64)).pin_memory().numpy().view(np.uint64)
pin_out = torch.empty((1, B, n), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
k = 77
ev.keygen_rotations([k])


def t(label, fn, reps=5):
    fn(); ev.sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    ev.sync()
    dt = (time.perf_counter() - t0) / reps
    print(f"{label:40s} {dt * 1e3:8.2f} ms  -> {B / dt:9.0f} /s", flush=True)
    return dt


ct = ev.encrypt(pin_in)
ev.sync()
t("encrypt pageable", lambda: ev.encrypt(slots))
t("encrypt pinned (async)", lambda: ev.encrypt(pin_in, async_=True))
t("rotate", lambda: ev.rotate(ct, k))
t("decrypt pageable", lambda: ev.decrypt(ct))
t("decrypt pinned (async)", lambda: ev.decrypt(ct, out=pin_out, async_=True))
for ch in (1, 4, 8, 16):
    bounds = [(B * i // ch, B * (i + 1) // ch) for i in range(ch)]

    def step():
        for r0, r1 in bounds:
            c = ev.encrypt(pin_in[:, r0:r1], async_=True)
            r = ev.rotate(c, k)
            ev.decrypt(r, out=pin_out[:, r0:r1], async_=True)
    t(f"e2e chunks={ch}", step)
for ch in (8,):
    bounds = [(B * i // ch, B * (i + 1) // ch) for i in range(ch)]

    def step2():
        cs = [ev.encrypt(pin_in[:, r0:r1], async_=True) for r0, r1 in bounds]
        rs = ev.rotate_many(cs, k)
        for (r0, r1), r in zip(bounds, rs):
            ev.decrypt(r, out=pin_out[:, r0:r1], async_=True)
    t(f"e2e enc/dec chunks={ch} + rotate_many", step2)

# per-kernel breakdown of encrypt / decrypt (single stream, isolated kernel times)
import ctypes  # noqa: E402
lib = ev.lib
for label, fn in (("encrypt", lambda: ev.encrypt(pin_in, async_=True)), ("decrypt", lambda: ev.decrypt(ct, out=pin_out, async_=True))):
    fn(); ev.sync()
    lib.call("fhe_prof_enable", ev.ctx, 1)
    fn(); ev.sync()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.call("fhe_prof_report", ev.ctx, buf, len(buf))
    lib.call("fhe_prof_enable", ev.ctx, 0)
    print(label, buf.value.decode().strip().replace("\n", " | "))
