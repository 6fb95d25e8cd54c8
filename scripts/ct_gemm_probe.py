"""k_ct_gemm (fhe_ct_gemm) against the multiply-add chain it replaces, at the shapes of
configs[3]'s ConvPack stages (K = 27 columns -> 8 channels; 8 -> 32), ring 2^14, L = 6,
64 images (32 row pairs).  Prints one JSON object."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03494_b200.abi import cuda_library  # noqa: E402
from paper_2102_03494_b200.params import make_params  # noqa: E402
from paper_2102_03494_b200.rlwe import Evaluator  # noqa: E402

P = make_params(8192, [65537], levels=6, q_bits=60)
ev = Evaluator(P, cuda_library())
R = 32
rng = np.random.default_rng(0)
out = {"ring_n": P.n, "L": P.L, "row_pairs": R, "cases": []}
for K, O in ((27, 8), (8, 32), (16, 64)):
    cts = [ev.encrypt(rng.integers(0, 3, size=(1, R, P.n)).astype(np.uint64)) for _ in range(K)]
    w = rng.integers(-127, 128, size=(K, O)).tolist()

    def gemm():
        return ev.ct_gemm(cts, w)

    def chain():
        res = []
        for o in range(O):
            acc = ev.mul_scalar(cts[0], w[0][o])
            for k in range(1, K):
                acc = ev.add(acc, ev.mul_scalar(cts[k], w[k][o]))
            res.append(acc)
        return res

    a, b = gemm(), chain()
    same = all(np.array_equal(ev.read(x), ev.read(y)) for x, y in zip(a[:2], b[:2]))
    del a, b
    t = {}
    for name, fn, reps in (("ct_gemm", gemm, 5), ("mul_scalar+add chain", chain, 2)):
        fn()
        ev.sync()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        ev.sync()
        t[name] = (time.perf_counter() - t0) / reps
    words = R * 2 * P.L * P.n
    gemm_bytes = (K * -(-O // 8) + O) * words * 8
    out["cases"].append({"K": K, "O": O, "equal_words": bool(same),
                         "ct_gemm_ms": 1e3 * t["ct_gemm"], "chain_ms": 1e3 * t["mul_scalar+add chain"],
                         "speedup": t["mul_scalar+add chain"] / t["ct_gemm"],
                         "ct_gemm_gbs": gemm_bytes / t["ct_gemm"] / 1e9,
                         "ct_gemm_gmac_s": K * O * words / t["ct_gemm"] / 1e9})
    del cts
print(json.dumps(out))
