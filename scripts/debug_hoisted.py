import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03494_b200.params import make_params
from paper_2102_03494_b200.rlwe import Evaluator
from paper_2102_03494_b200.abi import cuda_library
P = make_params(1024, [65537], levels=4, q_bits=55)
gp = Evaluator(P, cuda_library())
rng = np.random.default_rng(1)
for R in (1, 2):
    s = np.stack([rng.integers(0, ti, size=(R, P.n), dtype=np.uint64) for ti in P.t]).astype(np.uint64)
    c = gp.encrypt(s)
    for ks in ([1], [1, 5], [3, 1]):
        hs = gp.rotate_hoisted(c, ks)
        for k, h in zip(ks, hs):
            a, b = gp.read(gp.rotate(c, k)), gp.read(h)
            diff = np.argwhere(a != b)
            print("R", R, "ks", ks, "k", k, "equal", not len(diff), "first diffs", diff[:3].tolist(), "ndiff", len(diff),
                  "dec ok", np.array_equal(gp.decrypt(h), gp.decrypt(gp.rotate(c, k))))
