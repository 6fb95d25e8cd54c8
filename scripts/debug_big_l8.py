import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03494_b200.params import make_params
from paper_2102_03494_b200.rlwe import Evaluator
from paper_2102_03494_b200.abi import Library, cuda_library
golden = Library("oracle/_golden/libgolden_rlwe.so")
cl = cuda_library()


def run(L, R, ksb=None, label=""):
    if ksb:
        os.environ["FHE_KS_BATCH"] = str(ksb)
    else:
        os.environ.pop("FHE_KS_BATCH", None)
    P = make_params(32768, [786433, 1179649], levels=L, q_bits=60 if L > 4 else 50, p_bits=61 if L > 4 else 51)
    gd, gp = Evaluator(P, golden), Evaluator(P, cl)
    rng = np.random.default_rng(1)
    s = np.stack([rng.integers(0, ti, size=(R, P.n), dtype=np.uint64) for ti in P.t]).astype(np.uint64)
    cg = gd.encrypt(s, nonce=3)
    cc = gp.new_ct(R)
    gp.write(cc, gd.read(cg))
    og, oc = gd.rotate(cg, 1), gp.rotate(cc, 1)
    a, b = gd.read(og), gp.read(oc)
    bad = [i for i in range(a.shape[0]) if not np.array_equal(a[i], b[i])]
    print(label, "L", L, "R", R, "ksb", ksb, "rotate(1) equal:", not bad, "bad phys cts:", bad, flush=True)


run(8, 1, label="a")
run(3, 6, label="b")
run(8, 6, 12, label="c")
run(8, 6, 3, label="d")
run(5, 1, label="e")
run(4, 1, label="f")
