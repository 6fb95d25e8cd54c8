"""Small-ring workload for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python scripts/sanitize_smoke.py [small|ring14|cluster]

Exercises every kernel family of the library once: encode, encrypt (sync and
pinned-async), rotations (single, multi-key, rotate-and-add, hoisted), the key
inner product and ModDown, ct x pt (plain and fused HMA), scalar multiply,
add_plain, square + relinearization, mod switch, hoisted dot, decrypt.  Checks
the decrypted slots against plain modular arithmetic so a silent corruption
under the sanitizer also fails.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_03494_b200.params import make_params  # noqa: E402
from paper_2102_03494_b200.rlwe import Evaluator  # noqa: E402

CASES = {
    "small": (1024, [65537], 3, 50),       # n = 2^11, one CTA per row
    "ring14": (8192, [65537], 3, 50),      # n = 2^14, the configs[1] row kernels
    "cluster": (16384, [65537], 2, 50),    # n = 2^15, 2-CTA cluster rows (DSMEM)
}


def main(which):
    n_slots, t, L, qb = CASES[which]
    P = make_params(n_slots, t, levels=L, q_bits=qb, seed=11)
    ev = Evaluator(P)
    rng = np.random.default_rng(5)
    R = 2
    tt = P.t[0]
    a = rng.integers(0, tt, size=(1, R, P.n), dtype=np.uint64)
    b = rng.integers(0, tt, size=(1, R, P.n), dtype=np.uint64)
    w = rng.integers(0, tt, size=(1, P.n), dtype=np.uint64)
    ca, cb = ev.encrypt(a), ev.encrypt(b)
    pt = ev.encode(w)
    A, B, Wt = a.astype(object), b.astype(object), w.astype(object)[:, None, :]
    N = P.n_slots

    def roll(x, k):
        return np.concatenate([np.roll(x[..., :N], -k, axis=-1), np.roll(x[..., N:], -k, axis=-1)], axis=-1)

    def check(ct, want, what):
        got = ev.decrypt(ct).astype(object)
        if not np.array_equal(got, want % tt):
            raise SystemExit(f"sanitize_smoke[{which}]: {what} decrypts wrong")

    check(ev.add(ca, cb), A + B, "add")
    check(ev.mul_plain(ca, pt), A * Wt, "mul_plain")
    acc = ev.encrypt(b)
    ev.mul_plain_acc(ca, pt, acc)
    check(acc, B + A * Wt, "mul_plain_acc")
    check(ev.mul_scalar(ca, -3), A * -3, "mul_scalar")
    check(ev.add_plain(ca, pt), A + Wt, "add_plain")
    check(ev.rotate(ca, 3), roll(A, 3), "rotate")
    r1, r2 = ev.rotate_multi([ca, cb], [1, N - 1])
    check(r1, roll(A, 1), "rotate_multi[0]")
    check(r2, roll(B, N - 1), "rotate_multi[1]")
    (ra,) = ev.rotate_add_many([ca], 5)
    check(ra, A + roll(A, 5), "rotate_add")
    hs = ev.rotate_hoisted(ca, [2, 7])
    check(hs[1], roll(A, 7), "rotate_hoisted")
    check(ev.mod_switch(ca), A, "mod_switch")
    if P.b:
        check(ev.square(ca), A * A, "square")
    ks = [0, 2, 7]
    gs = [pow(5, k, 2 * P.n) for k in ks]
    (hd,) = ev.hoisted_dot([ca, hs[0], hs[1]], gs, [pt])
    want = sum(roll(A, k) * roll(np.broadcast_to(Wt, A.shape), k) for k in ks)
    check(hd, want, "hoisted_dot")
    ev.sync()
    print(f"sanitize_smoke[{which}] ok")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
