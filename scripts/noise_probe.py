"""Noise-budget probe for the cfg0 circuit shape (parameter selection evidence).

Runs the multiplicative chain of the FFConv MNIST network on one ciphertext
(full plaintext multiplies, rotate-and-sum trees, one-hot masks, combine chains,
squares) and prints the remaining invariant-noise budget after each stage, for
several plaintext-prime sizes and q chains.  Output: one JSON line per setting.
"""

import json
import math
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03494_b200.params import RlweParams, ntt_primes  # noqa: E402
from paper_2102_03494_b200.rlwe import Evaluator  # noqa: E402


def probe(t_bits, q_bits, L, combine_len=(168, 100), modswitch=False):
    n_slots = 8192
    two_n = 4 * n_slots
    t = ntt_primes(t_bits, 1, two_n)
    q = ntt_primes(q_bits, L, two_n, exclude=t)
    p = ntt_primes(min(q_bits + 1, 61), 1, two_n, exclude=t + q)
    b = ntt_primes(60, L + 1, two_n, exclude=t + q + p)
    P = RlweParams(log_n=14, q=tuple(q), p=tuple(p), t=tuple(t), b=tuple(b))
    ev = Evaluator(P)
    rng = np.random.default_rng(0)
    n = P.n
    T = t[0]
    log = []

    def rec(name, ct):
        log.append((name, round(float(ev.noise_budget(ct).min()), 1), ct.level))

    def rand_pt():
        return ev.encode(rng.integers(0, T, size=(1, n)).astype(np.uint64))

    def onehot():
        v = np.zeros((1, n), dtype=np.uint64)
        v[0, 0] = 1
        v[0, n_slots] = 1
        return ev.encode(v)

    def rs(ct, m):
        for h in reversed(range((m - 1).bit_length())):
            ct = ev.add(ct, ev.rotate(ct, 1 << h))
        return ct

    def chain(ct, k):
        acc = ct
        for i in range(k):
            acc = ev.add(acc, ev.rotate(ct, 1 + (i % 97)))
        return acc

    x = ev.encrypt(rng.integers(0, 256, size=(1, 1, n)).astype(np.uint64))
    rec("fresh", x)
    y = rs(ev.mul_plain(x, rand_pt()), 841)
    rec("w1 dot+rs", y)
    y = ev.mul_plain(y, onehot())
    rec("w1 mask", y)
    y = chain(y, combine_len[0])
    rec("w1 combine", y)
    y = ev.add(ev.mul_scalar(y, 127), ev.mul_scalar(ev.rotate(y, 1), -113))
    rec("w2 scalar", y)
    y = chain(y, 4)
    rec("combine5", y)
    y = ev.square(y)
    rec("square1", y)
    y = rs(ev.mul_plain(y, rand_pt()), 845)
    rec("fc1 dot+rs", y)
    y = ev.mul_plain(y, onehot())
    rec("fc1 mask", y)
    y = chain(y, combine_len[1] - 1)
    rec("fc1 combine", y)
    y = ev.square(y)
    rec("square2", y)
    y = rs(ev.mul_plain(y, rand_pt()), 100)
    rec("fc2 dot+rs", y)
    return {"t_bits": t_bits, "q_bits": q_bits, "L": L, "logQ": round(sum(math.log2(v) for v in q), 1),
            "logQP": round(P.log_qp, 1), "stages": log}


if __name__ == "__main__":
    settings = [(20, 58, 5), (20, 58, 6), (25, 58, 6), (25, 60, 6), (30, 60, 6), (30, 60, 7)]
    if len(sys.argv) > 1:
        settings = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]]
    for tb, qb, L in settings:
        print(json.dumps(probe(tb, qb, L)), flush=True)
