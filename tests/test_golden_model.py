"""Golden RLWE model properties (CPU): determinism of the sampler streams,
noise bookkeeping, modulus switching, and errors at the boundary."""

import numpy as np
import pytest

from paper_2102_03494_b200.abi import FheError
from paper_2102_03494_b200.params import make_params
from paper_2102_03494_b200.rlwe import Evaluator


def test_encryption_is_a_pure_function_of_seed_and_nonce(golden_lib):
    P = make_params(16, [65537], levels=3, q_bits=50)
    a, b = Evaluator(P, golden_lib), Evaluator(P, golden_lib)
    s = np.arange(2 * 32, dtype=np.uint64).reshape(1, 2, 32)
    assert np.array_equal(a.read(a.encrypt(s, nonce=5)), b.read(b.encrypt(s, nonce=5)))
    assert not np.array_equal(a.read(a.encrypt(s, nonce=5)), a.read(a.encrypt(s, nonce=6)))


def test_noise_budget_and_mod_switch(golden_lib):
    P = make_params(64, [65537], levels=4, q_bits=50)
    ev = Evaluator(P, golden_lib)
    rng = np.random.default_rng(0)
    s = rng.integers(0, 65537, size=(1, 1, 128)).astype(np.uint64)
    ct = ev.encrypt(s)
    b0 = ev.noise_budget(ct).min()
    assert b0 > 150
    pt = ev.encode(rng.integers(0, 65537, size=(1, 128)).astype(np.uint64))
    m = ev.mul_plain(ct, pt)
    assert ev.noise_budget(m).min() < b0 - 10
    down = ev.mod_switch(ct)
    assert down.level == 3 and np.array_equal(ev.decrypt(down), s)
    r = ev.rotate(down, 5)
    assert np.array_equal(ev.decrypt(r)[0, 0, :59], s[0, 0, 5:64])


def test_boundary_errors(golden_lib):
    P = make_params(8, [97], levels=2, q_bits=40)
    ev = Evaluator(P, golden_lib)
    ct = ev.encrypt(np.zeros((1, 1, 16), dtype=np.uint64))
    with pytest.raises(FheError):
        ev.rotate(ct, 0)
    with pytest.raises(FheError):
        ev.rotate(ct, 8)
    low = ev.mod_switch(ct)
    with pytest.raises(FheError):
        ev.mod_switch(low)
    with pytest.raises(FheError):
        ev.add(ct, low)


def test_empty_batches_golden(golden_lib):
    """Zero-length batch calls are no-ops that return empty lists (the same calls run
    against the CUDA library in test_gpu_parity.py::test_empty_batches)."""
    P = make_params(16, [65537], levels=3, q_bits=50)
    ev = Evaluator(P, golden_lib)
    ct = ev.encrypt(np.zeros((1, 1, 32), dtype=np.uint64))
    assert ev.rotate_many([], 3) == []
    assert ev.rotate_multi([], []) == []
    assert ev.rotate_hoisted(ct, []) == []
    assert ev.mul_plain_many([], []) == []
    assert ev.add_many([], []) == []


def _slots(P, R, rng, bound=None):
    return np.stack([rng.integers(0, bound or ti, size=(R, P.n), dtype=np.uint64) for ti in P.t]).astype(np.uint64)


def test_composite_operators_equal_their_sequences(golden_lib):
    """fhe_rotate_and_sum / fhe_combine / fhe_ct_gemm are the reference's rotate_and_sum
    (hesim.py:347-366), combine_to_dense (packing.py:350-368) and conv_conv channel sums
    (engine.py:178-197): their words equal the primitive sequences and their slots the
    reference semantics."""
    P = make_params(64, [65537], levels=3, q_bits=50)
    ev = Evaluator(P, golden_lib)
    N, t = P.n_slots, 65537
    rng = np.random.default_rng(4)
    # rotate_and_sum over a 37-slot payload (zero tail): slot 0 = sum of the payload
    s = np.zeros((1, 2, P.n), dtype=np.uint64)
    s[0, :, :37] = rng.integers(0, t, size=(2, 37))
    s[0, 1, N:N + 37] = rng.integers(0, t, size=37)
    a = ev.encrypt(s)
    out = ev.rotate_and_sum([a], 37)[0]
    acc = a
    for h in reversed(range(6)):
        acc = ev.add(acc, ev.rotate(acc, 1 << h))
    assert np.array_equal(ev.read(out), ev.read(acc))
    dec = ev.decrypt(out)
    assert int(dec[0, 0, 0]) == int(s[0, 0, :37].astype(object).sum() % t)
    assert int(dec[0, 1, N]) == int(s[0, 1, N:N + 37].astype(object).sum() % t)
    assert np.array_equal(ev.read(ev.rotate_and_sum([a], 1)[0]), ev.read(a))
    # combine: unequal lengths, odd count
    lengths = [5, 3, 7, 2, 4]
    payloads, cts = [], []
    for ln in lengths:
        v = np.zeros((1, 1, P.n), dtype=np.uint64)
        v[0, 0, :ln] = rng.integers(1, t, size=ln)
        v[0, 0, N:N + ln] = rng.integers(1, t, size=ln)
        payloads.append(v)
        cts.append(ev.encrypt(v))
    comb = ev.decrypt(ev.combine(cts, lengths))
    off = 0
    for v, ln in zip(payloads, lengths):
        assert np.array_equal(comb[0, 0, off:off + ln], v[0, 0, :ln])
        assert np.array_equal(comb[0, 0, N + off:N + off + ln], v[0, 0, N:N + ln])
        off += ln
    assert not comb[0, 0, off:N].any()
    assert np.array_equal(ev.read(ev.combine(cts[:1], lengths[:1])), ev.read(cts[0]))
    # ct_gemm: K = 3 inputs, O = 10 outputs (two output tiles), signed weights
    ins = [_slots(P, 2, rng) for _ in range(3)]
    cin = [ev.encrypt(x) for x in ins]
    w = rng.integers(-127, 128, size=(3, 10))
    outs = ev.ct_gemm(cin, w.tolist())
    for o, co in enumerate(outs):
        seq = ev.mul_scalar(cin[0], int(w[0, o]))
        for k in (1, 2):
            seq = ev.add(seq, ev.mul_scalar(cin[k], int(w[k, o])))
        assert np.array_equal(ev.read(co), ev.read(seq))
        want = sum(ins[k].astype(object) * int(w[k, o]) for k in range(3)) % t
        assert np.array_equal(ev.decrypt(co).astype(object), want)


def test_composite_operator_errors(golden_lib):
    P = make_params(8, [97], levels=2, q_bits=40)
    ev = Evaluator(P, golden_lib)
    a = ev.encrypt(np.zeros((1, 1, 16), dtype=np.uint64))
    with pytest.raises(FheError):
        ev.rotate_and_sum([a], 9)                  # span > N
    with pytest.raises(FheError):
        ev.combine([a, a], [5, 4])                 # 9 slots > N = 8
    with pytest.raises(FheError):
        ev.combine([a, a], [0, 4])                 # empty payload


def test_debug_rotate_stages_are_the_rotation(golden_lib):
    """The stages fhe_debug_rotate_stages exposes recombine into fhe_rotate's output:
    ModDown(acc) + tau_g(c0) (the GPU parity test compares the stages themselves)."""
    P = make_params(32, [65537], levels=3, q_bits=50)
    ev = Evaluator(P, golden_lib)
    rng = np.random.default_rng(8)
    ct = ev.encrypt(_slots(P, 1, rng))
    digits, ext, acc = ev.debug_rotate_stages(ct, 5)
    l, n = ct.level, P.n
    assert digits.shape == (1, l, n) and ext.shape == (1, l, l + 1, n) and acc.shape == (1, 2, l + 1, n)
    for j in range(l):
        assert not ext[0, j, j].any()                       # diagonal: read from the input
        assert int(digits[0, j].max()) < int(P.q[j])
    # c1 of the rotation is ModDown(acc[1]): (acc_i - [special row lifted]_i) / P mod q_i in the NTT domain,
    # so in the coefficient domain P * c1 + lift(special) == acc; check one prime at one evaluation-free point:
    # the sum of all NTT values of a row is n * coefficient 0
    out = ev.read(ev.rotate(ct, 5))[0]
    Pm = int(P.p[0])
    for i in range(l):
        q = int(P.q[i])
        r0 = int(acc[0, 1, l, 0])
        r0 = r0 - Pm if r0 > (Pm - 1) // 2 else r0
        lhs = (sum(int(v) for v in acc[0, 1, i]) - n * r0) % q
        rhs = (Pm * sum(int(v) for v in out[1, i])) % q
        assert lhs == rhs
