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
