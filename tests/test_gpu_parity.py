"""GPU kernels vs the golden C model: ciphertext words bit-exact after every op.

Both libraries implement include/ffconv_he.h; each test feeds the SAME input
words to both and compares outputs word for word, plus decrypted slots against
plain modular arithmetic (the reference slot semantics, hesim.py:244-345).
"""

import dataclasses

import numpy as np
import pytest

from paper_2102_03494_b200.params import make_params
from paper_2102_03494_b200.rlwe import Evaluator

pytestmark = pytest.mark.gpu

CASES = [
    # (n_slots, t factors, levels, q_bits)
    (4, [97], 3, 40),
    (64, [65537], 4, 50),
    (1024, [786433, 65537], 4, 55),
    (8192, [65537], 5, 55),
    (8192, [1099511922689], 4, 40),
    # lazy-bound classes of the butterfly schedule (LIM = 2^clz(q)): q < 2^58 never reduces a
    # forward stage, 60-bit primes (LIM = 16) every other one, the 61-bit special prime
    # (LIM = 8) nearly all; 7 levels of 61-bit primes (LIM = 8 everywhere) take the
    # canonical-ModUp and the rescale-addend fallbacks ((l + 2) q >= 2^64)
    (1024, [65537], 3, 58),
    (8192, [65537], 3, 60),
    (64, [65537], 7, 61),
    # many levels: key-switch paths at l = 12 (templated inner product, runtime-l special rows)
    (64, [65537], 12, 40),
    # rings 2^15 / 2^16: one row per thread-block cluster of 2 / 4 CTAs (DSMEM NTT)
    (16384, [65537], 3, 50),
    (32768, [786433], 3, 50),
]
BIG = CASES[-2:]


def _pair(case, golden_lib, cuda_lib):
    n_slots, t, L, qb = case
    P = make_params(n_slots, t, levels=L, q_bits=qb)
    if qb == 61:                      # 61-bit q: the largest of the L + 1 primes is the special one
        ps = sorted(P.q + P.p, reverse=True)
        P = dataclasses.replace(P, q=tuple(ps[1:]), p=(ps[0],))
    return Evaluator(P, golden_lib), Evaluator(P, cuda_lib), P


def _rand_slots(P, R, rng):
    return np.stack([rng.integers(0, ti, size=(R, P.n), dtype=np.uint64) for ti in P.t]).astype(np.uint64)


@pytest.fixture(params=CASES, ids=lambda c: f"N{c[0]}-T{len(c[1])}-L{c[2]}")
def pair(request, golden_lib, cuda_lib):
    return _pair(request.param, golden_lib, cuda_lib)


def test_encode_and_encrypt_bit_exact(pair):
    gd, gp, P = pair
    rng = np.random.default_rng(1)
    s = _rand_slots(P, 2, rng)
    pg, pc = gd.encode(s[:, 0]), gp.encode(s[:, 0])
    assert np.array_equal(gd.pt_words(pg), gp.pt_words(pc))
    cg, cc = gd.encrypt(s, nonce=7), gp.encrypt(s, nonce=7)
    assert np.array_equal(gd.read(cg), gp.read(cc))
    assert np.array_equal(gp.decrypt(cc), s)
    assert np.array_equal(gd.decrypt(cg), s)


def test_ops_bit_exact(pair):
    gd, gp, P = pair
    rng = np.random.default_rng(2)
    R = 2
    a_s, b_s = _rand_slots(P, R, rng), _rand_slots(P, R, rng)
    ag, bg = gd.encrypt(a_s, nonce=1), gd.encrypt(b_s, nonce=2)
    ac, bc = gp.new_ct(R), gp.new_ct(R)
    gp.write(ac, gd.read(ag))
    gp.write(bc, gd.read(bg))
    pts = _rand_slots(P, 1, rng)[:, 0]
    ptg, ptc = gd.encode(pts), gp.encode(pts)
    t = np.array(P.t, dtype=object)[:, None, None]

    def same(xg, xc, expect=None):
        assert np.array_equal(gd.read(xg), gp.read(xc))
        if expect is not None:
            assert np.array_equal(gp.decrypt(xc).astype(object), expect)

    A, B = a_s.astype(object), b_s.astype(object)
    same(gd.add(ag, bg), gp.add(ac, bc), (A + B) % t)
    same(gd.mul_plain(ag, ptg), gp.mul_plain(ac, ptc), (A * pts.astype(object)[:, None, :]) % t)
    same(gd.mul_scalar(ag, -5), gp.mul_scalar(ac, -5), (A * -5) % t)
    # fused HMA: acc += a * pt in place == add(acc, mul_plain(a, pt))
    accg, accc = gd.encrypt(b_s, nonce=2), gp.new_ct(R)
    gp.write(accc, gd.read(accg))
    gd.mul_plain_acc(ag, ptg, accg)
    gp.mul_plain_acc(ac, ptc, accc)
    same(accg, accc, (B + A * pts.astype(object)[:, None, :]) % t)
    assert np.array_equal(gp.read(accc), gp.read(gp.add(bc, gp.mul_plain(ac, ptc))))
    same(gd.add_plain(ag, ptg), gp.add_plain(ac, ptc), (A + pts.astype(object)[:, None, :]) % t)
    N = P.n_slots
    for k in sorted({1, N // 2 + 1, N - 1} & set(range(1, N))):
        rolled = np.concatenate([np.roll(A[..., :N], -k, axis=-1), np.roll(A[..., N:], -k, axis=-1)], axis=-1)
        same(gd.rotate(ag, k), gp.rotate(ac, k), rolled)
    same(gd.mod_switch(ag), gp.mod_switch(ac), A)
    same(gd.square(ag), gp.square(ac), (A * A) % t)


def test_rotate_many_matches_single(golden_lib, cuda_lib):
    gd, gp, P = _pair(CASES[2], golden_lib, cuda_lib)
    rng = np.random.default_rng(3)
    cts = [gp.encrypt(_rand_slots(P, 1 + i % 2, rng)) for i in range(5)]
    many = gp.rotate_many(cts, 3)
    for c, m in zip(cts, many):
        assert np.array_equal(gp.read(gp.rotate(c, 3)), gp.read(m))


def test_chain_noise_and_decrypt(golden_lib, cuda_lib):
    """A multiplicative chain on the GPU decrypts exactly and agrees word for word."""
    gd, gp, P = _pair(CASES[3], golden_lib, cuda_lib)
    rng = np.random.default_rng(4)
    s = _rand_slots(P, 1, rng)
    cg = gd.encrypt(s, nonce=3)
    cc = gp.new_ct(1)
    gp.write(cc, gd.read(cg))
    pt = _rand_slots(P, 1, rng)[:, 0]
    pg, pc = gd.encode(pt), gp.encode(pt)
    for step in range(2):
        cg, cc = gd.mul_plain(cg, pg), gp.mul_plain(cc, pc)
        cg, cc = gd.rotate(cg, 5 + step), gp.rotate(cc, 5 + step)
        cg, cc = gd.square(cg), gp.square(cc)
    assert np.array_equal(gd.read(cg), gp.read(cc))
    assert np.array_equal(gd.decrypt(cg), gp.decrypt(cc))


def test_rotate_multi_matches_single(golden_lib, cuda_lib):
    gd, gp, P = _pair(CASES[3], golden_lib, cuda_lib)
    rng = np.random.default_rng(6)
    cts = [gp.encrypt(_rand_slots(P, 1 + i % 3, rng)) for i in range(6)]
    ks = [1, 4095, 3, 3, 8191, 77]
    multi = gp.rotate_multi(cts, ks)
    for c, k, m in zip(cts, ks, multi):
        assert np.array_equal(gp.read(gp.rotate(c, k)), gp.read(m))
    # and the golden model agrees word for word
    cg = gd.new_ct(cts[1].rows)
    gd.write(cg, gp.read(cts[1]))
    assert np.array_equal(gd.read(gd.rotate(cg, 4095)), gp.read(multi[1]))


@pytest.mark.parametrize("case", BIG, ids=lambda c: f"N{c[0]}")
def test_cluster_rings_fused_paths_bit_exact(case, golden_lib, cuda_lib):
    """Cluster-row paths that gather across CTAs: fused rotate-and-add (automorphism
    of the addend in the ModDown epilogue) and per-ciphertext keys."""
    gd, gp, P = _pair(case, golden_lib, cuda_lib)
    rng = np.random.default_rng(8)
    N = P.n_slots
    s = _rand_slots(P, 2, rng)
    cg = gd.encrypt(s, nonce=5)
    cc = gp.new_ct(2)
    gp.write(cc, gd.read(cg))
    k = N // 4 + 3
    (og,), (oc,) = gd.rotate_add_many([cg], k), gp.rotate_add_many([cc], k)
    assert np.array_equal(gd.read(og), gp.read(oc))
    A = s.astype(object)
    rolled = np.concatenate([np.roll(A[..., :N], -k, axis=-1), np.roll(A[..., N:], -k, axis=-1)], axis=-1)
    t = np.array(P.t, dtype=object)[:, None, None]
    assert np.array_equal(gp.decrypt(oc).astype(object), (A + rolled) % t)
    ks = [1, N - 1]
    mg, mc = gd.rotate_multi([cg, cg], ks), gp.rotate_multi([cc, cc], ks)
    for x, y in zip(mg, mc):
        assert np.array_equal(gd.read(x), gp.read(y))


@pytest.mark.parametrize("case", [CASES[2], BIG[1]], ids=lambda c: f"N{c[0]}")
def test_key_cache_eviction_bit_exact(case, golden_lib, cuda_lib, monkeypatch):
    """Rotation keys are regenerated on demand: with a key budget of a few keys,
    many distinct steps (per-ciphertext keys, several sub-batches) still give the
    golden model's words."""
    n_slots, t, L, qb = case
    P = make_params(n_slots, t, levels=L, q_bits=qb)
    key_mb = L * 2 * (L + 1) * 2 * n_slots * 8 / 2 ** 20
    monkeypatch.setenv("FHE_KEY_BUDGET_MB", str(max(1, int(3 * key_mb))))
    monkeypatch.setenv("FHE_KS_BATCH", "4")
    gd, gp = Evaluator(P, golden_lib), Evaluator(P, cuda_lib)
    rng = np.random.default_rng(9)
    s = _rand_slots(P, 1, rng)
    cg = gd.encrypt(s, nonce=11)
    cc = gp.new_ct(1)
    gp.write(cc, gd.read(cg))
    N = P.n_slots
    ks = [int(k) for k in rng.choice(np.arange(1, N), size=14, replace=False)]
    multi = gp.rotate_multi([cc] * len(ks), ks)
    for k, m in zip(ks, multi):
        assert np.array_equal(gd.read(gd.rotate(cg, k)), gp.read(m)), k
    # evicted keys come back bit-identical
    again = gp.rotate_multi([cc] * 3, ks[:3])
    for a, m in zip(again, multi[:3]):
        assert np.array_equal(gp.read(a), gp.read(m))


def test_lane_reuses_fresh_key_bit_exact(golden_lib, cuda_lib, monkeypatch):
    """A key generated for the first sub-batch (stream 0) and reused from the cache
    by the next sub-batch on the second stream: the second stream must wait for the
    generation (ring 2^16, L = 8, sub-batches of 3 physical ciphertexts)."""
    monkeypatch.setenv("FHE_KS_BATCH", "3")
    P = make_params(32768, [786433, 1179649], levels=8, q_bits=60, p_bits=61)
    gd, gp = Evaluator(P, golden_lib), Evaluator(P, cuda_lib)
    rng = np.random.default_rng(12)
    s = _rand_slots(P, 6, rng)
    cg = gd.encrypt(s, nonce=3)
    cc = gp.new_ct(6)
    gp.write(cc, gd.read(cg))
    for k in (1, 12345):
        assert np.array_equal(gd.read(gd.rotate(cg, k)), gp.read(gp.rotate(cc, k))), k


def test_pinned_async_encrypt_decrypt_match_sync(golden_lib, cuda_lib):
    """Page-locked host buffers take the asynchronous copy-stream path (several calls
    in flight); results equal the synchronous pageable path word for word."""
    import torch
    gd, gp, P = _pair(CASES[3], golden_lib, cuda_lib)
    rng = np.random.default_rng(13)
    R = 6
    s = _rand_slots(P, R, rng)
    pin_in = torch.from_numpy(s.view(np.int64)).pin_memory().numpy().view(np.uint64)
    pin_out = torch.empty(s.shape, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    cts = [gp.encrypt(pin_in[:, r:r + 2], nonce=100 + r, async_=True) for r in range(0, R, 2)]
    rs = gp.rotate_many(cts, 9)
    for r, c in zip(range(0, R, 2), rs):
        gp.decrypt(c, out=pin_out[:, r:r + 2], async_=True)
    gp.sync()
    for r, c in zip(range(0, R, 2), cts):
        ref = gp.encrypt(np.ascontiguousarray(s[:, r:r + 2]), nonce=100 + r)
        assert np.array_equal(gp.read(ref), gp.read(c))
    N = P.n_slots
    A = s
    exp = np.concatenate([np.roll(A[..., :N], -9, axis=-1), np.roll(A[..., N:], -9, axis=-1)], axis=-1)
    assert np.array_equal(pin_out, exp)


@pytest.mark.parametrize("case", [CASES[2], CASES[4], BIG[1]], ids=lambda c: f"N{c[0]}")
def test_rotate_hoisted_bit_exact(case, golden_lib, cuda_lib, monkeypatch):
    """Rotations of one ciphertext sharing one ModUp equal separate golden rotations
    word for word (several source sub-batches and item chunks at FHE_KS_BATCH=3)."""
    monkeypatch.setenv("FHE_KS_BATCH", "3")
    gd, gp, P = _pair(case, golden_lib, cuda_lib)
    rng = np.random.default_rng(14)
    R = 2
    s = _rand_slots(P, R, rng)
    cg = gd.encrypt(s, nonce=21)
    cc = gp.new_ct(R)
    gp.write(cc, gd.read(cg))
    N = P.n_slots
    ks = sorted({1, 2, N // 2 - 1, N - 1, int(rng.integers(1, N))})
    outs = gp.rotate_hoisted(cc, ks)
    for k, o in zip(ks, outs):
        assert np.array_equal(gd.read(gd.rotate(cg, k)), gp.read(o)), k


def test_empty_batches(golden_lib, cuda_lib):
    """Zero-length batch calls launch nothing and return empty lists (both libraries)."""
    gd, gp, P = _pair(CASES[1], golden_lib, cuda_lib)
    for ev in (gd, gp):
        ct = ev.encrypt(_rand_slots(P, 1, np.random.default_rng(9)))
        assert ev.rotate_many([], 3) == []
        assert ev.rotate_multi([], []) == []
        assert ev.rotate_hoisted(ct, []) == []
        assert ev.mul_plain_many([], []) == []
        assert ev.add_many([], []) == []


COMPOSITE_CASES = [CASES[1], CASES[2], CASES[4], CASES[6], CASES[7], CASES[-2]]


@pytest.mark.parametrize("case", COMPOSITE_CASES, ids=lambda c: f"N{c[0]}-T{len(c[1])}-L{c[2]}-q{c[3]}")
def test_composite_operators_bit_exact(case, golden_lib, cuda_lib):
    """fhe_rotate_and_sum, fhe_combine and fhe_ct_gemm: GPU words equal the
    golden model's, which equal the reference sequences (tests/test_golden_model.py)."""
    gd, gp, P = _pair(case, golden_lib, cuda_lib)
    rng = np.random.default_rng(11)
    N = P.n_slots

    def mirror(slots, nonce):
        g = gd.encrypt(slots, nonce=nonce)
        c = gp.new_ct(slots.shape[1])
        gp.write(c, gd.read(g))
        return g, c

    # rotate_and_sum over several objects with different row counts, span not a power of two
    span = max(2, min(N, 37))
    objs = [mirror(_rand_slots(P, 1 + i % 2, rng), 20 + i) for i in range(3)]
    for og, oc in zip(gd.rotate_and_sum([g for g, _ in objs], span), gp.rotate_and_sum([c for _, c in objs], span)):
        assert np.array_equal(gd.read(og), gp.read(oc))
    og, oc = gd.rotate_and_sum([objs[0][0]], 1)[0], gp.rotate_and_sum([objs[0][1]], 1)[0]
    assert np.array_equal(gd.read(og), gp.read(oc))
    # combine: unequal lengths, odd count (a block that moves up a level unchanged)
    lengths = [max(1, N // 16), max(1, N // 32), max(1, N // 8), 1, max(1, N // 16)]
    if sum(lengths) > N:
        lengths = [1, 1, 1]
    blocks = [mirror(_rand_slots(P, 2, rng), 40 + i) for i in range(len(lengths))]
    assert np.array_equal(gd.read(gd.combine([g for g, _ in blocks], lengths)),
                          gp.read(gp.combine([c for _, c in blocks], lengths)))
    assert np.array_equal(gd.read(gd.combine([blocks[0][0]], lengths[:1])), gp.read(gp.combine([blocks[0][1]], lengths[:1])))
    # ct_gemm: K = 11 inputs (more than one lazy-accumulation chunk at 61 bits), O = 10 (two tiles)
    K, O = 11, 10
    ins = [mirror(_rand_slots(P, 2, rng), 60 + k) for k in range(K)]
    w = rng.integers(-127, 128, size=(K, O))
    w[0, 0] = -(1 << 62)                              # full-range int64 weights reduce per prime
    for og, oc in zip(gd.ct_gemm([g for g, _ in ins], w.tolist()), gp.ct_gemm([c for _, c in ins], w.tolist())):
        assert np.array_equal(gd.read(og), gp.read(oc))


def test_ct_gemm_wide_k_on_gpu(golden_lib, cuda_lib):
    """More inputs than one launch's pointer table (GEMM_MAXK = 64): chained accumulating launches."""
    gd, gp, P = _pair(CASES[1], golden_lib, cuda_lib)
    rng = np.random.default_rng(12)
    K, O = 70, 3
    base = [_rand_slots(P, 1, rng) for _ in range(K)]
    gi = [gd.encrypt(s, nonce=100 + k) for k, s in enumerate(base)]
    ci = []
    for g in gi:
        c = gp.new_ct(1)
        gp.write(c, gd.read(g))
        ci.append(c)
    w = rng.integers(-(1 << 40), 1 << 40, size=(K, O))
    for og, oc in zip(gd.ct_gemm(gi, w.tolist()), gp.ct_gemm(ci, w.tolist())):
        assert np.array_equal(gd.read(og), gp.read(oc))


@pytest.mark.parametrize("case", [CASES[1], CASES[4], CASES[6], CASES[7], CASES[8], CASES[-2]],
                         ids=lambda c: f"N{c[0]}-T{len(c[1])}-L{c[2]}-q{c[3]}")
def test_key_switch_stages_bit_exact(case, golden_lib, cuda_lib):
    """Parity after every KERNEL of a rotation, not only after the primitive: the digits
    (k_rot_gather_intt), the extended digits (k_modup), the key inner products
    (k_ks_inner) and the special row in coefficient form (k_ks_special) equal the golden
    model's intermediates word for word."""
    gd, gp, P = _pair(case, golden_lib, cuda_lib)
    rng = np.random.default_rng(21)
    s = _rand_slots(P, 2, rng)
    cg = gd.encrypt(s, nonce=9)
    cc = gp.new_ct(2)
    gp.write(cc, gd.read(cg))
    k = max(1, P.n_slots // 2 - 1)
    for name, g, c in zip(("digits", "ext", "acc"), gd.debug_rotate_stages(cg, k), gp.debug_rotate_stages(cc, k)):
        assert np.array_equal(g, c), name
    # and a lower level (fewer digits than the keys were generated for)
    if P.L > 2:
        lg, lc = gd.mod_switch(cg), gp.mod_switch(cc)
        for name, g, c in zip(("digits", "ext", "acc"), gd.debug_rotate_stages(lg, 1), gp.debug_rotate_stages(lc, 1)):
            assert np.array_equal(g, c), name


def test_cfg1_full_batch_properties(golden_lib, cuda_lib):
    """configs[1] at its full size: ring 2^14, 4 x 40-bit q + a 42-bit special prime, 1024 physical
    ciphertexts in one call (8 key-switch sub-batches of 128 on two lanes).  The golden model is too
    slow for all of them, so the whole batch is checked through size-independent properties of the
    reference rotation (hesim.py:244-261: a cyclic shift of each slot row) and a sample of
    ciphertexts from every sub-batch word for word against the golden model."""
    P = make_params(8192, [1099511922689], levels=4, q_bits=40, p_bits=42)
    gd, gp = Evaluator(P, golden_lib), Evaluator(P, cuda_lib)
    B, N, t, k = 1024, P.n_slots, P.t[0], 5203
    rng = np.random.default_rng(21)
    A = rng.integers(0, t, size=(1, B, P.n), dtype=np.uint64)
    Bm = rng.integers(0, t, size=(1, B, P.n), dtype=np.uint64)

    def roll(X, s):
        return np.concatenate([np.roll(X[..., :N], -s, axis=-1), np.roll(X[..., N:], -s, axis=-1)], axis=-1)

    ca, cb = gp.encrypt(A), gp.encrypt(Bm)
    ra, rb = gp.rotate(ca, k), gp.rotate(cb, k)
    # the reference's slot semantics on every ciphertext of the batch
    assert np.array_equal(gp.decrypt(ra), roll(A, k))
    # round trip: rotating on by N - k restores every slot vector
    assert np.array_equal(gp.decrypt(gp.rotate(ra, N - k)), A)
    # linearity: rot(a) + rot(b) and rot(a + b) hold the same slots
    want = roll((A + Bm) % np.uint64(t), k)
    assert np.array_equal(gp.decrypt(gp.add(ra, rb)), want)
    assert np.array_equal(gp.decrypt(gp.rotate(gp.add(ca, cb), k)), want)
    # one call over many objects equals the single-object call (sub-batching is invisible)
    parts = [gp.encrypt(A[:, r0:r0 + 256], nonce=1000 + r0) for r0 in range(0, B, 256)]
    many = gp.rotate_many(parts, k)
    for r0, m in zip(range(0, B, 256), many):
        assert np.array_equal(gp.decrypt(m), roll(A[:, r0:r0 + 256], k))
    # word-for-word against the golden model: first / last ciphertext of sub-batches on both lanes
    rows = [0, 127, 128, 383, 640, 1023]
    win, wout = gp.read(ca), gp.read(ra)
    cg = gd.new_ct(len(rows))
    gd.write(cg, win[rows])
    assert np.array_equal(gd.read(gd.rotate(cg, k)), wout[rows])
