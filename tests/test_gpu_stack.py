"""The reference-facing API on the sm_100a CUDA library (B200 only).

* every reference primitive sequence (hesim_sequences.json) decrypts, counts and
  tracks depth as the reference did;
* random FFConv-shaped networks (networks.json): logits, per-step op counts,
  depths and per-layer tensors equal the reference's, and the output
  ciphertexts equal the golden model's word for word;
* BASELINE configs[0] end to end: logits equal run_reference (fixture) for two
  synthetic images in one ciphertext row pair, under 5-prime plaintext CRT.
"""

import os

import numpy as np
import pytest

from paper_2102_03494_b200.hesim import HeContext
from paper_2102_03494_b200.planner import build_plan
from paper_2102_03494_b200.runner import inference_params, run_encrypted, scheme_for

from _shared import cfg0_network, load, network_from_fixture, reference_step_totals, replay, scheme_from, step_totals

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_sequences_on_gpu(cuda_lib):
    for case in load("hesim_sequences.json"):
        ctx = HeContext(scheme_from(case["n_slots"], case["t_factors"], levels=8), lib=cuda_lib, debug_checks=True)
        ct = replay(ctx, case)
        assert [int(v) for v in ctx.decrypt(ct)] == case["expect"]
        c = ctx.counters
        assert [c.mul_pc, c.add_cc, c.rot, c.mul_cc, c.assembly_mul_pc] == case["counters"]
        assert (ct.depth, ct.assembly_depth) == (case["depth"], case["assembly_depth"])


def test_networks_on_gpu_match_reference_and_golden(cuda_lib, golden_lib):
    for k, fx in enumerate(load("networks.json")):
        net, ws = network_from_fixture(fx)
        plan = build_plan(net, "explicit")
        x = np.array(fx["inputs"])
        gpu = HeContext(net.scheme, batch=2, lib=cuda_lib)
        res = run_encrypted(net, plan, ws, x, ctx=gpu, capture_layers=True)
        assert [[int(v) for v in row] for row in res.logits] == fx["logits"]
        assert step_totals(res.steps) == reference_step_totals(fx["rows"])
        assert (res.depth, res.assembly_depth) == (fx["depth"], fx["assembly_depth"])
        for (idx, got), r0, r1 in zip(res.layer_outputs, fx["layer_outputs"][0], fx["layer_outputs"][1]):
            assert np.asarray(got[0]).astype(str).tolist() == r0
            assert np.asarray(got[1]).astype(str).tolist() == r1
        if k < 4:
            gold = HeContext(net.scheme, batch=2, lib=golden_lib)
            res_g = run_encrypted(net, plan, ws, x, ctx=gold)
            for a, b in zip(res.value.cts, res_g.value.cts):
                assert np.array_equal(gpu.evaluator.read(a.handle), gold.evaluator.read(b.handle))


def test_cfg0_end_to_end_on_gpu(cuda_lib):
    from paper_2102_03494_b200.hesim import SchemeParams
    net0, ws, xs, meta = cfg0_network(SchemeParams(n_slots=8192, t=(1 << 61) - 1))
    plan0 = build_plan(net0, "explicit")
    rp = inference_params(net0, plan0, ws, input_bound=255)
    assert len(rp.t) == 5 and rp.L == 6 and rp.log_qp <= 438
    net, _, _, _ = cfg0_network(scheme_for(rp))
    plan = build_plan(net, "explicit")
    ctx = HeContext(net.scheme, batch=2, lib=cuda_lib)
    res = run_encrypted(net, plan, ws, xs, ctx=ctx)
    for row, want in zip(res.logits, meta["logits"]):
        assert [str(int(v)) for v in row] == want
    c = res.counters
    assert (c.mul_pc, c.add_cc, c.rot, c.mul_cc, c.assembly_mul_pc) == (458, 4894, 4889, 2, 438)
    assert min(ctx.noise_budget(ct) for ct in res.value.cts) > 5


def test_hoisted_schedule_on_gpu(cuda_lib, golden_lib):
    """schedule='hoisted': same logits as the reference, ciphertexts equal the
    golden model's word for word (k_hoisted_dot vs the golden loop)."""
    for fx in load("networks.json")[:4]:
        net, ws = network_from_fixture(fx)
        plan = build_plan(net, "explicit")
        x = np.array(fx["inputs"])
        gpu = HeContext(net.scheme, batch=2, lib=cuda_lib, schedule="hoisted", hoist_levels=3)
        gold = HeContext(net.scheme, batch=2, lib=golden_lib, schedule="hoisted", hoist_levels=3)
        a = run_encrypted(net, plan, ws, x, ctx=gpu)
        b = run_encrypted(net, plan, ws, x, ctx=gold)
        assert [[int(v) for v in row] for row in a.logits] == fx["logits"]
        for u, v in zip(a.value.cts, b.value.cts):
            assert np.array_equal(gpu.evaluator.read(u.handle), gold.evaluator.read(v.handle))


def test_cfg0_hoisted_on_gpu(cuda_lib):
    from paper_2102_03494_b200.hesim import SchemeParams
    net0, ws, xs, meta = cfg0_network(SchemeParams(n_slots=8192, t=(1 << 61) - 1))
    rp = inference_params(net0, build_plan(net0, "explicit"), ws, input_bound=255)
    net, _, _, _ = cfg0_network(scheme_for(rp))
    plan = build_plan(net, "explicit")
    ctx = HeContext(net.scheme, batch=2, lib=cuda_lib, schedule="hoisted")
    res = run_encrypted(net, plan, ws, xs, ctx=ctx)
    for row, want in zip(res.logits, meta["logits"]):
        assert [str(int(v)) for v in row] == want
    assert res.counters.rot < 4889 // 2
    assert min(ctx.noise_budget(ct) for ct in res.value.cts) > 5


def test_h_im2col_moves_hoisted_on_gpu(cuda_lib, golden_lib):
    """H-Im2Col moves (packing.py:249-279) with every rotation of one masked source
    sharing one ModUp: plaintext im2col, the reference's counts, golden words."""
    from paper_2102_03494_b200.packing import (ChannelPacked, KernelSpec, conv_unpack, dense_pack,
                                               h_im2col_from_conv, h_im2col_from_dense, plain_im2col)
    rng = np.random.default_rng(31)
    x = rng.integers(-5, 6, size=(2, 3, 5, 5))
    k = KernelSpec(d=2, stride=1, out_channels=1)
    words = []
    sch = scheme_from(128, [65537], levels=4)          # one key seed for both libraries
    for lib in (cuda_lib, golden_lib):
        ctx = HeContext(sch, batch=2, lib=lib)
        cols = h_im2col_from_dense(dense_pack(x, ctx), k, ctx)
        assert np.array_equal(conv_unpack(cols, ctx).astype(np.int64), plain_im2col(x, k))
        assert ctx.counters.rot == ctx.counters.add_cc == 16 * 12
        words.append([ctx.evaluator.read(c.handle) for c in cols.cts])
    for a, b in zip(*words):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("idx", range(6))
def test_extra_networks_on_gpu(cuda_lib, golden_lib, idx):
    """avg-pool (engine.py:271-279), DP-DP and in-network HIm2Col plans on the B200:
    the reference's logits, counts, depths and per-layer tensors, and the golden
    model's ciphertext words."""
    from test_host_stack import _check_network
    fx = load("networks_extra.json")[idx]
    sch = scheme_from(fx["n_slots"], fx["t_factors"], levels=8)
    res = _check_network(fx, HeContext(sch, batch=2, lib=cuda_lib))
    gold = _check_network(fx, HeContext(sch, batch=2, lib=golden_lib))
    ev = res.value.cts[0]._ctx.evaluator
    evg = gold.value.cts[0]._ctx.evaluator
    for a, b in zip(res.value.cts, gold.value.cts):
        assert np.array_equal(ev.read(a.handle), evg.read(b.handle))


def test_cfg3_end_to_end_on_gpu(cuda_lib):
    """BASELINE configs[3] (CIFAR-shaped, ring 2^16 on thread-block clusters, avg-pool,
    ffconv-default plan) on one row pair: both images' logits equal the reference's
    run_reference (tests/golden/cfg3.json), op counts and depths equal its report."""
    import sys
    sys.path.insert(0, ROOT)
    from bench import cfg3_setup
    net, plan, ws, xs, rp, ref = cfg3_setup(2, seed=20210205)
    ctx = HeContext(net.scheme, batch=2, lib=cuda_lib)
    res = run_encrypted(net, plan, ws, xs, ctx=ctx)
    assert [[int(v) for v in row] for row in res.logits] == ref
    meta = load("cfg3.json")
    assert step_totals(res.steps) == reference_step_totals(meta["count_rows"])
    assert (res.depth, res.assembly_depth) == (meta["depth"], meta["assembly_depth"])
    assert len(ctx.rotation_steps) < 200            # tree combine: ~log2 keys per combine (7,259 as a chain)


@pytest.mark.parametrize("variant", range(8))
def test_cfg4_variants_logits_on_gpu(cuda_lib, variant):
    """BASELINE configs[4]: every rank/packing variant on one row pair decrypts to the
    oracle's direct-loop logits, with the reference's rotation counts."""
    import sys
    sys.path.insert(0, ROOT)
    from bench import ABLATION, REF_ROTATIONS, _oracle_logits, ablation_setup
    name, first = ABLATION[variant]
    net, plan, ws, xs, rp = ablation_setup(first, 2, seed=20210205)
    ctx = HeContext(net.scheme, batch=2, lib=cuda_lib)
    res = run_encrypted(net, plan, ws, xs, ctx=ctx)
    assert [[int(v) for v in row] for row in res.logits] == _oracle_logits(net, ws, xs)
    assert res.counters.rot == REF_ROTATIONS[name]


@pytest.mark.parametrize("schedule", ["reference", "hoisted"])
def test_cfg0_level_schedule_on_gpu(cuda_lib, schedule):
    """Level schedule (HeContext(level_schedule=True)): q primes are dropped between and
    inside plan steps once the noise model allows; the logits stay the reference's, the
    op counts are unchanged and the budget is not exhausted."""
    from paper_2102_03494_b200.hesim import SchemeParams
    net0, ws, xs, meta = cfg0_network(SchemeParams(n_slots=8192, t=(1 << 61) - 1))
    rp = inference_params(net0, build_plan(net0, "explicit"), ws, input_bound=255)
    net, _, _, _ = cfg0_network(scheme_for(rp))
    plan = build_plan(net, "explicit")
    ctx = HeContext(net.scheme, batch=2, lib=cuda_lib, schedule=schedule, level_schedule=True)
    res = run_encrypted(net, plan, ws, xs, ctx=ctx)
    for row, want in zip(res.logits, meta["logits"]):
        assert [str(int(v)) for v in row] == want
    assert max(ct.handle.level for ct in res.value.cts) < rp.L
    assert ctx.last_noise_budget > 3
    if schedule == "reference":
        c = res.counters
        assert (c.mul_pc, c.add_cc, c.rot, c.mul_cc, c.assembly_mul_pc) == (458, 4894, 4889, 2, 438)


def test_captured_plan_replay_on_gpu(cuda_lib):
    """Plan capture + CUDA-graph replay (runner.CapturedPlan): the walk is recorded once on
    an all-zero example batch and replayed for new images; every replay decrypts to the
    reference's logits, and the replay issues no per-op launches from Python."""
    import ctypes
    from paper_2102_03494_b200.runner import CapturedPlan
    for fx in load("networks.json")[:4]:
        net, ws = network_from_fixture(fx)
        plan = build_plan(net, "explicit")
        x = np.array(fx["inputs"])
        ctx = HeContext(net.scheme, batch=2, lib=cuda_lib)
        cp = CapturedPlan(net, plan, ws, np.zeros_like(x), ctx)
        assert cp.nodes > 10
        ev = ctx.evaluator
        n0 = ctypes.c_uint64()
        cuda_lib.call("fhe_launch_count", ev.ctx, ctypes.byref(n0))
        got = cp.run(x)
        n1 = ctypes.c_uint64()
        cuda_lib.call("fhe_launch_count", ev.ctx, ctypes.byref(n1))
        assert [[int(v) for v in row] for row in got] == fx["logits"]
        assert [[int(v) for v in row] for row in cp.run(x[::-1].copy())] == fx["logits"][::-1]
        # encrypt + copy of every input ciphertext, one graph launch, decrypt of every logit
        # ciphertext: a few launches per boundary ciphertext, none per plan op
        from paper_2102_03494_b200.runner import _packed_cts
        boundary = len(list(_packed_cts(cp.packed))) + len(list(_packed_cts(cp.result.value)))
        assert n1.value - n0.value <= 8 * boundary + 8
