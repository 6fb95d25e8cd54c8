"""Generate golden fixtures by running the REFERENCE implementation itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fixtures.py

Reads the reference read-only (cipherpack, pure Python) in this container and
writes small fixtures next to this file; /root/reference does not exist on the
GPU box, so tests only ever read the committed fixtures:

  hesim_sequences.json  random primitive sequences through the reference
                        HeContext (hesim.py:186-366) at batching-compatible t,
                        with decrypted results, counters and depths
  networks.json         random 1-2 conv networks + square + fc (the reference's
                        test-strategy shape, tests/conftest.py:68-125) with
                        weights, inputs, plan steps, measured report rows,
                        depths, run_reference layer outputs and logits
  networks_extra.json   the same record for hand-picked networks covering
                        avg-pool, DP-DP and in-network HIm2Col steps
  cfg0.npz / cfg0.json  BASELINE configs[0]: the FFConv MNIST network on
                        seeded synthetic images: weights, inputs, reference
                        logits, count-only report, and the reference's own
                        encrypted logits with and without the FC->FC slot-0
                        mask fix
  cfg3.npz / cfg3.json  BASELINE configs[3] as SURVEY.md 8(d) pins it (valid
                        convs, 2^15 slots, ffconv-default): weights, two seeded
                        N(0.5, 0.25) CIFAR-shaped inputs, the reference's
                        run_reference logits and its count-only report
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from cipherpack import engine as ref_engine  # noqa: E402
from cipherpack import runner as ref_runner  # noqa: E402
from cipherpack.hesim import HeContext, SchemeParams  # noqa: E402
from cipherpack.netspec import LayerSpec, NetworkSpec  # noqa: E402
from cipherpack.packing import TensorShape  # noqa: E402
from cipherpack.planner import build_plan  # noqa: E402
from cipherpack.factorize import quantize_matrix  # noqa: E402
from cipherpack.weights import WeightSet, WeightTensor, random_weights, required_tensors  # noqa: E402

from paper_2102_03494_b200.params import ntt_primes  # noqa: E402


def crt_t(n_slots: int, bound: int, bits: int = 20):
    cands = ntt_primes(bits, 32, 4 * n_slots)
    ts, total = [], 1
    for p in cands:
        ts.append(p)
        total *= p
        if total > 2 * bound + 2:
            return ts
    raise ValueError("bound too large")


# ------------------------------------------------------------ primitives
def hesim_sequences(trials=300, seed=11):
    rng = np.random.default_rng(seed)
    choices = [(4, [97]), (8, [97]), (8, [97, 65537]), (16, [65537]), (32, [786433]), (64, [65537, 786433])]
    out = []
    for trial in range(trials):
        n, fs = choices[int(rng.integers(0, len(choices)))]
        t = math.prod(fs)
        ctx = HeContext(SchemeParams(n_slots=n, t=t))
        bound = (t - 1) // 2
        x = [int(v) for v in rng.integers(-min(bound, 2 ** 62), min(bound, 2 ** 62) + 1, size=n)]
        ct = ctx.encrypt(x)
        ops = []
        for _ in range(int(rng.integers(1, 6))):
            op = int(rng.integers(0, 6))
            if op == 0:
                k = int(rng.integers(0, n))
                ct = ctx.rotate(ct, k)
                ops.append(["rotate", k])
            elif op == 1:
                pv = [int(v) for v in rng.integers(-min(bound, 1000), min(bound, 1000) + 1, size=n)]
                assembly = bool(rng.random() < 0.2)
                ct = ctx.mul_plain(ct, ctx.encode(pv), assembly=assembly)
                ops.append(["mul_plain", pv, assembly])
            elif op == 2:
                y = [int(v) for v in rng.integers(-min(bound, 2 ** 62), min(bound, 2 ** 62) + 1, size=n)]
                ct = ctx.add_cc(ct, ctx.encrypt(y))
                ops.append(["add_cc", y])
            elif op == 3:
                ct = ctx.square(ct)
                ops.append(["square"])
            elif op == 4:
                pv = [int(v) for v in rng.integers(-min(bound, 1000), min(bound, 1000) + 1, size=n)]
                ct = ctx.add_plain(ct, ctx.encode(pv))
                ops.append(["add_plain", pv])
            else:
                m = int(rng.integers(1, n + 1))
                masked = [1] * m + [0] * (n - m)
                ct = ctx.mul_plain(ct, ctx.encode(masked))
                ct = ctx.rotate_and_sum(ct, m)
                ops.append(["mask_rotate_and_sum", m])
        c = ctx.counters
        out.append({"n_slots": n, "t_factors": fs, "x": x, "ops": ops,
                    "expect": [int(v) for v in ctx.decrypt(ct)],
                    "counters": [c.mul_pc, c.add_cc, c.rot, c.mul_cc, c.assembly_mul_pc],
                    "depth": ct.depth, "assembly_depth": ct.assembly_depth,
                    "elided": ctx.elided_rotations})
    return out


# ------------------------------------------------------------- networks
PATTERNS = ("dp-hi2c-cp", "cp-hi2c-cp", "dp-dp", "cp-hi2c-dp")


def _random_layers(rng, shape):
    def conv(cur):
        d = int(rng.integers(1, min(3, cur.w, cur.h) + 1))
        stride = int(rng.integers(1, 3))
        if (cur.w - d) // stride + 1 < 1 or (cur.h - d) // stride + 1 < 1:
            stride = 1
        oc = int(rng.integers(1, 4))
        if rng.random() < 0.5:
            rank = int(rng.integers(1, min(d * d * cur.c, oc) + 1))
            pat = str(rng.choice(PATTERNS))
            if pat.startswith("cp") and d == 1 and stride > 1:
                stride = 1
            return LayerSpec(kind="ffconv", d=d, stride=stride, out_channels=oc, rank=rank, packing_hint=pat)
        hint = str(rng.choice(["dense", "conv"]))
        if hint == "conv" and d == 1 and stride > 1:
            stride = 1
        return LayerSpec(kind="conv", d=d, stride=stride, out_channels=oc, packing_hint=hint)

    layers = [conv(shape)]
    cur = NetworkSpec._apply(layers[0], shape)
    if rng.random() < 0.4 and min(cur.w, cur.h) >= 2:
        layers.append(conv(cur))
        cur = NetworkSpec._apply(layers[-1], cur)
    layers.append(LayerSpec(kind="square"))
    layers.append(LayerSpec(kind="fc", out_channels=int(rng.integers(2, 5))))
    return layers


def _ws_json(ws):
    return {name: {"values": ws[name].values.tolist(), "bits": ws[name].bits, "scale": ws[name].scale}
            for name in ws.names()}


def _rows_json(report):
    return [{"name": r.name, "op": r.op, "pattern": r.pattern,
             "measured": [r.measured.mul_pc, r.measured.add_cc, r.measured.rot],
             "assembly": r.measured_assembly, "squarings": r.measured_squarings} for r in report.rows]


def networks(count=14, seed=23, n_slots=64):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        w, h, c = int(rng.integers(3, 8)), int(rng.integers(3, 8)), int(rng.integers(1, 3))
        shape = TensorShape(w=w, h=h, c=c)
        try:
            layers = _random_layers(rng, shape)
            prov = NetworkSpec(scheme=SchemeParams(n_slots=n_slots, t=(1 << 61)), input_shape=shape,
                               layers=tuple(layers))
        except Exception:
            continue
        ws = random_weights(prov, rng, bound=3)
        bound = max(e.static_bound for e in ref_runner.static_bounds(prov, ws, input_bound=7))
        fs = crt_t(n_slots, bound)
        net = NetworkSpec(scheme=SchemeParams(n_slots=n_slots, t=math.prod(fs)), input_shape=shape,
                          layers=tuple(layers))
        plan = build_plan(net, "explicit")
        xs = rng.integers(0, 8, size=(2, c, h, w))
        logits, per_img_layers = [], []
        res = None
        for x in xs:
            res = ref_runner.run_encrypted(net, plan, ws, x, capture_layers=True)
            assert res.logits.tolist() == res.reference_logits.tolist()
            logits.append([int(v) for v in res.logits])
            _, ref_layers, _ = ref_runner.run_reference(net, ws, x)
            per_img_layers.append([np.asarray(t, dtype=object).astype(str).tolist() for t in ref_layers])
        out.append({
            "n_slots": n_slots, "t_factors": fs, "input_shape": [w, h, c],
            "layers": [{k: v for k, v in l.__dict__.items() if v is not None} for l in layers],
            "weights": _ws_json(ws), "inputs": xs.tolist(),
            "plan": [[s.op, s.layer_index, s.pattern] for s in plan.steps],
            "rows": _rows_json(res.report), "depth": res.depth, "assembly_depth": res.assembly_depth,
            "logits": logits, "layer_outputs": per_img_layers,
        })
    return out


# Hand-picked networks for the plan steps the random ones never produce: avg-pool
# (engine.py:271-279), DP-DP, an in-network HIm2Col from a dense layout, and a
# pooled CP -> DP chain (lola-default gives DP-DP twice around the pool).
EXTRA_NETWORKS = [
    ("avgpool-dense", "explicit", (6, 6, 1), [
        dict(kind="conv", d=2, stride=1, out_channels=2, packing_hint="dense"), dict(kind="avgpool", d=2, stride=2),
        dict(kind="square"), dict(kind="fc", out_channels=3)]),
    ("dp-dp", "explicit", (6, 5, 2), [
        dict(kind="ffconv", d=3, stride=1, out_channels=3, rank=2, packing_hint="dp-dp"), dict(kind="square"),
        dict(kind="fc", out_channels=2)]),
    ("him2col-dense", "explicit", (7, 7, 1), [
        dict(kind="conv", d=2, stride=1, out_channels=2, packing_hint="dense"),
        dict(kind="conv", d=2, stride=1, out_channels=2, packing_hint="conv"), dict(kind="square"),
        dict(kind="fc", out_channels=3)]),
    ("cp-avgpool-dp", "explicit", (7, 7, 2), [
        dict(kind="ffconv", d=2, stride=1, out_channels=3, rank=2, packing_hint="cp-hi2c-cp"), dict(kind="square"),
        dict(kind="avgpool", d=2, stride=2),
        dict(kind="ffconv", d=2, stride=1, out_channels=2, rank=1, packing_hint="dp-hi2c-cp"),
        dict(kind="fc", out_channels=2)]),
    ("cp-avgpool-dp-lola", "lola-default", (7, 7, 2), [
        dict(kind="ffconv", d=2, stride=1, out_channels=3, rank=2, packing_hint="cp-hi2c-cp"), dict(kind="square"),
        dict(kind="avgpool", d=2, stride=2),
        dict(kind="ffconv", d=2, stride=1, out_channels=2, rank=1, packing_hint="dp-hi2c-cp"),
        dict(kind="fc", out_channels=2)]),
    ("conv-avgpool-him2col", "explicit", (8, 8, 1), [
        dict(kind="conv", d=3, stride=1, out_channels=2, packing_hint="conv"), dict(kind="avgpool", d=2, stride=2),
        dict(kind="conv", d=2, stride=1, out_channels=2, packing_hint="conv"), dict(kind="square"),
        dict(kind="fc", out_channels=2)]),
]


def networks_extra(seed=29, n_slots=256):
    rng = np.random.default_rng(seed)
    out = []
    for name, strategy, (w, h, c), layer_docs in EXTRA_NETWORKS:
        layers = tuple(LayerSpec(**d) for d in layer_docs)
        shape = TensorShape(w=w, h=h, c=c)
        prov = NetworkSpec(scheme=SchemeParams(n_slots=n_slots, t=(1 << 61)), input_shape=shape, layers=layers)
        ws = random_weights(prov, rng, bound=3)
        bound = max(e.static_bound for e in ref_runner.static_bounds(prov, ws, input_bound=7))
        fs = crt_t(n_slots, bound)
        net = NetworkSpec(scheme=SchemeParams(n_slots=n_slots, t=math.prod(fs)), input_shape=shape, layers=layers)
        plan = build_plan(net, strategy)
        xs = rng.integers(0, 8, size=(2, c, h, w))
        logits, per_img_layers, res = [], [], None
        for x in xs:
            res = ref_runner.run_encrypted(net, plan, ws, x, capture_layers=True)
            assert res.logits.tolist() == res.reference_logits.tolist()
            logits.append([int(v) for v in res.logits])
            _, ref_layers, _ = ref_runner.run_reference(net, ws, x)
            per_img_layers.append([np.asarray(t, dtype=object).astype(str).tolist() for t in ref_layers])
        out.append({
            "name": name, "strategy": strategy,
            "n_slots": n_slots, "t_factors": fs, "input_shape": [w, h, c], "layers": layer_docs,
            "weights": _ws_json(ws), "inputs": xs.tolist(),
            "plan": [[s.op, s.layer_index, s.pattern] for s in plan.steps],
            "rows": _rows_json(res.report), "depth": res.depth, "assembly_depth": res.assembly_depth,
            "logits": logits, "layer_outputs": per_img_layers,
        })
    return out


# ------------------------------------------------------------------ cfg0
def cfg0(images=2, seed=20210205):
    rng = np.random.default_rng(seed)
    layers = (LayerSpec(kind="ffconv", d=5, stride=2, out_channels=5, rank=2, packing_hint="dp-hi2c-cp"),
              LayerSpec(kind="square"), LayerSpec(kind="fc", out_channels=100), LayerSpec(kind="square"),
              LayerSpec(kind="fc", out_channels=10))
    shape = TensorShape(w=29, h=29, c=1)
    prov = NetworkSpec(scheme=SchemeParams(n_slots=8192, t=(1 << 61)), input_shape=shape, layers=layers)
    ws = WeightSet()
    for name, shp in required_tensors(prov).items():
        if name.endswith(".bias"):
            ws.add(WeightTensor(name=name, values=np.zeros(shp, dtype=np.int64), bits=8, scale=1.0))
        else:
            q, s = quantize_matrix(rng.normal(0.0, 0.1, size=shp), 8)
            ws.add(WeightTensor(name=name, values=q, bits=8, scale=s))
    pix = np.round(rng.random(size=(images, 1, 28, 28)) * 255).astype(np.int64)
    xs = np.zeros((images, 1, 29, 29), dtype=np.int64)
    xs[:, :, :28, :28] = pix
    bounds = [e.static_bound for e in ref_runner.static_bounds(prov, ws, input_bound=255)]
    logits = []
    maxima = None
    for x in xs:
        lg, _, mx = ref_runner.run_reference(prov, ws, x)
        logits.append([str(int(v)) for v in lg])
        maxima = mx if maxima is None else [max(a, b) for a, b in zip(maxima, mx)]
    plan = build_plan(prov, "explicit")
    counts = ref_runner.run_encrypted(prov, plan, ws, None, track_values=False)
    # the reference's own encrypted path on image 0 at the product's CRT modulus
    fs = ntt_primes(30, 5, 4 * 8192)
    net = NetworkSpec(scheme=SchemeParams(n_slots=8192, t=math.prod(fs)), input_shape=shape, layers=layers)
    plan_t = build_plan(net, "explicit")
    unpatched = ref_runner.run_encrypted(net, plan_t, ws, xs[0], check_ledger=False)
    orig_fc = ref_runner.fc_dense

    def fc_masked(x, w, bias, ctx):
        outs, phases = orig_fc(x, w, bias, ctx)
        return [ref_engine._mask_slot0(ctx, o) for o in outs], phases

    ref_runner.fc_dense = fc_masked
    try:
        patched = ref_runner.run_encrypted(net, plan_t, ws, xs[0], check_ledger=False)
    finally:
        ref_runner.fc_dense = orig_fc
    assert [int(v) for v in patched.logits] == [int(v) for v in logits[0]]
    np.savez_compressed(os.path.join(HERE, "cfg0.npz"), inputs=xs,
                        **{name.replace(".", "_"): ws[name].values for name in ws.names()})
    meta = {
        "seed": seed, "sigma": 0.1, "layers": [{k: v for k, v in l.__dict__.items() if v is not None} for l in layers],
        "input_shape": [29, 29, 1], "scales": {name: ws[name].scale for name in ws.names()},
        "logits": logits, "layer_max_bits": [round(math.log2(max(m, 1)), 2) for m in maxima],
        "static_bound_bits": [round(math.log2(max(b, 1)), 2) for b in bounds],
        "count_rows": _rows_json(counts.report), "depth": counts.depth, "assembly_depth": counts.assembly_depth,
        "crt_t": fs,
        "reference_encrypted_unpatched": [str(int(v)) for v in unpatched.logits],
        "reference_encrypted_patched": [str(int(v)) for v in patched.logits],
    }
    with open(os.path.join(HERE, "cfg0.json"), "w") as fh:
        json.dump(meta, fh, indent=1)



# ------------------------------------------------------------------ cfg3
CFG3_LAYERS = (
    dict(kind="ffconv", d=3, stride=1, out_channels=32, rank=8),
    dict(kind="square"), dict(kind="avgpool", d=2, stride=2),
    dict(kind="ffconv", d=3, stride=1, out_channels=64, rank=16),
    dict(kind="square"), dict(kind="avgpool", d=2, stride=2),
    dict(kind="fc", out_channels=10),
)


def cfg3(images=2, seed=20210316):
    rng = np.random.default_rng(seed)
    layers = tuple(LayerSpec(**d) for d in CFG3_LAYERS)
    shape = TensorShape(w=32, h=32, c=3)
    prov = NetworkSpec(scheme=SchemeParams(n_slots=32768, t=(1 << 61)), input_shape=shape, layers=layers)
    ws = WeightSet()
    for name, shp in required_tensors(prov).items():
        if name.endswith(".bias"):
            ws.add(WeightTensor(name=name, values=np.zeros(shp, dtype=np.int64), bits=8, scale=1.0))
        else:
            q, s = quantize_matrix(rng.normal(0.0, 0.05, size=shp), 8)
            ws.add(WeightTensor(name=name, values=q, bits=8, scale=s))
    xs = np.round(np.clip(rng.normal(0.5, 0.25, size=(images, 3, 32, 32)), 0.0, 1.0) * 255).astype(np.int64)
    bounds = [e.static_bound for e in ref_runner.static_bounds(prov, ws, input_bound=255)]
    logits, maxima = [], None
    for x in xs:
        lg, _, mx = ref_runner.run_reference(prov, ws, x)
        logits.append([str(int(v)) for v in lg])
        maxima = mx if maxima is None else [max(a, b) for a, b in zip(maxima, mx)]
    plan = build_plan(prov, "ffconv-default")
    counts = ref_runner.run_encrypted(prov, plan, ws, None, track_values=False)
    np.savez_compressed(os.path.join(HERE, "cfg3.npz"), inputs=xs,
                        **{name.replace(".", "_"): ws[name].values for name in ws.names()})
    meta = {
        "seed": seed, "sigma": 0.05, "layers": list(CFG3_LAYERS), "input_shape": [32, 32, 3],
        "n_slots": 32768, "strategy": "ffconv-default",
        "scales": {name: ws[name].scale for name in ws.names()},
        "logits": logits, "layer_max_bits": [round(math.log2(max(m, 1)), 2) for m in maxima],
        "static_bound_bits": [round(math.log2(max(b, 1)), 2) for b in bounds],
        "plan": [[st.op, st.layer_index, st.pattern] for st in plan.steps],
        "count_rows": _rows_json(counts.report), "depth": counts.depth, "assembly_depth": counts.assembly_depth,
    }
    with open(os.path.join(HERE, "cfg3.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def weight_file():
    """A CPKW0001 file written by the reference (weights.py:102-124)."""
    from cipherpack.weights import save_weights as ref_save
    ws = WeightSet([WeightTensor(name="layer0.weight", values=np.arange(-12, 12).reshape(2, 3, 4), bits=8,
                                 scale=0.125),
                    WeightTensor(name="layer0.bias", values=np.array([7, -3]), bits=8, scale=1.0)])
    ref_save(ws, os.path.join(HERE, "weights_ref.cpkw"))


if __name__ == "__main__":
    if sys.argv[1:] == ["cfg3"]:
        cfg3()
        sys.exit(0)
    if sys.argv[1:] == ["extra"]:
        with open(os.path.join(HERE, "networks_extra.json"), "w") as fh:
            json.dump(networks_extra(), fh)
        sys.exit(0)
    with open(os.path.join(HERE, "hesim_sequences.json"), "w") as fh:
        json.dump(hesim_sequences(), fh)
    with open(os.path.join(HERE, "networks.json"), "w") as fh:
        json.dump(networks(), fh)
    with open(os.path.join(HERE, "networks_extra.json"), "w") as fh:
        json.dump(networks_extra(), fh)
    cfg0()
    cfg3()
    weight_file()
    print("fixtures written to", HERE)
