"""Helpers shared by the CPU (golden-model) and GPU parity tests."""

from __future__ import annotations

import json
import math
import os

import numpy as np

from paper_2102_03494_b200.hesim import HeContext, SchemeParams
from paper_2102_03494_b200.netspec import LayerSpec, NetworkSpec, WeightSet, WeightTensor
from paper_2102_03494_b200.packing import TensorShape
from paper_2102_03494_b200.params import make_params

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def scheme_from(n_slots, factors, levels=6, q_bits=50, seed=None):
    rp = make_params(n_slots, factors, levels=levels, q_bits=q_bits, seed=seed)
    return SchemeParams(n_slots=n_slots, t=math.prod(factors), t_factors=tuple(factors), rlwe=rp)


def replay(ctx, case, encrypt=None):
    """Run a hesim_sequences.json case through any HeContext-like object."""
    enc = encrypt or ctx.encrypt
    n = case["n_slots"]
    ct = enc(case["x"])
    for op in case["ops"]:
        kind = op[0]
        if kind == "rotate":
            ct = ctx.rotate(ct, op[1])
        elif kind == "mul_plain":
            ct = ctx.mul_plain(ct, ctx.encode(op[1]), assembly=op[2])
        elif kind == "add_cc":
            ct = ctx.add_cc(ct, enc(op[1]))
        elif kind == "square":
            ct = ctx.square(ct)
        elif kind == "add_plain":
            ct = ctx.add_plain(ct, ctx.encode(op[1]))
        elif kind == "mask_rotate_and_sum":
            m = op[1]
            ct = ctx.mul_plain(ct, ctx.encode([1] * m + [0] * (n - m)))
            ct = ctx.rotate_and_sum(ct, m)
    return ct


def network_from_fixture(fx, scheme=None, seed=None):
    w, h, c = fx["input_shape"]
    layers = tuple(LayerSpec(**l) for l in fx["layers"])
    if scheme is None:
        scheme = scheme_from(fx["n_slots"], fx["t_factors"], seed=seed)
    net = NetworkSpec(scheme, TensorShape(w, h, c), layers)
    ws = WeightSet()
    for name, v in fx["weights"].items():
        ws.add(WeightTensor(name, np.array(v["values"], dtype=np.int64), v["bits"], v["scale"]))
    return net, ws


def cfg0_network(scheme):
    meta = load("cfg0.json")
    z = np.load(os.path.join(GOLD, "cfg0.npz"))
    layers = tuple(LayerSpec(**l) for l in meta["layers"])
    net = NetworkSpec(scheme, TensorShape(29, 29, 1), layers)
    ws = WeightSet()
    for name, scale in meta["scales"].items():
        ws.add(WeightTensor(name, z[name.replace(".", "_")].astype(np.int64), 8, scale))
    return net, ws, z["inputs"], meta


def step_totals(records):
    """label -> (mul_pc, add_cc, rot, assembly, squarings) summed over phases."""
    out = {}
    for r in records:
        tot = [0, 0, 0, 0, 0]
        for _, c in r.phases:
            tot = [tot[0] + c.mul_pc, tot[1] + c.add_cc, tot[2] + c.rot, tot[3] + c.assembly_mul_pc,
                   tot[4] + c.mul_cc]
        out[r.label] = tot
    return out


def reference_step_totals(rows):
    out = {}
    for r in rows:
        parts = r["name"].split(":")
        label = ":".join(parts[:2]) if parts[0].startswith("layer") else parts[0]
        t = out.setdefault(label, [0, 0, 0, 0, 0])
        m = r["measured"]
        out[label] = [t[0] + m[0], t[1] + m[1], t[2] + m[2], t[3] + r["assembly"], t[4] + r["squarings"]]
    return out
