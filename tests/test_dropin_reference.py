"""The drop-in, driven from the reference's side: cipherpack's own plan walker
(/root/reference/pkg/src/cipherpack/runner.py:290-409), with its one context
construction (runner.py:297) swapped for this package's HeContext on the golden
backend.  Everything else -- the reference's planner,
packing, engine, ledger and cost report -- runs unmodified on real RLWE
ciphertexts.  Skipped where the reference is absent (the GPU box)."""

import os
import sys

import numpy as np
import pytest

from _shared import load

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "cipherpack")),
                                reason="the reference (cipherpack) is not present")


def _ref_network(fx):
    from cipherpack.hesim import SchemeParams
    from cipherpack.netspec import LayerSpec, NetworkSpec
    from cipherpack.packing import TensorShape
    from cipherpack.weights import WeightSet, WeightTensor
    w, h, c = fx["input_shape"]
    net = NetworkSpec(scheme=SchemeParams(n_slots=fx["n_slots"], t=int(np.prod([int(f) for f in fx["t_factors"]],
                                                                                  dtype=object))),
                      input_shape=TensorShape(w=w, h=h, c=c), layers=tuple(LayerSpec(**l) for l in fx["layers"]))
    ws = WeightSet()
    for name, v in fx["weights"].items():
        ws.add(WeightTensor(name=name, values=np.array(v["values"], dtype=np.int64), bits=v["bits"],
                            scale=v["scale"]))
    return net, ws


@pytest.mark.parametrize("which", ["networks.json", "networks_extra.json"])
def test_reference_runner_on_the_b200_context(which, golden_lib, monkeypatch):
    monkeypatch.syspath_prepend(REF)
    import cipherpack.runner as ref_runner
    from cipherpack.planner import build_plan
    from paper_2102_03494_b200.dropin import make_context
    from paper_2102_03494_b200.hesim import HeContext
    made = []
    for fx in load(which):
        net, ws = _ref_network(fx)
        plan = build_plan(net, fx.get("strategy", "explicit"))

        def factory(scheme, plan=plan):          # the runner.py:297 hook
            ctx = make_context(scheme, plan=plan, lib=golden_lib)
            made.append(ctx)
            return ctx

        monkeypatch.setattr(ref_runner, "HeContext", factory)
        for x, want, layers in zip(fx["inputs"], fx["logits"], fx["layer_outputs"]):
            res = ref_runner.run_encrypted(net, plan, ws, np.array(x), capture_layers=True)
            assert isinstance(made[-1], HeContext)
            assert [int(v) for v in res.logits] == want
            assert res.logits.tolist() == res.reference_logits.tolist()
            assert [[r.measured.mul_pc, r.measured.add_cc, r.measured.rot] for r in res.report.rows] == \
                [r["measured"] for r in fx["rows"]]
            assert (res.depth, res.assembly_depth) == (fx["depth"], fx["assembly_depth"])
            for (_, got), ref in zip(res.layer_outputs, layers):
                assert np.asarray(got, dtype=object).astype(str).tolist() == ref
    assert made and all(m.params.t_factors for m in made)
