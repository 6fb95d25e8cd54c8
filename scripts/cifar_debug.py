"""configs[3] diagnostics: per-layer noise budget and decrypted values (mod the first
plaintext prime) of the GPU run against the slot oracle's run on the same image."""
import json, multiprocessing as mp, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import bench  # noqa: E402
from paper_2102_03494_b200 import runner  # noqa: E402

SCHED = os.environ.get("SCHED", "reference")


def oracle_layers(t0):
    from oracle.slot_oracle import Params, SlotContext
    net, plan, ws, xs, rp, ref = bench.cfg3_setup(1, seed=bench.CFG1["seed"])
    res = runner.run_encrypted(net, plan, ws, xs[0], ctx=SlotContext(Params(net.scheme.n_slots, t0)),
                               capture_layers=True)
    return [(i, np.asarray(v, dtype=object) % t0) for i, v in res.layer_outputs], [int(v) % t0 for v in res.logits]


def main():
    from paper_2102_03494_b200.abi import cuda_library
    from paper_2102_03494_b200.hesim import HeContext
    net, plan, ws, xs, rp, ref = bench.cfg3_setup(2, seed=bench.CFG1["seed"])
    t0 = rp.t[0]
    pool = mp.Pool(1)
    job = pool.apply_async(oracle_layers, (t0,))
    ctx = HeContext(net.scheme, batch=2, lib=cuda_library(), schedule=SCHED)
    budgets = []
    orig = runner._tensor

    def tensor_with_budget(value, c):
        cts = [value.ct] if hasattr(value, "ct") else list(value.cts)
        budgets.append(min(c.noise_budget(x) for x in cts[:4]))
        return orig(value, c)

    runner._tensor = tensor_with_budget
    t = time.time()
    res = runner.run_encrypted(net, plan, ws, xs, ctx=ctx, capture_layers=True)
    print("gpu run", round(time.time() - t, 1), "s", flush=True)
    o_layers, o_logits = job.get()
    out = []
    for (i, got), (j, want), b in zip(res.layer_outputs, o_layers, budgets):
        g0 = np.asarray(got, dtype=object)[0] % t0
        ok = bool(np.array_equal(g0, want))
        bad = int(np.sum(g0 != want))
        out.append({"layer": i, "noise_budget_bits": round(b, 1), "match_mod_t0": ok, "mismatches": bad,
                    "size": int(np.asarray(want).size)})
        print(out[-1], flush=True)
    lg = [int(v) % t0 for v in np.asarray(res.logits)[0]]
    print("logits mod t0 match:", lg == o_logits)
    print("logits vs fixture:", [[int(v) for v in r] for r in np.asarray(res.logits).tolist()] == ref)
    with open("gpurun_out/cifar_debug.json", "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
