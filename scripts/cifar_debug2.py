"""configs[3]: find the first HeContext call whose output loses noise budget abnormally."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import bench  # noqa: E402
from paper_2102_03494_b200 import runner  # noqa: E402
from paper_2102_03494_b200.hesim import HeContext  # noqa: E402
from paper_2102_03494_b200.abi import cuda_library  # noqa: E402


class Stop(Exception):
    pass


def main():
    net, plan, ws, xs, rp, ref = bench.cfg3_setup(2, seed=bench.CFG1["seed"])
    ctx = HeContext(net.scheme, batch=2, lib=cuda_library(), schedule=os.environ.get("SCHED", "reference"))
    calls = [0]

    def first_ct(x):
        if isinstance(x, (list, tuple)):
            return first_ct(x[0]) if x else None
        return x if hasattr(x, "handle") else None

    def wrap(name):
        fn = getattr(ctx, name)

        def inner(*a, **k):
            out = fn(*a, **k)
            calls[0] += 1
            ins = [first_ct(v) for v in a if first_ct(v) is not None and getattr(first_ct(v), "handle", None) is not None]
            o = first_ct(out)
            if o is None or o.handle is None:
                return out
            bo = ctx.noise_budget(o)
            bi = min([ctx.noise_budget(i) for i in ins[:2]] or [999])
            outs = out if isinstance(out, (list, tuple)) else [out]
            blast = ctx.noise_budget(outs[-1]) if len(outs) > 1 and outs[-1].handle is not None else bo
            if bo < 150 or blast < 150 or bi - min(bo, blast) > 80:
                extra = {kk: (v if isinstance(v, (int, str)) else (len(v) if isinstance(v, (list, tuple)) else type(v).__name__))
                         for kk, v in zip(range(len(a)), a)}
                print(f"ANOMALY call#{calls[0]} {name}: in {bi:.1f} -> out first {bo:.1f} last {blast:.1f}; args {extra}",
                      flush=True)
                if isinstance(a[-1], (list, tuple)) and a[-1] and isinstance(a[-1][0], int):
                    print("  steps", a[-1][:20], flush=True)
                raise Stop()
            if calls[0] % 200 == 0:
                print(f"call#{calls[0]} {name}: in {bi:.1f} -> out {bo:.1f}/{blast:.1f}", flush=True)
            return out
        setattr(ctx, name, inner)

    for nm in ("rotate", "mul_plain", "mul_scalar", "add_cc", "add_plain", "square", "rotate_and_sum",
               "mul_plain_many", "rotate_many", "hoisted_dot", "rotate_multi", "add_cc_many", "rotate_and_sum_many",
               "_rotate_add_many"):
        wrap(nm)
    t = time.time()
    try:
        runner.run_encrypted(net, plan, ws, xs, ctx=ctx)
        print("completed without anomaly")
    except Stop:
        pass
    print("elapsed", round(time.time() - t, 1), flush=True)


if __name__ == "__main__":
    main()
