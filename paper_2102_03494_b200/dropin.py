"""The drop-in hook for the reference's plan walker.

`cipherpack.runner.run_encrypted` builds its evaluation context at one line
(/root/reference/pkg/src/cipherpack/runner.py:297, `ctx = HeContext(net.scheme)`)
and then only calls context methods.  `make_context`
turns the reference's `SchemeParams` into this package's GPU `HeContext`, which
has the same methods, counters, depth bookkeeping and errors, so the line becomes

    ctx = make_context(net.scheme, plan=plan)

(INTEGRATION.md section 2).  Everything else in the reference -- planner, packing,
engine, ledger, report -- runs unchanged on top of it.
"""

from __future__ import annotations

import math

from .hesim import HeContext, SchemeParams
from .params import factor_plaintext_modulus


def make_context(scheme, *, plan=None, t_factors=None, lib=None, batch: int = 1, levels: int | None = None,
                 q_bits: int = 60, **kw) -> HeContext:
    """A GPU HeContext for a reference (or product) SchemeParams.

    t_factors: the prime factorization of scheme.t (plaintext CRT); recovered by
    factoring when omitted.  plan: the reference PackingPlan the context will run;
    when given, the q chain is sized for it by the product's noise model
    (runner.inference_params), else `levels` (default 4) q primes are used and the
    decryption noise guard raises NoiseBudgetError if that is too short."""
    factors = tuple(int(f) for f in (t_factors or getattr(scheme, "t_factors", None)
                                     or factor_plaintext_modulus(scheme.t, scheme.n_slots)))
    ours = SchemeParams(n_slots=scheme.n_slots, t=scheme.t, rotation_weight=scheme.rotation_weight,
                        t_factors=factors, rlwe=getattr(scheme, "rlwe", None))
    if levels is None and plan is not None and ours.rlwe is None:
        from .runner import _noise_bits
        # the reference engine's column stage is a masked constant plaintext multiply and
        # its FC outputs are not masked (engine.py:189-195, 241-260)
        need = _noise_bits(plan, math.log2(max(factors)), mask_fc=False, plain_conv_conv=True)
        levels = max(2, math.ceil(need / q_bits))
    return HeContext(ours, lib=lib, batch=batch, levels=levels, q_bits=q_bits if levels else None, **kw)
