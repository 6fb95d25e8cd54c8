"""Plan execution on the GPU evaluator.

Mirror of `cipherpack.runner.run_encrypted` (/root/reference/pkg/src/cipherpack/runner.py:290-433):
the same plan walk (step ops -> packing/engine calls), per-step measured
counters, depth bookkeeping and logits extraction, for a batch of images per
context.  Differences:

* the context is the sm_100a RNS-BFV evaluator; its parameters are chosen here
  (`inference_params`): plaintext CRT primes sized from the static worst-case
  logit bound (runner.py:233-266) and a q chain sized by a per-op noise model;
* the plaintext reference computation and the run ledger (runner.py:301-313)
  are not part of this path -- parity is checked by tests against the oracle;
* FC outputs that are later combined are masked to slot 0 (`mask_fc`, the F4
  fix); with mask_fc=False the reference's own (diverging)
  encrypted result is reproduced.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .engine import (
    BiasVector,
    WeightMatrix,
    avg_pool_weights,
    conv_conv,
    conv_dense,
    conv_dense_to_channels,
    factored_conv,
    fc_dense,
    packed_depth,
    square_layer,
)
from .hesim import HeContext, OpCounters, SchemeParams
from .netspec import NetworkSpec, WeightSet, validate_weights
from .packing import (
    ChannelPacked,
    DensePacked,
    KernelSpec,
    channel_unpack,
    channels_to_dense,
    conv_pack,
    dense_pack,
    dense_unpack,
    h_grouping,
    h_grouping_from_dense,
    h_im2col_from_conv,
    h_im2col_from_dense,
    plain_im2col,
)
from .params import RlweParams, ntt_primes
from .planner import (
    COMBINE, CONV_COLUMNS, CONV_DENSE, FC, FFCONV, GROUP_CONV, GROUP_DENSE, HIM2COL_CONV, HIM2COL_DENSE,
    PACK_COLUMNS, PACK_DENSE, SQUARE, PackingPlan,
)


def weights_to_matrix(w4d: np.ndarray) -> np.ndarray:
    """(d, d, in_c, out_c) filters -> K x O_c, rows channel-major (ch, ky, kx) (factorize.py:47-58)."""
    d1, d2, ic, oc = w4d.shape
    if d1 != d2:
        raise ValueError(f"kernel must be square, got {d1}x{d2}")
    return w4d.transpose(2, 0, 1, 3).reshape(d1 * d2 * ic, oc)


def _conv_w(ws, i):
    t = ws[f"layer{i}.weight"]
    return WeightMatrix(weights_to_matrix(t.values), t.bits, t.scale)


def _ff_w(ws, i):
    a, b = ws[f"layer{i}.w1"], ws[f"layer{i}.w2"]
    return (WeightMatrix(weights_to_matrix(a.values), a.bits, a.scale),
            WeightMatrix(weights_to_matrix(b.values), b.bits, b.scale))


def _fc_w(ws, i):
    t, b = ws[f"layer{i}.weight"], ws[f"layer{i}.bias"]
    return WeightMatrix(t.values, t.bits, t.scale), BiasVector(b.values, b.scale)


# ----------------------------------------------------------- static bounds

def _max_col_l1(m) -> int:
    return int(np.max(np.sum(np.abs(np.asarray(m).astype(object)), axis=0))) if np.size(m) else 0


def static_bounds(net: NetworkSpec, ws: WeightSet, input_bound: int) -> list[int]:
    """Worst-case |value| after every layer for inputs in [-input_bound, input_bound]
    (runner.py:233-266)."""
    b = int(input_bound)
    out = []
    for i, layer in enumerate(net.layers):
        if layer.kind == "conv":
            b *= _max_col_l1(weights_to_matrix(ws[f"layer{i}.weight"].values))
        elif layer.kind == "ffconv":
            b *= _max_col_l1(weights_to_matrix(ws[f"layer{i}.w1"].values))
            b *= _max_col_l1(weights_to_matrix(ws[f"layer{i}.w2"].values))
        elif layer.kind == "square":
            b *= b
        elif layer.kind == "avgpool":
            b *= layer.d * layer.d
        elif layer.kind == "fc":
            bias = ws[f"layer{i}.bias"].values
            b = b * _max_col_l1(ws[f"layer{i}.weight"].values) + (int(np.max(np.abs(bias))) if bias.size else 0)
        out.append(b)
    return out


# ----------------------------------------------------------- parameters

# Per-op invariant-noise cost in bits (t_bits = log2 of the plaintext prime).
# Calibrated with scripts/noise_probe.py on a B200 (profiles/noise_probe_r01.jsonl):
# at t = 30 bits the cfg0 chain measured fresh 35, dot+rotate-and-sum 43, slot
# mask 32, assembly chain 6, 1x1 scalar stage 4, combine 2-6, square 41 bits.
# Each term below is the measurement + 1 bit; 12 bits of margin on top.
def _step_noise_bits(plan: PackingPlan, k: int, t_bits: float, mask_fc: bool, plain_conv_conv: bool = False) -> float:
    """Invariant-noise bits plan step k adds (the per-op costs above).
    plain_conv_conv: the column stage multiplies by a masked constant plaintext
    (the reference engine, engine.py:189-195) instead of a scalar (engine.conv_conv
    here): about a slot mask's noise per stage instead of a few bits."""
    dot, mask, chain, square = t_bits + 14, t_bits + 3, 7, t_bits + 12
    cols = mask + 4 if plain_conv_conv else 5
    step = plan.steps[k]
    op, need = step.op, 0.0
    if op == CONV_DENSE or (op == FFCONV and step.pattern in ("DP-HI2C-CP", "DP-DP")):
        need += dot + mask + chain
    if op == FFCONV:
        need += cols                                  # 1x1 stage
        if step.pattern in ("CP-HI2C-CP", "CP-HI2C-DP"):
            need += cols
        if step.pattern == "DP-DP":
            need += dot + mask + chain
    if op == CONV_COLUMNS:
        need += cols + 3
    if op in (HIM2COL_DENSE, HIM2COL_CONV, GROUP_DENSE):
        need += mask + chain
    if op == SQUARE:
        need += square
    if op == FC:
        need += dot
        nxt = plan.steps[k + 1].op if k + 1 < len(plan.steps) else None
        if mask_fc and nxt == COMBINE:
            need += mask
    if op == COMBINE:
        need += chain
    return need


def _noise_bits(plan: PackingPlan, t_bits: float, mask_fc: bool, plain_conv_conv: bool = False) -> float:
    """Bits of q the whole plan needs: fresh encryption + every step + 12 bits of margin."""
    need = t_bits + 6                                 # fresh encryption
    for k in range(len(plan.steps)):
        need += _step_noise_bits(plan, k, t_bits, mask_fc, plain_conv_conv)
    return need + 12.0


# Level schedule (HeContext(level_schedule=True)).  BFV modulus switching keeps the noise
# budget: switching Q -> Q/q_last divides the noise by q_last and adds a rounding term of
# about the fresh-encryption noise.  So once the plan's steps have added more than
# log2(q_last) + SLACK bits of noise since encryption, the last prime can be dropped
# for free, and every later key switch runs at fewer primes (its cost grows as l^2).
LEVEL_SLACK_BITS = 12.0


def _target_level(q: tuple, level: int, consumed: float) -> int:
    """The lowest level reachable by dropping primes from `level` whose bits sum to at
    most consumed - LEVEL_SLACK_BITS (never below 2)."""
    room = consumed - LEVEL_SLACK_BITS
    drop = 0
    while level - drop > 2 and room >= math.log2(q[level - drop - 1]):
        room -= math.log2(q[level - drop - 1])
        drop += 1
    return level - drop


def inference_params(net: NetworkSpec, plan: PackingPlan, ws: WeightSet, input_bound: int, *,
                     t_bits: int = 30, q_bits: int = 60, mask_fc: bool = True, seed: int | None = None) -> RlweParams:
    """Plaintext CRT primes covering 2 * static bound, and a q chain for the plan."""
    n_slots = net.scheme.n_slots
    two_n = 4 * n_slots
    bound = max(static_bounds(net, ws, input_bound) + [input_bound, 1])
    cands = ntt_primes(t_bits, 64, two_n)
    ts, total = [], 1
    for p in cands:
        ts.append(p)
        total *= p
        if total > 2 * bound:
            break
    need = _noise_bits(plan, math.log2(ts[0]), mask_fc)
    L = max(2, math.ceil(need / q_bits))
    q = ntt_primes(q_bits, L, two_n, exclude=ts)
    p = ntt_primes(min(q_bits + 1, 61), 1, two_n, exclude=ts + q)
    b = ntt_primes(60, L + 1, two_n, exclude=ts + q + p)
    if sum(math.log2(x) for x in b) < sum(math.log2(x) for x in q) + math.log2(2 * n_slots) + t_bits + 4:
        b = ntt_primes(60, L + 2, two_n, exclude=ts + q + p)
    kw = {} if seed is None else {"seed": seed}
    return RlweParams(log_n=n_slots.bit_length(), q=tuple(q), p=tuple(p), t=tuple(ts), b=tuple(b), **kw)


def default_context(net: NetworkSpec, plan: PackingPlan, input_tensor=None, *, batch: int | None = None,
                    q_bits: int = 60, mask_fc: bool = True, lib=None) -> HeContext:
    """A GPU HeContext for net.scheme whose q chain is sized for this plan (the noise
    model of `inference_params` at the scheme's own plaintext factors) unless the
    scheme pins its RlweParams.  t must factor into batching-compatible primes."""
    x = None if input_tensor is None else np.asarray(input_tensor)
    if batch is None:
        shape_rank = 3
        batch = x.shape[0] if x is not None and x.ndim == shape_rank + 1 else 1
    if net.scheme.rlwe is not None:
        return HeContext(net.scheme, batch=batch, lib=lib)
    t_bits = math.log2(max(net.scheme.factors()))
    levels = max(2, math.ceil(_noise_bits(plan, t_bits, mask_fc) / q_bits))
    return HeContext(net.scheme, batch=batch, lib=lib, levels=levels, q_bits=q_bits)


def scheme_for(params: RlweParams, rotation_weight: float = 10.0) -> SchemeParams:
    """A SchemeParams whose t is the CRT product of the chosen plaintext primes."""
    return SchemeParams(n_slots=params.n_slots, t=params.t_product, rotation_weight=rotation_weight,
                        t_factors=params.t, rlwe=params)


# ----------------------------------------------------------- execution

@dataclass
class StepRecord:
    label: str
    op: str
    pattern: str | None
    phases: list          # [(name, OpCounters)]


@dataclass
class RunResult:
    logits: np.ndarray | None          # (B, n_out) object ints, or (n_out,) for batch 1
    steps: list
    counters: OpCounters
    depth: int
    assembly_depth: int
    layer_depths: list = field(default_factory=list)
    layer_outputs: list = field(default_factory=list)
    elided_rotations: int = 0
    value: object = None               # the final packed value (device handles)


def _logits(value, ctx):
    batch = getattr(ctx, "batch", 1)

    def dec(ct, k):
        if hasattr(ctx, "decrypt_slots"):         # only the payload slots leave the device
            v = np.asarray(ctx.decrypt_slots(ct, k), dtype=object)
            return v[None] if v.ndim == 1 else v
        v = np.asarray(ctx.decrypt(ct), dtype=object)
        v = v[None] if v.ndim == 1 else v
        return v[:, :k]

    if isinstance(value, DensePacked):
        out = dec(value.ct, value.occupied)
    elif isinstance(value, ChannelPacked):
        out = np.concatenate([dec(c, value.rows) for c in value.cts], axis=1)
    else:
        raise ValueError(f"cannot extract logits from {type(value)!r}")
    return out[0] if batch == 1 else out


def _logits_layout(net: NetworkSpec, plan: PackingPlan) -> tuple[int, int]:
    """(logit ciphertexts, payload slots per ciphertext) of a plan's final value,
    from a count-only walk (no device work)."""
    ctx = HeContext(net.scheme)
    res = run_encrypted(net, plan, _zero_weights(net), None, ctx=ctx, track_values=False)
    v = res.value
    if isinstance(v, DensePacked):
        return 1, v.occupied
    return len(v.cts), v.rows


def _zero_weights(net: NetworkSpec) -> WeightSet:
    from .netspec import required_tensors, WeightTensor
    ws = WeightSet()
    for name, shape in required_tensors(net).items():
        ws.add(WeightTensor(name, np.zeros(shape, dtype=np.int64), 8, 1.0))
    return ws


def _tensor(value, ctx):
    if isinstance(value, DensePacked):
        return dense_unpack(value, ctx)
    if isinstance(value, ChannelPacked):
        return channel_unpack(value, ctx)
    return None


def pack_input(net: NetworkSpec, plan: PackingPlan, input_tensor, ctx):
    """Client side of the plan's first step: encrypt the input(s) in the layout
    the plan starts from (runner.py:342-352)."""
    step = plan.steps[0]
    x = np.asarray(input_tensor)
    if step.op == PACK_DENSE:
        return dense_pack(x, ctx)
    if step.op == PACK_COLUMNS:
        ow, oh = step.kernel.out_dims(step.in_shape)
        return conv_pack(plain_im2col(x, step.kernel), ctx, (ow, oh))
    raise ValueError(f"plan does not start with a packing step: {step.op}")


def run_encrypted(net: NetworkSpec, plan: PackingPlan, weights: WeightSet, input_tensor, *,
                  ctx=None, track_values: bool = True, capture_layers: bool = False,
                  mask_fc: bool = True, packed=None, decrypt: bool = True) -> RunResult:
    """Walk the plan over an evaluation context (runner.py:290-409).

    input_tensor: (c, h, w) for a batch-1 context or (B, c, h, w).
    ctx: any object with the HeContext interface; default: a GPU HeContext on
    net.scheme (its parameters must then be batching-compatible).
    packed: an already encrypted input (from pack_input); decrypt=False leaves
    the logits encrypted (RunResult.value) -- together they bracket the
    server-side evaluation only."""
    validate_weights(net, weights)
    if plan.net != net:
        raise ValueError("plan was built for a different network")
    if ctx is None:
        ctx = default_context(net, plan, input_tensor)
    x_in = None
    if track_values and packed is None:
        x_in = np.asarray(input_tensor)
        shape = (net.input_shape.c, net.input_shape.h, net.input_shape.w)
        if x_in.shape[-3:] != shape:
            raise ValueError(f"input shape {x_in.shape} does not match (c, h, w) = {shape}")
    records, layer_depths, layer_outputs = [], [], []
    value = None
    sched = bool(getattr(ctx, "level_schedule", False)) and track_values
    if sched:
        t_bits = math.log2(max(ctx.params.factors()))
        qs, top, consumed = ctx.evaluator.params.q, ctx.evaluator.L, 0.0
    for k, step in enumerate(plan.steps):
        if sched:
            ctx.noise_consumed = consumed            # the engine's in-step level_down reads it
        before = ctx.counters.copy()
        d_before = packed_depth(value) if value is not None else (0, 0)
        phases = None
        op = step.op
        if packed is not None and k == 0 and op in (PACK_DENSE, PACK_COLUMNS):
            value = packed
        elif op == PACK_DENSE:
            value = dense_pack(x_in if track_values else np.zeros((step.in_shape.c, step.in_shape.h,
                                                                   step.in_shape.w), dtype=np.int64),
                               ctx, tracked=track_values)
        elif op == PACK_COLUMNS:
            ow, oh = step.kernel.out_dims(step.in_shape)
            cols = (plain_im2col(x_in, step.kernel) if track_values else
                    np.zeros((ow * oh, step.kernel.k_columns(step.in_shape.c)), dtype=np.int64))
            value = conv_pack(cols, ctx, (ow, oh), tracked=track_values)
        elif op == COMBINE:
            value = channels_to_dense(value, ctx)
        elif op == HIM2COL_DENSE:
            value = h_im2col_from_dense(value, step.kernel, ctx)
        elif op == HIM2COL_CONV:
            value = h_im2col_from_conv(value, step.kernel, ctx)
        elif op == GROUP_DENSE:
            value = h_grouping_from_dense(value, KernelSpec(1, 1), ctx)
        elif op == GROUP_CONV:
            value = h_grouping(value, KernelSpec(1, 1))
        elif op == SQUARE:
            value, phases = square_layer(value, ctx)
        elif op in (CONV_DENSE, CONV_COLUMNS):
            i = step.layer_index
            w = avg_pool_weights(step.kernel, step.in_shape.c) if step.pooling else _conv_w(weights, i)
            value, phases = (conv_dense(value, w, step.kernel, ctx) if op == CONV_DENSE
                             else conv_conv(value, w, ctx))
        elif op == FC:
            w, bias = _fc_w(weights, step.layer_index)
            nxt = plan.steps[k + 1].op if k + 1 < len(plan.steps) else None
            outs, phases = fc_dense(value, w, bias, ctx, mask_outputs=mask_fc and nxt == COMBINE)
            value = ChannelPacked(tuple(outs), (1, 1))
        elif op == FFCONV:
            value, phases = _run_ffconv(step, value, weights, ctx)
        else:
            raise ValueError(f"cannot execute step {op!r}")
        if sched and op not in (PACK_DENSE, PACK_COLUMNS):
            consumed += _step_noise_bits(plan, k, t_bits, mask_fc)
            value = _switch_value(value, ctx, _target_level(qs, top, consumed))
        if phases is None:
            phases = [("total", ctx.counters - before)]
        else:
            phases = [(p.name, p.counters) for p in phases]
        records.append(StepRecord(step.label(), op, step.pattern, phases))
        if step.layer_index is not None and op in (SQUARE, CONV_DENSE, CONV_COLUMNS, FC, FFCONV):
            d_after = packed_depth(value)
            layer_depths.append({"layer_index": step.layer_index, "op": op, "pattern": step.pattern,
                                 "depth_delta": d_after[0] - d_before[0],
                                 "assembly_delta": d_after[1] - d_before[1]})
            if capture_layers and track_values:
                layer_outputs.append((step.layer_index, _tensor(value, ctx)))
    if sched:
        ctx.noise_consumed = None
    logits = _logits(value, ctx) if (track_values and decrypt) else None
    depth, adepth = packed_depth(value)
    return RunResult(logits, records, ctx.counters.copy(), depth, adepth, layer_depths, layer_outputs,
                     ctx.elided_rotations, value)


def _packed_cts(value):
    if isinstance(value, DensePacked):
        return [value.ct]
    return list(value.cts)


class CapturedPlan:
    """One plan walk's device work, recorded once as a CUDA graph and replayed.

    The op sequence of a walk is data-independent (the reference's count-only walk,
    runner.py:290-293, proves it), so the launches of `run_encrypted` on a packed
    input can be captured (fhe_capture_begin/end) and replayed for every new input of
    the same shape: a replay copies the new encrypted input into the captured input
    ciphertexts and launches the graph -- no Python plan walk, no per-op launches.
    A warm-up walk first creates the keys, plaintexts and workspaces the capture
    needs and measures the ciphertext memory the arena must hold.  Op counters and
    depths are those of the captured walk (`self.result`)."""

    def __init__(self, net: NetworkSpec, plan: PackingPlan, weights: WeightSet, example, ctx, *,
                 mask_fc: bool = True, arena_margin: float = 1.25):
        self.net, self.plan, self.weights, self.ctx = net, plan, weights, ctx
        ev = ctx.evaluator
        ev.peak_bytes(reset=True)
        warm = pack_input(net, plan, example, ctx)
        run_encrypted(net, plan, weights, None, ctx=ctx, packed=warm, decrypt=False, mask_fc=mask_fc)
        ev.sync()
        peak = ev.peak_bytes()
        del warm
        self.packed = pack_input(net, plan, example, ctx)      # the buffers the graph reads
        ev.sync()
        # the arena's extents split and coalesce, so the walk's peak plus a margin holds it;
        # a walk that still outgrows it is captured again with a larger arena
        for attempt in range(3):
            ev.capture_begin(int(peak * arena_margin * (1 << attempt)) + (64 << 20))
            err = None
            try:
                self.result = run_encrypted(net, plan, weights, None, ctx=ctx, packed=self.packed, decrypt=False,
                                            mask_fc=mask_fc)
            except Exception as e:          # noqa: BLE001 - re-raised below unless it is the arena
                err = e
            finally:
                try:
                    self.graph = ev.capture_end()
                except Exception:           # noqa: BLE001 - the walk's own error is the one to report
                    if err is None:
                        raise
            if err is None:
                break
            if "arena exhausted" not in str(err) or attempt == 2:
                raise err
        self.nodes = self.graph.nodes(ev)

    def replay(self, packed=None):
        """Run the captured walk on `packed` (same shape as the example's), or again
        on the current contents of the captured input; returns the encrypted value."""
        ev = self.ctx.evaluator
        if packed is not None:
            for dst, src in zip(_packed_cts(self.packed), _packed_cts(packed)):
                ev.copy(src.handle, dst.handle)
        ev.launch(self.graph)
        return self.result.value

    def run(self, images):
        """Host images -> encrypt -> replay -> decrypted logits."""
        self.replay(pack_input(self.net, self.plan, images, self.ctx))
        return _logits(self.result.value, self.ctx)


def _switch_value(value, ctx, level: int):
    """Modulus-switch every ciphertext of a packed value down to `level` (uncounted,
    as in hesim.HeContext.mod_switch)."""
    def down(ct):
        while ct.tracked and ct.handle.level > level:
            ct = ctx.mod_switch(ct)
        return ct
    if isinstance(value, DensePacked):
        return DensePacked(down(value.ct), value.shape)
    if isinstance(value, ChannelPacked):
        return ChannelPacked(tuple(down(c) for c in value.cts), value.spatial)
    from .packing import ConvPacked
    if isinstance(value, ConvPacked):
        return ConvPacked(tuple(down(c) for c in value.cts), value.spatial)
    return value


def _run_ffconv(step, value, ws, ctx):
    w1, w2 = _ff_w(ws, step.layer_index)
    pat = step.pattern
    if pat in ("DP-HI2C-CP", "CP-HI2C-CP"):
        return factored_conv(value, w1, w2, step.kernel, pat, ctx)
    rank_k = KernelSpec(step.kernel.d, step.kernel.stride, step.rank)
    one = KernelSpec(1, 1, step.kernel.out_channels)
    if pat == "DP-DP":
        mid, p1 = conv_dense(value, w1, rank_k, ctx)
        out, p2 = conv_dense(mid, w2, one, ctx)
        names = ["w1-dots", "w1-assembly", "w2-dots", "w2-assembly"]
        return out, [type(p)(n, p.counters) for p, n in zip(p1 + p2, names)]
    if pat == "CP-HI2C-DP":
        mid, p1 = conv_conv(value, w1, ctx)
        before = ctx.counters.copy()
        dense_mid = channels_to_dense(mid, ctx)
        comb = ctx.counters - before
        out, p2 = conv_dense(dense_mid, w2, one, ctx)
        from .engine import PhaseCost
        phases = [PhaseCost("w1", p1[0].counters), PhaseCost("mid-combine", comb),
                  PhaseCost("w2-dots", p2[0].counters), PhaseCost("w2-assembly", p2[1].counters)]
        return out, phases
    raise ValueError(f"unknown factorized pattern {pat!r}")
