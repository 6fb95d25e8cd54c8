"""Layer evaluation over packed ciphertexts.

Mirror of `cipherpack.engine` (/root/reference/pkg/src/cipherpack/engine.py):
same functions, arguments, phase names and exact operation counts.  Two things
are organised for the GPU:

* independent primitives of one layer are issued as batches (all dot products
  of an output channel share one ct x pt launch sequence and one key-switching
  launch sequence per rotate-and-sum level) through the context's `*_many`
  forms; with a context that lacks them (e.g. the reference's own HeContext or
  the slot oracle) the same code issues them one by one;
* conv_conv multiplies by the weight as a constant (`ctx.mul_scalar`) instead of
  a masked constant plaintext: ConvPacked columns are zero past the S rows
  (packing.py:96-98), so the decrypted slots are identical, the noise growth is
  ~log2|w| bits instead of ~log2(t sqrt(n)), and no plaintext is encoded.

FC outputs that feed a combine are masked to slot 0 (`mask_outputs`), the fix
for the reference's FC -> FC divergence (engine.py:241-260 leaves
partial sums in slots >= 1 that combine_to_dense then adds into the payload).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .hesim import OpCounters, rotations_for_span
from .packing import (
    ChannelPacked,
    ConvPacked,
    DensePacked,
    KernelSpec,
    _add_many,
    _mul_plain_many,
    _rotate_multi,
    combine_to_dense,
    h_grouping,
    source_slots,
    tree_combine,
)


@dataclass(frozen=True)
class WeightMatrix:
    """K x O_c quantized weights; real value = entry * scale (engine.py:46-66)."""

    entries: np.ndarray
    bits: int = 8
    scale: float = 1.0

    def __post_init__(self):
        if self.entries.ndim != 2:
            raise ValueError("weight matrix must be 2D")
        if self.entries.size and int(np.max(np.abs(self.entries.astype(object)))) >= 2 ** (self.bits - 1):
            raise ValueError(f"entries exceed {self.bits}-bit signed range")

    @property
    def k(self) -> int:
        return self.entries.shape[0]

    @property
    def out_channels(self) -> int:
        return self.entries.shape[1]


@dataclass(frozen=True)
class BiasVector:
    entries: np.ndarray
    scale: float = 1.0


@dataclass(frozen=True)
class PhaseCost:
    name: str
    counters: OpCounters


def _phase(ctx, name: str, before) -> PhaseCost:
    return PhaseCost(name, ctx.counters - before)


def _plain(ctx, tracked: bool, fill):
    if not tracked:
        return None
    buf = np.zeros(ctx.params.n_slots, dtype=np.int64)
    fill(buf)
    return ctx.encode(buf)


def _scatter_plain(ctx, indices, values, tracked: bool):
    def fill(b):
        b[indices] = values
    return _plain(ctx, tracked, fill)


def _prefix_values(ctx, values, tracked: bool):
    def fill(b):
        b[: len(values)] = values
    return _plain(ctx, tracked, fill)


def _slot0_mask(ctx, tracked: bool):
    def fill(b):
        b[0] = 1
    return _plain(ctx, tracked, fill)


def _rotate_and_sum_many(ctx, cts, m: int):
    if hasattr(ctx, "rotate_and_sum_many"):
        return ctx.rotate_and_sum_many(cts, m)
    return [ctx.rotate_and_sum(c, m) for c in cts]


# --------------------------------------------------------------- dense style

def _group_size(ctx) -> int:
    """How many independent outputs to keep in flight (device memory bound)."""
    return max(1, int(getattr(ctx, "group_size", 1 << 30)))


def _dense_dots(x: DensePacked, w: WeightMatrix, kernel: KernelSpec, ctx, o: int, s0: int, s1: int, hoist=None):
    """Dot products of outputs (o, s0..s1-1): scatter the filter column to each
    patch, multiply, rotate-and-sum over the occupied span; result in slot 0
    (engine.py:104-121)."""
    idx = source_slots(x.shape, kernel)
    if w.k != idx.shape[1]:
        raise ValueError(f"weight matrix has {w.k} rows, kernel needs {idx.shape[1]}")
    col = w.entries[:, o]
    tracked = x.ct.tracked
    pvs = [_scatter_plain(ctx, idx[s], col, tracked) for s in range(s0, s1)]
    return _products_and_sums(ctx, x.ct, pvs, x.occupied, hoist)


# cost of one ct x pt GEMM term relative to one key-switched rotation of the same
# ciphertext (2 l n MACs vs (l^2 + 3l + 2) n-point NTTs): conservatively 1/64
GEMM_TERM_COST = 1.0 / 64


def hoist_depth(outputs: int, rounds: int, max_levels: int) -> int:
    """Tree levels to hoist for `outputs` trees over one input: maximise the
    rotations saved (outputs * h) minus the input rotations (2^h - 1) and the
    extra GEMM terms (outputs * (2^h - 1) * GEMM_TERM_COST)."""
    best, best_gain = 0, 0.0
    for h in range(1, min(max_levels, rounds) + 1):
        gain = outputs * h - (2 ** h - 1) - outputs * (2 ** h - 1) * GEMM_TERM_COST
        if gain > best_gain:
            best, best_gain = h, gain
    return best


class _Hoist:
    """Rotations of one shared input by every subset sum of the top h steps of a
    rotate-and-sum tree, computed once per layer and reused by all its outputs."""

    def __init__(self, ctx, ct, m: int, outputs: int):
        r = (m - 1).bit_length()
        self.h = hoist_depth(outputs, r, int(getattr(ctx, "hoist_levels", 7)))
        self.tail = [1 << i for i in reversed(range(r - self.h))]      # remaining steps, largest first
        ks = [0]
        for i in range(self.h):
            step = 1 << (r - 1 - i)
            ks = ks + [k + step for k in ks]
        self.ks = ks
        if len(ks) <= 1:
            rot = []
        elif hasattr(ctx, "rotate_hoisted"):          # one shared ModUp for all of them
            rot = ctx.rotate_hoisted(ct, ks[1:])
        else:
            rot = _rotate_multi(ctx, [ct] * (len(ks) - 1), ks[1:])
        self.rotated = [ct] + list(rot)


def _hoisted(ctx) -> bool:
    return getattr(ctx, "schedule", "reference") == "hoisted" and hasattr(ctx, "hoisted_dot")


def level_down(ctx, cts, extra_bits: float):
    """Level schedule inside a plan step (HeContext(level_schedule=True)): the runner
    records the model's noise consumption before the step (ctx.noise_consumed); once
    the step's own operations so far (`extra_bits`) let the budget absorb dropping
    q primes, the ciphertexts are modulus-switched before the rotation-heavy part."""
    if not getattr(ctx, "level_schedule", False) or getattr(ctx, "noise_consumed", None) is None:
        return cts
    cts = list(cts)
    if not cts or not cts[0].tracked:
        return cts
    from .runner import _target_level
    ev = ctx.evaluator
    target = _target_level(ev.params.q, ev.L, ctx.noise_consumed + extra_bits)
    out = []
    for c in cts:
        while c.handle.level > target:
            c = ctx.mod_switch(c)
        out.append(c)
    return out


def _t_bits(ctx) -> float:
    import math
    return math.log2(max(ctx.params.factors())) if hasattr(ctx.params, "factors") else 0.0


def _products_and_sums(ctx, ct, pvs, m: int, hoist):
    """rotate_and_sum(ct * pv, m) for every pv.  Reference schedule: one product
    and ceil(log2 m) rotate-add levels each.  Hoisted schedule: the top h levels of
    every tree as one ct x pt GEMM over the shared input's rotations."""
    if hoist is None or hoist.h == 0:
        prods = level_down(ctx, _mul_plain_many(ctx, [ct] * len(pvs), pvs), _t_bits(ctx) + 8)
        return _rotate_and_sum_many(ctx, prods, m)
    outs = ctx.hoisted_dot(hoist.rotated, hoist.ks, pvs)
    for step in hoist.tail:
        outs = ctx._rotate_add_many(outs, step)
    return outs


def _mask_slot0_many(ctx, cts):
    tracked = bool(cts) and cts[0].tracked
    mask = _slot0_mask(ctx, tracked)
    return _mul_plain_many(ctx, cts, [mask] * len(cts), assembly=True)


def _dense_assemble(x, w, kernel, ctx, blocks):
    """Dot products + slot-0 masks + combine, in output groups so that only a
    bounded number of per-output ciphertexts is alive.  `blocks` lists the
    output ranges (start, stop) that are combined into one ciphertext each,
    in output order.  Every ciphertext equals the one the reference's phase
    order (all dots, then all masks, then the combines) produces; the phase
    counters are accumulated separately."""
    n = ctx.params.n_slots
    rows = len(source_slots(x.shape, kernel))       # outputs per channel
    g = _group_size(ctx)
    hoist = None
    dots, asm = OpCounters(), OpCounters()
    results = []
    for b0, b1 in blocks:
        acc = None
        s0 = b0
        while s0 < b1:
            o = s0 // rows
            s1 = min(b1, (o + 1) * rows, s0 + g)
            before = ctx.counters.copy()
            if hoist is None and _hoisted(ctx) and x.ct.tracked:
                hoist = _Hoist(ctx, x.ct, x.occupied, w.out_channels * rows)
            outs = _dense_dots(x, w, kernel, ctx, o, s0 - o * rows, s1 - o * rows, hoist)
            dots = dots + (ctx.counters - before)
            before = ctx.counters.copy()
            masked = level_down(ctx, _mask_slot0_many(ctx, outs), 2 * _t_bits(ctx) + 17)   # dot + mask
            # the group's outputs as one contiguous block (tree: log2 keys), then placed
            # at its offset in the block: len - 1 + 1 rotations, as the chain's
            group, _ = tree_combine(ctx, masked, [1] * len(masked))
            if acc is None:
                acc = group
            else:
                acc = ctx.add_cc(acc, ctx.rotate(group, (n - (s0 - b0)) % n))
            asm = asm + (ctx.counters - before)
            s0 = s1
        results.append(acc)
    return results, PhaseCost("dot-products", dots), PhaseCost("assembly", asm)


def conv_dense(x: DensePacked, w: WeightMatrix, kernel: KernelSpec, ctx):
    """Dense in, dense out.  Dot phase (O, O*r, O*r); assembly: O masks plus
    O-1 rotations/additions (engine.py:133-151)."""
    total = w.out_channels * len(source_slots(x.shape, kernel))
    if total > ctx.params.n_slots:
        raise ValueError(f"{total} outputs exceed {ctx.params.n_slots} slots")
    (ct,), dots, asm = _dense_assemble(x, w, kernel, ctx, [(0, total)])
    return DensePacked(ct, kernel.out_shape(x.shape)), [dots, asm]


def conv_dense_to_channels(x: DensePacked, w: WeightMatrix, kernel: KernelSpec, ctx):
    """Dense in, one ciphertext per output channel; assembly O masks and O - O_c
    rotations/additions (engine.py:154-171)."""
    ow, oh = kernel.out_dims(x.shape)
    rows = ow * oh
    blocks = [(o * rows, (o + 1) * rows) for o in range(w.out_channels)]
    chans, dots, asm = _dense_assemble(x, w, kernel, ctx, blocks)
    return ChannelPacked(tuple(chans), (ow, oh)), [dots, asm]


# -------------------------------------------------------------- column style

def conv_conv(x: ConvPacked, w: WeightMatrix, ctx):
    """Output channel o = sum_k w[k, o] * column_k; exactly (O_c*K, O_c*(K-1), 0)
    (engine.py:178-197)."""
    if w.k != x.k:
        raise ValueError(f"weight matrix has {w.k} rows but input has {x.k} columns")
    before = ctx.counters.copy()
    if hasattr(ctx, "ct_gemm"):
        # one ct-GEMM pass: every column is read once per tile of outputs (fhe_ct_gemm)
        outs = ctx.ct_gemm(list(x.cts), [[int(w.entries[k, o]) for o in range(w.out_channels)] for k in range(x.k)])
        if outs is not None:
            return ChannelPacked(tuple(outs), x.spatial), [_phase(ctx, "channel-sums", before)]
    chans = []
    for o in range(w.out_channels):
        terms = [_scalar_term(ctx, x, k, int(w.entries[k, o])) for k in range(x.k)]
        acc = terms[0]
        for term in terms[1:]:
            acc = ctx.add_cc(acc, term)
        chans.append(acc)
    return ChannelPacked(tuple(chans), x.spatial), [_phase(ctx, "channel-sums", before)]


def _scalar_term(ctx, x: ConvPacked, k: int, value: int):
    ct = x.cts[k]
    if hasattr(ctx, "mul_scalar"):
        return ctx.mul_scalar(ct, value)
    # contexts without a constant multiply: the reference's masked constant plaintext
    pv = _prefix_values(ctx, [value] * x.rows, ct.tracked)
    return ctx.mul_plain(ct, pv)


# ------------------------------------------------------------ factorized layer

FACTORIZED_PATTERNS = ("DP-HI2C-CP", "CP-HI2C-CP")


def factored_conv(x, w1: WeightMatrix, w2: WeightMatrix, kernel: KernelSpec, pattern: str, ctx):
    """Two-stage low-rank convolution, two multiplicative levels (engine.py:207-234)."""
    if w1.out_channels != w2.k:
        raise ValueError("factor ranks do not line up")
    transition = KernelSpec(d=1, stride=1, out_channels=w2.out_channels)
    if pattern == "DP-HI2C-CP":
        if not isinstance(x, DensePacked):
            raise ValueError("DP-HI2C-CP needs a dense input")
        ch1, ph1 = conv_dense_to_channels(x, w1, kernel, ctx)
    elif pattern == "CP-HI2C-CP":
        if not isinstance(x, ConvPacked):
            raise ValueError("CP-HI2C-CP needs a column-packed input")
        ch1, ph1 = conv_conv(x, w1, ctx)
    else:
        raise ValueError(f"unsupported pattern {pattern!r}; expected one of {FACTORIZED_PATTERNS}")
    ch2, ph2 = conv_conv(h_grouping(ch1, transition), w2, ctx)
    return ch2, ([PhaseCost(f"w1-{p.name}", p.counters) for p in ph1]
                 + [PhaseCost(f"w2-{p.name}", p.counters) for p in ph2])


# ----------------------------------------------------- fc, pooling, activation

def fc_dense(x: DensePacked, w: WeightMatrix, bias: BiasVector | None, ctx, mask_outputs: bool = False):
    """Row-major matrix-vector product: per output one plaintext multiply and a
    rotate-and-sum, bias added as a free constant (engine.py:241-260).  With
    mask_outputs each result is then masked to slot 0 (assembly ledger)."""
    m = x.occupied
    if w.k != m:
        raise ValueError(f"weight matrix has {w.k} rows but payload is {m}")
    if bias is not None and bias.entries.shape[0] != w.out_channels:
        raise ValueError("bias length does not match output count")
    tracked = x.ct.tracked
    g = _group_size(ctx)
    rows, masks = OpCounters(), OpCounters()
    outs = []
    hoist = None
    for o0 in range(0, w.out_channels, g):
        o1 = min(w.out_channels, o0 + g)
        before = ctx.counters.copy()
        if hoist is None and _hoisted(ctx) and tracked:
            hoist = _Hoist(ctx, x.ct, m, w.out_channels)
        pvs = [_prefix_values(ctx, w.entries[:, o], tracked) for o in range(o0, o1)]
        red = _products_and_sums(ctx, x.ct, pvs, m, hoist)
        if bias is not None:
            red = [ctx.add_plain(r, _scatter_plain(ctx, [0], [int(bias.entries[o])], tracked))
                   for o, r in zip(range(o0, o1), red)]
        rows = rows + (ctx.counters - before)
        if mask_outputs:
            before = ctx.counters.copy()
            red = level_down(ctx, _mask_slot0_many(ctx, red), 2 * _t_bits(ctx) + 17)
            masks = masks + (ctx.counters - before)
        outs.extend(red)
    phases = [PhaseCost("row-products", rows)]
    if mask_outputs:
        phases.append(PhaseCost("slot0-masks", masks))
    return outs, phases


def avg_pool_weights(window: KernelSpec, channels: int) -> WeightMatrix:
    """Pooling as a constant-1 convolution per channel (engine.py:271-279)."""
    k = window.d * window.d
    entries = np.zeros((k * channels, channels), dtype=np.int64)
    for ch in range(channels):
        entries[ch * k:(ch + 1) * k, ch] = 1
    return WeightMatrix(entries=entries, bits=2, scale=1.0 / k)


def square_layer(x, ctx):
    """Slot-wise square of every constituent ciphertext (engine.py:282-295)."""
    before = ctx.counters.copy()
    if isinstance(x, DensePacked):
        out = DensePacked(ctx.square(x.ct), x.shape)
    elif isinstance(x, ChannelPacked):
        out = ChannelPacked(tuple(ctx.square(c) for c in x.cts), x.spatial)
    elif isinstance(x, ConvPacked):
        out = ConvPacked(tuple(ctx.square(c) for c in x.cts), x.spatial)
    else:
        raise TypeError(f"not a packed tensor: {type(x)!r}")
    return out, [_phase(ctx, "square", before)]


def packed_depth(x) -> tuple[int, int]:
    """(depth, assembly_depth), max over ciphertexts (engine.py:298-310)."""
    if isinstance(x, DensePacked):
        cts = [x.ct]
    elif isinstance(x, (ChannelPacked, ConvPacked)):
        cts = list(x.cts)
    elif isinstance(x, (list, tuple)):
        cts = list(x)
    elif hasattr(x, "depth"):
        cts = [x]
    else:
        raise TypeError(f"not a packed tensor: {type(x)!r}")
    return max(c.depth for c in cts), max(c.assembly_depth for c in cts)


__all__ = [
    "WeightMatrix", "BiasVector", "PhaseCost", "conv_dense", "conv_dense_to_channels", "conv_conv",
    "factored_conv", "fc_dense", "avg_pool_weights", "square_layer", "packed_depth", "rotations_for_span",
    "FACTORIZED_PATTERNS",
]
