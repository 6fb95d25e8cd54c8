"""Image-parallel execution across ranks (one process per GPU).

The path has no exchange step: images shard contiguously by
rank and every rank evaluates its shard independently.  Collectives are used
only at the ends of the job, as the north_star prescribes:

* scatter: rank 0 (the client, which holds the input images) encrypts every
  rank's input batch and sends the ciphertext words; ranks r > 0 import them;
* gather: ranks send their encrypted logits back; rank 0 decrypts.

Transfers go through torch.distributed point-to-point ops on tensors that alias
the ciphertext words -- device tensors over NCCL (NVLink) on GPUs, host tensors
over gloo in the CPU tests.  Each end is one batched exchange
(`batch_isend_irecv`): rank 0's sends to all ranks are in flight together.
All ranks derive keys from the same seed (`shared_seed`, checked by
`check_shared_keys`), so every rank's evaluation keys match the client's secret.
"""

from __future__ import annotations

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) of `total` items for `rank`; sizes differ by <= 1."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _words_tensor(ev, ct, device):
    import torch
    return torch.empty(ev.words(ct), dtype=torch.int64, device=device)


def _stream_sync(device):
    """NCCL ops run on torch's current stream; the library copies on its own
    stream, so order them explicitly (no-op for CPU tensors / gloo)."""
    import torch
    if str(device).startswith("cuda"):
        torch.cuda.current_stream(torch.device(device)).synchronize()


def shared_seed(rank: int, world: int) -> int:
    """A fresh random key seed drawn by rank 0 (the client) and broadcast, so every
    rank regenerates the client's evaluation keys.  (Every rank that holds the seed
    can also derive the secret key: this harness trades that for on-GPU key
    regeneration.)"""
    import secrets
    import torch.distributed as dist
    obj = [secrets.randbits(64) if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    return int(obj[0])


def check_shared_keys(ctx, world: int) -> None:
    """Raise unless every rank's context derives its keys from the same seed."""
    import torch.distributed as dist
    if world <= 1 or getattr(ctx, "_keys_shared", False):
        return
    seeds = [None] * world
    dist.all_gather_object(seeds, int(ctx.evaluator.params.seed))
    if len(set(seeds)) != 1:
        raise ValueError("ranks use different key seeds; build every rank's parameters with shared_seed()")
    ctx._keys_shared = True                      # checked once per context


def _cts_of(packed):
    from .packing import ChannelPacked, ConvPacked, DensePacked
    if isinstance(packed, DensePacked):
        return [packed.ct]
    if isinstance(packed, (ConvPacked, ChannelPacked)):
        return list(packed.cts)
    raise TypeError(f"not a packed tensor: {type(packed)!r}")


def _exchange(pairs, device):
    """Run (op, tensor, peer) point-to-point transfers as one batch (NCCL groups
    them, so all ranks' transfers are in flight together)."""
    import torch.distributed as dist
    if not pairs:
        return
    ops = [dist.P2POp(dist.isend if op == "send" else dist.irecv, t, peer) for op, t, peer in pairs]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    _stream_sync(device)


def _template(net, plan, ctx):
    """Packed-input shapes of the plan's first step without encrypting anything."""
    from .packing import conv_pack, dense_pack
    from .planner import PACK_DENSE
    step = plan.steps[0]
    zeros = np.zeros((step.in_shape.c, step.in_shape.h, step.in_shape.w), dtype=np.int64)
    if step.op == PACK_DENSE:
        return dense_pack(zeros, ctx, tracked=False)
    ow, oh = step.kernel.out_dims(step.in_shape)
    return conv_pack(np.zeros((ow * oh, step.kernel.k_columns(step.in_shape.c)), dtype=np.int64), ctx,
                     (ow, oh), tracked=False)


def scatter_packed(net, plan, ctx, images, rank: int, world: int, device):
    """Rank 0 (the client) packs and encrypts each rank's image batch and sends the
    ciphertext words to it, all ranks' transfers in one batched exchange; returns
    this rank's packed input.  `images`: the whole job on rank 0, ignored
    elsewhere.  Every rank's batch must have ctx.batch images."""
    from .packing import ConvPacked, DensePacked
    from .runner import pack_input
    check_shared_keys(ctx, world)
    ev = ctx.evaluator
    if rank == 0:
        mine, pairs = None, []
        for r in range(world):
            lo, hi = shard_range(len(images), r, world)
            packed = pack_input(net, plan, images[lo:hi], ctx)
            if r == 0:
                mine = packed
                continue
            for c in _cts_of(packed):
                buf = _words_tensor(ev, c.handle, device)
                ev.export_words(c.handle, buf.data_ptr())
                pairs.append(("send", buf, r))
        _exchange(pairs, device)
        return mine
    template = _template(net, plan, ctx)
    hs, pairs = [], []
    for _ in _cts_of(template):
        h = ev.new_ct(ctx.rows, ev.L)
        buf = _words_tensor(ev, h, device)
        hs.append((h, buf))
        pairs.append(("recv", buf, 0))
    _exchange(pairs, device)
    for h, buf in hs:
        ev.import_words(h, buf.data_ptr())
    cts = [ctx._wrap(h, 0) for h, _ in hs]
    if isinstance(template, DensePacked):
        return DensePacked(cts[0], template.shape)
    return ConvPacked(tuple(cts), template.spatial)


def gather_logits(ctx, value, rank: int, world: int, device):
    """Every rank sends its encrypted logits to rank 0 in one batched exchange;
    rank 0 decrypts them all.  Returns the (images, outputs) logits on rank 0 (in
    shard order), None elsewhere."""
    from .packing import ChannelPacked, DensePacked
    from .runner import _logits
    ev = ctx.evaluator
    cts = _cts_of(value)
    if rank != 0:
        pairs = []
        for c in cts:
            buf = _words_tensor(ev, c.handle, device)
            ev.export_words(c.handle, buf.data_ptr())
            pairs.append(("send", buf, 0))
        _exchange(pairs, device)
        return None
    incoming, pairs = [], []
    for r in range(1, world):
        got = []
        for c in cts:
            h = ev.new_ct(ctx.rows, c.handle.level)
            buf = _words_tensor(ev, h, device)
            got.append((h, buf, c))
            pairs.append(("recv", buf, r))
        incoming.append(got)
    _exchange(pairs, device)
    parts = [np.atleast_2d(_logits(value, ctx))]
    for got in incoming:
        wrapped = []
        for h, buf, c in got:
            ev.import_words(h, buf.data_ptr())
            wrapped.append(ctx._wrap(h, c.depth, c.assembly_depth))
        other = (ChannelPacked(tuple(wrapped), value.spatial) if isinstance(value, ChannelPacked)
                 else DensePacked(wrapped[0], value.shape))
        parts.append(np.atleast_2d(_logits(other, ctx)))
    return np.concatenate(parts, axis=0)
