"""Image-parallel execution across ranks (one process per GPU).

The path has no exchange step: images shard contiguously by
rank and every rank evaluates its shard independently.  Collectives are used
only at the ends of the job, as the north_star prescribes:

* scatter: rank 0 (the client, which holds the input images) encrypts every
  rank's input batch and sends the ciphertext words; ranks r > 0 import them;
* gather: ranks send their encrypted logits back; rank 0 decrypts.

Transfers go through torch.distributed point-to-point ops on tensors that alias
the ciphertext words -- device tensors over NCCL (NVLink) on GPUs, host tensors
over gloo in the CPU tests.  All ranks derive keys from the same seed, so every
rank's evaluation keys match the client's secret.
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


def send_ct(ev, ct, dst: int, device):
    import torch.distributed as dist
    buf = _words_tensor(ev, ct, device)
    ev.export_words(ct, buf.data_ptr())        # synchronous on the library stream
    dist.send(buf, dst)


def recv_ct(ev, rows: int, level: int, src: int, device):
    import torch.distributed as dist
    ct = ev.new_ct(rows, level)
    buf = _words_tensor(ev, ct, device)
    dist.recv(buf, src)
    _stream_sync(device)                       # the received words must land before the copy-in
    ev.import_words(ct, buf.data_ptr())
    return ct


def scatter_packed(net, plan, ctx, images, rank: int, world: int, device):
    """Rank 0 packs (encrypts) each rank's image batch and sends it; returns this
    rank's packed input.  `images`: the whole job on rank 0, ignored elsewhere.
    Every rank's batch must have ctx.batch images."""
    from .packing import ConvPacked, DensePacked
    from .runner import pack_input
    ev = ctx.evaluator
    if rank == 0:
        mine = None
        for r in range(world):
            lo, hi = shard_range(len(images), r, world)
            packed = pack_input(net, plan, images[lo:hi], ctx)
            if r == 0:
                mine = packed
                continue
            cts = [packed.ct] if isinstance(packed, DensePacked) else list(packed.cts)
            for c in cts:
                send_ct(ev, c.handle, r, device)
        return mine
    step = plan.steps[0]
    template = pack_input(net, plan, np.zeros((ctx.batch,) + (step.in_shape.c, step.in_shape.h, step.in_shape.w),
                                              dtype=np.int64), ctx)
    if isinstance(template, DensePacked):
        h = recv_ct(ev, ctx.rows, ev.L, 0, device)
        return DensePacked(ctx._wrap(h, 0), template.shape)
    cts = tuple(ctx._wrap(recv_ct(ev, ctx.rows, ev.L, 0, device), 0) for _ in template.cts)
    return ConvPacked(cts, template.spatial)


def gather_logits(ctx, value, rank: int, world: int, device):
    """Every rank sends its encrypted logits to rank 0, which decrypts them all.
    Returns the (images, outputs) logits on rank 0 (in shard order), None elsewhere."""
    from .packing import ChannelPacked, DensePacked
    from .runner import _logits
    ev = ctx.evaluator
    cts = list(value.cts) if isinstance(value, ChannelPacked) else [value.ct]
    if rank != 0:
        for c in cts:
            send_ct(ev, c.handle, 0, device)
        return None
    parts = [np.atleast_2d(_logits(value, ctx))]
    for r in range(1, world):
        got = [ctx._wrap(recv_ct(ev, ctx.rows, c.handle.level, r, device), c.depth, c.assembly_depth)
               for c in cts]
        other = (ChannelPacked(tuple(got), value.spatial) if isinstance(value, ChannelPacked)
                 else DensePacked(got[0], value.shape))
        parts.append(np.atleast_2d(_logits(other, ctx)))
    return np.concatenate(parts, axis=0)
