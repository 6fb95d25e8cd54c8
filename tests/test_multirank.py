"""The N > 1 path on CPU: world_size 2 over gloo, golden model as the backend.

Rank 0 encrypts both ranks' images and scatters the ciphertext words, each rank
evaluates its shard, rank 0 gathers the encrypted logits and decrypts; the
result must equal the reference's logits for every image (networks.json)."""

import json
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2102_03494_b200.shard import shard_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_range_partitions():
    for total in (1, 7, 256, 1000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def _worker(rank, world, port, out_path, golden_path):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2102_03494_b200.abi import Library
    from paper_2102_03494_b200.hesim import HeContext
    from paper_2102_03494_b200.planner import build_plan
    from paper_2102_03494_b200.runner import run_encrypted
    from paper_2102_03494_b200.shard import gather_logits, scatter_packed, shared_seed
    from _shared import load, network_from_fixture
    fx = load("networks.json")[0]
    net, ws = network_from_fixture(fx, seed=shared_seed(rank, world))
    plan = build_plan(net, "explicit")
    images = np.concatenate([np.array(fx["inputs"])] * world)        # 2 images per rank
    ctx = HeContext(net.scheme, batch=2, lib=Library(golden_path))
    packed = scatter_packed(net, plan, ctx, images if rank == 0 else None, rank, world, "cpu")
    res = run_encrypted(net, plan, ws, None, ctx=ctx, packed=packed, decrypt=False)
    logits = gather_logits(ctx, res.value, rank, world, "cpu")
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump([[int(v) for v in row] for row in logits], fh)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_gloo(world, tmp_path, golden_lib):
    out = tmp_path / "logits.json"
    port = 29500 + (os.getpid() * 7 + world) % 1000
    mp.spawn(_worker, args=(world, port, str(out), golden_lib.path), nprocs=world, join=True)
    from _shared import load
    fx = load("networks.json")[0]
    got = json.loads(out.read_text())
    assert got == fx["logits"] * world


def _mismatch_worker(rank, world, port, out_path):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2102_03494_b200.shard import check_shared_keys

    class _Ev:
        class params:
            seed = 1000 + rank

    class _Ctx:
        evaluator = _Ev()

    try:
        check_shared_keys(_Ctx(), world)
        msg = "no error"
    except ValueError as e:
        msg = str(e)
    if rank == 0:
        with open(out_path, "w") as fh:
            fh.write(msg)
    dist.destroy_process_group()


def test_ranks_with_different_key_seeds_are_rejected(tmp_path):
    out = tmp_path / "msg.txt"
    port = 28500 + os.getpid() % 1000
    mp.spawn(_mismatch_worker, args=(2, port, str(out)), nprocs=2, join=True)
    assert "different key seeds" in out.read_text()
