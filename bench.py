#!/usr/bin/env python
"""Benchmark driver (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload rotation|inference]

Workloads (BASELINE.json configs):
  rotation   configs[1]: ring 2^14, 4 x ~40-bit q primes + 1 special prime, a batch
             of 1024 ciphertexts per GPU with slot values uniform in {-1,0,1},
             t = 1099511922689.  A step = one key-switched rotation of every
             ciphertext by a seeded step k in [1, 8192).  Also reported: ct x pt
             multiply-accumulate and rescale (modulus switch) rates.
  inference  configs[2]: the FFConv MNIST-shaped network on synthetic images,
             sharded image-wise across ranks (added with the host stack).

`value` is device-timed (CUDA events on the library's stream, max over ranks);
`e2e` is the same metric through the public API from pinned host slot vectors
(encrypt -> rotate -> decrypt, host<->device copies inside the timed region).
--impl reference times the reference's own CPU algorithm for the path (the
numpy port in oracle/slot_oracle.py, all host cores) on the same config.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG1 = dict(n_slots=8192, t=1099511922689, L=4, q_bits=40, batch=1024, seed=20210205)


# ------------------------------------------------------------------ helpers
def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def rotation_params():
    from paper_2102_03494_b200.params import RlweParams, ntt_primes
    two_n = 4 * CFG1["n_slots"]
    t = CFG1["t"]
    q = ntt_primes(CFG1["q_bits"], CFG1["L"], two_n, exclude=[t])
    p = ntt_primes(CFG1["q_bits"] + 2, 1, two_n, exclude=[t] + q)
    return RlweParams(log_n=14, q=tuple(q), p=tuple(p), t=(t,), b=(), seed=CFG1["seed"])


def rotation_config(world: int) -> dict:
    """configs[1] workload identity, printed by both arms."""
    P = rotation_params()
    return {"workload": "configs[1] primitive microbench: 1024 ciphertexts per GPU, one seeded rotation "
                        "step per batch", "ring_n": P.n, "L": P.L, "K": 1, "dnum": P.L,
            "q_bits": [round(math.log2(x), 2) for x in P.q], "t": P.t[0], "batch_per_gpu": CFG1["batch"],
            "rotation_step": rotation_step(), "l2": "inputs 1 GiB per batch > 126 MB L2 (no flush needed)",
            "parallelism": f"dp{world} (independent ciphertexts, no collective)"}


def algorithmic_counts(n: int, l: int):
    """Per-ciphertext algorithmic modmuls / bytes per kernel of one key-switched
    rotation (hybrid KS, one prime per digit, one special prime)."""
    ntt = (n // 2) * int(math.log2(n))
    w = 8
    return {
        "k_rot_gather_intt": (l * ntt, (2 * l * n + 2 * l * n + l * n) * w),
        "k_modup": (l * l * ntt, (l * n + l * l * n) * w),          # read the l digits, write l^2 extended rows
        "k_ks_inner": (2 * l * l * n, (l * l * n + 2 * l * n) * w),
        "k_ks_special": (2 * ntt + 2 * l * n, (2 * l * n + 2 * n) * w),
        "k_rescale(moddown)": (2 * l * ntt + 2 * l * n, (2 * n + 2 * l * n + l * n + 2 * l * n) * w),
    }


def kernel_counts(n: int, l: int):
    """algorithmic_counts plus the fused ModDown (k_moddown = the q primes' inner
    product + the ModDown rescale, the default path)."""
    c = algorithmic_counts(n, l)
    w = 8
    ntt = (n // 2) * int(math.log2(n))
    c["k_moddown"] = (c["k_ks_inner"][0] + c["k_rescale(moddown)"][0],
                      (l * l * n + 2 * n + l * n + 2 * l * n) * w)
    return c


def rotation_modmuls(n, l):
    return sum(v[0] for v in algorithmic_counts(n, l).values())


def rotation_bytes(n, l, batch):
    key = 2 * l * (l + 1) * n * 8
    return 2 * (2 * l * n * 8) + key / batch


def parse_prof(text: str):
    out = {}
    for line in text.strip().splitlines():
        name, calls, ms = line.rsplit(" ", 2)
        out[name] = (int(calls), float(ms))
    return out


# ------------------------------------------------------------- CPU baselines
def _cpu_rotations(args):
    """Reference algorithm (slot oracle) rotations over `count` slot vectors, by the
    configs[1] step.  The vectors are encrypted before the timer starts; only the
    rotations are timed (in this process)."""
    count, reps, seed = args
    from oracle.slot_oracle import Params, SlotContext
    ctx = SlotContext(Params(CFG1["n_slots"], CFG1["t"]))
    rng = np.random.default_rng(seed)
    cts = [ctx.encrypt(rng.integers(-1, 2, size=CFG1["n_slots"])) for _ in range(count)]
    k = rotation_step()
    t0 = time.perf_counter()
    for _ in range(reps):
        cts = [ctx.rotate(c, k) for c in cts]
    return count * reps, time.perf_counter() - t0


def rotation_step() -> int:
    """The configs[1] step: one seeded k in [1, 8192) per batch (same for both arms)."""
    return int(np.random.default_rng(CFG1["seed"]).integers(1, CFG1["n_slots"]))


def cpu_baseline_rotation(cores: int = 1, seconds: float = 2.0):
    """rotations/s of the reference algorithm over the configs[1] batch on `cores`
    processes: each worker rotates its share of the 1024 vectors `reps` times and
    times itself; rate = all rotations / the slowest worker's rotation time."""
    # calibrate reps so the sample is a bounded amount of CPU work
    n, dt = _cpu_rotations((64, 1, 1))
    per = dt / n
    count = CFG1["batch"]
    reps = max(1, int(seconds * max(1, cores) / max(per * count, 1e-9)))
    if cores <= 1:
        done, el = _cpu_rotations((count, reps, 7))
        rate = done / el
    else:
        import multiprocessing as mp
        chunk = max(1, count // cores)
        with mp.Pool(cores) as pool:
            res = pool.map(_cpu_rotations, [(chunk, reps, 7 + i) for i in range(cores)])
        rate = sum(r[0] for r in res) / max(r[1] for r in res)
    return rate, (f"{count} slot vectors x {reps} rotation rounds by k = {rotation_step()} (N=8192, "
                  f"t=1099511922689), {max(1, cores)} worker process(es), vectors built before the timer")


# --------------------------------------------------------------- our arm
def run_rotation(args, rank, world, local_rank):
    import torch
    from paper_2102_03494_b200.abi import cuda_library
    from paper_2102_03494_b200.rlwe import Evaluator

    torch.cuda.set_device(local_rank)
    lib = cuda_library()
    P = rotation_params()
    ev = Evaluator(P, lib, device=local_rank)
    stream_ptr = ctypes.c_void_p()
    lib.call("fhe_ctx_stream", ev.ctx, ctypes.byref(stream_ptr))
    stream = torch.cuda.ExternalStream(stream_ptr.value, device=local_rank)

    B = CFG1["batch"]
    n = P.n
    rng = np.random.default_rng(CFG1["seed"] + rank)
    slots = np.mod(rng.integers(-1, 2, size=(1, B, n)), P.t[0]).astype(np.uint64)
    ct = ev.encrypt(slots)
    k = rotation_step()
    pt = ev.encode(np.mod(rng.integers(-1, 2, size=(1, n)), P.t[0]).astype(np.uint64))
    ev.keygen_rotations([k])
    ev.sync()

    # roofline denominator: the faster of the two Shoup forms the library issues
    # (exact quotient; approximate quotient = the NTT butterflies' form)
    peaks = {}
    for kind, name in ((0, "shoup_exact"), (1, "shoup_approx")):
        peak = ctypes.c_double()
        lib.call("fhe_peak_modmul_kind", ev.ctx, 20000, kind, ctypes.byref(peak))
        peaks[name] = peak.value
    peak_modmul = max(peaks.values())

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        ev.sync()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{local_rank}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    holder = {}

    def rot_step():
        holder["r"] = ev.rotate(ct, k)

    cnt0 = ctypes.c_uint64()
    lib.call("fhe_launch_count", ev.ctx, ctypes.byref(cnt0))
    with ClockSampler(local_rank) as clk:
        rot_ms = timed(rot_step, args.steps, args.warmup)
    cnt1 = ctypes.c_uint64()
    lib.call("fhe_launch_count", ev.ctx, ctypes.byref(cnt1))
    launches = int((cnt1.value - cnt0.value) * args.steps / (args.steps + args.warmup))

    # secondary rates: HMA (acc += ct * pt, one fused in-place kernel) and rescale
    acc = {"a": ev.zero(B)}

    def hma_step():
        ev.mul_plain_acc(ct, pt, acc["a"])

    hma_ms = timed(hma_step, args.steps, args.warmup)

    def ms_step():
        holder["m"] = ev.mod_switch(ct)

    resc_ms = timed(ms_step, args.steps, args.warmup)

    # per-kernel live timing (separate pass, same command) for the roofline
    lib.call("fhe_prof_enable", ev.ctx, 1)
    for _ in range(max(1, args.steps)):
        rot_step()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.call("fhe_prof_report", ev.ctx, buf, len(buf))
    lib.call("fhe_prof_enable", ev.ctx, 0)
    prof = parse_prof(buf.value.decode())
    counts = kernel_counts(n, P.L)
    steps_prof = max(1, args.steps)
    kern = {}
    for name, (calls, ms) in prof.items():
        mm, by = counts.get(name, (0, 0))
        kern[name] = {"calls": calls, "ms": ms, "modmul_per_s": mm * B * steps_prof / (ms * 1e-3) if ms else 0.0,
                      "gbs": by * B * steps_prof / (ms * 1e-3) / 1e9 if ms else 0.0}
    dominant = max(kern, key=lambda x: kern[x]["ms"]) if kern else None

    # e2e: host slots -> encrypt -> rotate -> decrypt -> host.  Page-locked buffers make the
    # library's encrypt/decrypt asynchronous (copies on its copy stream), so the batch is
    # issued in chunks whose H2D/D2H overlap the other chunks' evaluation.
    host_in = torch.from_numpy(slots.view(np.int64)).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    in_np, out_np = host_in.numpy().view(np.uint64), host_out.numpy().view(np.uint64)
    e2e_chunks = _env_int("BENCH_E2E_CHUNKS", 4)    # measured: 4 chunks 93.8K, 8 89.5K, 16 83.2K rot/s
    bounds = [(B * i // e2e_chunks, B * (i + 1) // e2e_chunks) for i in range(e2e_chunks)]

    # "overlap" (default): software-pipelined across steps.  Step i's rotate_many is issued first, then
    # step i + 1's chunked encryptions (their H2D copies run on the library's copy stream under step
    # i's key switch; the encryption kernels queue behind it), then step i's decryptions (their D2H
    # copies run under step i + 1's kernels).  Every step still copies its whole input from page-locked
    # host memory and reads its whole result back; prologue and drain are inside the timed region.
    # "phases": all encryptions, one rotate_many, all decryptions, nothing carried across steps.
    # "pipeline": chunk by chunk encrypt -> rotate -> decrypt (measured slowest: 81.7K vs 84.8K rot/s).
    e2e_mode = os.environ.get("BENCH_E2E_MODE", "overlap")

    def enc_chunks():
        return [ev.encrypt(in_np[:, r0:r1], async_=True) for r0, r1 in bounds]

    def dec_chunks(rs):
        for (r0, r1), r in zip(bounds, rs):
            ev.decrypt(r, out=out_np[:, r0:r1], async_=True)

    def e2e_run(steps):
        if e2e_mode == "overlap":
            cs = enc_chunks()
            for i in range(steps):
                rs = ev.rotate_many(cs, k)             # one key-switching launch sequence
                cs = enc_chunks() if i + 1 < steps else None
                dec_chunks(rs)
            return
        for _ in range(steps):
            if e2e_mode == "phases":
                dec_chunks(ev.rotate_many(enc_chunks(), k))
                continue
            for r0, r1 in bounds:
                c = ev.encrypt(in_np[:, r0:r1], async_=True)
                ev.decrypt(ev.rotate(c, k), out=out_np[:, r0:r1], async_=True)

    def e2e_timed(steps):
        e2e_run(2)
        ev.sync()
        out_np[...] = 0
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e2e_run(steps)
        ev.sync()
        s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([s], device=f"cuda:{local_rank}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            s = float(t.item())
        return s

    e2e_steps = max(1, min(args.steps, 10))
    e2e_s = e2e_timed(e2e_steps)
    e2e_serial = None
    if e2e_mode == "overlap":                          # the unpipelined figure beside it
        e2e_mode = "phases"
        e2e_serial = world * B * e2e_steps / e2e_timed(e2e_steps)
        e2e_mode = "overlap"

    # the e2e output is the rotated input, slot for slot (both rows)
    N = P.n_slots
    exp = np.concatenate([np.roll(slots[0, :4, :N], -k, axis=-1), np.roll(slots[0, :4, N:], -k, axis=-1)], axis=-1)
    e2e_ok = bool(np.array_equal(out_np[0, :4], exp))
    rot_rate = world * B * args.steps / (rot_ms * 1e-3)
    per_rot_mm = rotation_modmuls(n, P.L)
    result = {
        "metric": "key-switched rotations/s (ring 2^14, 4x40-bit q + 1 special prime, hybrid KS)",
        "value": rot_rate,
        "unit": "rotations/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": rot_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (seeded slot values uniform in {-1,0,1})",
        "config": rotation_config(world),
        "rates": {
            "rotations_per_s": rot_rate,
            "hma_per_s": world * B * args.steps / (hma_ms * 1e-3),
            "rescale_per_s": world * B * args.steps / (resc_ms * 1e-3),
            "rotation_modmul_per_s": rot_rate / world * per_rot_mm,
            "rotation_frac_of_int_peak": rot_rate / world * per_rot_mm / peak_modmul,
            "rotation_hbm_gbs": rot_rate / world * rotation_bytes(n, P.L, B) / 1e9,
        },
        "kernels": kern,
        "gpu_launches": launches,
        "e2e": {"value": world * B * e2e_steps / e2e_s, "unit": "rotations/s",
                "h2d_bytes_per_step": int(slots.nbytes), "d2h_bytes_per_step": int(slots.nbytes),
                "mode": e2e_mode, "chunks": e2e_chunks, "steps": e2e_steps,
                "path": {"overlap": "Evaluator encrypt(page-locked host slots, chunked) -> rotate_many -> "
                                    "decrypt(page-locked host, chunked), software-pipelined across steps: step "
                                    "i + 1's H2D and step i - 1's D2H run under step i's key switch",
                         "phases": "Evaluator encrypt(page-locked host slots, chunked) -> rotate_many -> "
                                   "decrypt(page-locked host, chunked)",
                         }.get(e2e_mode, "per chunk: Evaluator encrypt(page-locked host slots) -> rotate -> "
                                         "decrypt(page-locked host)")
                        + "; copies on the library's H2D/D2H streams",
                "unpipelined_value": e2e_serial,
                "check": e2e_ok},
        "clocks": clk.summary(),
    }
    if dominant:
        d = kern[dominant]
        result["roofline"] = {
            "kernel": dominant, "bound": "int", "achieved": d["modmul_per_s"] / 1e9,
            "peak": peak_modmul / 1e9, "unit": "Gmodmul/s", "frac": d["modmul_per_s"] / peak_modmul,
            "peak_source": "measured live: k_peak_modmul (chained 64-bit Shoup modmuls, all SMs; the faster of "
                           "the exact- and approximate-quotient forms)",
            "peaks_gmodmul": {k: v / 1e9 for k, v in peaks.items()},
            "hbm_gbs": d["gbs"], "hbm_peak_gbs": _hbm_peak(),
            "traffic": (_ncu_traffic(dominant) or {}).get("bytes_per_launch"),
            "traffic_source": (_ncu_traffic(dominant) or {}).get("source"),
            "algorithmic": "per ciphertext: l*l NTTs of (n/2)log2(n) modmuls (k_modup); see DESIGN.md section 3",
        }
    # the HBM-bound primitive of configs[1]: the fused HMA streams ct, acc in and acc out (3 x 2 l n words per
    # ciphertext; the one plaintext of the batch, l n words, stays in L2)
    hma_bytes = 3 * 2 * P.L * n * 8
    hma_gbs = B * args.steps / (hma_ms * 1e-3) * hma_bytes / 1e9
    result["roofline_hma"] = {
        "kernel": "k_mul_plain (acc += ct * pt, in place)", "bound": "hbm", "achieved": hma_gbs,
        "peak": _hbm_peak(), "unit": "GB/s", "frac": hma_gbs / _hbm_peak(),
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (driver-written copy bandwidth), else the recipe's fallback",
        "traffic": None,
        "algorithmic": f"per ciphertext: ct read + acc read + acc write = {hma_bytes} B (plaintext L2-resident)"}
    return result


# ------------------------------------------------------------ inference arm
def cfg0_setup(images: int, seed: int, offset: int = 0):
    """BASELINE configs[0]/[2] network on seeded synthetic MNIST-shaped images:
    28x28 pixels round(U[0,1]*255), zero-padded to 29x29 (valid convs);
    weights N(0, 0.1) -> 8-bit symmetric quantization; zero biases."""
    from paper_2102_03494_b200.hesim import SchemeParams
    from paper_2102_03494_b200.netspec import LayerSpec, NetworkSpec, synthetic_weights
    from paper_2102_03494_b200.packing import TensorShape
    from paper_2102_03494_b200.planner import build_plan
    from paper_2102_03494_b200.runner import inference_params, scheme_for

    layers = (LayerSpec("ffconv", d=5, stride=2, out_channels=5, rank=2, packing_hint="dp-hi2c-cp"),
              LayerSpec("square"), LayerSpec("fc", out_channels=100), LayerSpec("square"),
              LayerSpec("fc", out_channels=10))
    shape = TensorShape(29, 29, 1)
    prov = NetworkSpec(SchemeParams(n_slots=8192, t=(1 << 61) - 1), shape, layers)
    ws = synthetic_weights(prov, np.random.default_rng(seed), sigma=0.1)
    rp = inference_params(prov, build_plan(prov, "explicit"), ws, input_bound=255, seed=CFG1["seed"])
    net = NetworkSpec(scheme_for(rp), shape, layers)
    plan = build_plan(net, "explicit")
    rng = np.random.default_rng(seed + 1)
    pix = np.round(rng.random(size=(offset + images, 1, 28, 28)) * 255).astype(np.int64)[offset:]
    xs = np.zeros((images, 1, 29, 29), dtype=np.int64)
    xs[:, :, :28, :28] = pix
    return net, plan, ws, xs, rp


CIFAR_LAYERS = (
    # configs[3] as SURVEY.md 8(d) pins it: valid convolutions at 2^15 slots (ring 2^16),
    # "3x3 low-rank conv 3->8 then 1x1 8->32" = ffconv(d=3, r=8, O=32), x^2, 2x2 avg-pool,
    # ffconv(d=3, r=16, O=64), x^2, 2x2 avg-pool, FC 2304->10; planner "ffconv-default"
    dict(kind="ffconv", d=3, stride=1, out_channels=32, rank=8),
    dict(kind="square"), dict(kind="avgpool", d=2, stride=2),
    dict(kind="ffconv", d=3, stride=1, out_channels=64, rank=16),
    dict(kind="square"), dict(kind="avgpool", d=2, stride=2),
    dict(kind="fc", out_channels=10),
)


def cfg3_setup(images: int, seed: int, offset: int = 0):
    """BASELINE configs[3] on CIFAR-shaped images: weights N(0, 0.05) -> 8-bit and the
    first two inputs from the committed fixture (tests/golden/cfg3.npz, made by the
    reference's own code), further images seeded round(clip(N(0.5, 0.25), 0, 1) * 255);
    zero biases.  Returns the reference logits of the fixture images in range."""
    from paper_2102_03494_b200.hesim import SchemeParams
    from paper_2102_03494_b200.netspec import LayerSpec, NetworkSpec, WeightSet, WeightTensor
    from paper_2102_03494_b200.packing import TensorShape
    from paper_2102_03494_b200.planner import build_plan
    from paper_2102_03494_b200.runner import inference_params, scheme_for

    gold = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(gold, "cfg3.json")) as fh:
        meta = json.load(fh)
    z = np.load(os.path.join(gold, "cfg3.npz"))
    layers = tuple(LayerSpec(**d) for d in meta["layers"])
    shape = TensorShape(32, 32, 3)
    ws = WeightSet()
    for name, scale in meta["scales"].items():
        ws.add(WeightTensor(name, z[name.replace(".", "_")].astype(np.int64), 8, scale))
    prov = NetworkSpec(SchemeParams(n_slots=meta["n_slots"], t=(1 << 61) - 1), shape, layers)
    rp = inference_params(prov, build_plan(prov, meta["strategy"]), ws, input_bound=255, seed=CFG1["seed"])
    net = NetworkSpec(scheme_for(rp), shape, layers)
    plan = build_plan(net, meta["strategy"])
    fx = z["inputs"].astype(np.int64)
    extra = max(0, offset + images - len(fx))
    rng = np.random.default_rng(seed + 1)
    more = np.round(np.clip(rng.normal(0.5, 0.25, size=(extra, 3, 32, 32)), 0.0, 1.0) * 255).astype(np.int64)
    xs = np.concatenate([fx, more])[offset:offset + images]
    ref = [[int(v) for v in row] for row in meta["logits"]][offset:offset + images]
    return net, plan, ws, xs, rp, ref


def run_cifar(args, rank, world, local_rank):
    """configs[3] on a bounded sample: `--images` images (default 2 = one row pair)
    per rank, decrypted logits compared with the reference algorithm."""
    import torch
    from paper_2102_03494_b200.abi import cuda_library
    from paper_2102_03494_b200.hesim import HeContext
    from paper_2102_03494_b200.runner import pack_input, run_encrypted
    from paper_2102_03494_b200.shard import shard_range
    torch.cuda.set_device(local_rank)
    lib = cuda_library()
    lo, hi = shard_range(args.images, rank, world)
    per_rank = hi - lo
    net, plan, ws, xs, rp, ref_logits = cfg3_setup(per_rank, seed=CFG1["seed"], offset=lo)
    ctx = HeContext(net.scheme, batch=min(args.chunk, per_rank), lib=lib, schedule=args.schedule,
                    level_schedule=args.level_schedule)
    ev = ctx.evaluator
    stream_ptr = ctypes.c_void_p()
    lib.call("fhe_ctx_stream", ev.ctx, ctypes.byref(stream_ptr))
    stream = torch.cuda.ExternalStream(stream_ptr.value, device=local_rank)
    chunk = ctx.batch
    parts = []
    for i in range(0, per_rank, chunk):
        sub = xs[i:i + chunk]
        if len(sub) < chunk:                                   # ragged tail: zero images
            sub = np.concatenate([sub, np.zeros((chunk - len(sub),) + sub.shape[1:], dtype=sub.dtype)])
        parts.append(pack_input(net, plan, sub, ctx))
    ev.sync()
    if world > 1:
        torch.distributed.barrier()
    rot0 = ctx.counters.rot
    cnt0 = ctypes.c_uint64()
    lib.call("fhe_launch_count", ev.ctx, ctypes.byref(cnt0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = os.environ.get("FHE_BENCH_PROF") == "1"      # per-kernel breakdown (single stream, slower)
    if prof:
        lib.call("fhe_prof_enable", ev.ctx, 1)
    t0 = time.perf_counter()
    results = []
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for packed in parts:
            results.append(run_encrypted(net, plan, ws, None, ctx=ctx, packed=packed, decrypt=False))
        e1.record(stream)
        e1.synchronize()
    res = results[-1]
    ms = e0.elapsed_time(e1)
    wall = time.perf_counter() - t0
    breakdown = None
    if prof:
        buf = ctypes.create_string_buffer(1 << 16)
        lib.call("fhe_prof_report", ev.ctx, buf, len(buf))
        lib.call("fhe_prof_enable", ev.ctx, 0)
        breakdown = {k: {"calls": c, "ms": round(m, 3)} for k, (c, m) in parse_prof(buf.value.decode()).items()}
    cnt1 = ctypes.c_uint64()
    lib.call("fhe_launch_count", ev.ctx, ctypes.byref(cnt1))
    logits = np.concatenate([np.atleast_2d(_decrypt_logits(r, ctx)) for r in results])[:per_rank]
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local_rank}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    got = [[int(v) for v in row] for row in np.atleast_2d(np.asarray(logits)).tolist()]
    # every image against the oracle's direct loops (the fixture images are also pinned
    # to the reference's own run_reference logits, tests/golden/cfg3.json)
    want = _oracle_logits(net, ws, xs) if os.environ.get("BENCH_CIFAR_ORACLE", "1") == "1" else None
    kb = ctypes.c_uint64()
    lib.call("fhe_ctx_key_bytes", ev.ctx, ctypes.byref(kb))
    rots = ctx.counters.rot - rot0
    return {
        "images_per_s": args.images / (ms * 1e-3), "ms": ms, "wall_s": wall, "images_per_rank": per_rank,
        "schedule": args.schedule, "crt_primes": len(rp.t), "L": rp.L, "log_qp": round(rp.log_qp, 1),
        "ring": rp.n, "logical_rotations": rots,
        "physical_rotations_per_s": rots * rp.T * ctx.rows / (ms * 1e-3),
        "gpu_launches": int(cnt1.value - cnt0.value), "key_bytes_resident": int(kb.value),
        "depth": res.depth, "assembly_depth": res.assembly_depth, "clocks": clk.summary(),
        # images with a fixture (the reference's run_reference logits): exact comparison
        "logits_checked": len(ref_logits),
        "logits_match_reference": got[:len(ref_logits)] == ref_logits if ref_logits else None,
        "oracle_images_checked": len(want) if want is not None else 0,
        "logits_match_oracle": got == want if want is not None else None,
        "distinct_rotation_keys": len(ctx.rotation_steps),
        "logits_sample": [str(int(v)) for v in np.asarray(logits)[0][:3]],
        "kernel_ms": breakdown,
    }


ABLATION = [
    # (name, first layer spec) -- the configs[4] variants: unfactorized 5x5 conv vs FFConv ranks,
    # each under DensePack and ConvPack, followed by square, fc100, square, fc10
    ("conv-dense", dict(kind="conv", d=5, stride=2, out_channels=5, packing_hint="dense")),
    ("conv-cp", dict(kind="conv", d=5, stride=2, out_channels=5, packing_hint="conv")),
    ("ffconv-r1-dp", dict(kind="ffconv", d=5, stride=2, out_channels=5, rank=1, packing_hint="dp-hi2c-cp")),
    ("ffconv-r2-dp", dict(kind="ffconv", d=5, stride=2, out_channels=5, rank=2, packing_hint="dp-hi2c-cp")),
    ("ffconv-r4-dp", dict(kind="ffconv", d=5, stride=2, out_channels=5, rank=4, packing_hint="dp-hi2c-cp")),
    ("ffconv-r1-cp", dict(kind="ffconv", d=5, stride=2, out_channels=5, rank=1, packing_hint="cp-hi2c-cp")),
    ("ffconv-r2-cp", dict(kind="ffconv", d=5, stride=2, out_channels=5, rank=2, packing_hint="cp-hi2c-cp")),
    ("ffconv-r4-cp", dict(kind="ffconv", d=5, stride=2, out_channels=5, rank=4, packing_hint="cp-hi2c-cp")),
]


# logical rotations per image of each variant in the reference's own report (SURVEY.md
# section 8(d), configs[4]); the F4 slot-0 masks are plaintext products and add none
REF_ROTATIONS = {"conv-dense": 10463, "conv-cp": 1173, "ffconv-r1-dp": 3031, "ffconv-r2-dp": 4889,
                 "ffconv-r4-dp": 8605, "ffconv-r1-cp": 1173, "ffconv-r2-cp": 1173, "ffconv-r4-cp": 1173}


def ablation_setup(first, images, seed, offset=0):
    from paper_2102_03494_b200.hesim import SchemeParams
    from paper_2102_03494_b200.netspec import LayerSpec, NetworkSpec, synthetic_weights
    from paper_2102_03494_b200.packing import TensorShape
    from paper_2102_03494_b200.planner import build_plan
    from paper_2102_03494_b200.runner import inference_params, scheme_for
    layers = (LayerSpec(**first), LayerSpec("square"), LayerSpec("fc", out_channels=100), LayerSpec("square"),
              LayerSpec("fc", out_channels=10))
    shape = TensorShape(29, 29, 1)
    prov = NetworkSpec(SchemeParams(n_slots=8192, t=(1 << 61) - 1), shape, layers)
    ws = synthetic_weights(prov, np.random.default_rng(seed), sigma=0.1)
    rp = inference_params(prov, build_plan(prov, "explicit"), ws, input_bound=255, seed=CFG1["seed"])
    net = NetworkSpec(scheme_for(rp), shape, layers)
    rng = np.random.default_rng(seed + 1)
    pix = np.round(rng.random(size=(offset + images, 1, 28, 28)) * 255).astype(np.int64)[offset:]
    xs = np.zeros((images, 1, 29, 29), dtype=np.int64)
    xs[:, :, :28, :28] = pix
    return net, build_plan(net, "explicit"), ws, xs, rp


def run_ablation(args, rank, world, local_rank):
    """configs[4]: rotation count and latency per variant (images sharded over ranks)."""
    import torch
    from paper_2102_03494_b200.abi import cuda_library
    from paper_2102_03494_b200.hesim import HeContext
    from paper_2102_03494_b200.runner import pack_input, run_encrypted
    from paper_2102_03494_b200.shard import shard_range
    torch.cuda.set_device(local_rank)
    lib = cuda_library()
    lo, hi = shard_range(args.images, rank, world)
    per_rank = hi - lo
    out = {}
    for name, first in ABLATION:
        net, plan, ws, xs, rp = ablation_setup(first, per_rank, seed=CFG1["seed"], offset=lo)
        chunk = min(args.chunk, per_rank)
        ctx = HeContext(net.scheme, batch=chunk, lib=lib, level_schedule=args.level_schedule)
        chunks = [xs[i:i + chunk] for i in range(0, per_rank, chunk)]
        if len(chunks[-1]) < chunk:
            pad = np.zeros((chunk - len(chunks[-1]),) + xs.shape[1:], dtype=xs.dtype)
            chunks[-1] = np.concatenate([chunks[-1], pad])
        packed = [pack_input(net, plan, c, ctx) for c in chunks]
        run_encrypted(net, plan, ws, None, ctx=ctx, packed=packed[0], decrypt=False)     # warm-up: keys, plaintexts
        ctx.evaluator.sync()
        if world > 1:
            torch.distributed.barrier()
        c0 = ctx.counters.copy()
        t0 = time.perf_counter()
        results = []
        for p in packed:
            res = run_encrypted(net, plan, ws, None, ctx=ctx, packed=p, decrypt=False)
            results.append(res)
        ctx.evaluator.sync()
        el = time.perf_counter() - t0
        # every image's logits against the oracle (outside the timed region)
        got = [row for r in results for row in np.atleast_2d(_decrypt_logits(r, ctx)).tolist()][:per_rank]
        want = _oracle_logits(net, ws, xs)
        match = [[int(v) for v in g] for g in got] == want
        if world > 1:
            t = torch.tensor([el], device=f"cuda:{local_rank}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        d = ctx.counters - c0
        per_chunk = len(packed)
        out[name] = {"rotations_per_image": d.rot // per_chunk, "mul_pc_per_image": d.mul_pc // per_chunk,
                     "add_cc_per_image": d.add_cc // per_chunk, "assembly_masks_per_image": d.assembly_mul_pc // per_chunk,
                     "crt_primes": len(rp.t), "L": rp.L, "images_per_s": args.images / el,
                     "latency_ms_per_batch": 1e3 * el / per_chunk, "batch": chunk,
                     "depth": res.depth, "assembly_depth": res.assembly_depth,
                     "reference_rotations_per_image": REF_ROTATIONS[name],
                     "logits_checked": len(want), "logits_match": match,
                     "distinct_rotation_keys": len(ctx.rotation_steps)}
        del ctx, packed, res
    return out




def rotation_modmuls_L(n, l):
    return rotation_modmuls(n, l)


def run_inference(args, rank, world, local_rank, images_total=None, steps=None, warmup=None, schedule=None):
    """configs[2]: `images_total` images sharded contiguously over ranks, each
    rank's shard evaluated in rounds of `chunk` images.  value: evaluation of
    resident encrypted inputs (CUDA events, max over ranks).  e2e: rank 0 holds
    the host images, encrypts and scatters them (NCCL), every rank evaluates,
    rank 0 gathers the encrypted logits and decrypts them to host."""
    import torch
    from paper_2102_03494_b200.abi import cuda_library
    from paper_2102_03494_b200.hesim import HeContext
    from paper_2102_03494_b200.runner import pack_input, run_encrypted
    from paper_2102_03494_b200.shard import gather_logits, scatter_packed, shard_range

    torch.cuda.set_device(local_rank)
    device = f"cuda:{local_rank}"
    lib = cuda_library()
    images_total = images_total or args.images
    steps = steps if steps is not None else args.steps
    warmup = warmup if warmup is not None else args.warmup
    lo, hi = shard_range(images_total, rank, world)
    per_rank = hi - lo
    chunk = min(args.chunk, per_rank)
    rounds = -(-per_rank // chunk)
    net, plan, ws, xs_all, rp = cfg0_setup(images_total, seed=CFG1["seed"])
    schedule = schedule or args.schedule
    ctx = HeContext(net.scheme, batch=chunk, lib=lib, schedule=schedule, level_schedule=args.level_schedule)
    ev = ctx.evaluator
    stream_ptr = ctypes.c_void_p()
    lib.call("fhe_ctx_stream", ev.ctx, ctypes.byref(stream_ptr))
    stream = torch.cuda.ExternalStream(stream_ptr.value, device=local_rank)

    def round_images(k):
        """every rank's k-th chunk, concatenated in rank order (rank 0's view)."""
        parts = []
        for r in range(world):
            a, b = shard_range(images_total, r, world)
            sub = xs_all[a:b][k * chunk:(k + 1) * chunk]
            if len(sub) < chunk:                               # ragged tail: pad with zero images
                sub = np.concatenate([sub, np.zeros((chunk - len(sub),) + sub.shape[1:], dtype=sub.dtype)])
            parts.append(sub)
        return np.concatenate(parts)

    def scatter_round(k):
        if world == 1:
            return pack_input(net, plan, round_images(k), ctx)
        return scatter_packed(net, plan, ctx, round_images(k) if rank == 0 else None, rank, world, device)

    packed = [scatter_round(k) for k in range(rounds)]

    def evaluate(ps):
        return [run_encrypted(net, plan, ws, None, ctx=ctx, packed=p, decrypt=False) for p in ps]

    for _ in range(max(1, warmup)):
        evaluate(packed[:1])
    ev.sync()
    if world > 1:
        torch.distributed.barrier()
    peak_mm = 0.0
    for kind in (0, 1):
        pk = ctypes.c_double()
        lib.call("fhe_peak_modmul_kind", ev.ctx, 20000, kind, ctypes.byref(pk))
        peak_mm = max(peak_mm, pk.value)
    cnt0 = ctypes.c_uint64()
    lib.call("fhe_launch_count", ev.ctx, ctypes.byref(cnt0))
    mm0 = ctypes.c_double()
    lib.call("fhe_work_modmuls", ev.ctx, ctypes.byref(mm0))
    rot0 = ctx.counters.rot
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            evaluate(packed)
        e1.record(stream)
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    cnt1 = ctypes.c_uint64()
    lib.call("fhe_launch_count", ev.ctx, ctypes.byref(cnt1))
    mm1 = ctypes.c_double()
    lib.call("fhe_work_modmuls", ev.ctx, ctypes.byref(mm1))
    rots = ctx.counters.rot - rot0
    if world > 1:
        t = torch.tensor([ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    # e2e: host images on rank 0 -> encrypt + scatter -> evaluate -> gather + decrypt
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    round_logits = []
    for k in range(rounds):
        res = run_encrypted(net, plan, ws, None, ctx=ctx, packed=scatter_round(k), decrypt=False)
        lg = gather_logits(ctx, res.value, rank, world, device) if world > 1 else _decrypt_logits(res, ctx)
        round_logits.append(lg)
    ev.sync()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    # every image's decrypted logits against the oracle (the reference's direct-loop
    # network, runner.py:197-226 restated in oracle/slot_oracle.py), on rank 0
    check = None
    if rank == 0:
        got = {}
        for k, lg in enumerate(round_logits):
            lg = np.atleast_2d(lg)
            for r in range(world):
                a, b = shard_range(images_total, r, world)
                for j in range(chunk):
                    idx = a + k * chunk + j
                    if idx < b:
                        got[idx] = [int(v) for v in lg[r * chunk + j]]
        want = _oracle_logits(net, ws, xs_all)
        bad = [i for i in range(images_total) if got.get(i) != want[i]]
        check = {"images_checked": len(got), "logits_match": not bad and len(got) == images_total,
                 "mismatched_images": bad[:8],
                 "oracle": "oracle/slot_oracle.run_reference_ints (reference runner.py:197-226 restated)"}
    first_logits = round_logits[0] if round_logits else None
    # per-kernel breakdown of one chunk (single-stream, isolated kernel times)
    lib.call("fhe_prof_enable", ev.ctx, 1)
    evaluate(packed[:1])
    buf = ctypes.create_string_buffer(1 << 16)
    lib.call("fhe_prof_report", ev.ctx, buf, len(buf))
    lib.call("fhe_prof_enable", ev.ctx, 0)
    breakdown = {k: {"calls": c, "ms": round(m, 3)} for k, (c, m) in parse_prof(buf.value.decode()).items()}
    # physical ciphertext rotations: logical rotations x CRT primes x row pairs
    phys_rot = rots * rp.T * ctx.rows
    mm = mm1.value - mm0.value          # algorithmic modmuls the library issued (fhe_work_modmuls)
    # bytes crossing PCIe in the e2e loop: the encrypted inputs' slot residues (rank 0
    # encrypts every rank's batch: T x R x n words per input ciphertext) and the logit
    # slot ranges read back (fhe_decrypt_slots: T x R x 2 x m words per logit ciphertext)
    from paper_2102_03494_b200.runner import _logits_layout
    in_cts = 1 if plan.steps[0].op == "pack-dense" else plan.steps[0].kernel.k_columns(plan.steps[0].in_shape.c)
    n_logit_cts, m_logit = _logits_layout(net, plan)
    in_bytes = rounds * world * in_cts * rp.T * ctx.rows * rp.n * 8
    out_bytes = rounds * world * n_logit_cts * rp.T * ctx.rows * 2 * m_logit * 8
    return {
        "schedule": schedule, "level_schedule": bool(args.level_schedule),
        "images_per_s": images_total * steps / (ms * 1e-3),
        "ms_per_step": ms / steps,
        "e2e_images_per_s": images_total / e2e_s,
        "per_rank_images": per_rank, "chunk": chunk, "rounds": rounds,
        "crt_primes": len(rp.t), "t_bits": round(math.log2(rp.t[0]), 2), "L": rp.L,
        "log_qp": round(rp.log_qp, 1), "logical_rotations_per_chunk": rots // max(1, steps * rounds),
        "physical_rotations_per_s": world * phys_rot / (ms * 1e-3),
        "modmul_per_s_per_gpu": mm / (ms * 1e-3),
        "roofline": {"bound": "int", "achieved": mm / (ms * 1e-3) / 1e9, "peak": peak_mm / 1e9, "unit": "Gmodmul/s",
                     "frac": mm / (ms * 1e-3) / peak_mm,
                     "algorithmic": "whole evaluation: (n/2)log2(n) per row (I)NTT at the row's level, key inner "
                                    "products, ModDown scaling, hoisted-dot MACs (elementwise ops not counted)"},
        "gpu_launches": int(cnt1.value - cnt0.value),
        "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": int(out_bytes),
        "clocks": clk.summary(),
        "logits_sample": [str(int(v)) for v in np.atleast_2d(first_logits)[0][:3]] if first_logits is not None else None,
        "logits_check": check,
        "kernel_ms_one_chunk": breakdown,
    }


def run_latency(args, local_rank, schedule="reference"):
    """configs[0]: one synthetic image, end to end on one GPU -- host pixels -> encrypt ->
    evaluate -> decrypt -> host logits -- and the device time of the evaluation alone
    (CUDA events); a warm-up run first builds keys and plaintexts."""
    import torch
    from paper_2102_03494_b200.abi import cuda_library
    from paper_2102_03494_b200.hesim import HeContext
    from paper_2102_03494_b200.runner import pack_input, run_encrypted
    torch.cuda.set_device(local_rank)
    lib = cuda_library()
    net, plan, ws, xs, rp = cfg0_setup(1, seed=CFG1["seed"])
    ctx = HeContext(net.scheme, batch=1, lib=lib, schedule=schedule, level_schedule=args.level_schedule)
    ev = ctx.evaluator
    stream_ptr = ctypes.c_void_p()
    lib.call("fhe_ctx_stream", ev.ctx, ctypes.byref(stream_ptr))
    stream = torch.cuda.ExternalStream(stream_ptr.value, device=local_rank)
    run_encrypted(net, plan, ws, xs[0], ctx=ctx)                    # warm-up: keys, plaintexts
    packed = pack_input(net, plan, xs[0], ctx)
    ev.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run_encrypted(net, plan, ws, None, ctx=ctx, packed=packed, decrypt=False)
    e1.record(stream)
    e1.synchronize()
    dev_ms = e0.elapsed_time(e1)
    t0 = time.perf_counter()
    res = run_encrypted(net, plan, ws, xs[0], ctx=ctx)
    e2e_ms = 1e3 * (time.perf_counter() - t0)
    want = _oracle_logits(net, ws, xs)[0]
    ok = [int(v) for v in res.logits] == want
    # the same walk captured once as a CUDA graph and replayed (runner.CapturedPlan)
    from paper_2102_03494_b200.runner import CapturedPlan
    graph = {}
    try:
        cp = CapturedPlan(net, plan, ws, np.zeros_like(xs[0]), ctx)
        cp.run(xs[0])                                               # warm replay
        ev.sync()
        e0.record(stream)
        cp.replay()
        e1.record(stream)
        e1.synchronize()
        g_dev = e0.elapsed_time(e1)
        t0 = time.perf_counter()
        lg = cp.run(xs[0])
        g_e2e = 1e3 * (time.perf_counter() - t0)
        graph = {"device_ms": g_dev, "e2e_ms": g_e2e, "nodes": cp.nodes,
                 "logits_match": [int(v) for v in np.atleast_1d(lg)] == want}
    except Exception as exc:                                        # noqa: BLE001 -- reported, not fatal
        graph = {"error": str(exc)[:300]}
    return {"workload": "configs[0]: one 28x28 image (zero-padded to 29x29), batch 1", "schedule": schedule,
            "level_schedule": bool(args.level_schedule), "device_ms": dev_ms, "e2e_ms": e2e_ms,
            "logits_match": ok, "crt_primes": rp.T, "L": rp.L, "graph_replay": graph}


def _oracle_logits(net, ws, xs):
    """Reference logits of every image (object ints) from the oracle's direct loops."""
    from oracle.slot_oracle import run_reference_ints
    layers = [{k: v for k, v in l.__dict__.items() if v is not None} for l in net.layers]
    wd = {}
    for name in ws.names():
        i, key = name[len("layer"):].split(".")
        wd.setdefault(int(i), {})[key] = ws[name].values
    return [[int(v) for v in run_reference_ints(layers, wd, x)[0]] for x in xs]


def _decrypt_logits(res, ctx):
    from paper_2102_03494_b200.runner import _logits
    return np.atleast_2d(_logits(res.value, ctx))


def cpu_baseline_inference(images: int = 1):
    """Reference algorithm on the host: the product's plan walk over the slot
    oracle (np.int64 slot engine), one run per plaintext CRT prime, 1 core."""
    from oracle.slot_oracle import Params, SlotContext
    from paper_2102_03494_b200.runner import run_encrypted
    net, plan, ws, xs, rp = cfg0_setup(images, seed=CFG1["seed"])
    t0 = time.perf_counter()
    for x in xs:
        for ti in rp.t:
            ctx = SlotContext(Params(8192, ti))
            run_encrypted(net, plan, ws, x, ctx=ctx)
    el = time.perf_counter() - t0
    return images / el, f"{images} image(s) x {len(rp.t)} CRT primes, cfg0 plan on the slot oracle"


def _cpu_inference_task(args):
    img_idx, ti = args
    from oracle.slot_oracle import Params, SlotContext
    from paper_2102_03494_b200.runner import run_encrypted
    net, plan, ws, xs, rp = cfg0_setup(1, seed=CFG1["seed"], offset=img_idx)
    run_encrypted(net, plan, ws, xs[0], ctx=SlotContext(Params(8192, ti)))
    return 1


def _ncu_traffic(kernel: str):
    """dram__bytes_read + dram__bytes_write per launch of `kernel` from the newest
    committed `ncu --set full` summary in profiles/ (None if absent)."""
    import glob
    import re
    base = kernel.split("(")[0]
    paths = glob.glob(os.path.join(ROOT, "profiles", f"r[0-9][0-9]_{base}.txt")) + \
        glob.glob(os.path.join(ROOT, "profiles", "r*_prof_top.txt"))
    for path in sorted(paths, key=os.path.basename, reverse=True):
        text = open(path).read()
        if base not in "\n".join(text.splitlines()[:6]):
            continue
        vals = {}
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            m = re.search(name + r"\s+([0-9.]+)\s+(\w+)", text)
            if m:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m.group(2), 1)
                vals[name] = float(m.group(1)) * scale
        if len(vals) == 2:
            return {"bytes_per_launch": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                    "source": os.path.relpath(path, ROOT)}
    return None


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh).get("hbm_gbs")
    except OSError:
        return 6650.0


def run_reference_arm(args, rank, world):
    if rank != 0:
        return None
    cores = os.cpu_count() or 1
    if args.workload == "inference":
        import multiprocessing as mp
        _, _, _, _, rp = cfg0_setup(1, seed=CFG1["seed"])
        sample = max(cores, 8)
        tasks = [(i, ti) for i in range(sample) for ti in rp.t]
        rates = []
        with mp.Pool(cores) as pool:
            for it in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                pool.map(_cpu_inference_task, tasks)
                el = time.perf_counter() - t0
                if it >= args.warmup:
                    rates.append(sample / el)
        v = statistics.median(rates)
        return {
            "impl": "reference", "metric": "encrypted-image inferences/s (FFConv MNIST-shaped HECNN, cfg2)",
            "value": v, "unit": "images/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sample / v, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": "configs[2] (reference slot-engine algorithm, one run per CRT prime)"},
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": cores, "kind": "port",
                             "sample": f"{sample} images x {len(rp.t)} CRT primes per step"},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "the reference is a slot simulator with no cryptography",
        }
    rates = []
    for _ in range(args.warmup):
        cpu_baseline_rotation(cores, seconds=0.5)
    for _ in range(args.steps):
        r, sample = cpu_baseline_rotation(cores, seconds=1.0)
        rates.append(r)
    v = statistics.median(rates)
    return {
        "impl": "reference",
        "metric": "key-switched rotations/s (ring 2^14, 4x40-bit q + 1 special prime, hybrid KS)",
        "value": v, "unit": "rotations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * CFG1["batch"] / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": rotation_config(world),
        "cpu_baseline": {"value": v, "unit": "rotations/s", "cores": cores, "kind": "port", "sample": sample,
                         "algorithm": "reference slot engine (oracle/slot_oracle.py restates hesim.py:244-261): "
                                      "np.roll of an int64 slot vector"},
        "e2e": {"value": v, "unit": "rotations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference is a slot simulator: its rotation is np.roll, not a key-switched RLWE rotation",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["rotation", "inference", "ablation", "cifar", "latency"], default="rotation")
    ap.add_argument("--images", type=int, default=256, help="inference: images per step (whole job)")
    ap.add_argument("--chunk", type=int, default=None,
                    help="inference: images per plan walk (measured at 256 images: 64 -> 7.24, 128 -> 7.27, 256 -> 7.28 images/s)")
    ap.add_argument("--no-inference", action="store_true", help="rotation workload: skip the inference sample")
    ap.add_argument("--schedule", choices=["reference", "hoisted"], default="reference",
                    help="inference: rotate-and-sum schedule (hoisted = top levels as a ct x pt GEMM)")
    ap.add_argument("--no-level-schedule", dest="level_schedule", action="store_false",
                    help="inference: keep every ciphertext at the top level (no modulus switching between steps)")
    args = ap.parse_args()
    if args.chunk is None:                      # configs[3] / configs[4] keep the 64-image walks they were measured with
        args.chunk = 128 if args.workload in ("rotation", "inference") else 64
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    rank, world, local_rank = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1), _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        res = run_reference_arm(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    if args.workload == "ablation":
        abl = run_ablation(args, rank, world, local_rank)
        if rank == 0:
            best = max(abl.values(), key=lambda v: v["images_per_s"])
            print(json.dumps({
                "metric": "encrypted-image inferences/s per packing/rank variant (configs[4] ablation)",
                "value": best["images_per_s"], "unit": "images/s (best variant)", "n_gpus": world,
                "steps": 1, "warmup": 1, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u64", "data": "synthetic (seeded images)",
                "config": {"workload": f"configs[4]: {args.images} images, chunks of {args.chunk}"},
                "variants": abl}), flush=True)
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()
        return
    if args.workload == "cifar":
        if "--images" not in sys.argv:
            args.images = 2
        cf = run_cifar(args, rank, world, local_rank)
        if rank == 0:
            print(json.dumps({
                "metric": "encrypted-image inferences/s (FFConv CIFAR-shaped HECNN, configs[3])",
                "value": cf["images_per_s"], "unit": "images/s", "n_gpus": world, "steps": 1, "warmup": 0,
                "ms_per_step": cf["ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u64", "data": "synthetic (seeded N(0.5,0.25) images)",
                "config": {"workload": f"configs[3] sample: {args.images} images (BASELINE: 64), ring 2^16",
                           "parallelism": f"dp{world} (image shards, no collective)"},
                "cifar": cf, "gpu_launches": cf["gpu_launches"], "clocks": cf["clocks"]}), flush=True)
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()
        return
    if args.workload == "latency":
        if rank == 0:
            lat = {s: run_latency(args, local_rank, schedule=s) for s in ("reference", "hoisted")}
            print(json.dumps({"metric": "configs[0] single-image latency (ms, end to end)",
                              "value": lat["reference"]["e2e_ms"], "unit": "ms", "n_gpus": 1,
                              "higher_is_better": False, "latency": lat}), flush=True)
        return
    if args.workload == "inference":
        inf = run_inference(args, rank, world, local_rank)
        res = {
            "metric": "encrypted-image inferences/s (FFConv MNIST-shaped HECNN, cfg2)",
            "value": inf["images_per_s"], "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": inf["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded images)",
            "config": {"workload": f"configs[2]: {args.images} images, chunks of {inf['chunk']}",
                       "parallelism": f"dp{world} (image shards, no collective)"},
            "inference": inf, "gpu_launches": inf["gpu_launches"], "clocks": inf["clocks"],
            "e2e": {"value": inf["e2e_images_per_s"], "unit": "images/s",
                    "h2d_bytes_per_step": inf["h2d_bytes_per_step"], "d2h_bytes_per_step": inf["d2h_bytes_per_step"]},
        }
        if rank == 0:
            print(json.dumps(res), flush=True)
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()
        return
    res = run_rotation(args, rank, world, local_rank)
    if not args.no_inference:
        # secondary line item: configs[2], the full 256-image batch sharded over the ranks,
        # one timed step, every image's logits checked against the oracle
        inf = run_inference(args, rank, world, local_rank, images_total=256, steps=1, warmup=1,
                            schedule="reference")
        res["inference"] = inf
        res["rates"]["images_per_s"] = inf["images_per_s"]
        hinf = run_inference(args, rank, world, local_rank, images_total=256, steps=1, warmup=1,
                             schedule="hoisted")
        res["inference_hoisted"] = {k: hinf[k] for k in ("schedule", "images_per_s", "e2e_images_per_s",
                                                         "logical_rotations_per_chunk", "roofline",
                                                         "kernel_ms_one_chunk", "logits_check")}
        res["rates"]["images_per_s_hoisted"] = hinf["images_per_s"]
        if world == 1:
            res["latency_cfg0"] = run_latency(args, local_rank)
    if rank == 0 and world == 1:
        rate, sample = cpu_baseline_rotation(1, seconds=3.0)
        res["cpu_baseline"] = {"value": rate, "unit": "rotations/s", "cores": 1, "kind": "port",
                               "sample": sample,
                               "note": "reference slot-engine algorithm (np.roll), no cryptography"}
        if not args.no_inference:
            irate, isample = cpu_baseline_inference(1)
            res["cpu_baseline_inference"] = {"value": irate, "unit": "images/s", "cores": 1, "kind": "port",
                                             "sample": isample}
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
