"""Reference-facing slot API, backed by the sm_100a RNS-BFV evaluator.

Mirrors `cipherpack.hesim` (/root/reference/pkg/src/cipherpack/hesim.py) name for
name: `SchemeParams`, `OpCounters`, `PlainVector`, `SlotCiphertext`, `HeContext`,
`rotations_for_span`, `merge_contexts` and the three error types, with the same
argument meaning, counter/depth semantics and error behaviour.  What changes is
underneath: a tracked `SlotCiphertext` holds a device handle to real BFV
ciphertexts instead of a numpy slot array.

Differences a caller can observe, all deliberate:

* one context evaluates `batch` images at once; every primitive acts on all of
  them (images 2r and 2r+1 share the two batching rows of row-pair r);
* `encrypt`/`decrypt` accept/return one slot vector per image when batch > 1;
* `ct.slots` is a decrypting property (test convenience, costs a decrypt);
* the `rotate_and_sum` zero-tail precondition is checked on the device for every
  call (a decrypt of the operand and a scan of slots >= m, no host round trip);
  a violation raises `PreconditionError` at the next synchronizing call
  (decrypt, `check()`), or immediately with `debug_checks=True`;
* every decryption checks the noise budget on the device and raises
  `NoiseBudgetError` instead of returning garbage slots;
* t must factor into primes = 1 mod 2N (SIMD batching); a composite t is given
  through `SchemeParams.t_factors` and evaluated by plaintext CRT.
"""

from __future__ import annotations

import collections
import hashlib
import math
from dataclasses import dataclass, field, replace

import numpy as np

from .params import RlweParams, batching_compatible, make_params

_INT64_T_LIMIT = 1 << 62


class CapacityError(ValueError):
    """Payload does not fit into the available slots."""


class EncodingOverflowError(ValueError):
    """A signed value falls outside the representable range (-t/2, t/2)."""


class PreconditionError(ValueError):
    """An operation's slot-content precondition is violated."""


class NoiseBudgetError(ValueError):
    """A decrypted ciphertext had no noise budget left: its slots are not the
    encrypted values (the q chain is too short for the computation)."""


@dataclass(frozen=True)
class SchemeParams:
    """Slot count N and plaintext modulus t (reference: hesim.py:61-95).

    t_factors optionally lists the prime factorization of t used for plaintext
    CRT; rlwe optionally pins the full RNS-BFV parameter set.
    """

    n_slots: int
    t: int
    rotation_weight: float = 10.0
    noise_budget_bits: int | None = None
    security_bits: int | None = None
    t_factors: tuple | None = None
    rlwe: RlweParams | None = field(default=None, compare=False)

    def __post_init__(self):
        if self.n_slots < 2 or (self.n_slots & (self.n_slots - 1)) != 0:
            raise ValueError(f"n_slots must be a power of two >= 2, got {self.n_slots}")
        if self.t < 2:
            raise ValueError(f"plaintext modulus must be >= 2, got {self.t}")
        if not self.rotation_weight > 0:
            raise ValueError("rotation_weight must be positive")
        if self.t_factors is not None:
            object.__setattr__(self, "t_factors", tuple(int(f) for f in self.t_factors))
            if math.prod(self.t_factors) != self.t:
                raise ValueError("t_factors do not multiply to t")

    @property
    def int64_storage(self) -> bool:
        return self.t <= _INT64_T_LIMIT

    @property
    def max_value(self) -> int:
        return (self.t - 1) // 2

    def factors(self) -> tuple[int, ...]:
        if self.t_factors is not None:
            return self.t_factors
        return (self.t,)


@dataclass
class OpCounters:
    """Additive tallies of homomorphic operations (reference: hesim.py:97-134)."""

    mul_pc: int = 0
    add_cc: int = 0
    rot: int = 0
    mul_cc: int = 0
    assembly_mul_pc: int = 0

    def copy(self) -> "OpCounters":
        return replace(self)

    def __sub__(self, other: "OpCounters") -> "OpCounters":
        return OpCounters(*(getattr(self, f) - getattr(other, f) for f in _FIELDS))

    def __add__(self, other: "OpCounters") -> "OpCounters":
        return OpCounters(*(getattr(self, f) + getattr(other, f) for f in _FIELDS))

    def merge(self, other: "OpCounters") -> None:
        for f in _FIELDS:
            setattr(self, f, getattr(self, f) + getattr(other, f))


_FIELDS = ("mul_pc", "add_cc", "rot", "mul_cc", "assembly_mul_pc")


class PlainVector:
    """Unencrypted slot vector, canonical residues in [0, t) (hesim.py:137-151).

    The device encoding is created on first use and cached by content.
    """

    __slots__ = ("_slots", "params", "_key", "_small")

    def __init__(self, slots: np.ndarray | None, params: SchemeParams, small: np.ndarray | None = None):
        # `small`: the same vector as centered int64 values when every |v| < 2^62 (weights,
        # masks); the canonical residue array is then built only if someone asks for it
        self._slots = slots
        self.params = params
        self._key = None
        self._small = small

    @property
    def slots(self) -> np.ndarray:
        if self._slots is None:
            t = self.params.t
            if self.params.int64_storage:
                self._slots = np.mod(self._small, t).astype(np.int64)
            else:
                v = self._small.astype(object)
                self._slots = np.where(v < 0, v + t, v)
        return self._slots

    def centered(self) -> np.ndarray:
        if self._small is not None:
            return self._small
        lift = (self.params.t + 1) // 2
        out = self.slots.astype(np.int64, copy=True) if self.params.int64_storage else self.slots.copy()
        out[self.slots >= lift] -= self.params.t
        return out

    def content_key(self) -> bytes:
        if self._key is None:
            if self._small is not None:
                data = b"i64" + self._small.tobytes()
            else:
                arr = np.asarray(self.slots)
                if arr.dtype == object:
                    c = self.centered()
                    if all(abs(int(x)) < 2 ** 62 for x in (c.min(), c.max())):
                        data = b"i64" + c.astype(np.int64).tobytes()
                    else:
                        data = np.array([str(int(v)) for v in arr]).astype("S").tobytes()
                else:
                    data = b"i64" + self.centered().astype(np.int64).tobytes()
            self._key = hashlib.blake2b(data, digest_size=16).digest()
        return self._key


class SlotCiphertext:
    """Packed ciphertext: device handle plus depth counters (hesim.py:154-171).

    `handle is None` marks a count-only ciphertext.
    """

    __slots__ = ("handle", "depth", "params", "assembly_depth", "_ctx")

    def __init__(self, handle, depth: int, params: SchemeParams, assembly_depth: int = 0, ctx=None):
        self.handle = handle
        self.depth = depth
        self.params = params
        self.assembly_depth = assembly_depth
        self._ctx = ctx

    @property
    def tracked(self) -> bool:
        return self.handle is not None

    @property
    def slots(self):
        """Residues in [0, t) (decrypts; test/debug convenience)."""
        if self.handle is None:
            return None
        return self._ctx._residues(self)

    @property
    def level(self) -> int:
        return self.handle.level


def rotations_for_span(m: int) -> int:
    """ceil(log2 m): rotate-and-sum cost over an m-slot payload (hesim.py:369-373)."""
    if m < 1:
        raise ValueError("span must be positive")
    return (m - 1).bit_length()


def default_rlwe(params: SchemeParams, levels: int | None = None, q_bits: int | None = None) -> RlweParams:
    """RNS-BFV parameters for a SchemeParams."""
    if params.rlwe is not None:
        return params.rlwe
    factors = params.factors()
    for f in factors:
        if not batching_compatible(f, params.n_slots):
            raise ValueError(
                f"plaintext modulus factor {f} does not admit SIMD batching over {params.n_slots} slots "
                f"(needs a prime = 1 mod {4 * params.n_slots} below 2^61); pass t_factors or rlwe")
    qb = q_bits or (55 if params.n_slots >= 1024 else 50)
    return make_params(params.n_slots, factors, levels=levels or 4, q_bits=qb)


class HeContext:
    """One evaluation context: scheme parameters, counters, and a GPU evaluator.

    batch: images evaluated by every call (two per batching-row pair).
    lib:   the ABI implementation; default is the CUDA build (raises if absent).
    """

    def __init__(self, params: SchemeParams, *, batch: int = 1, lib=None, levels: int | None = None,
                 q_bits: int | None = None, debug_checks: bool = False, pt_cache: bool = True,
                 schedule: str = "reference", hoist_levels: int = 7, precondition_checks: bool = True,
                 level_schedule: bool = False):
        if batch < 1:
            raise ValueError("batch must be >= 1")
        self.params = params
        self.counters = OpCounters()
        self.elided_rotations = 0
        self.batch = batch
        self.rows = (batch + 1) // 2
        self.debug_checks = debug_checks
        self.precondition_checks = precondition_checks
        # runner.run_encrypted drops q primes between plan steps once the noise model says
        # the budget allows it (runner._target_level): same slots, cheaper key switches
        self.level_schedule = level_schedule
        self.noise_consumed = None
        self.last_noise_budget = None
        # distinct rotation steps used (= Galois keys a real evaluation needs)
        self.rotation_steps: set[int] = set()
        self._lib = lib
        self._levels = levels
        self._q_bits = q_bits
        self._ev = None
        # device plaintexts by content, LRU-bounded (FHE_PT_CACHE_GB, default 16): the
        # CIFAR-shaped network scatters ~20,000 distinct plaintexts per image batch
        self._pt_cache = collections.OrderedDict() if pt_cache else None
        self._pt_cache_bytes = 0
        if schedule not in ("reference", "hoisted"):
            raise ValueError("schedule must be 'reference' or 'hoisted'")
        # "hoisted": the top hoist_levels levels of rotate-and-sum trees that share
        # one input are evaluated as rotations of the input + a ct x pt GEMM
        # (engine._dense_dots / fc_dense); decrypted slots are identical, op counts differ
        self.schedule = schedule
        self.hoist_levels = hoist_levels

    # ------------------------------------------------------------------ device
    @property
    def evaluator(self):
        if self._ev is None:
            from .rlwe import Evaluator
            rp = default_rlwe(self.params, self._levels, self._q_bits)
            if rp.n_slots != self.params.n_slots:
                raise ValueError("rlwe parameters do not match n_slots")
            self._ev = Evaluator(rp, self._lib)
        return self._ev

    @property
    def group_size(self) -> int:
        """Independent outputs a layer keeps in flight: ~1/4 of a device-memory
        budget (FHE_GROUP_BUDGET_GB, default 24) over the bytes of one handle."""
        import os
        if self._ev is None:          # count-only walk: no device memory involved
            return 1 << 30
        ev = self._ev
        handle = ev.T * self.rows * 2 * ev.L * ev.n * 8
        budget = float(os.environ.get("FHE_GROUP_BUDGET_GB", "24")) * (1 << 30)
        return max(1, int(budget / (4 * handle)))

    def _wrap(self, handle, depth, assembly_depth=0) -> SlotCiphertext:
        return SlotCiphertext(handle, depth, self.params, assembly_depth, ctx=self)

    def _factor_residues(self, values: np.ndarray) -> np.ndarray:
        """signed ints (..., k) -> uint64 residues (T, ..., k)"""
        fs = self.evaluator.params.t
        if values.dtype != object and values.size and np.max(np.abs(values.astype(np.float64))) < 2 ** 62:
            v = values.astype(np.int64)
            return np.stack([np.mod(v, f).astype(np.uint64) for f in fs])
        v = values.astype(object)
        return np.stack([np.array((v % f).tolist(), dtype=np.uint64).reshape(v.shape) for f in fs])

    def _layout(self, per_image: np.ndarray) -> np.ndarray:
        """(T, batch, N) residues -> (T, R, 2N) row-pair layout."""
        T, B, N = per_image.shape
        out = np.zeros((T, self.rows, 2 * N), dtype=np.uint64)
        out[:, :, :N] = per_image[:, 0::2]
        if B > 1:
            out[:, : B // 2, N:] = per_image[:, 1::2]
        return out

    def _device_pt(self, pv: PlainVector):
        key = pv.content_key()
        cache = self._pt_cache
        if cache is not None and key in cache:
            cache.move_to_end(key)
            return cache[key]
        N = self.params.n_slots
        res = self._factor_residues(np.asarray(pv.centered()))          # (T, N)
        both = np.concatenate([res, res], axis=1)                        # replicate to row 1
        ev = self.evaluator
        pt = ev.encode(both)
        if cache is not None:
            import os
            size = ev.T * ev.L * ev.n * 8
            budget = float(os.environ.get("FHE_PT_CACHE_GB", "16")) * (1 << 30)
            while cache and self._pt_cache_bytes + size > budget:
                cache.popitem(last=False)
                self._pt_cache_bytes -= size
            cache[key] = pt
            self._pt_cache_bytes += size
        return pt

    def check(self) -> None:
        """Synchronize with the device and raise any deferred check failure:
        PreconditionError (a rotate_and_sum operand had nonzero slots >= m) or
        NoiseBudgetError (a decryption since the last check had no budget left)."""
        if self._ev is None:
            return
        budget, flags = self._ev.status(reset=True)
        self.last_noise_budget = budget
        # the distance to the nearest integer never exceeds 1/2, so an exhausted budget
        # reads as ~0 bits (uniform fractions); below 0.5 bits (|noise| > 0.35) the
        # ciphertext is one operation from garbage and is rejected as well
        if budget < 0.5:
            raise NoiseBudgetError(f"noise budget exhausted ({budget:.3f} bits left at decryption): the q chain "
                                   f"is too short for this computation; size it with runner.inference_params")
        if flags & 1:
            raise PreconditionError("rotate_and_sum: slots at index >= m must be zero "
                                    "(detected on the device at an earlier call)")

    def _residues(self, ct: SlotCiphertext):
        """Decrypted residues mod t, (N,) for batch 1 else (batch, N)."""
        ev = self.evaluator
        raw = ev.decrypt(ct.handle)                                      # (T, R, 2N) uint64
        self.check()
        N = self.params.n_slots
        per = np.empty((raw.shape[0], self.batch, N), dtype=np.uint64)
        per[:, 0::2] = raw[:, : (self.batch + 1) // 2, :N]
        if self.batch > 1:
            per[:, 1::2] = raw[:, : self.batch // 2, N:]
        out = self._crt(per)
        return out[0] if self.batch == 1 else out

    def _crt(self, per: np.ndarray) -> np.ndarray:
        """(T, ...) residues mod t_i -> (...) residues mod t (int64 when t fits)."""
        fs = self.evaluator.params.t
        if len(fs) == 1:
            return per[0].astype(np.int64) if self.params.int64_storage else per[0].astype(object)
        t = self.params.t
        acc = np.zeros(per.shape[1:], dtype=object)
        for f, r in zip(fs, per):
            mf = t // f
            acc = acc + r.astype(object) * (mf * pow(mf, -1, f))
        acc = acc % t
        return acc.astype(np.int64) if self.params.int64_storage else acc

    def decrypt_slots(self, ct: SlotCiphertext, m: int) -> np.ndarray:
        """decrypt(ct)[..., :m] without moving or reconstructing the other slots:
        centered values, (m,) for batch 1 else (batch, m).  The device decodes every
        slot; only the first m of each row cross to the host and go through CRT."""
        if not ct.tracked:
            raise ValueError("cannot decrypt a count-only ciphertext")
        N = self.params.n_slots
        if not 0 <= m <= N:
            raise ValueError(f"m must be in [0, {N}], got {m}")
        raw = self.evaluator.decrypt_slots(ct.handle, 0, m)               # (T, R, 2, m)
        self.check()
        per = np.empty((raw.shape[0], self.batch, m), dtype=np.uint64)
        per[:, 0::2] = raw[:, : (self.batch + 1) // 2, 0]
        if self.batch > 1:
            per[:, 1::2] = raw[:, : self.batch // 2, 1]
        res = np.asarray(self._crt(per)).astype(object)
        t = self.params.t
        res[res >= (t + 1) // 2] -= t
        return res[0] if self.batch == 1 else res

    # --------------------------------------------------------------- client
    def encode(self, values) -> PlainVector:
        """Encode signed integers into a plaintext slot vector (hesim.py:203-215)."""
        values = np.asarray(values)
        n, t = self.params.n_slots, self.params.t
        if values.size > n:
            raise CapacityError(f"{values.size} values exceed {n} slots")
        flat = values.ravel()
        if flat.size and flat.dtype != object:
            if flat.dtype.kind in "ib":
                big = int(np.max(np.abs(flat.astype(np.int64))))
            elif flat.dtype.kind == "u":
                big = int(flat.max())
            else:
                big = int(max(abs(int(x)) for x in flat.tolist()))
        else:
            big = int(max(abs(int(flat.min())), abs(int(flat.max())))) if flat.size else 0
        if flat.size and 2 * big >= t:
            raise EncodingOverflowError(f"|value| must be < t/2 = {t / 2}")
        if not flat.size or big < 2 ** 62:
            small = np.zeros(n, dtype=np.int64)       # centered values; residues built lazily
            small[: flat.size] = flat.astype(np.int64)
            return PlainVector(None, self.params, small=small)
        dtype = np.int64 if self.params.int64_storage else object
        slots = np.zeros(n, dtype=dtype)
        res = np.asarray(flat, dtype=object) % t
        slots[: flat.size] = res.astype(np.int64) if self.params.int64_storage else res
        return PlainVector(slots, self.params)

    def encrypt(self, values) -> SlotCiphertext:
        """One slot vector for every image ((k,)), or one per image ((batch, k))."""
        values = np.asarray(values)
        n, t = self.params.n_slots, self.params.t
        per_image = values.ndim == 2
        if per_image and values.shape[0] != self.batch:
            raise ValueError(f"expected {self.batch} slot vectors, got {values.shape[0]}")
        k = values.shape[-1] if values.ndim else values.size
        if k > n:
            raise CapacityError(f"{k} values exceed {n} slots")
        if values.size and int(2 * np.max(np.abs(values.astype(object)))) >= t:
            raise EncodingOverflowError(f"|value| must be < t/2 = {t / 2}")
        mat = np.zeros((self.batch, n), dtype=values.dtype if values.dtype != object else object)
        if per_image:
            mat[:, :k] = values
        elif values.size:
            mat[:, :k] = values.ravel()[None, :]
        res = self._factor_residues(mat)                                  # (T, batch, N)
        handle = self.evaluator.encrypt(self._layout(res))
        return self._wrap(handle, 0)

    def encrypt_zero(self, tracked: bool = True) -> SlotCiphertext:
        if not tracked:
            return SlotCiphertext(None, 0, self.params)
        return self._wrap(self.evaluator.zero(self.rows), 0)

    def encrypt_untracked(self) -> SlotCiphertext:
        return SlotCiphertext(None, 0, self.params)

    def decrypt(self, ct: SlotCiphertext) -> np.ndarray:
        """Centered representatives in [-t/2, t/2), object array (hesim.py:231-238)."""
        if not ct.tracked:
            raise ValueError("cannot decrypt a count-only ciphertext")
        t = self.params.t
        res = np.asarray(self._residues(ct)).astype(object)
        res[res >= (t + 1) // 2] -= t
        return res

    def noise_budget(self, ct: SlotCiphertext) -> float:
        """Minimum remaining invariant-noise budget (bits) over all physical cts."""
        return float(np.min(self.evaluator.noise_budget(ct.handle)))

    # ----------------------------------------------------------- primitives
    def _align(self, a: SlotCiphertext, b: SlotCiphertext):
        """Bring two tracked cts to the same level (mod switch the higher)."""
        ha, hb = a.handle, b.handle
        while ha.level > hb.level:
            ha = self.evaluator.mod_switch(ha)
        while hb.level > ha.level:
            hb = self.evaluator.mod_switch(hb)
        return ha, hb

    def rotate(self, ct: SlotCiphertext, k: int, charge_identity: bool = False) -> SlotCiphertext:
        """Cyclic left rotation: output slot i = input slot (i+k) mod N (hesim.py:244-261)."""
        n = self.params.n_slots
        if not 0 <= k < n:
            raise ValueError(f"rotation amount must be in [0, {n}), got {k}")
        if k != 0 or charge_identity:
            self.counters.rot += 1
        if k == 0:
            if not charge_identity:
                self.elided_rotations += 1
            return ct
        self.rotation_steps.add(k)
        if not ct.tracked:
            return SlotCiphertext(None, ct.depth, ct.params, ct.assembly_depth)
        return self._wrap(self.evaluator.rotate(ct.handle, k), ct.depth, ct.assembly_depth)

    def mul_plain(self, ct: SlotCiphertext, pv: PlainVector | None, assembly: bool = False) -> SlotCiphertext:
        """Slot-wise product mod t; one multiplicative level (hesim.py:263-283)."""
        if assembly:
            self.counters.assembly_mul_pc += 1
        else:
            self.counters.mul_pc += 1
        depth = ct.depth + (0 if assembly else 1)
        adepth = ct.assembly_depth + (1 if assembly else 0)
        if not ct.tracked:
            return SlotCiphertext(None, depth, ct.params, adepth)
        if pv is None:
            raise ValueError("tracked ciphertext requires a plaintext operand")
        out = self.evaluator.mul_plain(ct.handle, self._device_pt(pv))
        return self._wrap(out, depth, adepth)

    def mul_scalar(self, ct: SlotCiphertext, w: int) -> SlotCiphertext:
        """mul_plain by the constant-w plaintext, valid when every slot outside the
        constant's support is zero (ConvPacked columns, packing.py:96-98); tallied
        as one mul_pc like the reference's masked-constant multiply (engine.py:192-193)."""
        self.counters.mul_pc += 1
        depth = ct.depth + 1
        if not ct.tracked:
            return SlotCiphertext(None, depth, ct.params, ct.assembly_depth)
        return self._wrap(self.evaluator.mul_scalar(ct.handle, int(w)), depth, ct.assembly_depth)

    def add_cc(self, a: SlotCiphertext, b: SlotCiphertext) -> SlotCiphertext:
        """Slot-wise sum mod t; depth is the max of the operands (hesim.py:304-316)."""
        if a.params != b.params:
            raise ValueError("ciphertexts come from different schemes")
        self.counters.add_cc += 1
        depth = max(a.depth, b.depth)
        adepth = max(a.assembly_depth, b.assembly_depth)
        if not (a.tracked and b.tracked):
            return SlotCiphertext(None, depth, a.params, adepth)
        ha, hb = self._align(a, b)
        return self._wrap(self.evaluator.add(ha, hb), depth, adepth)

    def add_plain(self, ct: SlotCiphertext, pv: PlainVector | None) -> SlotCiphertext:
        """Plaintext addition; uncounted (hesim.py:318-326)."""
        if not ct.tracked:
            return ct
        if pv is None:
            raise ValueError("tracked ciphertext requires a plaintext operand")
        out = self.evaluator.add_plain(ct.handle, self._device_pt(pv))
        return self._wrap(out, ct.depth, ct.assembly_depth)

    def square(self, ct: SlotCiphertext) -> SlotCiphertext:
        """Slot-wise square mod t (ct x ct multiply + relinearization) (hesim.py:328-345)."""
        self.counters.mul_cc += 1
        depth = ct.depth + 1
        if not ct.tracked:
            return SlotCiphertext(None, depth, ct.params, ct.assembly_depth)
        return self._wrap(self.evaluator.square(ct.handle), depth, ct.assembly_depth)

    def mod_switch(self, ct: SlotCiphertext) -> SlotCiphertext:
        """BFV modulus switch (drop one prime); no reference counterpart, uncounted."""
        if not ct.tracked:
            return ct
        return self._wrap(self.evaluator.mod_switch(ct.handle), ct.depth, ct.assembly_depth)

    def rotate_and_sum(self, ct: SlotCiphertext, m: int) -> SlotCiphertext:
        """slot 0 <- sum of the first m slots; ceil(log2 m) rotations/additions (hesim.py:347-366)."""
        return self.rotate_and_sum_many([ct], m)[0]

    # --------------------------------------------------- batched primitives
    # Same counters and results as issuing the calls one by one; the device
    # work of each list is one launch sequence.
    def mul_plain_many(self, cts, pvs, assembly: bool = False):
        cts = list(cts)
        pvs = list(pvs)
        if assembly:
            self.counters.assembly_mul_pc += len(cts)
        else:
            self.counters.mul_pc += len(cts)
        tracked = [c.tracked for c in cts]
        if not any(tracked):
            return [SlotCiphertext(None, c.depth + (0 if assembly else 1), c.params,
                                   c.assembly_depth + (1 if assembly else 0)) for c in cts]
        if not all(tracked):
            raise ValueError("mixed tracked/untracked operands")
        if any(p is None for p in pvs):
            raise ValueError("tracked ciphertext requires a plaintext operand")
        outs = self.evaluator.mul_plain_many([c.handle for c in cts], [self._device_pt(p) for p in pvs])
        return [self._wrap(o, c.depth + (0 if assembly else 1), c.assembly_depth + (1 if assembly else 0))
                for o, c in zip(outs, cts)]

    def rotate_many(self, cts, k: int):
        cts = list(cts)
        n = self.params.n_slots
        if not 0 <= k < n:
            raise ValueError(f"rotation amount must be in [0, {n}), got {k}")
        if k == 0:
            self.elided_rotations += len(cts)
            return cts
        self.counters.rot += len(cts)
        self.rotation_steps.add(k)
        if not cts[0].tracked:
            return [SlotCiphertext(None, c.depth, c.params, c.assembly_depth) for c in cts]
        groups: dict[int, list[int]] = {}
        for i, c in enumerate(cts):
            groups.setdefault(c.handle.level, []).append(i)
        outs = [None] * len(cts)
        for idx in groups.values():
            res = self.evaluator.rotate_many([cts[i].handle for i in idx], k)
            for i, h in zip(idx, res):
                outs[i] = self._wrap(h, cts[i].depth, cts[i].assembly_depth)
        return outs

    def hoisted_dot(self, rotated, ks, pvs):
        """out[s] = sum_k rotated[k] * rot_{ks[k]}(pvs[s]) where rotated[k] =
        rotate(x, ks[k]) (ks[0] = 0): equal, slot for slot, to sum_k rotate(x * pv_s, ks[k]).
        Counts len(ks) plaintext products and len(ks) - 1 additions per output."""
        rotated, ks, pvs = list(rotated), [int(k) for k in ks], list(pvs)
        S, K = len(pvs), len(ks)
        self.counters.mul_pc += S * K
        self.counters.add_cc += S * (K - 1)
        depth = max(r.depth for r in rotated) + 1
        adepth = max(r.assembly_depth for r in rotated)
        if not rotated[0].tracked:
            return [SlotCiphertext(None, depth, rotated[0].params, adepth) for _ in pvs]
        if any(p is None for p in pvs):
            raise ValueError("tracked ciphertext requires a plaintext operand")
        two_n = 4 * self.params.n_slots
        gs = [pow(5, k, two_n) for k in ks]
        level = min(r.handle.level for r in rotated)
        hs = []
        for r in rotated:
            h = r.handle
            while h.level > level:
                h = self.evaluator.mod_switch(h)
            hs.append(h)
        outs = self.evaluator.hoisted_dot(hs, gs, [self._device_pt(p) for p in pvs])
        return [self._wrap(o, depth, adepth) for o in outs]

    def rotate_multi(self, cts, ks):
        """rotate(cts[i], ks[i]) for every i: same counters and results, one
        batched launch sequence (each ciphertext with its own key)."""
        cts, ks = list(cts), [int(k) for k in ks]
        n = self.params.n_slots
        for k in ks:
            if not 0 <= k < n:
                raise ValueError(f"rotation amount must be in [0, {n}), got {k}")
        outs = list(cts)
        live = [i for i, k in enumerate(ks) if k != 0]
        self.elided_rotations += len(cts) - len(live)
        self.counters.rot += len(live)
        self.rotation_steps.update(ks[i] for i in live)
        if not live:
            return outs
        if not cts[live[0]].tracked:
            for i in live:
                outs[i] = SlotCiphertext(None, cts[i].depth, cts[i].params, cts[i].assembly_depth)
            return outs
        groups: dict[int, list[int]] = {}
        for i in live:
            groups.setdefault(cts[i].handle.level, []).append(i)
        for idx in groups.values():
            res = self.evaluator.rotate_multi([cts[i].handle for i in idx], [ks[i] for i in idx])
            for i, h in zip(idx, res):
                outs[i] = self._wrap(h, cts[i].depth, cts[i].assembly_depth)
        return outs

    def rotate_hoisted(self, ct, ks, charge_identity: bool = False):
        """[rotate(ct, k, charge_identity) for k in ks]: same counters, objects and
        decrypted slots; the nonzero steps share one digit decomposition + ModUp on
        the device (fhe_rotate_hoisted), ciphertext words equal separate rotations."""
        ks = [int(k) for k in ks]
        n = self.params.n_slots
        for k in ks:
            if not 0 <= k < n:
                raise ValueError(f"rotation amount must be in [0, {n}), got {k}")
        outs = [ct] * len(ks)
        for k in ks:
            if k != 0 or charge_identity:
                self.counters.rot += 1
            elif not charge_identity:
                self.elided_rotations += 1
        live = sorted({k for k in ks if k != 0})
        self.rotation_steps.update(live)
        if not live:
            return outs
        if not ct.tracked:
            return [ct if k == 0 else SlotCiphertext(None, ct.depth, ct.params, ct.assembly_depth) for k in ks]
        hs = dict(zip(live, self.evaluator.rotate_hoisted(ct.handle, live)))
        return [ct if k == 0 else self._wrap(hs[k], ct.depth, ct.assembly_depth) for k in ks]

    def add_cc_many(self, a, b):
        a, b = list(a), list(b)
        self.counters.add_cc += len(a)
        if not a[0].tracked:
            return [SlotCiphertext(None, max(x.depth, y.depth), x.params, max(x.assembly_depth, y.assembly_depth))
                    for x, y in zip(a, b)]
        pairs = [self._align(x, y) for x, y in zip(a, b)]
        outs = self.evaluator.add_many([p[0] for p in pairs], [p[1] for p in pairs])
        return [self._wrap(o, max(x.depth, y.depth), max(x.assembly_depth, y.assembly_depth))
                for o, x, y in zip(outs, a, b)]

    def rotate_and_sum_many(self, cts, m: int):
        n = self.params.n_slots
        if not 1 <= m <= n:
            raise ValueError(f"m must be in [1, {n}], got {m}")
        cts = list(cts)
        if (self.debug_checks or self.precondition_checks) and m < n:
            tracked = [ct for ct in cts if ct.tracked]
            for ct in tracked:
                self.evaluator.check_zero_tail(ct.handle, m)
            if self.debug_checks and tracked:
                self.check()                       # immediate, like the reference (hesim.py:360-361)
        rounds = (m - 1).bit_length()
        if rounds == 0:
            return cts
        # ceil(log2 m) rotations and additions per ciphertext (hesim.py:363-365); the device
        # runs every level as one fused launch sequence inside one call (fhe_rotate_and_sum)
        self.counters.rot += rounds * len(cts)
        self.counters.add_cc += rounds * len(cts)
        self.rotation_steps.update(1 << h for h in range(rounds))
        if not cts[0].tracked:
            return [SlotCiphertext(None, c.depth, c.params, c.assembly_depth) for c in cts]
        groups: dict[int, list[int]] = {}
        for i, c in enumerate(cts):
            groups.setdefault(c.handle.level, []).append(i)
        outs = [None] * len(cts)
        for idx in groups.values():
            res = self.evaluator.rotate_and_sum([cts[i].handle for i in idx], m)
            for i, h in zip(idx, res):
                outs[i] = self._wrap(h, cts[i].depth, cts[i].assembly_depth)
        return outs

    def combine(self, cts, lengths):
        """Concatenate slot-0-anchored payloads as a pairwise tree in one device call
        (fhe_combine; packing.tree_combine states the schedule): len - 1 rotations and
        additions, as the reference's chain (packing.py:350-368).  Returns None when the
        operands cannot go down in one call (mixed levels or tracking)."""
        cts, lengths = list(cts), [int(v) for v in lengths]
        n = self.params.n_slots
        if len(cts) < 2 or any(v < 1 for v in lengths) or sum(lengths) > n:
            return None
        tracked = [c.tracked for c in cts]
        if any(tracked) != all(tracked):
            return None
        if tracked[0] and len({c.handle.level for c in cts}) != 1:
            return None
        lens, steps = lengths, []
        while len(lens) > 1:
            nxt = []
            for k in range(0, len(lens) - 1, 2):
                steps.append(n - lens[k])
                nxt.append(lens[k] + lens[k + 1])
            if len(lens) % 2:
                nxt.append(lens[-1])
            lens = nxt
        self.counters.rot += len(steps)
        self.counters.add_cc += len(steps)
        self.rotation_steps.update(steps)
        depth = max(c.depth for c in cts)
        adepth = max(c.assembly_depth for c in cts)
        if not tracked[0]:
            return SlotCiphertext(None, depth, cts[0].params, adepth)
        return self._wrap(self.evaluator.combine([c.handle for c in cts], lengths), depth, adepth)

    def ct_gemm(self, cts, w):
        """out[o] = sum_k w[k][o] * cts[k] in one device pass (fhe_ct_gemm): the ConvPack
        channel sums of engine.py:178-197, tallied as the reference tallies them --
        O*K constant multiplies and O*(K-1) additions.  Valid where mul_scalar is (every
        slot outside the constants' support is zero).  Returns None when the operands
        cannot go down in one call."""
        cts = list(cts)
        K, O = len(cts), len(w[0])
        tracked = [c.tracked for c in cts]
        if any(tracked) != all(tracked):
            return None
        if tracked[0] and len({c.handle.level for c in cts}) != 1:
            return None
        self.counters.mul_pc += O * K
        self.counters.add_cc += O * (K - 1)
        depth = max(c.depth for c in cts) + 1
        adepth = max(c.assembly_depth for c in cts)
        if not tracked[0]:
            return [SlotCiphertext(None, depth, cts[0].params, adepth) for _ in range(O)]
        outs = self.evaluator.ct_gemm([c.handle for c in cts], w)
        return [self._wrap(o, depth, adepth) for o in outs]

    def _rotate_add_many(self, cts, k: int):
        """acc + rotate(acc, k) for every acc: one rotation and one addition each
        (counted as such), fused on the device."""
        self.counters.rot += len(cts)
        self.counters.add_cc += len(cts)
        self.rotation_steps.add(k)
        if not cts[0].tracked:
            return [SlotCiphertext(None, c.depth, c.params, c.assembly_depth) for c in cts]
        groups: dict[int, list[int]] = {}
        for i, c in enumerate(cts):
            groups.setdefault(c.handle.level, []).append(i)
        outs = [None] * len(cts)
        for idx in groups.values():
            res = self.evaluator.rotate_add_many([cts[i].handle for i in idx], k)
            for i, h in zip(idx, res):
                outs[i] = self._wrap(h, cts[i].depth, cts[i].assembly_depth)
        return outs


def merge_contexts(target: HeContext, *others: HeContext) -> HeContext:
    """Fold counters of per-thread contexts into one (hesim.py:376-383)."""
    for other in others:
        if other.params != target.params:
            raise ValueError("contexts use different scheme parameters")
        target.counters.merge(other.counters)
        target.elided_rotations += other.elided_rotations
    return target
