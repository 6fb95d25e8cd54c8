"""Thin object layer over the C ABI: contexts, ciphertext and plaintext handles.

`Evaluator` owns one fhe_ctx (keys, tables, CUDA stream) and hands out
`Ciphertext` / `Plaintext` objects whose device memory is released by a
finalizer.  It speaks residues: slot arrays are uint64 [T][R][n] (one slot
vector per plaintext modulus, per row pair, both rows concatenated).  The
reference-facing API (SchemeParams / HeContext with signed values, counters and
depth) is built on top of it in `hesim.py`.
"""

from __future__ import annotations

import ctypes
import math
import weakref

import numpy as np

from .abi import Library, cuda_library, handle_array, u64_ptr
from .params import RlweParams


class _Handle:
    __slots__ = ("ptr", "_fin", "__weakref__")

    def __init__(self, ptr, destroy, owner):
        self.ptr = ptr
        # keep the owning context alive for as long as the handle lives
        self._fin = weakref.finalize(self, _destroy, destroy, ptr, owner)


def _destroy(fn, ptr, _owner):
    fn(ptr)


class Ciphertext(_Handle):
    """T x R physical BFV ciphertexts at one level (device resident)."""

    __slots__ = ("rows", "level")

    def __init__(self, ev: "Evaluator", rows: int, level: int):
        ptr = ctypes.c_void_p()
        ev.lib.call("fhe_ct_create", ev.ctx, rows, level, ctypes.byref(ptr))
        super().__init__(ptr.value, ev.lib.dll.fhe_ct_destroy, ev._keepalive)
        self.rows = rows
        self.level = level


class Plaintext(_Handle):
    __slots__ = ()

    def __init__(self, ev: "Evaluator"):
        ptr = ctypes.c_void_p()
        ev.lib.call("fhe_pt_create", ev.ctx, ctypes.byref(ptr))
        super().__init__(ptr.value, ev.lib.dll.fhe_pt_destroy, ev._keepalive)


class Graph(_Handle):
    """A captured launch sequence (CUDA graph) and the device arena it writes."""

    __slots__ = ()

    def __init__(self, ev: "Evaluator", ptr):
        super().__init__(ptr, ev.lib.dll.fhe_graph_destroy, ev._keepalive)

    def nodes(self, ev: "Evaluator") -> int:
        v = ctypes.c_uint64()
        ev.lib.call("fhe_graph_nodes", self.ptr, ctypes.byref(v))
        return v.value


class _CtxOwner:
    """Destroys the fhe_ctx once the evaluator and every handle are gone."""

    def __init__(self, lib: Library, ptr):
        self.lib, self.ptr = lib, ptr

    def __del__(self):
        if self.ptr:
            self.lib.dll.fhe_ctx_destroy(self.ptr)
            self.ptr = None


class Evaluator:
    def __init__(self, params: RlweParams, lib: Library | None = None, device: int = 0):
        self.params = params
        self.lib = lib if lib is not None else cuda_library()
        st = params.to_struct(device)
        ptr = ctypes.c_void_p()
        self.lib.call("fhe_ctx_create", ctypes.byref(st), ctypes.byref(ptr))
        self.ctx = ptr.value
        self._keepalive = _CtxOwner(self.lib, self.ctx)
        self._nonce = 0
        self.n = params.n
        self.T = params.T
        self.L = params.L

    # -- objects --------------------------------------------------------
    def new_ct(self, rows: int, level: int | None = None) -> Ciphertext:
        return Ciphertext(self, rows, self.L if level is None else level)

    def zero(self, rows: int, level: int | None = None) -> Ciphertext:
        ct = self.new_ct(rows, level)
        self.lib.call("fhe_ct_zero", self.ctx, ct.ptr)
        return ct

    def words(self, ct: Ciphertext) -> int:
        return self.T * ct.rows * 2 * ct.level * self.n

    def read(self, ct: Ciphertext) -> np.ndarray:
        out = np.empty(self.words(ct), dtype=np.uint64)
        self.lib.call("fhe_ct_read", self.ctx, ct.ptr, u64_ptr(out))
        return out.reshape(self.T * ct.rows, 2, ct.level, self.n)

    def write(self, ct: Ciphertext, words: np.ndarray) -> None:
        w = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1)
        if w.size != self.words(ct):
            raise ValueError("word count does not match the ciphertext shape")
        self.lib.call("fhe_ct_write", self.ctx, ct.ptr, u64_ptr(w))

    def export_words(self, ct: Ciphertext, ptr: int) -> None:
        """Copy the ciphertext words into caller-owned device memory at `ptr`."""
        self.lib.call("fhe_ct_to_device", self.ctx, ct.ptr, ctypes.c_void_p(ptr))

    def import_words(self, ct: Ciphertext, ptr: int) -> None:
        self.lib.call("fhe_ct_from_device", self.ctx, ct.ptr, ctypes.c_void_p(ptr))

    def encode(self, slots: np.ndarray) -> Plaintext:
        s = np.ascontiguousarray(slots, dtype=np.uint64)
        if s.shape != (self.T, self.n):
            raise ValueError(f"plaintext slots must have shape {(self.T, self.n)}")
        pt = Plaintext(self)
        self.lib.call("fhe_encode", self.ctx, u64_ptr(s), pt.ptr)
        return pt

    def pt_words(self, pt: Plaintext) -> np.ndarray:
        out = np.empty(self.T * self.L * self.n, dtype=np.uint64)
        self.lib.call("fhe_pt_read", self.ctx, pt.ptr, u64_ptr(out))
        return out.reshape(self.T, self.L, self.n)

    def encrypt(self, slots: np.ndarray, nonce: int | None = None, async_: bool = False) -> Ciphertext:
        """Encrypt [T][R][n] residues.  With a page-locked `slots` buffer and
        async_=True the host->device copy runs on the library's copy stream and
        the call returns at once: `slots` must stay untouched until sync().
        Otherwise the call returns only after the input has been read."""
        s = np.ascontiguousarray(slots, dtype=np.uint64)
        if s.ndim != 3 or s.shape[0] != self.T or s.shape[2] != self.n:
            raise ValueError(f"slots must have shape (T={self.T}, R, n={self.n})")
        if nonce is None:
            nonce = self._nonce
            if nonce > 0xFFFFFFFF:
                raise RuntimeError("encryption nonces exhausted (2^32 encryptions per context)")
            self._nonce += 1
        ct = self.new_ct(s.shape[1])
        self.lib.call("fhe_encrypt", self.ctx, u64_ptr(s), nonce & 0xFFFFFFFF, ct.ptr)
        if not async_:
            self.sync()
        return ct

    def decrypt(self, ct: Ciphertext, out: np.ndarray | None = None, async_: bool = False) -> np.ndarray:
        """Decrypted [T][R][n] residues.  With a page-locked `out` and async_=True
        the device->host copy is only enqueued: `out` is valid after sync()."""
        if out is None:
            out = np.empty((self.T, ct.rows, self.n), dtype=np.uint64)
        elif out.dtype != np.uint64 or out.size != self.T * ct.rows * self.n or not out.flags["C_CONTIGUOUS"]:
            raise ValueError("decrypt: out must be a contiguous uint64 array of T*R*n words")
        self.lib.call("fhe_decrypt", self.ctx, ct.ptr, u64_ptr(out))
        if not async_:
            self.sync()
        return out.reshape(self.T, ct.rows, self.n)

    def decrypt_slots(self, ct: Ciphertext, lo: int, cnt: int) -> np.ndarray:
        """Residues of slots [lo, lo + cnt) of both rows: [T][R][2][cnt] (synchronous)."""
        out = np.empty((self.T, ct.rows, 2, cnt), dtype=np.uint64)
        self.lib.call("fhe_decrypt_slots", self.ctx, ct.ptr, int(lo), int(cnt), u64_ptr(out))
        return out

    def check_zero_tail(self, ct: Ciphertext, m: int) -> None:
        """Enqueue the rotate_and_sum precondition check (slots >= m zero); a
        violation shows up in status()."""
        self.lib.call("fhe_check_zero_tail", self.ctx, ct.ptr, int(m))

    def status(self, reset: bool = True) -> tuple[float, int]:
        """(smallest noise budget in bits seen by decryptions since the last
        reset, sticky check flags); synchronizes the context's stream."""
        d, f = ctypes.c_uint32(), ctypes.c_uint32()
        self.lib.call("fhe_status", self.ctx, ctypes.byref(d), ctypes.byref(f), int(reset))
        # distance d / 2^32 to the nearest integer: budget = -log2(2 d / 2^32)
        budget = 31.0 - math.log2(d.value) if d.value else 32.0
        return budget, f.value

    def decrypt_raw(self, ct: Ciphertext) -> np.ndarray:
        out = np.empty((self.T * ct.rows, ct.level, self.n), dtype=np.uint64)
        self.lib.call("fhe_decrypt_raw", self.ctx, ct.ptr, u64_ptr(out))
        return out

    def noise_budget(self, ct: Ciphertext) -> np.ndarray:
        """Exact remaining invariant-noise budget in bits, per physical ct:
        -log2(2 max|v|) with t x / Q = m + v, i.e. log2(Q) - 1 - log2 max|[t x]_Q|."""
        raw = self.decrypt_raw(ct)
        q = [int(v) for v in self.params.q[: ct.level]]
        Q = 1
        for v in q:
            Q *= v
        basis = [(Q // qi) * pow(Q // qi, -1, qi) for qi in q]
        out = np.empty(raw.shape[0])
        for ci in range(raw.shape[0]):
            t = int(self.params.t[ci // ct.rows])
            x = np.zeros(self.n, dtype=object)
            for i, bi in enumerate(basis):
                x = x + raw[ci, i].astype(object) * bi
            z = (x * t) % Q
            z = np.where(z > Q // 2, Q - z, z)
            worst = max(int(v) for v in z)
            out[ci] = math.log2(Q) - 1 - (math.log2(worst) if worst else 0.0)
        return out.reshape(self.T, ct.rows)

    # -- evaluation -------------------------------------------------------
    def add(self, a: Ciphertext, b: Ciphertext, out: Ciphertext | None = None) -> Ciphertext:
        out = out or self.new_ct(a.rows, a.level)
        self.lib.call("fhe_add", self.ctx, a.ptr, b.ptr, out.ptr)
        return out

    def mul_plain(self, a: Ciphertext, pt: Plaintext, out: Ciphertext | None = None) -> Ciphertext:
        out = out or self.new_ct(a.rows, a.level)
        self.lib.call("fhe_mul_plain", self.ctx, a.ptr, pt.ptr, out.ptr)
        return out

    def mul_plain_acc(self, a: Ciphertext, pt: Plaintext, acc: Ciphertext) -> Ciphertext:
        """acc += a * pt in place (fused HMA); returns acc."""
        self.lib.call("fhe_mul_plain_acc", self.ctx, a.ptr, pt.ptr, acc.ptr)
        return acc

    def mul_scalar(self, a: Ciphertext, w: int, out: Ciphertext | None = None) -> Ciphertext:
        out = out or self.new_ct(a.rows, a.level)
        self.lib.call("fhe_mul_scalar", self.ctx, a.ptr, int(w), out.ptr)
        return out

    def add_plain(self, a: Ciphertext, pt: Plaintext, out: Ciphertext | None = None) -> Ciphertext:
        out = out or self.new_ct(a.rows, a.level)
        self.lib.call("fhe_add_plain", self.ctx, a.ptr, pt.ptr, out.ptr)
        return out

    def rotate(self, a: Ciphertext, k: int) -> Ciphertext:
        out = self.new_ct(a.rows, a.level)
        self.lib.call("fhe_rotate", self.ctx, a.ptr, int(k), out.ptr)
        return out

    def mod_switch(self, a: Ciphertext) -> Ciphertext:
        out = self.new_ct(a.rows, a.level - 1)
        self.lib.call("fhe_mod_switch", self.ctx, a.ptr, out.ptr)
        return out

    def square(self, a: Ciphertext) -> Ciphertext:
        out = self.new_ct(a.rows, a.level)
        self.lib.call("fhe_square", self.ctx, a.ptr, out.ptr)
        return out

    def rotate_many(self, cts, k: int) -> list[Ciphertext]:
        outs = [self.new_ct(c.rows, c.level) for c in cts]
        self.lib.call("fhe_rotate_many", self.ctx, handle_array([c.ptr for c in cts]),
                      handle_array([o.ptr for o in outs]), len(cts), int(k))
        return outs

    def rotate_add_many(self, cts, k: int) -> list[Ciphertext]:
        """out[i] = cts[i] + rotate(cts[i], k), fused."""
        outs = [self.new_ct(c.rows, c.level) for c in cts]
        self.lib.call("fhe_rotate_add_many", self.ctx, handle_array([c.ptr for c in cts]),
                      handle_array([o.ptr for o in outs]), len(cts), int(k))
        return outs

    def rotate_multi(self, cts, ks) -> list[Ciphertext]:
        outs = [self.new_ct(c.rows, c.level) for c in cts]
        arr = (ctypes.c_uint32 * len(ks))(*[int(k) for k in ks])
        self.lib.call("fhe_rotate_multi", self.ctx, handle_array([c.ptr for c in cts]),
                      handle_array([o.ptr for o in outs]), arr, len(cts))
        return outs

    def rotate_hoisted(self, ct, ks) -> list[Ciphertext]:
        """rotate(ct, k) for every k, one shared digit decomposition + ModUp."""
        outs = [self.new_ct(ct.rows, ct.level) for _ in ks]
        arr = (ctypes.c_uint32 * len(ks))(*[int(k) for k in ks])
        self.lib.call("fhe_rotate_hoisted", self.ctx, ct.ptr, arr, len(ks), handle_array([o.ptr for o in outs]))
        return outs

    def hoisted_dot(self, R, gs, pts) -> list[Ciphertext]:
        """out[s] = sum_k R[k] * tau_{gs[k]}(pts[s])."""
        outs = [self.new_ct(R[0].rows, R[0].level) for _ in pts]
        arr = (ctypes.c_uint32 * len(gs))(*[int(g) for g in gs])
        self.lib.call("fhe_hoisted_dot", self.ctx, handle_array([r.ptr for r in R]), arr, len(R),
                      handle_array([p.ptr for p in pts]), len(pts), handle_array([o.ptr for o in outs]))
        return outs

    def mul_plain_many(self, cts, pts) -> list[Ciphertext]:
        outs = [self.new_ct(c.rows, c.level) for c in cts]
        self.lib.call("fhe_mul_plain_many", self.ctx, handle_array([c.ptr for c in cts]),
                      handle_array([p.ptr for p in pts]), handle_array([o.ptr for o in outs]),
                      len(cts))
        return outs

    def add_many(self, a, b) -> list[Ciphertext]:
        outs = [self.new_ct(c.rows, c.level) for c in a]
        self.lib.call("fhe_add_many", self.ctx, handle_array([c.ptr for c in a]),
                      handle_array([c.ptr for c in b]), handle_array([o.ptr for o in outs]),
                      len(a))
        return outs

    def rotate_and_sum(self, cts, span: int) -> list[Ciphertext]:
        """slot 0 of out[i] <- sum of the first `span` slots of cts[i]; every tree level is
        one fused rotate-and-add launch sequence over all objects (fhe_rotate_and_sum)."""
        outs = [self.new_ct(c.rows, c.level) for c in cts]
        self.lib.call("fhe_rotate_and_sum", self.ctx, handle_array([c.ptr for c in cts]),
                      handle_array([o.ptr for o in outs]), len(cts), int(span))
        return outs

    def combine(self, cts, lengths) -> Ciphertext:
        """Tree concatenation of slot-0-anchored payloads (fhe_combine)."""
        out = self.new_ct(cts[0].rows, cts[0].level)
        arr = (ctypes.c_uint32 * len(lengths))(*[int(v) for v in lengths])
        self.lib.call("fhe_combine", self.ctx, handle_array([c.ptr for c in cts]), arr, len(cts), out.ptr)
        return out

    def ct_gemm(self, cts, w) -> list[Ciphertext]:
        """out[o] = sum_k w[k][o] * cts[k] (fhe_ct_gemm); w is a K x O integer matrix."""
        K, O = len(cts), len(w[0])
        flat = [int(w[k][o]) for k in range(K) for o in range(O)]
        arr = (ctypes.c_int64 * len(flat))(*flat)
        outs = [self.new_ct(cts[0].rows, cts[0].level) for _ in range(O)]
        self.lib.call("fhe_ct_gemm", self.ctx, handle_array([c.ptr for c in cts]), K, arr, O,
                      handle_array([o.ptr for o in outs]))
        return outs

    def debug_rotate_stages(self, ct: Ciphertext, k: int):
        """(digits [c][l][n], ext [c][l][l+1][n], acc [c][2][l+1][n]) of rotate(ct, k)'s key
        switch, c = T * rows physical ciphertexts (fhe_debug_rotate_stages; tests only)."""
        c, l = self.T * ct.rows, ct.level
        digits = np.empty((c, l, self.n), dtype=np.uint64)
        ext = np.empty((c, l, l + 1, self.n), dtype=np.uint64)
        acc = np.empty((c, 2, l + 1, self.n), dtype=np.uint64)
        self.lib.call("fhe_debug_rotate_stages", self.ctx, ct.ptr, int(k), u64_ptr(digits), u64_ptr(ext), u64_ptr(acc))
        return digits, ext, acc

    def copy(self, src: Ciphertext, dst: Ciphertext) -> None:
        """dst <- src words on the device (same rows and level), asynchronous."""
        self.lib.call("fhe_ct_copy", self.ctx, src.ptr, dst.ptr)

    def peak_bytes(self, reset: bool = False) -> int:
        v = ctypes.c_uint64()
        self.lib.call("fhe_ctx_peak_bytes", self.ctx, ctypes.byref(v), int(reset))
        return v.value

    def capture_begin(self, arena_bytes: int) -> None:
        self.lib.call("fhe_capture_begin", self.ctx, int(arena_bytes))

    def capture_end(self) -> "Graph":
        ptr = ctypes.c_void_p()
        self.lib.call("fhe_capture_end", self.ctx, ctypes.byref(ptr))
        return Graph(self, ptr.value)

    def launch(self, graph: "Graph") -> None:
        self.lib.call("fhe_graph_launch", self.ctx, graph.ptr)

    def keygen_rotations(self, steps) -> None:
        arr = (ctypes.c_uint32 * len(steps))(*[int(s) for s in steps])
        self.lib.call("fhe_keygen_rotations", self.ctx, arr, len(steps))

    def key_bytes(self) -> int:
        v = ctypes.c_uint64()
        self.lib.call("fhe_ctx_key_bytes", self.ctx, ctypes.byref(v))
        return v.value

    def sync(self) -> None:
        self.lib.call("fhe_sync", self.ctx)
