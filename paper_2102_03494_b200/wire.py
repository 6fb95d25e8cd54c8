"""File and wire formats on the inference path.

* CPKW0001 weight files -- the reference's format (weights.py:1-26): magic,
  uint32 manifest length, JSON manifest (name, shape, bits, scale, offset, and a
  sha256 of the data section), then little-endian int32 tensors in row-major
  order.  Files written by the reference load here and vice versa.
* FFCT0001 ciphertext blobs -- one ciphertext object as bytes for storage or
  host-side transport: magic, uint32 header length, JSON header (ring, level,
  row pairs, plaintext moduli, a digest of the parameter set), then the NTT-domain
  words [T*R][2][level][n] as little-endian uint64.  Loading checks the header
  against the receiving evaluator's parameters.
"""

from __future__ import annotations

import hashlib
import json
import struct

import numpy as np

from .netspec import WeightFileError, WeightSet, WeightTensor

WEIGHT_MAGIC = b"CPKW0001"
CT_MAGIC = b"FFCT0001"
_I32 = (-(1 << 31), (1 << 31) - 1)


def save_weights(ws: WeightSet, path) -> None:
    blobs, entries, offset = [], [], 0
    for name in ws.names():
        t = ws[name]
        v = np.asarray(t.values)
        if v.size and (v.min() < _I32[0] or v.max() > _I32[1]):
            raise WeightFileError(f"{name}: entries exceed int32")
        blob = v.astype("<i4").tobytes(order="C")
        entries.append({"name": name, "shape": list(v.shape), "bits": int(t.bits), "scale": repr(float(t.scale)),
                        "offset": offset})
        blobs.append(blob)
        offset += len(blob)
    data = b"".join(blobs)
    manifest = json.dumps({"tensors": entries, "sha256": hashlib.sha256(data).hexdigest()},
                          sort_keys=True).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(WEIGHT_MAGIC + struct.pack("<I", len(manifest)) + manifest + data)


def load_weights(path) -> WeightSet:
    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:8] != WEIGHT_MAGIC:
        raise WeightFileError(f"{path}: not a weight file (bad magic)")
    if len(raw) < 12:
        raise WeightFileError(f"{path}: truncated header")
    (mlen,) = struct.unpack("<I", raw[8:12])
    try:
        manifest = json.loads(raw[12:12 + mlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise WeightFileError(f"{path}: corrupt manifest: {exc}") from exc
    data = raw[12 + mlen:]
    if hashlib.sha256(data).hexdigest() != manifest.get("sha256"):
        raise WeightFileError(f"{path}: data checksum mismatch (corrupt file)")
    ws = WeightSet()
    for e in manifest["tensors"]:
        shape = tuple(e["shape"])
        count = int(np.prod(shape)) if shape else 1
        lo, hi = e["offset"], e["offset"] + 4 * count
        if hi > len(data):
            raise WeightFileError(f"{path}: tensor {e['name']!r} overruns the file")
        vals = np.frombuffer(data[lo:hi], dtype="<i4").astype(np.int64).reshape(shape)
        ws.add(WeightTensor(e["name"], vals, int(e["bits"]), float(e["scale"])))
    return ws


def _params_digest(params) -> str:
    h = hashlib.sha256()
    for part in (params.log_n, params.q, params.p, params.t, params.b, params.seed):
        h.update(repr(part).encode())
    return h.hexdigest()[:32]


def ct_to_bytes(ev, ct) -> bytes:
    words = ev.read(ct)
    header = json.dumps({"log_n": ev.params.log_n, "level": ct.level, "rows": ct.rows, "T": ev.T,
                         "t": [str(x) for x in ev.params.t], "params": _params_digest(ev.params)},
                        sort_keys=True).encode("utf-8")
    return CT_MAGIC + struct.pack("<I", len(header)) + header + words.astype("<u8").tobytes()


def ct_from_bytes(ev, blob: bytes):
    if blob[:8] != CT_MAGIC:
        raise ValueError("not a ciphertext blob (bad magic)")
    (hlen,) = struct.unpack("<I", blob[8:12])
    header = json.loads(blob[12:12 + hlen].decode("utf-8"))
    if header["params"] != _params_digest(ev.params):
        raise ValueError("ciphertext was produced under different parameters")
    ct = ev.new_ct(int(header["rows"]), int(header["level"]))
    words = np.frombuffer(blob[12 + hlen:], dtype="<u8").astype(np.uint64)
    if words.size != ev.words(ct):
        raise ValueError("ciphertext blob has the wrong number of words")
    ev.write(ct, words)
    return ct
