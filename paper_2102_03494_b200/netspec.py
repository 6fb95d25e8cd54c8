"""Network descriptions and weight sets.

Mirrors the parts of `cipherpack.netspec` (/root/reference/pkg/src/cipherpack/netspec.py)
and `cipherpack.weights` (weights.py) that the encrypted-inference path consumes:
`LayerSpec`, `NetworkSpec` with eager shape validation and the slot-capacity
check (netspec.py:63-121), the JSON document form (netspec.py:1-18, 124-172),
`WeightTensor` / `WeightSet` with the runner's tensor naming (weights.py:17-25),
`required_tensors`, `validate_weights`, `random_weights` (weights.py:156-194).
The CPKW0001 binary file format and the CLI are out of scope.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np

from .hesim import SchemeParams
from .packing import KernelSpec, TensorShape

LAYER_KINDS = ("conv", "ffconv", "fc", "square", "avgpool")
FFCONV_PATTERNS = ("dp-hi2c-cp", "cp-hi2c-cp", "dp-dp", "cp-hi2c-dp")


class NetworkError(ValueError):
    """Schema or shape violation, naming the offending layer."""


class WeightFileError(ValueError):
    pass


@dataclass(frozen=True)
class LayerSpec:
    kind: str
    d: int | None = None
    stride: int = 1
    out_channels: int | None = None
    rank: int | None = None
    packing_hint: str | None = None

    def kernel(self) -> KernelSpec:
        if self.kind not in ("conv", "ffconv", "avgpool"):
            raise NetworkError(f"layer kind {self.kind} has no kernel")
        return KernelSpec(d=self.d, stride=self.stride, out_channels=self.out_channels or 1)


def _next_shape(layer: LayerSpec, shape: TensorShape) -> TensorShape:
    kind = layer.kind
    if kind == "square":
        return shape
    if kind == "fc":
        if not layer.out_channels:
            raise ValueError("fc needs out_channels")
        return TensorShape(1, 1, layer.out_channels)
    if kind == "avgpool":
        if not layer.d:
            raise ValueError("avgpool needs a window size d")
        return KernelSpec(layer.d, layer.stride, shape.c).out_shape(shape)
    if kind in ("conv", "ffconv"):
        if not layer.d or not layer.out_channels:
            raise ValueError("conv needs d and out_channels")
        kernel = layer.kernel()
        if kind == "ffconv":
            k = kernel.k_columns(shape.c)
            if layer.rank is None:
                raise ValueError("ffconv needs a rank")
            if not 1 <= layer.rank <= min(k, layer.out_channels):
                raise ValueError(f"rank {layer.rank} outside [1, {min(k, layer.out_channels)}]")
        elif layer.rank is not None:
            raise ValueError("rank is only meaningful for ffconv layers")
        if layer.packing_hint is not None:
            allowed = FFCONV_PATTERNS if kind == "ffconv" else ("dense", "conv")
            if layer.packing_hint not in allowed:
                raise ValueError(f"packing_hint must be one of {allowed}")
        return kernel.out_shape(shape)
    raise ValueError(f"unknown layer kind {kind!r}")


@dataclass(frozen=True)
class NetworkSpec:
    scheme: SchemeParams
    input_shape: TensorShape
    layers: tuple
    version: int = 1

    def __post_init__(self):
        self.layer_shapes()

    def layer_shapes(self) -> list[TensorShape]:
        n = self.scheme.n_slots
        shape = self.input_shape
        if shape.size > n:
            raise NetworkError(f"input of {shape.size} elements exceeds {n} slots")
        out = []
        for i, layer in enumerate(self.layers):
            try:
                shape = _next_shape(layer, shape)
            except (ValueError, TypeError) as exc:
                raise NetworkError(f"layer {i} ({layer.kind}): {exc}") from exc
            if shape.size > n:
                raise NetworkError(f"layer {i} ({layer.kind}): output of {shape.size} elements exceeds {n} slots")
            out.append(shape)
        return out


def network_from_dict(doc: dict) -> NetworkSpec:
    try:
        version, sch, shp, lays = doc["version"], doc["scheme"], doc["input_shape"], doc["layers"]
    except (KeyError, TypeError) as exc:
        raise NetworkError(f"missing required field: {exc}") from exc
    if version != 1:
        raise NetworkError(f"unsupported version {version!r}")
    t = sch["t"]
    if isinstance(t, list):
        factors = tuple(int(f) for f in t)
        tval = math.prod(factors)
    elif isinstance(t, str):
        factors, tval = None, int(t)
    else:
        raise NetworkError("scheme.t must be a decimal string or a list of factor strings")
    scheme = SchemeParams(n_slots=int(sch["N"]), t=tval, rotation_weight=float(sch.get("rotation_weight", 10.0)),
                          t_factors=factors)
    layers = []
    for i, ld in enumerate(lays):
        if not isinstance(ld, dict) or "kind" not in ld:
            raise NetworkError(f"layer {i}: expected an object with a 'kind'")
        if ld["kind"] not in LAYER_KINDS:
            raise NetworkError(f"layer {i}: unknown kind {ld['kind']!r}")
        layers.append(LayerSpec(ld["kind"], ld.get("d"), int(ld.get("stride", 1)), ld.get("out_channels"),
                                ld.get("rank"), ld.get("packing_hint")))
    return NetworkSpec(scheme, TensorShape(int(shp["w"]), int(shp["h"]), int(shp["c"])), tuple(layers))


def network_to_dict(net: NetworkSpec) -> dict:
    t = [str(f) for f in net.scheme.t_factors] if net.scheme.t_factors else str(net.scheme.t)
    return {
        "version": net.version,
        "scheme": {"N": net.scheme.n_slots, "t": t, "rotation_weight": net.scheme.rotation_weight},
        "input_shape": {"w": net.input_shape.w, "h": net.input_shape.h, "c": net.input_shape.c},
        "layers": [{k: v for k, v in (("kind", l.kind), ("d", l.d), ("stride", l.stride),
                                      ("out_channels", l.out_channels), ("rank", l.rank),
                                      ("packing_hint", l.packing_hint)) if v is not None}
                   for l in net.layers],
    }


def load_network(path) -> NetworkSpec:
    with open(path, "r", encoding="utf-8") as fh:
        try:
            doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise NetworkError(f"{path}: not valid JSON: {exc}") from exc
    return network_from_dict(doc)


def save_network(net: NetworkSpec, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(network_to_dict(net), fh, indent=2, sort_keys=True)
        fh.write("\n")


# ------------------------------------------------------------------ weights

@dataclass(frozen=True)
class WeightTensor:
    name: str
    values: np.ndarray
    bits: int
    scale: float


class WeightSet:
    """Ordered named integer tensors (weights.py:59-99)."""

    def __init__(self, tensors=None):
        self._t: dict[str, WeightTensor] = {}
        for t in tensors or []:
            self.add(t)

    def add(self, t: WeightTensor) -> None:
        if t.name in self._t:
            raise WeightFileError(f"duplicate tensor {t.name!r}")
        self._t[t.name] = t

    def __contains__(self, name) -> bool:
        return name in self._t

    def __getitem__(self, name) -> WeightTensor:
        try:
            return self._t[name]
        except KeyError:
            raise WeightFileError(f"missing tensor {name!r}") from None

    def names(self) -> list[str]:
        return list(self._t)


def required_tensors(net: NetworkSpec) -> dict:
    """name -> shape: conv (d, d, in_c, out_c); ffconv w1 (d, d, in_c, r), w2 (1, 1, r, out_c);
    fc weight (m, out_c), bias (out_c,) (weights.py:156-173)."""
    shapes, cur = {}, net.input_shape
    for i, layer in enumerate(net.layers):
        if layer.kind == "conv":
            shapes[f"layer{i}.weight"] = (layer.d, layer.d, cur.c, layer.out_channels)
        elif layer.kind == "ffconv":
            shapes[f"layer{i}.w1"] = (layer.d, layer.d, cur.c, layer.rank)
            shapes[f"layer{i}.w2"] = (1, 1, layer.rank, layer.out_channels)
        elif layer.kind == "fc":
            shapes[f"layer{i}.weight"] = (cur.size, layer.out_channels)
            shapes[f"layer{i}.bias"] = (layer.out_channels,)
        cur = _next_shape(layer, cur)
    return shapes


def validate_weights(net: NetworkSpec, ws: WeightSet) -> None:
    for name, shape in required_tensors(net).items():
        if name not in ws:
            raise WeightFileError(f"{name}: tensor missing from weight file")
        if ws[name].values.shape != shape:
            raise WeightFileError(f"{name}: expected shape {shape}, found {ws[name].values.shape}")


def random_weights(net: NetworkSpec, rng: np.random.Generator, bits: int = 8, bound: int | None = None) -> WeightSet:
    """Uniform integer weights in [-bound, bound] (weights.py:186-194)."""
    limit = bound if bound is not None else 2 ** (bits - 1) - 1
    ws = WeightSet()
    for name, shape in required_tensors(net).items():
        ws.add(WeightTensor(name, rng.integers(-limit, limit + 1, size=shape), bits, 1.0 / max(limit, 1)))
    return ws


def quantize_matrix(w: np.ndarray, bits: int):
    """Symmetric per-tensor quantization, round half away from zero
    (factorize.py:115-128): returns (int entries, scale)."""
    w = np.asarray(w, dtype=np.float64)
    peak = float(np.max(np.abs(w))) if w.size else 0.0
    if peak == 0.0:
        return np.zeros_like(w, dtype=np.int64), 1.0
    scale = peak / (2 ** (bits - 1) - 1)
    q = np.sign(w / scale) * np.floor(np.abs(w / scale) + 0.5)
    return q.astype(np.int64), scale


def synthetic_weights(net: NetworkSpec, rng: np.random.Generator, sigma: float, bits: int = 8) -> WeightSet:
    """BASELINE weights: N(0, sigma) per tensor -> 8-bit symmetric quantization;
    biases zero."""
    ws = WeightSet()
    for name, shape in required_tensors(net).items():
        if name.endswith(".bias"):
            ws.add(WeightTensor(name, np.zeros(shape, dtype=np.int64), bits, 1.0))
            continue
        q, scale = quantize_matrix(rng.normal(0.0, sigma, size=shape), bits)
        ws.add(WeightTensor(name, q, bits, scale))
    return ws
