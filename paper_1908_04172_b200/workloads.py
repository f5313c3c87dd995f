# SPDX-License-Identifier: Apache-2.0
"""BASELINE.json workloads as reference-format models (JSON manifest + f32
blob, the format load_model parses: henet/graph.hpp:236-295) and parameter
sets.  Shared by the parity tests and bench.py so both arms run the identical
graph, weights and parameters.

Parameters (BASELINE.md s2 / SURVEY H1): the chains are the largest primes
= 1 mod 2N below 2^b; contexts are built by field assignment because scale 2^24
exceeds the 24-bit primes (the checked constructor would reject it).
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

# N = 8192, chain [30, 24 x 5] bits + 30-bit special, scale 2^24 (configs 1-3, 5a)
N8192 = dict(
    n=8192,
    chain=[1073692673, 16760833, 16580609, 16515073, 16465921, 16384001],
    special=1073643521,
    scale=float(2 ** 24),
)
# N = 16384, chain [40, 30 x 7] + 40-bit special, scale 2^30 (configs 4, 5b) -- 40-bit
# limbs are outside what the round-1 kernels implement.
N16384 = dict(
    n=16384,
    chain=[1099510054913, 1073643521, 1073479681, 1073184769, 1073053697, 1072857089, 1072496641, 1071513601],
    special=1099508121601,
    scale=float(2 ** 30),
)


# The reference's own parameter presets, make_parameters (henet/params.hpp:74-101): P11 has
# no special prime (0 here); P12-P14 use primes above 2^30 (u64 residues on the GPU path).
PRESETS = {
    "P11": dict(n=2048, chain=[18014398509404161], special=0, scale=float(2 ** 24)),
    "P12": dict(n=4096, chain=[1073750017, 1073815553, 1073872897], special=1099511799809, scale=float(2 ** 30)),
    "P13": dict(n=8192, chain=[1125899906990081, 1099511922689, 1099512004609, 1099512266753, 1099512299521,
                              1099512365057], special=1125899907219457, scale=float(2 ** 40)),
    "P14": dict(n=16384, chain=[1125899908022273, 1099511922689, 1099512938497, 1099514314753, 1099514478593,
                               1099515691009, 1099515789313, 1099515985921], special=1125899908612097,
                scale=float(2 ** 40)),
}


class Blob:
    """Mirror of the reference's BlobBuilder layout (henet/models.hpp:22-61): one
    little-endian f32 blob, entries at 4-byte offsets."""

    def __init__(self):
        self.parts: List[bytes] = []
        self.offset = 0
        self.table = {}

    def add(self, name: str, shape: List[int], values: np.ndarray) -> None:
        v = np.ascontiguousarray(values, dtype="<f4").reshape(-1)
        assert v.size == int(np.prod(shape))
        self.table[name] = {"offset": self.offset, "shape": list(shape)}
        b = v.tobytes()
        self.parts.append(b)
        self.offset += len(b)

    def bytes(self) -> bytes:
        return b"".join(self.parts)


def _node(nid, op, inputs=(), attrs=None, weight_ref="", bias_ref=""):
    n = {"id": nid, "op": op}
    if inputs:
        n["inputs"] = list(inputs)
    if attrs:
        n["attrs"] = attrs
    if weight_ref:
        n["weight_ref"] = weight_ref
    if bias_ref:
        n["bias_ref"] = bias_ref
    return n


@dataclass
class Workload:
    name: str
    manifest: str
    blob: bytes
    input_shape: List[int]
    packing: int           # 0 real, 1 complex
    batch: int             # images per ciphertext
    patch_terminal_rescale: bool = False  # config 1: force one rescale per output

    @property
    def input_count(self) -> int:
        return int(np.prod(self.input_shape))


def _gauss(rng: np.random.Generator, shape, sigma) -> np.ndarray:
    return (rng.standard_normal(int(np.prod(shape))) * sigma).astype(np.float32)


def dense_layer(seed: int = 1, k: int = 845, m: int = 100, batch: int = 4096, packing: int = 0,
                w_scale: float = 1.0) -> Workload:
    """Config 1: single encrypted dense layer 845 -> 100 with bias, W ~ N(0, 0.05^2),
    b ~ N(0, 0.01^2); one lazy rescale per output (patched plan).  packing=1: complex
    packing (two images per slot), the bias encoded by encode_vector.  w_scale = 0: all-zero
    weights (the output decrypts to the bias alone, proj/tests/test_graph.cpp:247)."""
    rng = np.random.default_rng(seed)
    blob = Blob()
    blob.add("fc_w", [k, m], (_gauss(rng, (k, m), 0.05) * np.float32(w_scale)).astype(np.float32))
    blob.add("fc_b", [m], _gauss(rng, (m,), 0.01))
    j = {
        "name": "dense-845-100",
        "packing": "complex" if packing else "real",
        "preset": "P13",
        "weights": blob.table,
        "nodes": [
            _node("input", "Input", attrs={"shape": [k]}),
            _node("fc", "Dot", ["input"], weight_ref="fc_w", bias_ref="fc_b"),
            _node("out", "Output", ["fc"]),
        ],
    }
    return Workload("c1_dense_845_100", json.dumps(j), blob.bytes(), [k], packing, batch, patch_terminal_rescale=True)


def cryptonets(seed: int = 2, batch: int = 4096, sigma: float = 0.05) -> Workload:
    """Config 2: conv 5x5/2 pad {0,0,1,1} 5 filters -> square -> flatten(845) ->
    dense 845->100 -> square -> dense 100->10 (make_cryptonets topology,
    henet/models.hpp:83-106) with N(0, sigma^2) weights."""
    rng = np.random.default_rng(seed)
    blob = Blob()
    blob.add("conv1_w", [5, 1, 5, 5], _gauss(rng, (5, 1, 5, 5), sigma))
    blob.add("fc1_w", [845, 100], _gauss(rng, (845, 100), sigma))
    blob.add("fc2_w", [100, 10], _gauss(rng, (100, 10), sigma))
    j = {
        "name": "cryptonets",
        "packing": "real",
        "preset": "P13",
        "weights": blob.table,
        "nodes": [
            _node("input", "Input", attrs={"shape": [1, 28, 28]}),
            _node("conv1", "Convolution", ["input"], {"stride": 2, "window": 5, "filters": 5, "pad": [0, 0, 1, 1]},
                  "conv1_w"),
            _node("act1", "Square", ["conv1"]),
            _node("flatten", "Reshape", ["act1"], {"shape": [845]}),
            _node("fc1", "Dot", ["flatten"], weight_ref="fc1_w"),
            _node("act2", "Square", ["fc1"]),
            _node("fc2", "Dot", ["act2"], weight_ref="fc2_w"),
            _node("out", "Output", ["fc2"]),
        ],
    }
    return Workload("c2_cryptonets", json.dumps(j), blob.bytes(), [1, 28, 28], 0, batch)


def cryptonets_relu(seed: int = 3, batch: int = 8192, sigma: float = 0.05, packing: int = 1) -> Workload:
    """Config 3: the CryptoNets-ReLU topology (henet/models.hpp:110-136)
    with biases and client-aided ReLU, complex packing (two images per slot)."""
    rng = np.random.default_rng(seed)
    blob = Blob()
    blob.add("conv1_w", [5, 1, 5, 5], _gauss(rng, (5, 1, 5, 5), sigma))
    blob.add("conv1_b", [5], _gauss(rng, (5,), 0.01))
    blob.add("fc1_w", [845, 100], _gauss(rng, (845, 100), sigma))
    blob.add("fc1_b", [100], _gauss(rng, (100,), 0.01))
    blob.add("fc2_w", [100, 10], _gauss(rng, (100, 10), sigma))
    blob.add("fc2_b", [10], _gauss(rng, (10,), 0.01))
    j = {
        "name": "cryptonets-relu",
        "packing": "complex" if packing else "real",
        "preset": "P13",
        "weights": blob.table,
        "nodes": [
            _node("input", "Input", attrs={"shape": [1, 28, 28]}),
            _node("conv1", "Convolution", ["input"], {"stride": 2, "window": 5, "filters": 5, "pad": [0, 0, 1, 1]},
                  "conv1_w", "conv1_b"),
            _node("act1", "Relu", ["conv1"]),
            _node("flatten", "Reshape", ["act1"], {"shape": [845]}),
            _node("fc1", "Dot", ["flatten"], weight_ref="fc1_w", bias_ref="fc1_b"),
            _node("act2", "Relu", ["fc1"]),
            _node("fc2", "Dot", ["act2"], weight_ref="fc2_w", bias_ref="fc2_b"),
            _node("out", "Output", ["fc2"]),
        ],
    }
    return Workload("c3_cryptonets_relu_complex" if packing else "c3_cryptonets_relu_real", json.dumps(j),
                    blob.bytes(), [1, 28, 28], packing, batch)


def toy_cryptonets(seed: int = 4, batch: int = 64) -> Workload:
    """Scaled-down conv->square->fc->square->fc (make_cryptonets_shaped_toy shape,
    henet/models.hpp:206-228) for fast parity runs."""
    rng = np.random.default_rng(seed)
    blob = Blob()
    blob.add("conv_w", [2, 1, 3, 3], _gauss(rng, (2, 1, 3, 3), 0.3))
    blob.add("fc1_w", [18, 4], _gauss(rng, (18, 4), 0.25))
    blob.add("fc2_w", [4, 2], _gauss(rng, (4, 2), 0.5))
    j = {
        "name": "cryptonets-toy",
        "packing": "real",
        "preset": "P13",
        "weights": blob.table,
        "nodes": [
            _node("input", "Input", attrs={"shape": [1, 8, 8]}),
            _node("conv", "Convolution", ["input"], {"stride": 2, "window": 3, "filters": 2}, "conv_w"),
            _node("act1", "Square", ["conv"]),
            _node("flatten", "Reshape", ["act1"], {"shape": [18]}),
            _node("fc1", "Dot", ["flatten"], weight_ref="fc1_w"),
            _node("act2", "Square", ["fc1"]),
            _node("fc2", "Dot", ["act2"], weight_ref="fc2_w"),
            _node("out", "Output", ["fc2"]),
        ],
    }
    return Workload("toy_cryptonets", json.dumps(j), blob.bytes(), [1, 8, 8], 0, batch)


def toy_cryptonets_relu(seed: int = 5, batch: int = 64, packing: int = 0) -> Workload:
    """The CryptoNets-ReLU topology (henet/models.hpp:110-136) scaled down like
    make_cryptonets_shaped_toy: conv 3x3/2 (2 filters, bias) -> Relu -> dense 18->4 (bias) ->
    Relu -> dense 4->2 (bias); client-aided refreshes, no rescales."""
    rng = np.random.default_rng(seed)
    blob = Blob()
    blob.add("conv_w", [2, 1, 3, 3], _gauss(rng, (2, 1, 3, 3), 0.3))
    blob.add("conv_b", [2], _gauss(rng, (2,), 0.05))
    blob.add("fc1_w", [18, 4], _gauss(rng, (18, 4), 0.25))
    blob.add("fc1_b", [4], _gauss(rng, (4,), 0.05))
    blob.add("fc2_w", [4, 2], _gauss(rng, (4, 2), 0.5))
    blob.add("fc2_b", [2], _gauss(rng, (2,), 0.05))
    j = {
        "name": "cryptonets-relu-toy",
        "packing": "complex" if packing else "real",
        "preset": "P11",
        "weights": blob.table,
        "nodes": [
            _node("input", "Input", attrs={"shape": [1, 8, 8]}),
            _node("conv", "Convolution", ["input"], {"stride": 2, "window": 3, "filters": 2}, "conv_w", "conv_b"),
            _node("act1", "Relu", ["conv"]),
            _node("flatten", "Reshape", ["act1"], {"shape": [18]}),
            _node("fc1", "Dot", ["flatten"], weight_ref="fc1_w", bias_ref="fc1_b"),
            _node("act2", "Relu", ["fc1"]),
            _node("fc2", "Dot", ["act2"], weight_ref="fc2_w", bias_ref="fc2_b"),
            _node("out", "Output", ["fc2"]),
        ],
    }
    return Workload("toy_cryptonets_relu", json.dumps(j), blob.bytes(), [1, 8, 8], packing, batch)


def synthetic_images(shape, batch: int, seed: int) -> np.ndarray:
    """(batch, elems) pixels uniform in [0, 1) (BASELINE configs 2/3)."""
    rng = np.random.default_rng(seed)
    return rng.random((batch, int(np.prod(shape))))


def random_ciphertexts(params: dict, count: int, seed: int, level: int = None) -> np.ndarray:
    """Seeded uniform residues with the shape of fresh ciphertexts, (count, 2, L, N) u64.
    Fresh RLWE ciphertexts are uniform mod q, so throughput runs use these."""
    rng = np.random.default_rng(seed)
    L = level or len(params["chain"])
    out = np.empty((count, 2, L, params["n"]), dtype=np.uint64)
    for i, q in enumerate(params["chain"][:L]):
        out[:, :, i, :] = rng.integers(0, q, size=(count, 2, params["n"]), dtype=np.uint64)
    return out


def wide_dense_weights(seed: int = 5, k: int = 4096, m: int = 4096) -> np.ndarray:
    """The c5b weight matrix, K x M row-major f32, W ~ N(0, 0.1^2)."""
    return np.asarray(_gauss(np.random.default_rng(seed), (k, m), 0.1), dtype=np.float32).reshape(k, m)


def wide_dense(seed: int = 5, k: int = 4096, m: int = 4096, batch: int = 8192) -> Workload:
    """Config 5b: wide dense layer k -> m on N=16384 batch-packed ciphertexts (40-bit limb 0),
    W ~ N(0, 0.1^2) (config 4/5 weight scale), one rescale per output (patched plan, as c1)."""
    blob = Blob()
    blob.add("fc_w", [k, m], wide_dense_weights(seed, k, m))
    j = {
        "name": f"dense-{k}-{m}",
        "packing": "real",
        "preset": "P14",
        "weights": blob.table,
        "nodes": [
            _node("input", "Input", attrs={"shape": [k]}),
            _node("fc", "Dot", ["input"], weight_ref="fc_w"),
            _node("out", "Output", ["fc"]),
        ],
    }
    return Workload(f"c5b_dense_{k}_{m}", json.dumps(j), blob.bytes(), [k], 0, batch, patch_terminal_rescale=True)


def mobilenet_block(seed: int = 6, hw: int = 56, cin: int = 16, expand: int = 96, cout: int = 24,
                    batch: int = 8192) -> Workload:
    """Config 4: MobileNetV2 inverted-residual block on (cin, hw, hw) activations: 1x1 expand
    cin->expand, ReLU6 (client-aided), 3x3 depthwise (as a block-diagonal full convolution:
    zero weights give exact zero residues), ReLU6, 1x1 project expand->cout.
    Weights ~ N(0, 0.1^2).  The reference graph has no ReLU6/depthwise op: ReLU6 runs through
    the NonlinearityProvider hook as a Relu node whose provider clips to [0, 6]."""
    rng = np.random.default_rng(seed)
    blob = Blob()
    blob.add("exp_w", [expand, cin, 1, 1], _gauss(rng, (expand, cin, 1, 1), 0.1))
    dw = np.zeros((expand, expand, 3, 3), np.float32)
    dwv = _gauss(rng, (expand, 3, 3), 0.1).reshape(expand, 3, 3)
    for c in range(expand):
        dw[c, c] = dwv[c]
    blob.add("dw_w", [expand, expand, 3, 3], dw)
    blob.add("proj_w", [cout, expand, 1, 1], _gauss(rng, (cout, expand, 1, 1), 0.1))
    j = {
        "name": "mobilenetv2-block",
        "packing": "real",
        "preset": "P14",
        "weights": blob.table,
        "nodes": [
            _node("input", "Input", attrs={"shape": [cin, hw, hw]}),
            _node("expand", "Convolution", ["input"], {"stride": 1, "window": 1, "filters": expand}, "exp_w"),
            _node("relu6a", "Relu", ["expand"]),
            _node("dw", "Convolution", ["relu6a"], {"stride": 1, "window": 3, "filters": expand, "pad": [1, 1, 1, 1]},
                  "dw_w"),
            _node("relu6b", "Relu", ["dw"]),
            _node("project", "Convolution", ["relu6b"], {"stride": 1, "window": 1, "filters": cout}, "proj_w"),
            _node("out", "Output", ["project"]),
        ],
    }
    return Workload("c4_mobilenetv2_block", json.dumps(j), blob.bytes(), [cin, hw, hw], 0, batch)
