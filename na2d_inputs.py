"""Seeded synthetic inputs and workload shapes for NA2D (shared by tests, bench and smoke).

This module holds NO arithmetic of the method: only the workload shapes (BASELINE.json
``configs``), a counter-free NumPy PCG64 generator, and bf16 round-to-nearest-even
encoding of the generated fp32 values.  Both the CUDA path and the oracle consume the
arrays it returns; neither is imported here.

Input recipe: Q, K, V, dO ~ N(0, 1) drawn in fp32 in that order,
rounded to bf16 (RNE) for the bf16 path; then the RPB table:
  * ``rpb="parity"``: N(0,1) * sqrt(d), so that under Eq. 2's bias-inside-scale reading the
    effective logit bias scale*B ~ N(0,1) (RPB bugs cannot hide under the tolerance);
  * ``rpb="swin"``:  truncated N(0, 0.02) at +-2 sigma (the Swin initialisation);
  * ``rpb=None``:   no bias (Table 7 "no positional information" variant).
Seed = 2204 + config index unless given.  The 8x8 config mirrors BASELINE config 1.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass(frozen=True)
class Shape:
    name: str
    B: int
    heads: int
    H: int
    W: int
    d: int
    kernel_size: int

    @property
    def units(self) -> int:
        return self.B * self.heads

    @property
    def queries(self) -> int:
        return self.B * self.heads * self.H * self.W

    def replace(self, **kw) -> "Shape":
        return dataclasses.replace(self, **kw)


# BASELINE.json "configs", restated as concrete tensors.  Config 3 assumes
# B=128 and config 5 assumes heads=2 (NAT-Tiny stage 1 at 800x1344).
CONFIGS: dict[str, Shape] = {
    "cfg1_8x8_k3": Shape("cfg1_8x8_k3", 1, 1, 8, 8, 32, 3),
    "cfg2_nat_tiny_s1": Shape("cfg2_nat_tiny_s1", 128, 2, 56, 56, 32, 7),
    "cfg3_nat_tiny_s2": Shape("cfg3_nat_tiny_s2", 128, 4, 28, 28, 32, 7),
    "cfg3_nat_tiny_s3": Shape("cfg3_nat_tiny_s3", 128, 8, 14, 14, 32, 7),
    "cfg3_nat_tiny_s4": Shape("cfg3_nat_tiny_s4", 128, 16, 7, 7, 32, 7),
    "cfg4_ade20k_128": Shape("cfg4_ade20k_128", 16, 2, 128, 128, 32, 7),
    "cfg5_coco_200x336": Shape("cfg5_coco_200x336", 2, 2, 200, 336, 32, 7),
}
CONFIG_SEED = {name: 2204 + i for i, name in enumerate(
    ["cfg1_8x8_k3", "cfg2_nat_tiny_s1", "cfg3_nat_tiny_s2", "cfg4_ade20k_128", "cfg5_coco_200x336"])}
for _n in ("cfg3_nat_tiny_s3", "cfg3_nat_tiny_s4"):
    CONFIG_SEED[_n] = CONFIG_SEED["cfg3_nat_tiny_s2"]


# Shape-generality workloads (not BASELINE configs): NAT-Tiny stage-1 geometry
# with other head dims, for bench lines of the tensor-core paths beyond d = 32.
EXTRA_WORKLOADS: dict[str, Shape] = {
    "f3_d16_s1": Shape("f3_d16_s1", 128, 2, 56, 56, 16, 7),
    "f3_d64_s1": Shape("f3_d64_s1", 128, 2, 56, 56, 64, 7),
}


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest bf16 value (ties to even), returned as fp32.  Encoding only."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    out = u.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(x), x, out)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16-representable fp32 array -> uint16 bit patterns."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def make_inputs(shape: Shape, seed: int | None = None, dtype: str = "bf16", rpb: str | None = "parity",
                batch_offset: int = 0, batch_count: int | None = None) -> dict:
    """Generate {q,k,v,dout,rpb} as fp32 NumPy arrays (bf16-representable when dtype='bf16').

    ``batch_offset/batch_count`` select a batch slice of the SAME global tensors (the draw
    is done per batch index from a seed derived from (seed, b)), so multi-GPU shards are
    slices of the 1-GPU input."""
    if seed is None:
        seed = CONFIG_SEED.get(shape.name, 2204)
    nb = shape.B - batch_offset if batch_count is None else batch_count
    per = (shape.heads, shape.H, shape.W, shape.d)
    qs, ks, vs, ds = [], [], [], []
    for b in range(batch_offset, batch_offset + nb):
        g = np.random.Generator(np.random.PCG64([seed, b]))
        qs.append(g.standard_normal(per, dtype=np.float32))
        ks.append(g.standard_normal(per, dtype=np.float32))
        vs.append(g.standard_normal(per, dtype=np.float32))
        ds.append(g.standard_normal(per, dtype=np.float32))
    out = {"q": np.stack(qs), "k": np.stack(ks), "v": np.stack(vs), "dout": np.stack(ds)}
    T = 2 * shape.kernel_size - 1
    g = np.random.Generator(np.random.PCG64([seed, 1 << 30]))
    if rpb == "parity":
        out["rpb"] = (g.standard_normal((shape.heads, T, T)) * np.sqrt(shape.d)).astype(np.float32)
    elif rpb == "swin":
        t = g.standard_normal((shape.heads, T, T))
        while np.any(np.abs(t) > 2.0):
            bad = np.abs(t) > 2.0
            t[bad] = g.standard_normal(int(bad.sum()))
        out["rpb"] = (0.02 * t).astype(np.float32)
    elif rpb is None:
        out["rpb"] = None
    else:
        raise ValueError(rpb)
    if dtype == "bf16":
        for n in ("q", "k", "v", "dout"):
            out[n] = bf16_round(out[n])
    elif dtype == "f16":  # fp16-representable (IEEE round to nearest even)
        for n in ("q", "k", "v", "dout"):
            out[n] = out[n].astype(np.float16).astype(np.float32)
    elif dtype != "f32":
        raise ValueError(dtype)
    return out
