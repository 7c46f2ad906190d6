"""Seeded synthetic inputs for the TRIOT hot path (BASELINE.json configs C1..C5).

This module is shared by the oracle side (tests, bench cpu_baseline) and the CUDA side
(tests, bench, smoke).  It holds NONE of the method's arithmetic: it only draws numbers
with numpy's PCG64 generator and states the shapes of the paper's workloads.
The recipes are the ones DESIGN.md §Inputs lists (BASELINE.json configs[0..4]).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    op: str                      # "embed" | "binary" | "ev"
    dtype: str                   # "f32" | "f64"
    shapes: dict = field(default_factory=dict)
    note: str = ""


CONFIGS = {
    "C1": Config("C1", "embed", "f64",
                 {"src": (4, 9, 7, 5), "dst": (8, 16, 8, 8)},
                 "zero-padded embed d=4, src uniform[0,1) seed 0 into the corner of dst"),
    "C2": Config("C2", "embed", "f32",
                 {"src": (384, 384, 384), "dst": (512, 512, 512)},
                 "FFT-padding embed d=3, src standard normal seed 1, full dst written"),
    "C3": Config("C3", "ev", "f64",
                 {"p": (16,) * 6},
                 "expected value of a d=6 PMF, uniform[0,1) seed 2 normalised to sum 1"),
    "C4": Config("C4", "binary", "f64",
                 {"a": (32, 48, 24, 40, 36), "b": (40, 32, 32, 32, 32),
                  "iter": (32, 32, 24, 32, 32)},
                 "C[t]=A[t]*B[t] over the min shape, A seed 3, B seed 4"),
    "C5": Config("C5", "embed", "f32",
                 {"src": (3,) * 14, "dst": (4,) * 14},
                 "d=14 tiny-extent embed, src uniform[-1,1) seed 5"),
}


# The paper's own Benchmarks 1-3, §8(f) NEXT-2/3.  The paper states shapes only; the
# element type (double, as in its listings) and the values (uniform[0,1),
# seeds 11-15) are this build's choice.
PAPER_BENCHMARKS = {
    "B1": Config("B1", "embed", "f64", {"src": (1024, 512, 256), "dst": (512, 512, 32)},
                 "Benchmark 1: copy (crop) a (2^10,2^9,2^8) tensor into (2^9,2^9,2^5)"),
    "B2": Config("B2", "dot", "f64", {"a": (1024, 512, 256), "b": (512, 512, 32)},
                 "Benchmark 2: inner product over the shared tuples"),
    "B3": Config("B3", "update", "f64",
                 {"x": (129, 32, 13, 16), "y": (253, 64, 64, 23), "z": (256, 39, 64, 33)},
                 "Benchmark 3: x[t] <- x[t] + y[t]*x[t] - z[t] over x's shape"),
}


def make_paper_inputs(name: str) -> dict:
    if name == "B1":
        return {"src": np.random.default_rng(11).random((1024, 512, 256)),
                "dst_shape": (512, 512, 32)}
    if name == "B2":
        return {"a": np.random.default_rng(12).random((1024, 512, 256)),
                "b": np.random.default_rng(13).random((512, 512, 32))}
    if name == "B3":
        return {"x": np.random.default_rng(14).random((129, 32, 13, 16)),
                "y": np.random.default_rng(15).random((253, 64, 64, 23)),
                "z": np.random.default_rng(16).random((256, 39, 64, 33))}
    raise KeyError(name)


def _np_dtype(s: str):
    return np.float32 if s == "f32" else np.float64


def make_inputs(name: str) -> dict:
    """Host (numpy) inputs of config `name`, exactly as DESIGN.md §Inputs states."""
    if name == "C1":
        src = np.random.default_rng(0).random((4, 9, 7, 5))
        return {"src": src, "dst_shape": (8, 16, 8, 8)}
    if name == "C2":
        src = np.random.default_rng(1).standard_normal((384,) * 3, dtype=np.float32)
        return {"src": src, "dst_shape": (512,) * 3}
    if name == "C3":
        u = np.random.default_rng(2).random((16,) * 6)
        return {"p": u / u.sum()}
    if name == "C4":
        a = np.random.default_rng(3).random((32, 48, 24, 40, 36))
        b = np.random.default_rng(4).random((40, 32, 32, 32, 32))
        return {"a": a, "b": b, "iter_shape": (32, 32, 24, 32, 32)}
    if name == "C5":
        src = (np.random.default_rng(5).random((3,) * 14, dtype=np.float32) * 2 - 1)
        return {"src": src.astype(np.float32), "dst_shape": (4,) * 14}
    raise KeyError(name)


def random_shape(rng: np.random.Generator, d: int, max_elems: int, lo: int = 1,
                 hi: int | None = None) -> tuple:
    """A random shape of dimension d with at most max_elems elements (ragged extents)."""
    if hi is None:
        hi = max(2, int(round(max_elems ** (1.0 / d))) + 2)
    while True:
        s = tuple(int(x) for x in rng.integers(lo, hi + 1, size=d))
        if math.prod(s) <= max_elems:
            return s


def random_values(rng: np.random.Generator, shape, dtype: str, kind: str = "uniform"):
    """Random values of the paper's kinds: uniform[0,1), normal, or small integers."""
    dt = _np_dtype(dtype)
    if kind == "uniform":
        return rng.random(shape, dtype=np.float64).astype(dt)
    if kind == "normal":
        return rng.standard_normal(shape).astype(dt)
    if kind == "int":
        return rng.integers(0, 256, size=shape).astype(dt)
    raise KeyError(kind)


def special_values(dtype: str) -> np.ndarray:
    """Bit patterns a raw move must preserve: NaN payloads, -0.0, subnormals, +-inf."""
    if dtype == "f32":
        bits = np.array([0x7FC00001, 0xFFC12345, 0x80000000, 0x00000001, 0x807FFFFF,
                         0x7F800000, 0xFF800000, 0x3F800000], dtype=np.uint32)
        return bits.view(np.float32)
    bits = np.array([0x7FF8000000000001, 0xFFF0000000ABCDEF, 0x8000000000000000,
                     0x0000000000000001, 0x800FFFFFFFFFFFFF, 0x7FF0000000000000,
                     0xFFF0000000000000, 0x3FF0000000000000], dtype=np.uint64)
    return bits.view(np.float64)
