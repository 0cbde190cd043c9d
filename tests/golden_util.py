"""Helpers for the golden fixtures in tests/golden/ (made by oracle/golden_gen.cpp)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
M64 = (1 << 64) - 1


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def unhex(s: str) -> np.ndarray:
    return np.frombuffer(bytes.fromhex(s), dtype=np.uint8).copy()


def splitmix64(i: np.ndarray) -> np.ndarray:
    z = i.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def grid_hash(values) -> int:
    """sum_i (uint32(v_i) + 0x9E37) * splitmix64(i) mod 2^64 (same as golden_gen.cpp)."""
    v = np.asarray(values).reshape(-1).astype(np.int64).astype(np.uint32).astype(np.uint64)
    with np.errstate(over="ignore"):
        terms = (v + np.uint64(0x9E37)) * splitmix64(np.arange(v.size, dtype=np.uint64))
        return int(np.sum(terms, dtype=np.uint64))
