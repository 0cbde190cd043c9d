"""Seeded synthetic inputs for the five BASELINE.json configs.

No public dataset is named by the reference or BASELINE.json; these stand in
with the configs' shapes, alphabets and mutation models.  Randomness is a
counter-based splitmix64 stream (pure numpy, platform independent), so the
same (config, seed) gives the same bytes here, on the GPU box and in the
oracle runs.  DNA is ASCII ``ACGT`` and protein-like sigma=20 is
``ACDEFGHIKLMNPQRSTVWY`` (as FASTA ingest would give, io.cpp:66); byte 0 never
occurs (model.hpp:33-34).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

DNA = np.frombuffer(b"ACGT", dtype=np.uint8)
PROTEIN = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", dtype=np.uint8)

_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z + _G
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def rand_u64(seed: int, stream: int, n: int) -> np.ndarray:
    """n 64-bit words of stream `stream` of seed `seed`."""
    with np.errstate(over="ignore"):
        key = _mix(np.array([(seed * 1_000_003 + stream * 7919) & ((1 << 64) - 1)], dtype=np.uint64))[0]
        return _mix(np.arange(n, dtype=np.uint64) + key)


def rand_unit(seed: int, stream: int, n: int) -> np.ndarray:
    return (rand_u64(seed, stream, n) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


def rand_index(seed: int, stream: int, n: int, k: int) -> np.ndarray:
    """Uniform integers in [0, k)."""
    hi = rand_u64(seed, stream, n) >> np.uint64(32)
    return ((hi * np.uint64(k)) >> np.uint64(32)).astype(np.int64)


def uniform(seed: int, stream: int, n: int, alphabet: np.ndarray) -> np.ndarray:
    return alphabet[rand_index(seed, stream, n, alphabet.size)]


def mutate_dna(x: np.ndarray, seed: int, p_sub: float, p_indel: float) -> np.ndarray:
    """Point substitutions (uniform other base) then single-base indels (half ins / half del)."""
    n = x.size
    code = np.searchsorted(DNA, x)  # DNA is sorted (A<C<G<T)
    sub = rand_unit(seed, 10, n) < p_sub
    shift = 1 + rand_index(seed, 11, n, 3)
    code = np.where(sub, (code + shift) % 4, code)
    y = DNA[code]
    if p_indel <= 0:
        return y
    u = rand_unit(seed, 12, n)
    dele = u < p_indel / 2
    ins = (u >= p_indel / 2) & (u < p_indel)
    ins_base = DNA[rand_index(seed, 13, n, 4)]
    # each position emits: nothing (deleted), itself, or itself + an inserted base
    keep = ~dele
    counts = keep.astype(np.int64) + ins.astype(np.int64)
    out = np.empty(int(counts.sum()), dtype=np.uint8)
    pos = np.cumsum(counts) - counts
    out[pos[keep]] = y[keep]
    out[pos[ins] + 1] = ins_base[ins]
    return out


@dataclass(frozen=True)
class Config:
    name: str
    w: int
    h: int
    r: int
    t_half: Optional[int]   # None = dense output
    description: str


CONFIGS = {
    "C1": Config("C1", 64, 1, 1, None, "LCS plot, uniform DNA m=n=2000, w=64, dense (seed 1)"),
    "C2": Config("C2", 100, 1, 2, None,
                 "alignment-score plot, x uniform DNA m=16384, y = x + 10% subs + 3% indels (seed 2), w=100, dense"),
    "C3": Config("C3", 128, 1, 1, 192, "LCS plot, uniform DNA m=n=65536, w=128, WLCS >= 96 (t_half 192)"),
    "C4": Config("C4", 64, 1, 2, 32,
                 "alignment-score plot, uniform sigma=20 m=n=262144, w=64, score >= 16 (t_half 32)"),
    "C5": Config("C5", 256, 1, 1, 360,
                 "LCS dot plot m=n=1048576, y = x with 30% of 5 kb blocks fresh + 5% subs (seed 5), w=256, "
                 "WLCS >= 180 (t_half 360)"),
}


def make_inputs(name: str, scale: float = 1.0) -> Tuple[np.ndarray, np.ndarray]:
    """(x, y) uint8 arrays of config `name`; `scale` < 1 shrinks m and n for quick tests."""
    if name == "C1":
        m = max(64, int(2000 * scale))
        return uniform(1, 0, m, DNA), uniform(1, 1, m, DNA)
    if name == "C2":
        m = max(100, int(16384 * scale))
        x = uniform(2, 0, m, DNA)
        return x, mutate_dna(x, 2, 0.10, 0.03)
    if name == "C3":
        m = max(128, int(65536 * scale))
        return uniform(3, 0, m, DNA), uniform(3, 1, m, DNA)
    if name == "C4":
        m = max(64, int(262144 * scale))
        return uniform(4, 0, m, PROTEIN), uniform(4, 1, m, PROTEIN)
    if name == "C5":
        m = max(256, int(1048576 * scale))
        x = uniform(5, 0, m, DNA)
        y = x.copy()
        block = 5000
        nblocks = (m + block - 1) // block
        nrep = int(round(0.30 * nblocks))
        order = np.argsort(rand_u64(5, 20, nblocks))
        fresh = uniform(5, 21, m, DNA)
        for b in np.sort(order[:nrep]):
            s, e = b * block, min(m, (b + 1) * block)
            y[s:e] = fresh[s:e]
        return x, mutate_dna(y, 5, 0.05, 0.0)
    raise KeyError(name)
