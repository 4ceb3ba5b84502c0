"""Seeded synthetic workloads shared by the tests, bench.py and smoke().

This module holds NO arithmetic of the method (no normalisation, encoding,
packing or scoring): it only draws the raw float32 database / query vectors
and holds the BASELINE.json configurations.  Both the CUDA path and the CPU
oracle consume exactly these arrays.

Generator ("Datasets"): the query has integer
components uniform in [-99, 99]; K_m planted matches are query + uniform
integer noise in [-2, 2] per component at uniformly random distinct
positions; the other K - K_m vectors are uniform integers in [-99, 99]^ell.
Stored as float32 (normalisation happens inside the library / oracle).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DATA_SEED_BASE = 260400546
KEY_SEED = 1
ENC_SEED_BASE = 1000


@dataclass(frozen=True)
class Config:
    name: str
    log_n: int          # ring degree 2^log_n
    dim: int            # VECTOR_DIM = N (block size)
    num_vectors: int    # K
    n1: int             # baby-step size
    limbs: int = 3      # L (R5)
    index: int = 1      # BASELINE.json configs[] position (+1): data seed offset
    planted: int = 3    # K_m
    special: int = 1    # K_sp special primes (R11; paper-depth profile 4, R31)
    digit_limbs: int = 1  # alpha limbs per key-switching digit (R11; paper-depth profile 4)

    @property
    def num_slots(self):
        return 1 << (self.log_n - 1)

    @property
    def groups(self):
        return -(-self.num_vectors // self.dim)

    @property
    def aggregates(self):
        M = self.num_slots // self.dim
        return -(-2 * self.groups // M)

    @property
    def data_seed(self):
        return DATA_SEED_BASE + self.index


# BASELINE.json "configs" (C1..C5); n1 = 128 for C4 chosen from the n1 sweep at 2^20 (R22).
CONFIGS = {
    "C1": Config("C1-toy", 12, 64, 256, 8, index=1),
    "C2": Config("C2", 15, 512, 1 << 14, 16, index=2),
    "C3": Config("C3", 15, 512, 1 << 17, 16, index=3),
    "C4": Config("C4", 16, 512, 1 << 20, 128, index=4),
    "C4n64": Config("C4-n64", 16, 512, 1 << 20, 64, index=4),
    "C4n16": Config("C4-n16", 16, 512, 1 << 20, 16, index=4),
    "C4n32": Config("C4-n32", 16, 512, 1 << 20, 32, index=4),
    "C4n128": Config("C4-n128", 16, 512, 1 << 20, 128, index=4),
    "C2n128": Config("C2-n128", 15, 512, 1 << 14, 128, index=2),
    "C4n256": Config("C4-n256", 16, 512, 1 << 20, 256, index=4),
    "C2n256": Config("C2-n256", 15, 512, 1 << 14, 256, index=2),
}
# SURVEY 8(d) "secondary": the paper's depth (depth 11, scale 45) as L = 12 limbs,
# alpha = 4 limbs per digit, K_sp = 4 special primes (R31), on C3 (P = 1) and the toy workload
CONFIGS["C3p"] = Config("C3-paper-depth", 15, 512, 1 << 17, 16, limbs=12, index=3, special=4, digit_limbs=4)
CONFIGS["C1p"] = Config("C1-paper-depth", 12, 64, 256, 8, limbs=12, index=1, special=4, digit_limbs=4)
for _n1 in (4, 8, 16, 32, 64):
    CONFIGS[f"C5n{_n1}"] = Config(f"C5-n1={_n1}", 15, 512, 1 << 17, _n1, index=5)


def make_dataset(num_vectors: int, dim: int, seed: int, planted: int = 3):
    """Return (db float32 [K, dim], query float32 [dim], planted_positions sorted).

    Draws are made in fixed-size chunks so the same seed gives the same rows
    whatever K is sampled from (rows [a, b) of a large K are reproducible
    without materialising the whole database: see ``dataset_rows``).
    """
    rng = np.random.default_rng(seed)
    query = rng.integers(-99, 100, size=dim).astype(np.float32)
    planted = min(planted, num_vectors)
    pos = np.sort(rng.choice(num_vectors, size=planted, replace=False)) if planted else np.zeros(0, np.int64)
    db = dataset_rows(num_vectors, dim, seed, 0, num_vectors, query=query, planted_pos=pos)
    return db, query, pos


def planted_positions(num_vectors: int, dim: int, seed: int, planted: int = 3):
    """The planted-match positions make_dataset(num_vectors, dim, seed) draws (no rows made)."""
    rng = np.random.default_rng(seed)
    rng.integers(-99, 100, size=dim)
    planted = min(planted, num_vectors)
    return np.sort(rng.choice(num_vectors, size=planted, replace=False)) if planted else np.zeros(0, np.int64)


_CHUNK = 4096


def dataset_rows(num_vectors, dim, seed, start, stop, query=None, planted_pos=None):
    """Rows [start, stop) of the database drawn by ``make_dataset``."""
    if query is None or planted_pos is None:
        rng = np.random.default_rng(seed)
        query = rng.integers(-99, 100, size=dim).astype(np.float32)
        planted = min(3, num_vectors)
        planted_pos = np.sort(rng.choice(num_vectors, size=planted, replace=False))
    out = np.empty((stop - start, dim), dtype=np.float32)
    c0 = start // _CHUNK
    c1 = -(-stop // _CHUNK)
    for c in range(c0, c1):
        rng = np.random.default_rng([seed, 1, c])
        lo = c * _CHUNK
        hi = min(lo + _CHUNK, num_vectors)
        block = rng.integers(-99, 100, size=(hi - lo, dim)).astype(np.float32)
        a, b = max(lo, start), min(hi, stop)
        out[a - start:b - start] = block[a - lo:b - lo]
    for idx, p in enumerate(planted_pos):
        if start <= p < stop:
            rng = np.random.default_rng([seed, 2, idx])
            out[p - start] = query + rng.integers(-2, 3, size=dim).astype(np.float32)
    return out

