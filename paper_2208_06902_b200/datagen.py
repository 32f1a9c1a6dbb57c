"""Seeded synthetic inputs (BASELINE.json configs C1-C5) — shared by tests, bench and smoke.

Holds none of the method's arithmetic: only numpy PCG64 draws.  The paper's workloads
are N = 1e8 synthetic float64 keys and 2e8 real uint64 keys; the BASELINE
configs stand in for them:

* C1 Uniform[0,1)          — P:604-606 uses Uniform(0, N)
* C2 Normal(0,1)           — P:608-610
* C3 LogNormal(0, 2)       — P:612-614 uses sigma = 0.5
* C4 root-dups i mod sqrt(n), shuffled — P:625-626
* C5 5-component Gaussian mixture — P:616-617 gives no parameters; BASELINE fixes them

``generate(name, n)`` draws the same distribution at any size (for parity cases the
oracle finishes quickly); at the default size it reproduces the BASELINE input bytes
exactly (SHA-256 pinned in tests/golden/inputs.txt).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    dtype: str
    k: int
    base_case: int
    seed: int
    desc: str


CONFIGS = {
    "C1": Config("C1", 1_000_000, "f64", 256, 4096, 42, "Uniform[0,1) float64, PCG64(42)"),
    "C2": Config("C2", 100_000_000, "f64", 1024, 4096, 1, "Normal(0,1) float64, PCG64(1)"),
    "C3": Config("C3", 100_000_000, "f64", 1024, 4096, 2, "LogNormal(0,2) float64, PCG64(2)"),
    "C4": Config("C4", 100_000_000, "u64", 1024, 4096, 3,
                 "root-dups i mod floor(sqrt(n)) uint64, shuffled PCG64(3)"),
    "C5": Config("C5", 200_000_000, "f64", 1024, 4096, 4,
                 "5-Gaussian mixture float64, PCG64(4)"),
}


# The paper's nine synthetic workloads, for the widening runs (SURVEY §8(f)
# NEXT #4): same draws at any size, PCG64(seed).  Readings where the paper is silent
# (DESIGN.md §4): Zipf(0.75) is drawn over the ranks 1..10^6 (float64 ranks); Root Dups and
# Two Dups keep the paper's index order (no shuffle); Mix Gauss uses C5's parameters.
PAPER_WORKLOADS = {
    "uniform": ("f64", "Uniform(0, N) float64 (P:604-606)"),
    "normal": ("f64", "Normal(0, 1) float64 (P:608-610)"),
    "lognormal": ("f64", "LogNormal(0, 0.5) float64 (P:612-614)"),
    "mixgauss": ("f64", "5-Gaussian mixture float64, C5 parameters (P:616-617)"),
    "exponential": ("f64", "Exponential(lambda = 2) float64 (P:619-620)"),
    "chisquared": ("f64", "Chi-squared(k = 4) float64 (P:621-622)"),
    "rootdups": ("u64", "A[i] = i mod floor(sqrt N) uint64, index order (P:625-626)"),
    "twodups": ("u64", "A[i] = (i^2 + N/2) mod N uint64, index order (P:627-628)"),
    "zipf": ("f64", "Zipf(s = 0.75) ranks 1..10^6 float64 (P:629-630)"),
}


def paper_workload(name: str, n: int, seed: int = 7) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(seed))
    if name == "uniform":
        return g.uniform(0.0, float(n), n)
    if name == "normal":
        return g.normal(0.0, 1.0, n)
    if name == "lognormal":
        return g.lognormal(0.0, 0.5, n)
    if name == "mixgauss":
        c = g.choice(5, size=n, p=[0.3, 0.2, 0.2, 0.2, 0.1])
        mu = np.array([0.0, 10.0, 20.0, 40.0, 80.0])
        sd = np.array([1.0, 0.5, 2.0, 0.1, 5.0])
        return g.normal(mu[c], sd[c])
    if name == "exponential":
        return g.exponential(0.5, n)
    if name == "chisquared":
        return g.chisquare(4.0, n)
    if name == "rootdups":
        r = max(1, int(np.floor(np.sqrt(n))))
        while r * r > n:
            r -= 1
        return np.arange(n, dtype=np.uint64) % np.uint64(max(r, 1))
    if name == "twodups":
        i = np.arange(n, dtype=np.uint64)
        return (i * i + np.uint64(n // 2)) % np.uint64(max(n, 1))
    if name == "zipf":
        ranks = np.arange(1, 10**6 + 1, dtype=np.float64)
        cdf = np.cumsum(ranks ** -0.75)
        cdf /= cdf[-1]
        return (np.searchsorted(cdf, g.random(n), side="right") + 1).astype(np.float64)
    raise KeyError(name)


def generate(name: str, n: int | None = None) -> np.ndarray:
    """Exact BASELINE generator call order; ``n`` overrides the size (same distribution)."""
    cfg = CONFIGS[name]
    n = cfg.n if n is None else int(n)
    if name == "C1":
        g = np.random.Generator(np.random.PCG64(cfg.seed))
        return g.random(n)
    if name == "C2":
        return np.random.Generator(np.random.PCG64(cfg.seed)).normal(0.0, 1.0, n)
    if name == "C3":
        return np.random.Generator(np.random.PCG64(cfg.seed)).lognormal(0.0, 2.0, n)
    if name == "C4":
        r = int(np.floor(np.sqrt(n))) if n > 0 else 1
        # exact integer sqrt for the default size (sqrt(1e8) = 1e4)
        while r * r > n:
            r -= 1
        while (r + 1) * (r + 1) <= n:
            r += 1
        x = np.arange(n, dtype=np.uint64) % np.uint64(max(r, 1))
        np.random.Generator(np.random.PCG64(cfg.seed)).shuffle(x)
        return x
    if name == "C5":
        g = np.random.Generator(np.random.PCG64(cfg.seed))
        c = g.choice(5, size=n, p=[0.3, 0.2, 0.2, 0.2, 0.1])
        mu = np.array([0.0, 10.0, 20.0, 40.0, 80.0])
        sd = np.array([1.0, 0.5, 2.0, 0.1, 5.0])
        return g.normal(mu[c], sd[c])
    raise KeyError(name)


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fuzz_array(rng: np.random.Generator, n: int, kind: str) -> np.ndarray:
    """Edge-case inputs for parity fuzzing (no method arithmetic)."""
    if kind == "uniform":
        return rng.random(n)
    if kind == "normal":
        return rng.normal(0.0, 1.0, n)
    if kind == "lognormal":
        return rng.lognormal(0.0, 2.0, n)
    if kind == "all_equal":
        return np.full(n, 3.25)
    if kind == "two_values":
        return np.where(rng.random(n) < 0.5, -1.0, 7.0)
    if kind == "signed_zeros":
        return np.where(rng.random(n) < 0.5, -0.0, 0.0) + 0.0 * rng.random(n)
    if kind == "zeros_mixed":
        v = rng.choice(np.array([-0.0, 0.0, 1.0, -1.0]), size=n)
        return v
    if kind == "denormals":
        return rng.random(n) * 5e-324 * 1e6 - 2e-318
    if kind == "infs":
        v = rng.normal(0.0, 1.0, n)
        if n > 2:
            idx = rng.choice(n, size=max(1, n // 50), replace=False)
            v[idx] = np.where(rng.random(idx.size) < 0.5, np.inf, -np.inf)
        return v
    if kind == "sorted":
        return np.sort(rng.normal(0.0, 1.0, n))
    if kind == "reverse":
        return np.sort(rng.normal(0.0, 1.0, n))[::-1].copy()
    if kind == "few_distinct":
        return rng.integers(0, 5, n).astype(np.float64)
    if kind == "root_dups_u64":
        r = max(1, int(np.sqrt(n)))
        x = np.arange(n, dtype=np.uint64) % np.uint64(r)
        rng.shuffle(x)
        return x
    if kind == "u64_big":
        return rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    if kind == "u64_above_2_53":
        return (np.uint64(2**60) + rng.integers(0, 2**20, n, dtype=np.uint64))
    if kind == "mixture":
        c = rng.choice(5, size=n, p=[0.3, 0.2, 0.2, 0.2, 0.1])
        mu = np.array([0.0, 10.0, 20.0, 40.0, 80.0])
        sd = np.array([1.0, 0.5, 2.0, 0.1, 5.0])
        return rng.normal(mu[c], sd[c])
    if kind == "exponential":
        return rng.exponential(0.5, n)
    raise KeyError(kind)


def stress_array(rng: np.random.Generator, n: int, kind: str) -> np.ndarray:
    """Inputs that load the base case's bins: tight clusters of near-equal keys (several keys
    per interpolation bin, in every order), one sign per window or windows through zero,
    u64 keys that collide in binary64.  Shuffled.  No method arithmetic."""
    if kind in ("clusters3", "clusters40", "neg_clusters"):
        c = 3 if kind != "clusters40" else 40
        m = (n + c - 1) // c
        centers = rng.random(m) * 1e3
        if kind == "neg_clusters":
            centers = -1.0 - centers
        v = np.repeat(centers, c)[:n] + rng.integers(0, 4, n) * 1e-9
    elif kind == "zero_straddle":
        v = rng.normal(0.0, 1e-300, n)
        v[rng.random(n) < 0.01] = 0.0
        v[rng.random(n) < 0.01] = -0.0
    elif kind == "u64_clusters":
        m = (n + 2) // 3
        centers = rng.integers(2**60, 2**63, m, dtype=np.uint64)
        v = np.repeat(centers, 3)[:n] + rng.integers(0, 8, n, dtype=np.uint64)
    else:
        raise KeyError(kind)
    rng.shuffle(v)
    return v


STRESS_KINDS = ["clusters3", "clusters40", "neg_clusters", "zero_straddle", "u64_clusters"]

FUZZ_KINDS = ["uniform", "normal", "lognormal", "all_equal", "two_values", "signed_zeros",
              "zeros_mixed", "denormals", "infs", "sorted", "reverse", "few_distinct",
              "root_dups_u64", "u64_big", "u64_above_2_53", "mixture", "exponential"]
