"""Seeded synthetic inputs shared by tests, bench and oracle checks.

This module holds NONE of the method's arithmetic (no CSR build, no operator, no sketch, no GCN).
It draws degree-corrected SBM multigraphs (Def. 5) shaped like the paper's
benchmark graphs (Table I / §V-A1) at the sizes BASELINE.json's configs name,
and returns a RAW edge list (duplicates, both orientations and self pairs left in, random order):
canonicalisation is the method's job.

The recipe (block sizes, power-law theta, mixture Omega, the "stated-edge" rescale) is written out
in DESIGN.md "Input recipe"; it stands in for the authors' own generator, whose graphs are not
available.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libdcsbm.so")
_lib = None


def build() -> str:
    """Compile synth/dcsbm.c (gcc, OpenMP) in-tree."""
    src = os.path.join(_HERE, "dcsbm.c")
    if (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-o", _LIB, src, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        _lib.dcsbm_sample.restype = ctypes.c_int
    return _lib


@dataclass(frozen=True)
class DCSBMConfig:
    """One BASELINE.json config (C1..C5) plus the method sizes that go with it."""
    name: str
    n: int
    k: int
    alpha: float          # Dirichlet concentration of block sizes
    gamma: float          # power-law exponent of expected degree
    dmin: float
    dmax: float
    rho: float            # within:between expected edge ratio
    m_stated: int         # stated undirected edge count (stated-edge rule)
    r: int                # sketch width (Eq. 5's L)
    dims: tuple           # GNN widths [L, L_1, ..., d] (Eq. 6)
    min_size: int = 20


# BASELINE.json configs[0..4]
CONFIGS = {
    "C1": DCSBMConfig("C1", 1_000, 11, 1.5, 2.5, 10, 100, 3.0, 10_000, 64, (64, 64, 32)),
    "C2": DCSBMConfig("C2", 50_000, 44, 1.5, 2.5, 10, 100, 2.5, 1_000_000, 64, (64, 64, 32)),
    "C3": DCSBMConfig("C3", 200_000, 70, 0.5, 2.1, 5, 300, 1.5, 4_000_000, 128, (128, 128, 64, 32)),
    "C4": DCSBMConfig("C4", 5_000_000, 500, 1.0, 2.3, 5, 1000, 2.0, 100_000_000, 128, (128, 128, 64)),
    "C5": DCSBMConfig("C5", 50_000_000, 4000, 1.0, 2.3, 4, 2000, 2.0, 1_000_000_000, 128, (128, 128, 64)),
}


@dataclass
class Graph:
    n: int
    src: np.ndarray       # int32[m] raw edge list (not canonical)
    dst: np.ndarray       # int32[m]
    labels: np.ndarray    # int32[n] planted block of each node
    info: dict


def _block_sizes(rng, n, k, alpha, min_size):
    min_size = min(min_size, n // k)
    p = rng.dirichlet(np.full(k, alpha))
    sizes = np.maximum(min_size, np.rint(p * n).astype(np.int64))
    sizes[np.argmax(sizes)] += n - sizes.sum()
    while sizes.min() < 1 or sizes.sum() != n:       # tiny-n safety
        sizes = np.maximum(1, sizes)
        sizes[np.argmax(sizes)] += n - sizes.sum()
    return sizes


def _powerlaw(rng, size, gamma, lo, hi):
    u = rng.random(size)
    a, b = lo ** (1.0 - gamma), hi ** (1.0 - gamma)
    return (a + u * (b - a)) ** (1.0 / (1.0 - gamma))


def generate(cfg: DCSBMConfig | str, seed: int = 0, rule: str = "stated", n: int | None = None) -> Graph:
    """Draw one seeded DC-SBM multigraph for a config.

    rule="stated": theta rescaled so the expected undirected edge count is cfg.m_stated (scaled by
    n/cfg.n if n overrides the node count); rule="law": the degree law as stated, unscaled.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    N = int(n if n is not None else cfg.n)
    m_target = cfg.m_stated * (N / cfg.n)
    K = min(cfg.k, max(1, N // 2))
    rng = np.random.Generator(np.random.PCG64(seed))
    sizes = _block_sizes(rng, N, K, cfg.alpha, cfg.min_size)
    block_start = np.zeros(K + 1, np.int64)
    block_start[1:] = np.cumsum(sizes)
    theta = _powerlaw(rng, N, cfg.gamma, cfg.dmin, cfg.dmax)
    if rule == "stated":
        theta *= (2.0 * m_target) / theta.sum()
    elif rule != "law":
        raise ValueError(rule)
    cum = np.zeros(N + 1, np.float64)
    cum[1:] = np.cumsum(theta)
    two_m = cum[-1]
    kappa = cum[block_start[1:]] - cum[block_start[:-1]]
    s = float((kappa ** 2).sum() / two_m)
    f_in = (cfg.rho * (two_m - s) - s) / ((1.0 + cfg.rho) * (two_m - s)) if two_m > s else 1.0
    f_in = float(np.clip(f_in, 0.0, 1.0))
    within = rng.poisson(f_in * kappa / 2.0).astype(np.int64)
    nglobal = max(1, int(min(256, (1.0 - f_in) * two_m / 2.0 // 200_000 + 1)))
    glob = rng.poisson(np.full(nglobal, (1.0 - f_in) * two_m / 2.0 / nglobal)).astype(np.int64)
    seg_count = np.concatenate([within, glob])
    seg_offset = np.zeros(len(seg_count) + 1, np.int64)
    seg_offset[1:] = np.cumsum(seg_count)
    perm = rng.permutation(N).astype(np.int32)
    m = int(seg_offset[-1])
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    lib = _load()
    P = ctypes.c_void_p
    rc = lib.dcsbm_sample(ctypes.c_int64(N), P(cum.ctypes.data), ctypes.c_int64(K), P(block_start.ctypes.data),
                          ctypes.c_int64(nglobal), P(seg_count.ctypes.data), P(seg_offset.ctypes.data),
                          P(perm.ctypes.data), ctypes.c_uint64(seed), P(src.ctypes.data), P(dst.ctypes.data))
    if rc != 0:
        raise RuntimeError("dcsbm_sample failed")
    labels = np.empty(N, np.int32)
    labels[perm] = np.repeat(np.arange(K, dtype=np.int32), sizes)
    info = dict(config=cfg.name, n=N, k=K, rule=rule, seed=seed, f_in=f_in, m_raw=m,
                expected_undirected=float(two_m / 2.0), theta_max=float(theta.max()), theta_min=float(theta.min()))
    return Graph(N, src, dst, labels, info)


def random_edges(n: int, m: int, seed: int, self_loops: float = 0.05, dup: float = 0.1):
    """Small uniform random raw edge list with deliberate self-loops and duplicates (edge-case input)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    src = rng.integers(0, n, m).astype(np.int32) if n > 0 else np.zeros(0, np.int32)
    dst = rng.integers(0, n, m).astype(np.int32) if n > 0 else np.zeros(0, np.int32)
    if m and n:
        k = int(self_loops * m)
        dst[:k] = src[:k]
        d = int(dup * m)
        if d and m > 2 * d:
            src[-d:], dst[-d:] = dst[k:k + d], src[k:k + d]
    return src, dst


def sample_rows(n: int, count: int, seed: int) -> np.ndarray:
    """Seeded sorted sample of distinct row ids (for sampled parity at full size)."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    count = min(count, n)
    return np.sort(rng.choice(n, size=count, replace=False)).astype(np.int64)


def sbm_params(cfg: DCSBMConfig | str, seed: int = 0, rule: str = "stated", n: int | None = None):
    """Parameters (c, theta, Omega) of the same degree-corrected SBM that `generate` draws from (Def. 5,
    PAPER.md:106-109): lambda_ij = theta_i theta_j Omega[c_i][c_j] with the mixture Omega_rs =
    f_in delta_rs / kappa_r + (1 - f_in) / 2m, node ids randomly permuted. Input for the Alg. 2 sampler."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    N = int(n if n is not None else cfg.n)
    m_target = cfg.m_stated * (N / cfg.n)
    K = min(cfg.k, max(1, N // 2))
    rng = np.random.Generator(np.random.PCG64(seed))
    sizes = _block_sizes(rng, N, K, cfg.alpha, cfg.min_size)
    theta = _powerlaw(rng, N, cfg.gamma, cfg.dmin, cfg.dmax)
    if rule == "stated":
        theta *= (2.0 * m_target) / theta.sum()
    block = np.repeat(np.arange(K, dtype=np.int32), sizes)
    two_m = float(theta.sum())
    kappa = np.bincount(block, weights=theta, minlength=K)
    s = float((kappa ** 2).sum() / two_m)
    f_in = (cfg.rho * (two_m - s) - s) / ((1.0 + cfg.rho) * (two_m - s)) if two_m > s else 1.0
    f_in = float(np.clip(f_in, 0.0, 1.0))
    omega = np.full((K, K), (1.0 - f_in) / two_m)
    omega[np.arange(K), np.arange(K)] += f_in / kappa
    perm = rng.permutation(N)
    c = np.empty(N, np.int32)
    th = np.empty(N, np.float64)
    c[perm] = block
    th[perm] = theta
    return c, th, omega
