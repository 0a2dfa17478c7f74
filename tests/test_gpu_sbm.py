"""GPU parity of NEXT-3 — Alg. 2, the exact SBM sampler (docs/SBM_SPEC.md) — through the C-ABI
(raftgp_sbm_sample) against the oracle: the edge lists must be IDENTICAL (integer output; every floating-point
decision is taken on bit-identical fp64 values), in (block pair, chunk, cell) order. Cases: DC-SBM parameters
of C1 and C2 (synth.sbm_params), random parameters with empty and one-node blocks, zero Omega entries, chunk
sizes from 2^4 (many chunk boundaries) to 2^20, and the capacity / retry protocol."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg(cuda_required):
    from paper_2312_01560_b200 import raftgp
    raftgp.load_library()
    return raftgp


@pytest.fixture(scope="module")
def ctx(rg):
    return rg.Context(0)


def _both(rg, ctx, c, th, om, seed, q):
    rs, rd = oracle.sbm_sample(c, th, om, seed, q=q)
    gs, gd = rg.raftgp_sbm_sample(ctx, torch.from_numpy(c).cuda(), torch.from_numpy(th).cuda(),
                                  torch.from_numpy(om).cuda(), seed, q=q)
    return rs, rd, gs.cpu().numpy(), gd.cpu().numpy()


def _check(rs, rd, gs, gd):
    assert gs.size == rs.size, f"{gs.size} vs {rs.size} edges"
    assert np.array_equal(gs, rs) and np.array_equal(gd, rd)


@pytest.mark.parametrize("cfg,n", [("C1", None), ("C2", 20000)])
@pytest.mark.parametrize("q", [6, 20])
def test_parity_dcsbm(rg, ctx, cfg, n, q):
    c, th, om = synth.sbm_params(cfg, 1, n=n)
    _check(*_both(rg, ctx, c, th, om, 7, q))


@pytest.mark.parametrize("seed", range(6))
def test_parity_random(rg, ctx, seed):
    rng = np.random.default_rng(seed)
    n, K = int(rng.integers(1, 400)), int(rng.integers(1, 12))
    c = rng.integers(0, K, n).astype(np.int32)
    if K > 2:
        c[c == 1] = 0                       # block 1 empty
        c[int(rng.integers(0, n))] = 2      # (possibly) a one-node block 2
    th = rng.uniform(0.2, 2.5, n)
    A = rng.uniform(0.0, 0.05, (K, K))
    om = (A + A.T) / 2
    om[rng.random((K, K)) < 0.2] = 0.0
    om = np.minimum(om, om.T)               # keep symmetric zeros
    _check(*_both(rg, ctx, c, th, om, seed, int(rng.choice([4, 5, 9, 20]))))


def test_dense_and_empty(rg, ctx):
    c, th, om = synth.sbm_params("C1", 2, n=300)
    _check(*_both(rg, ctx, c, th, om * 1e4, 3, 6))     # every cell is an edge
    rs, rd, gs, gd = _both(rg, ctx, c, th, om * 0.0, 3, 6)
    assert rs.size == 0 and gs.size == 0


def test_capacity_protocol_and_errors(rg, ctx):
    c, th, om = synth.sbm_params("C1", 0)
    ct, tt, ot = (torch.from_numpy(x).cuda() for x in (c, th, om))
    src, dst = rg.raftgp_sbm_sample(ctx, ct, tt, ot, 5, cap=10)      # too small: the binding retries
    rs, rd = oracle.sbm_sample(c, th, om, 5)
    assert np.array_equal(src.cpu().numpy(), rs) and np.array_equal(dst.cpu().numpy(), rd)
    bad = ot.clone()
    bad[0, 1] += 1.0
    with pytest.raises(rg.RaftGPError) as e:
        rg.raftgp_sbm_sample(ctx, ct, tt, bad, 5)
    assert e.value.code == rg.RAFTGP_ERR_PARAM
    with pytest.raises(rg.RaftGPError):
        rg.raftgp_sbm_sample(ctx, ct, -tt, ot, 5)
    with pytest.raises(rg.RaftGPError):
        rg.raftgp_sbm_sample(ctx, ct, tt, ot, 5, q=3)


def test_parity_diagonal_heavy(rg, ctx):
    """One dense block plus sparse ones: per-pair chunk sizes hit the 2^4 floor on the diagonal pair."""
    rng = np.random.default_rng(11)
    n, K = 600, 4
    c = np.where(rng.random(n) < 0.5, 0, rng.integers(1, K, n)).astype(np.int32)
    th = rng.uniform(0.5, 2.0, n)
    om = np.full((K, K), 0.002)
    om[0, 0] = 0.05
    for q in (4, 8, 20):
        _check(*_both(rg, ctx, c, th, om, 3, q))


_SLOT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth
from paper_2312_01560_b200 import raftgp as rg
ctx = rg.Context(0)
c, th, om = synth.sbm_params('C2', 2, n=20000)
for q in (6, 20):
    rs, rd = oracle.sbm_sample(c, th, om, 11, q=q)
    gs, gd = rg.raftgp_sbm_sample(ctx, torch.from_numpy(c).cuda(), torch.from_numpy(th).cuda(),
                                  torch.from_numpy(om).cuda(), 11, q=q)
    assert np.array_equal(gs.cpu().numpy(), rs) and np.array_equal(gd.cpu().numpy(), rd), q
print('ok', rs.size)
"""


@pytest.mark.parametrize("slots,log", [("0", None), ("1", None), ("3", None), ("1", "0"), ("2", "100")])
def test_parity_slot_paths(rg, slots, log):
    """The write pass emits the event cells recorded by the count walk (RAFTGP_SBM_SLOTS per chunk) and the
    events logged past them (RAFTGP_SBM_LOG entries); chunks whose events do not all fit are walked again.
    slots = 0 (every chunk walked twice), 1 and 3 (most events logged), no log (overflow chunks re-walked) and
    a log too small for the events (falls back to the re-walk) must all give the oracle's edge list."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RAFTGP_SBM_SLOTS=slots)
    if log is not None:
        env["RAFTGP_SBM_LOG"] = log
    r = subprocess.run([sys.executable, "-c", _SLOT_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_parity_many_blocks(rg, ctx):
    """K above the counting-sort limit (4096): member lists come from the CSR build path instead."""
    rng = np.random.default_rng(5)
    n, K = 6000, 4200
    c = rng.integers(0, K, n).astype(np.int32)
    th = rng.uniform(0.5, 3.0, n)
    om = np.full((K, K), 2e-3)
    np.fill_diagonal(om, 0.5)
    _check(*_both(rg, ctx, c, th, om, 3, 20))
