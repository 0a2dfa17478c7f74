"""The C-ABI from plain C: examples/raftgp_demo.c (built by __graft_entry__.build()) builds the CSR of a ring +
chords graph from host arrays, embeds it (NCut and Mod, GCN 64 -> 64 -> 32) and scores a labelling. Its
printout must match the Python binding on the same inputs exactly (same library, same kernels) and the
oracle (CSR size, modularity / NCut to 1e-12, unit rows)."""
import os
import subprocess

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ring_chords(n):
    i = np.arange(n, dtype=np.int64)
    src = np.repeat(i, 2).astype(np.int32)
    dst = np.empty(2 * n, np.int32)
    dst[0::2] = (i + 1) % n
    dst[1::2] = (7 * i + 3) % n
    return src, dst


@pytest.mark.parametrize("n", [1000, 4099])
def test_c_demo_matches_python_and_oracle(cuda_required, n):
    from paper_2312_01560_b200 import build as b
    from paper_2312_01560_b200 import raftgp as rg
    exe = b.build_demo()
    out = subprocess.run([exe, str(n), "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = {l.split()[0]: l.split() for l in out.stdout.strip().splitlines()}
    src, dst = _ring_chords(n)
    ref = oracle.build_csr(n, src, dst)
    assert int(lines["n"][3]) == ref.row_ptr[-1] and int(lines["n"][5]) == ref.row_ptr[-1]
    ctx = rg.Context(0)
    g = rg.raftgp_build_csr(ctx, n, torch.from_numpy(src), torch.from_numpy(dst))
    _, Z = rg.raftgp_embed_multi(g, ["ncut", "mod"], (64, 64, 32), 1)
    for v in ("ncut", "mod"):
        z = Z[v].cpu().numpy().astype(np.float64)
        s, sq, z00 = (float(x) for x in lines[v][2::2])
        assert s == float(f"{z.sum():.9e}") or abs(s - z.sum()) <= 1e-6 * max(1.0, abs(z.sum()))
        assert abs(sq - (z * z).sum()) <= 1e-6 * n and abs(sq - n) < 1e-3 * n   # unit rows
        assert z00 == float(f"{z[0, 0]:.9e}")
    lab = ((np.arange(n) * 4) // n).astype(np.int32)
    q, nc = float(lines["modularity"][1]), float(lines["modularity"][3])
    assert abs(q - oracle.modularity(ref, lab, 4)) < 1e-9
    assert abs(nc - oracle.ncut(ref, lab, 4)) < 1e-9
