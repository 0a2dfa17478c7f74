"""bench.py end to end on the GPU: the default one-GPU line (C2 for speed) carries the contract's keys, and
`--gpus 2` (self-spawned under torch.distributed.run; both ranks on this one GPU with gloo host barriers, the
functional mode RAFTGP_BENCH_ONE_GPU=1 -- not a measurement) runs the row-partitioned step and prints one line with
n_gpus = 2 and the exchange / partition block."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
QUICK = ["--config", "C2", "--steps", "2", "--warmup", "3", "--no-select", "--no-table1", "--no-sbm", "--no-stream",
         "--no-clocks"]


def _run(args, env=None):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, env=e, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-4000:]
    return json.loads(lines[0])


def test_bench_one_gpu_line(cuda_required):
    rec = _run(QUICK + ["--no-cpu-baseline"])
    assert rec["n_gpus"] == 1 and rec["value"] > 0 and rec["unit"] == "nnz*r/s"
    assert rec["roofline"]["bound"] == "hbm" and rec["roofline"]["achieved"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] > 0 and rec["gpu_launches"] > 0


def test_bench_two_ranks_one_gpu(cuda_required):
    rec = _run(["--gpus", "2", *QUICK, "--no-e2e"], {"RAFTGP_BENCH_BACKEND": "gloo", "RAFTGP_BENCH_ONE_GPU": "1"})
    assert rec["n_gpus"] == 2 and rec["value"] > 0
    d = rec["dist"]
    assert len(d["nnz_local"]) == 2 and sum(d["nnz_local"]) == rec["config"]["nnz"]
    assert d["egress_bytes_per_rank_per_step"] > 0
