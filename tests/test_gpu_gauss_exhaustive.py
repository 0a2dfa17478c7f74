"""The Gaussian generator's branch-free steps (gauss.cuh: div_rn_narrow, sqrt_rn_narrow, the select-based quadrant
map) against the generic IEEE forms (__fdiv_rn, __fsqrt_rn, switch) on EVERY input they can receive: all 2^24
values of u1 (radius, ln) and of k2 (sincos2pi). The sketch is then bit-identical to SKETCH_SPEC by construction
(the Theta bit-exactness tests against the oracle stay in test_gpu_parity.py)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_generator_steps_exhaustive(cuda_required, tmp_path):
    exe = str(tmp_path / "gauss_exhaustive")
    subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe,
                           os.path.join(HERE, "cuda", "gauss_exhaustive.cu")])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("radius 0 ln 0 sincos 0 "), out.stdout
