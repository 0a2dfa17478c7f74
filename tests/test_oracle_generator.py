"""Pins of the oracle's Gaussian generator (docs/SKETCH_SPEC.md; Eq. 5, Eq. 6 W^(k)).

What pins what (none of these re-types the oracle's code):
  * Philox words   — CUDA's own host-compiled curand_Philox4x32_10 (an independent implementation).
  * ln_spec/sincos — numpy's float64 log / cos / sin over EVERY 24-bit input the generator can produce.
  * Box–Muller + column layout — invariants z_a^2 + z_b^2 = -2 ln u1 and atan2(z_b, z_a) = 2 pi u2,
    with u1/u2 recomputed from the pinned Philox words.
  * Distribution   — moments and a KS test against N(0, 1/den) (variance reading #2/#4).
The fp32 bit pattern itself is fixed by the spec, not by the paper.
"""
import os
import subprocess

import numpy as np
import pytest
import scipy.stats

import oracle

CURAND_HARNESS = r"""
#include <cstdio>
#include <cstdint>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main() {
  unsigned a[6];
  while (scanf("%u %u %u %u %u %u", &a[0], &a[1], &a[2], &a[3], &a[4], &a[5]) == 6) {
    uint4 c = {a[0], a[1], a[2], a[3]}; uint2 k = {a[4], a[5]};
    uint4 o = curand_Philox4x32_10(c, k);
    printf("%u %u %u %u\n", o.x, o.y, o.z, o.w);
  }
  return 0;
}
"""


@pytest.fixture(scope="module")
def curand_philox(tmp_path_factory):
    d = tmp_path_factory.mktemp("curand")
    src = d / "h.cpp"
    src.write_text(CURAND_HARNESS)
    exe = d / "h"
    cuda_inc = "/usr/local/cuda/include"
    if not os.path.exists(os.path.join(cuda_inc, "curand_philox4x32_x.h")):
        pytest.skip("CUDA headers not present")
    subprocess.check_call(["g++", "-O1", "-I", cuda_inc, str(src), "-o", str(exe)])

    def run(rows):
        inp = "\n".join(" ".join(str(int(v)) for v in r) for r in rows) + "\n"
        out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout
        return np.array([[int(t) for t in line.split()] for line in out.strip().splitlines()], np.uint64)

    return run


def test_philox_matches_curand_host(curand_philox):
    rng = np.random.default_rng(1)
    rows = rng.integers(0, 2 ** 32, size=(3000, 6), dtype=np.uint64).tolist()
    rows += [[0] * 6, [0xFFFFFFFF] * 6, [1, 0, 0, 0, 0, 0], [0, 0, 0, 0, 1, 0], [5, 17, 0, 3, 0, 0]]
    ref = curand_philox(rows)
    mine = np.array([oracle.philox(r[:4], r[4:]) for r in rows], np.uint64)
    np.testing.assert_array_equal(mine, ref)


def test_ln_spec_all_inputs_vs_libm():
    k = np.arange(1, 2 ** 24 + 1, dtype=np.uint64)
    u = (k.astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)
    got = oracle.ln_spec(u).astype(np.float64)
    ref = np.log(u.astype(np.float64))
    err = np.abs(got - ref)
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    ulp[ref == 0] = 2.0 ** -149
    # accurate to a few fp32 ulp everywhere (accuracy only shapes the Gaussian; bits are fixed by the spec)
    assert np.max(err / np.maximum(ulp, 2.0 ** -30)) <= 4.0
    assert got[-1] == 0.0                      # u1 = 1 -> ln = 0 exactly -> R = 0


def test_sincos_spec_all_inputs_vs_libm():
    k2 = np.arange(0, 2 ** 24, dtype=np.uint32)
    c, s = oracle.sincos_spec(k2)
    ang = 2.0 * np.pi * (k2.astype(np.float64) / 2.0 ** 24)
    assert np.max(np.abs(c - np.cos(ang))) < 4e-7
    assert np.max(np.abs(s - np.sin(ang))) < 4e-7
    # exact quadrant structure: k2 = 0 -> (1, 0); quarter turns are sign-exact
    assert c[0] == 1.0 and s[0] == 0.0
    assert c[2 ** 22] == 0.0
    assert s[2 ** 22] == 1.0 and c[2 ** 23] == -1.0


@pytest.mark.parametrize("seed,tag,den", [(0, 0, 1), (123456789012345, 0, 1), (7, 3, 1)])
def test_box_muller_invariants_and_layout(seed, tag, den):
    rows, cols = 64, 16
    row0 = 2 ** 33 + 5 if seed == 7 else 0          # exercises hi32(i) in the counter
    Z = oracle.gaussian(seed, tag, row0, rows, cols, den).astype(np.float64)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for i in range(rows):
        gi = row0 + i
        for q in range(cols // 4):
            x = oracle.philox([q, gi & 0xFFFFFFFF, gi >> 32, tag], key).astype(np.uint64)
            for pair in range(2):
                xa, xb = int(x[2 * pair]), int(x[2 * pair + 1])
                u1 = ((xa >> 8) + 1) / 2.0 ** 24
                u2 = (xb >> 8) / 2.0 ** 24
                za, zb = Z[i, 4 * q + 2 * pair], Z[i, 4 * q + 2 * pair + 1]
                r2 = -2.0 * np.log(u1)
                assert abs(za * za + zb * zb - r2) <= 3e-6 * max(1.0, r2)
                if r2 > 1e-6:
                    ang = np.arctan2(zb, za) % (2 * np.pi)
                    d = abs(ang - 2 * np.pi * u2)
                    assert min(d, 2 * np.pi - d) < 2e-6 / np.sqrt(r2) + 1e-6


def test_sigma_scaling_is_exact():
    # den = 64 -> sigma = 0.125 exactly: the scaled draw is the unit draw times 2^-3, bit for bit
    a = oracle.gaussian(11, 0, 0, 40, 64, 1)
    b = oracle.gaussian(11, 0, 0, 40, 64, 64)
    np.testing.assert_array_equal(a * np.float32(0.125), b)


def test_theta_distribution_N_0_1_over_r():
    r = 128
    th = oracle.theta(8192, r, seed=0).astype(np.float64).ravel()      # 1,048,576 draws
    sd = 1.0 / np.sqrt(r)
    assert abs(th.mean()) < 5 * sd / np.sqrt(th.size)
    assert abs(th.var() / sd ** 2 - 1.0) < 5 * np.sqrt(2.0 / th.size)
    kurt = scipy.stats.kurtosis(th / sd)
    assert abs(kurt) < 5 * np.sqrt(24.0 / th.size)
    assert scipy.stats.kstest(th / sd, "norm").pvalue > 1e-4
    # columns are not correlated with each other (pairs share one Philox call)
    M = th.reshape(8192, r)
    C = np.corrcoef(M[:, :8].T)
    assert np.max(np.abs(C - np.eye(8))) < 5 / np.sqrt(8192)


def test_weights_variance_is_fan_in():
    W = oracle.weights(2, 128, 64, seed=0).astype(np.float64)
    assert abs(W.var() * 128 - 1.0) < 0.06
    W1 = oracle.weights(1, 128, 64, seed=0)
    assert not np.array_equal(W, W1)                 # tags separate the streams (reading #5)


def test_rows_are_addressed_globally():
    full = oracle.theta(50, 7, seed=3)
    part = oracle.theta(20, 7, seed=3, row_begin=30)
    np.testing.assert_array_equal(full[30:], part)
