"""CPU ORACLE for the RaftGP embedding hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may import this
package. The product package paper_2312_01560_b200/ never imports it and shares no code with it.

Thin ctypes wrapper over oracle/oracle.c (plain C, fp64; the Gaussian generator is fp32 bit-exact
per docs/SKETCH_SPEC.md). Every function cites the passage it follows in oracle.c's header.
Parity status of each function is listed in DESIGN.md §"Oracle pins"; none is "parity unpinned"
except the Θ/W bit pattern, which is fixed by the spec rather than by the paper (the paper names no
generator).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

NCUT, MOD, MOD_REDUCED, PROP = 0, 1, 2, 3
VARIANTS = {"ncut": NCUT, "mod": MOD, "mod_reduced": MOD_REDUCED}


def build() -> str:
    src = os.path.join(_HERE, "oracle.c")
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-o", _SO + ".tmp", src, "-lm"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        for name in ("oracle_gaussian", "oracle_build_csr", "oracle_apply", "oracle_project", "oracle_gcn",
                     "oracle_embed_rows", "oracle_modularity", "oracle_ncut", "oracle_local_modularity",
                     "oracle_kmeans2", "oracle_model_select", "oracle_split_stops", "oracle_sbm_sample"):
            getattr(_lib, name).restype = ctypes.c_int
    return _lib


def set_threads(k: int) -> None:
    """Threads of the oracle's row loops (0 = OpenMP default = all cores). Results are bit-identical for any k
    (each output row is computed sequentially by one thread; cross-row sums stay sequential)."""
    _L().oracle_set_threads(ctypes.c_int(int(k)))


def get_threads() -> int:
    return int(_L().oracle_get_threads())


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc)


# ------------------------------------------------------------------ generator (SKETCH_SPEC)
def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    _L().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def ln_spec(u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, np.float32)
    out = np.empty_like(u)
    _L().oracle_ln_spec_batch(_p(u), _p(out), ctypes.c_int64(u.size))
    return out


def sincos_spec(k2: np.ndarray):
    k2 = np.ascontiguousarray(k2, np.uint32)
    c = np.empty(k2.shape, np.float32)
    s = np.empty(k2.shape, np.float32)
    _L().oracle_sincos_spec_batch(_p(k2), _p(c), _p(s), ctypes.c_int64(k2.size))
    return c, s


def gaussian(seed: int, tag: int, row_begin: int, rows: int, cols: int, den: int) -> np.ndarray:
    """rows x cols block (global rows row_begin..) of the spec generator, fp32 bit-exact."""
    out = np.empty((rows, cols), np.float32)
    _check(_L().oracle_gaussian(ctypes.c_uint64(seed), ctypes.c_uint32(tag), ctypes.c_int64(row_begin),
                                ctypes.c_int64(rows), ctypes.c_int32(cols), ctypes.c_int32(den), _p(out)))
    return out


def theta(n: int, r: int, seed: int, row_begin: int = 0) -> np.ndarray:
    """Θ of Eq. 5 (tag 0, variance 1/r)."""
    return gaussian(seed, 0, row_begin, n, r, r)


def weights(k: int, fan_in: int, fan_out: int, seed: int) -> np.ndarray:
    """W^(k) of Eq. 6 (tag k, variance 1/fan_in)."""
    return gaussian(seed, k, 0, fan_in, fan_out, fan_in)


# ------------------------------------------------------------------ graph
class CSR:
    def __init__(self, n, row_ptr, col):
        self.n = int(n)
        self.row_ptr = row_ptr
        self.col = col

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    @property
    def deg(self):
        return np.diff(self.row_ptr).astype(np.int32)


def build_csr(n: int, src, dst) -> CSR:
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    m = src.size
    row_ptr = np.zeros(n + 1, np.int64)
    col = np.zeros(max(1, 2 * m), np.int32)
    nnz = ctypes.c_int64(0)
    _check(_L().oracle_build_csr(ctypes.c_int64(n), ctypes.c_int64(m), _p(src), _p(dst), _p(row_ptr), _p(col),
                                 ctypes.byref(nnz)))
    return CSR(n, row_ptr, col[: nnz.value].copy())


def apply(g: CSR, op: int, X: np.ndarray) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float64)
    if X.ndim == 1:
        return apply(g, op, X[:, None])[:, 0]
    out = np.empty_like(X)
    _check(_L().oracle_apply(ctypes.c_int64(g.n), _p(g.row_ptr), _p(g.col), ctypes.c_int(op),
                             ctypes.c_int32(X.shape[1]), _p(X), _p(out)))
    return out


def project(g: CSR, variant, r: int, seed: int) -> np.ndarray:
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    Y = np.empty((g.n, r), np.float64)
    _check(_L().oracle_project(ctypes.c_int64(g.n), _p(g.row_ptr), _p(g.col), ctypes.c_int(v), ctypes.c_int32(r),
                               ctypes.c_uint64(seed), _p(Y)))
    return Y


def gcn(g: CSR, dims, seed: int, Y: np.ndarray):
    """Returns [Z^(1), ..., Z^(K)] (Z^(K) = the embedding Z)."""
    dims = np.ascontiguousarray(dims, np.int32)
    K = len(dims) - 1
    Y = np.ascontiguousarray(Y, np.float64)
    tot = int(sum(int(d) for d in dims[1:]))
    Zc = np.empty(g.n * tot, np.float64)
    _check(_L().oracle_gcn(ctypes.c_int64(g.n), _p(g.row_ptr), _p(g.col), ctypes.c_int32(K), _p(dims),
                           ctypes.c_uint64(seed), _p(Y), _p(Zc)))
    out, off = [], 0
    for k in range(1, K + 1):
        out.append(Zc[off: off + g.n * dims[k]].reshape(g.n, dims[k]))
        off += g.n * dims[k]
    return out


def embed_rows(g: CSR, variant, r: int, dims, seed: int, rows):
    """(Y[rows], [Z^(k)[rows]]) via the receptive field; identical arithmetic to project + gcn."""
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    dims = np.ascontiguousarray(dims if dims is not None else [r], np.int32)
    K = len(dims) - 1
    rows = np.ascontiguousarray(rows, np.int64)
    S = rows.size
    Y = np.empty((S, r), np.float64)
    tot = int(sum(int(d) for d in dims[1:]))
    Zc = np.empty(max(1, S * tot), np.float64)
    _check(_L().oracle_embed_rows(ctypes.c_int64(g.n), _p(g.row_ptr), _p(g.col), ctypes.c_int(v), ctypes.c_int32(r),
                                  ctypes.c_int32(K), _p(dims), ctypes.c_uint64(seed), _p(rows), ctypes.c_int64(S),
                                  _p(Y), _p(Zc)))
    out, off = [], 0
    for k in range(1, K + 1):
        out.append(Zc[off: off + S * dims[k]].reshape(S, dims[k]))
        off += S * dims[k]
    return Y, out


# ------------------------------------------------------------------ scoring
def modularity(g: CSR, assign, k: int) -> float:
    a = np.ascontiguousarray(assign, np.int32)
    out = ctypes.c_double(0)
    _check(_L().oracle_modularity(ctypes.c_int64(g.n), _p(g.row_ptr), _p(g.col), _p(a), ctypes.c_int32(k),
                                  ctypes.byref(out)))
    return out.value


def ncut(g: CSR, assign, k: int) -> float:
    a = np.ascontiguousarray(assign, np.int32)
    out = ctypes.c_double(0)
    _check(_L().oracle_ncut(ctypes.c_int64(g.n), _p(g.row_ptr), _p(g.col), _p(a), ctypes.c_int32(k),
                            ctypes.byref(out)))
    return out.value


def local_modularity(g: CSR, nodes, block_of_node, k: int) -> float:
    nd = np.ascontiguousarray(nodes, np.int64)
    b = np.ascontiguousarray(block_of_node, np.int32)
    out = ctypes.c_double(0)
    _check(_L().oracle_local_modularity(ctypes.c_int64(g.n), _p(g.row_ptr), _p(g.col), _p(nd), ctypes.c_int64(nd.size),
                                        _p(b), ctypes.c_int32(k), ctypes.byref(out)))
    return out.value


# ------------------------------------------------------------------ Alg. 1 model selection (NEXT-1)
def kmeans2(Z: np.ndarray, members, max_iter: int = 100):
    """SELECT_SPEC §3: deterministic 2-means on the rows Z[members]. Returns (side uint8[len], iterations)."""
    Z = np.ascontiguousarray(Z, np.float32)
    U = np.ascontiguousarray(members, np.int32)
    side = np.zeros(max(1, U.size), np.uint8)
    it = _L().oracle_kmeans2(_p(Z), ctypes.c_int32(Z.shape[1]), _p(U), ctypes.c_int64(U.size),
                             ctypes.c_int32(max_iter), _p(side))
    return side[: U.size], int(it)


def model_select(g: CSR, Z: np.ndarray, eps: int = 5, max_iter: int = 100, rule=0):
    """Alg. 1 from U = V on the fp32 embedding Z. Returns (labels int32[n], K, stats)
    with canonical labels (SELECT_SPEC §5) and stats = dict(blocks, splits, kmeans_iters, depth).
    rule: 0 = "global" e = |E| (SELECT_SPEC §4 default), 1 = "local" 2e = degree sum of U."""
    rule = {"global": 0, "local": 1}.get(rule, rule)
    Z = np.ascontiguousarray(Z, np.float32)
    labels = np.zeros(max(1, g.n), np.int32)
    k = ctypes.c_int32(0)
    st = np.zeros(4, np.int64)
    _check(_L().oracle_model_select(ctypes.c_int64(g.n), _p(g.row_ptr), _p(g.col), _p(Z), ctypes.c_int32(Z.shape[1]),
                                    ctypes.c_int32(eps), ctypes.c_int32(max_iter), ctypes.c_int32(rule), _p(labels), ctypes.byref(k), _p(st)))
    return labels[: g.n], int(k.value), dict(zip(("blocks", "splits", "kmeans_iters", "depth"), (int(x) for x in st)))


def split_stops(g: CSR, members, side, eps: int = 5, rule=0) -> bool:
    """Alg. 1 lines 2+4 (SELECT_SPEC §4): True iff U = members, split by `side`, becomes a block."""
    rule = {"global": 0, "local": 1}.get(rule, rule)
    U = np.ascontiguousarray(members, np.int32)
    sd = np.ascontiguousarray(side, np.uint8)
    where = np.zeros(g.n + 1, np.int32)
    return bool(_L().oracle_split_stops(_p(g.row_ptr), _p(g.col), ctypes.c_int64(int(g.row_ptr[-1])), _p(U),
                                        ctypes.c_int64(U.size), _p(sd), ctypes.c_int32(eps), ctypes.c_int32(rule),
                                        _p(where)))


# ------------------------------------------------------------------ NEXT-2: Table I widths
def gcn_np(g: CSR, dims, seed: int, Y: np.ndarray):
    """Eq. 6 + row l2 normalisation for wide layers (Table I), the same
    steps as oracle_gcn but with numpy's fp64 matmul as the dense product (a library primitive) so that
    4096-wide stacks finish in seconds: Z^(k) = rownorm(tanh((P Z^(k-1)) W^(k))), P applied by oracle_apply.
    Pinned against the C oracle_gcn at small widths (tests/test_oracle_graph_ops.py)."""
    Z = np.ascontiguousarray(Y, np.float64)
    out = []
    for k in range(1, len(dims)):
        W = weights(k, int(dims[k - 1]), int(dims[k]), seed).astype(np.float64)
        H = np.tanh(apply(g, PROP, Z) @ W)
        nrm = np.sqrt((H * H).sum(axis=1))
        Z = np.where(nrm[:, None] > 0, H / np.where(nrm > 0, nrm, 1.0)[:, None], 0.0)
        out.append(Z)
    return out


# ------------------------------------------------------------------ NEXT-3: Alg. 2 SBM sampler
def _L_f64():
    lib = _L()
    lib.oracle_ln_spec64.restype = ctypes.c_double
    lib.oracle_ln_spec64.argtypes = [ctypes.c_double]
    lib.oracle_sbm_uniform.restype = ctypes.c_double
    lib.oracle_sbm_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
    lib.oracle_sbm_range_sum_hook.restype = ctypes.c_double
    lib.oracle_sbm_range_sum_hook.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_int64]
    return lib


def sbm_range_sum(theta_r, theta_s, omega: float, x: int, y: int) -> float:
    """SBM_SPEC §3 RangeSum over cells x..y of one block pair (theta_s=None: the diagonal pair of theta_r)."""
    tr = np.ascontiguousarray(theta_r, np.float64)
    ts = np.ascontiguousarray(theta_s if theta_s is not None else [0.0], np.float64)
    return _L_f64().oracle_sbm_range_sum_hook(int(theta_s is None), tr.size, tr.ctypes.data, ts.size if theta_s is not None else 0,
                                              ts.ctypes.data, float(omega), int(x), int(y))


def ln_spec64(u: float) -> float:
    """SBM_SPEC §6."""
    return _L_f64().oracle_ln_spec64(float(u))


def sbm_uniform(seed: int, p: int, k: int, d: int) -> float:
    """SBM_SPEC §5."""
    return _L_f64().oracle_sbm_uniform(seed, p, k, d)


def sbm_sample(c, theta, omega, seed: int, q: int = 20, cap=None):
    """Alg. 2 per docs/SBM_SPEC.md: returns (src, dst) int32 edge arrays in (pair, chunk,
    cell) order."""
    c = np.ascontiguousarray(c, np.int32)
    theta = np.ascontiguousarray(theta, np.float64)
    omega = np.ascontiguousarray(omega, np.float64)
    K = omega.shape[0]
    n = c.size
    m = ctypes.c_int64(0)
    cap = int(cap) if cap is not None else max(1024, int(4 * (theta.sum() ** 2) * omega.max() + 10 * n))
    while True:
        src = np.zeros(max(1, cap), np.int32)
        dst = np.zeros(max(1, cap), np.int32)
        _check(_L().oracle_sbm_sample(ctypes.c_int64(n), ctypes.c_int32(K), _p(c), _p(theta), _p(omega),
                                      ctypes.c_uint64(seed), ctypes.c_int32(q), _p(src), _p(dst),
                                      ctypes.c_int64(cap), ctypes.byref(m)))
        if m.value <= cap:
            return src[: m.value].copy(), dst[: m.value].copy()
        cap = m.value
