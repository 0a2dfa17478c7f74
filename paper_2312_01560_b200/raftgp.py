"""Thin Python binding of the C-ABI in include/raftgp.h (ctypes; argument marshalling only).

Every computation happens inside libraftgp.so (sm_100a kernels). PyTorch is used only to own device
memory and to supply the CUDA stream. There is no fallback: if the library is missing or no GPU is
present, calls raise.

Function names are the C-ABI names; `Context` and `Graph` wrap the two opaque handles.
"""
from __future__ import annotations

import atexit
import ctypes
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RAFTGP_LIB") or os.path.join(_HERE, "libraftgp.so")

RAFTGP_OK, RAFTGP_ERR_PARAM, RAFTGP_ERR_DATA = 0, 2, 3
RAFTGP_ERR_INTERNAL, RAFTGP_ERR_CUDA, RAFTGP_ERR_NOMEM, RAFTGP_ERR_COMM, RAFTGP_ERR_STATE = 4, 5, 6, 7, 8
RAFTGP_NCUT, RAFTGP_MOD, RAFTGP_MOD_REDUCED = 0, 1, 2
VARIANTS = {"ncut": RAFTGP_NCUT, "mod": RAFTGP_MOD, "mod_reduced": RAFTGP_MOD_REDUCED}
RAFTGP_LMOD_GLOBAL, RAFTGP_LMOD_LOCAL = 0, 1
LMOD_RULES = {"global": RAFTGP_LMOD_GLOBAL, "local": RAFTGP_LMOD_LOCAL}
RAFTGP_HOST_PTRS, RAFTGP_DEVICE_PTRS = 0, 1

# every symbol declared in include/raftgp.h
EXPORTS = (
    "raftgp_last_error", "raftgp_version", "raftgp_ctx_create", "raftgp_ctx_destroy", "raftgp_ctx_sync",
    "raftgp_ctx_stream", "raftgp_ctx_set_profiling", "raftgp_prof_kernels", "raftgp_prof_name", "raftgp_prof_read",
    "raftgp_prof_reset", "raftgp_launch_count", "raftgp_sketch_transform", "raftgp_build_csr", "raftgp_graph_info", "raftgp_graph_export",
    "raftgp_graph_local_degrees", "raftgp_graph_set_degrees", "raftgp_graph_set_order", "raftgp_graph_destroy", "raftgp_sketch",
    "raftgp_weights", "raftgp_project", "raftgp_gcn_transform", "raftgp_gcn_hop", "raftgp_gnn_embed",
    "raftgp_embed", "raftgp_embed_multi", "raftgp_feature_transform", "raftgp_modularity", "raftgp_ncut", "raftgp_local_modularity",
    "raftgp_model_select", "raftgp_gemm_tf32x3", "raftgp_sbm_sample", "raftgp_stream_create",
    "raftgp_stream_add_edges", "raftgp_stream_embedding", "raftgp_stream_graph", "raftgp_stream_destroy",
    "raftgp_stream_set_mode",
    "raftgp_build_embed", "raftgp_ctx_trim", "raftgp_feature_transform_push", "raftgp_gcn_hop_push",
    "raftgp_ipc_alloc", "raftgp_ipc_free", "raftgp_ipc_open", "raftgp_ipc_close", "raftgp_copy",
    "raftgp_nccl_unique_id", "raftgp_ctx_create_dist", "raftgp_ctx_rank", "raftgp_barrier", "raftgp_allgather",
    "raftgp_build_embed_loopback",
)

_lib = None
_exiting = False


def _mark_exit():
    global _exiting
    _exiting = True


atexit.register(_mark_exit)   # no library calls from __del__ once the interpreter (and CUDA) shut down
c_i32, c_i64, c_u32, c_u64, c_vp, c_dbl = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                           ctypes.c_void_p, ctypes.c_double)
P = ctypes.POINTER

_SIGS = {
    "raftgp_last_error": (ctypes.c_char_p, []),
    "raftgp_version": (ctypes.c_char_p, []),
    "raftgp_ctx_create": (ctypes.c_int, [ctypes.c_int, c_vp, P(c_vp)]),
    "raftgp_ctx_destroy": (ctypes.c_int, [c_vp]),
    "raftgp_ctx_sync": (ctypes.c_int, [c_vp]),
    "raftgp_ctx_stream": (ctypes.c_int, [c_vp, P(c_vp)]),
    "raftgp_ctx_trim": (ctypes.c_int, [c_vp, P(c_i64)]),
    "raftgp_ctx_set_profiling": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "raftgp_prof_kernels": (ctypes.c_int, []),
    "raftgp_prof_name": (ctypes.c_char_p, [ctypes.c_int]),
    "raftgp_prof_read": (ctypes.c_int, [c_vp, ctypes.c_int, P(c_dbl), P(c_i64)]),
    "raftgp_prof_reset": (ctypes.c_int, [c_vp]),
    "raftgp_launch_count": (ctypes.c_int, [c_vp, P(c_i64), ctypes.c_int]),
    "raftgp_build_csr": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_u32, P(c_vp)]),
    "raftgp_graph_info": (ctypes.c_int, [c_vp, P(c_i64), P(c_i64), P(c_i64), P(c_i64), P(c_i64)]),
    "raftgp_graph_export": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_u32]),
    "raftgp_graph_local_degrees": (ctypes.c_int, [c_vp, c_vp]),
    "raftgp_graph_set_degrees": (ctypes.c_int, [c_vp, c_vp]),
    "raftgp_graph_set_order": (ctypes.c_int, [c_vp, c_vp]),
    "raftgp_graph_destroy": (ctypes.c_int, [c_vp]),
    "raftgp_sketch": (ctypes.c_int, [c_vp, c_u64, c_u32, c_i64, c_i64, c_i32, c_i32, c_vp]),
    "raftgp_weights": (ctypes.c_int, [c_vp, c_u64, c_i32, c_i32, c_i32, c_vp]),
    "raftgp_sketch_transform": (ctypes.c_int, [c_vp, c_u64, c_i64, c_i32, c_vp, c_i32, c_vp]),
    "raftgp_project": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32, c_u64, c_vp]),
    "raftgp_gcn_transform": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_i32, c_vp]),
    "raftgp_gcn_hop": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_vp]),
    "raftgp_feature_transform_push": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_i32, c_u64, c_vp, c_i32]),
    "raftgp_gcn_hop_push": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_i32]),
    "raftgp_ipc_alloc": (ctypes.c_int, [c_vp, ctypes.c_size_t, P(c_vp), c_vp]),
    "raftgp_ipc_free": (ctypes.c_int, [c_vp, c_vp]),
    "raftgp_ipc_open": (ctypes.c_int, [c_vp, c_vp, P(c_vp)]),
    "raftgp_ipc_close": (ctypes.c_int, [c_vp, c_vp]),
    "raftgp_copy": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_size_t]),
    "raftgp_gnn_embed": (ctypes.c_int, [c_vp, c_i32, c_vp, c_u64, c_vp, c_vp, c_vp]),
    "raftgp_embed": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32, c_vp, c_u64, c_vp, c_vp, c_vp]),
    "raftgp_embed_multi": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_vp, c_u64, c_vp, c_vp]),
    "raftgp_feature_transform": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_i32, c_u64, c_vp]),
    "raftgp_modularity": (ctypes.c_int, [c_vp, c_vp, c_i32, P(c_dbl)]),
    "raftgp_ncut": (ctypes.c_int, [c_vp, c_vp, c_i32, P(c_dbl)]),
    "raftgp_local_modularity": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_i32, P(c_dbl)]),
    "raftgp_model_select": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, P(c_i32), c_vp]),
    "raftgp_gemm_tf32x3": (ctypes.c_int, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "raftgp_sbm_sample": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_u64, c_i32, c_vp, c_vp, c_i64, P(c_i64)]),
    "raftgp_stream_create": (ctypes.c_int, [c_vp, c_i32, c_vp, c_u64, P(c_vp)]),
    "raftgp_stream_add_edges": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_u32, c_vp]),
    "raftgp_stream_embedding": (ctypes.c_int, [c_vp, c_vp]),
    "raftgp_stream_graph": (ctypes.c_int, [c_vp, P(c_vp)]),
    "raftgp_stream_destroy": (ctypes.c_int, [c_vp]),
    "raftgp_stream_set_mode": (ctypes.c_int, [c_vp, c_i32]),
    "raftgp_build_embed": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_u32, c_i32, c_vp, c_i32, c_vp, c_u64, c_vp,
                                          P(c_vp)]),
    "raftgp_build_embed_loopback": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i64, c_vp, c_vp, c_u32, c_i32, c_vp, c_i32, c_vp,
                                                   c_u64, c_vp]),
    "raftgp_nccl_unique_id": (ctypes.c_int, [c_vp]),
    "raftgp_ctx_create_dist": (ctypes.c_int, [ctypes.c_int, c_vp, ctypes.c_int, ctypes.c_int, c_vp, P(c_vp)]),
    "raftgp_ctx_rank": (ctypes.c_int, [c_vp, P(ctypes.c_int), P(ctypes.c_int)]),
    "raftgp_barrier": (ctypes.c_int, [c_vp]),
    "raftgp_allgather": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_size_t]),
}


class RaftGPError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"raftgp status {code}: {msg}")
        self.code = code


def load_library(path: str = LIB_PATH):
    """Load libraftgp.so (raises if it has not been built: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _ck(rc: int):
    if rc != RAFTGP_OK:
        raise RaftGPError(rc, load_library().raftgp_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensors passed to raftgp must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _own(t: torch.Tensor, stream) -> torch.Tensor:
    """t as a contiguous tensor for a library call that reads it on `stream` (the context's stream). The caller keeps
    the returned tensor alive for the whole call. A copy made here runs on torch's current stream: when that is not
    the context's stream, the context's stream waits for it, and record_stream keeps the caching allocator from
    handing the copy's memory out again before the library's kernels have read it."""
    c = t.contiguous()
    if c is not t and c.is_cuda and stream is not None:
        cur = torch.cuda.current_stream(c.device)
        if stream.cuda_stream != cur.cuda_stream:
            stream.wait_stream(cur)
            c.record_stream(stream)
    return c


def _dev(t: torch.Tensor, what: str):
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    return t


# ------------------------------------------------------------------ context
class Context:
    """raftgp_ctx on one device, enqueuing on a torch CUDA stream (the current one by default). With `dist=(rank,
    world, uid)` the context joins a world-rank NCCL communicator (raftgp_ctx_create_dist; uid from
    raftgp_nccl_unique_id() on rank 0, passed to the others out of band)."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None, dist=None):
        lib = load_library()
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = c_vp()
        if dist is None:
            _ck(lib.raftgp_ctx_create(device, c_vp(self.stream.cuda_stream), ctypes.byref(h)))
        else:
            rank, world, uid = dist
            if len(uid) != 128:
                raise ValueError("the NCCL unique id has 128 bytes")
            ub = (ctypes.c_char * 128).from_buffer_copy(uid)
            _ck(lib.raftgp_ctx_create_dist(device, c_vp(self.stream.cuda_stream), int(rank), int(world), ub,
                                           ctypes.byref(h)))
        self.h = h

    def rank_world(self):
        r, w = ctypes.c_int(0), ctypes.c_int(1)
        _ck(load_library().raftgp_ctx_rank(self.h, ctypes.byref(r), ctypes.byref(w)))
        return r.value, w.value

    def barrier(self):
        """Stream-ordered barrier over the context's communicator (no-op on a one-rank context)."""
        _ck(load_library().raftgp_barrier(self.h))

    def allgather(self, send: torch.Tensor, recv: torch.Tensor):
        """ncclAllGather on the context stream: recv (world x send bytes) receives every rank's send block."""
        _ck(load_library().raftgp_allgather(self.h, _ptr(send), _ptr(recv), send.numel() * send.element_size()))

    def sync(self):
        _ck(load_library().raftgp_ctx_sync(self.h))

    def trim(self) -> int:
        """Release the cached workspace blocks to the device; returns the bytes released."""
        b = c_i64(0)
        _ck(load_library().raftgp_ctx_trim(self.h, ctypes.byref(b)))
        return b.value

    def set_profiling(self, on: bool = True):
        _ck(load_library().raftgp_ctx_set_profiling(self.h, int(on)))

    def prof_read(self) -> dict:
        """{kernel_name: (total_ms, launches)} of the launches recorded since the last reset."""
        lib = load_library()
        out = {}
        for k in range(lib.raftgp_prof_kernels()):
            ms, cnt = c_dbl(0), c_i64(0)
            _ck(lib.raftgp_prof_read(self.h, k, ctypes.byref(ms), ctypes.byref(cnt)))
            if cnt.value:
                out[lib.raftgp_prof_name(k).decode()] = (ms.value, cnt.value)
        return out

    def prof_reset(self):
        _ck(load_library().raftgp_prof_reset(self.h))

    def launch_count(self, reset: bool = False) -> int:
        v = c_i64(0)
        _ck(load_library().raftgp_launch_count(self.h, ctypes.byref(v), int(reset)))
        return v.value

    def close(self):
        if getattr(self, "h", None) is not None and _lib is not None and not _exiting:
            _lib.raftgp_ctx_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ graph
class Graph:
    """raftgp_graph: the canonical CSR of rows [row_begin, row_end) plus degree scalars, on device."""

    def __init__(self, ctx: Context, h):
        self.ctx = ctx
        self.h = h

    def info(self):
        v = [c_i64(0) for _ in range(5)]
        _ck(load_library().raftgp_graph_info(self.h, *[ctypes.byref(x) for x in v]))
        n, rb, re, nnz, two_e = (x.value for x in v)
        return dict(n=n, row_begin=rb, row_end=re, nnz_local=nnz, two_e=two_e)

    @property
    def n(self):
        return self.info()["n"]

    @property
    def rows(self):
        i = self.info()
        return i["row_end"] - i["row_begin"]

    def export(self):
        """Host copies (numpy) of the local row_ptr (int64), col_idx (int32) and degrees (int32)."""
        i = self.info()
        rows = i["row_end"] - i["row_begin"]
        rp = np.zeros(rows + 1, np.int64)
        col = np.zeros(max(1, i["nnz_local"]), np.int32)
        deg = np.zeros(max(1, rows), np.int32)
        _ck(load_library().raftgp_graph_export(self.h, c_vp(rp.ctypes.data), c_vp(col.ctypes.data),
                                               c_vp(deg.ctypes.data), RAFTGP_HOST_PTRS))
        return rp, col[: i["nnz_local"]], deg[:rows]

    def local_degrees(self) -> torch.Tensor:
        out = torch.empty(max(1, self.rows), dtype=torch.int32, device=self.ctx.device)
        _ck(load_library().raftgp_graph_local_degrees(self.h, _ptr(out)))
        return out[: self.rows]

    def set_degrees(self, deg_all: torch.Tensor):
        d = _own(_dev(deg_all, "deg_all"), self.ctx.stream)
        _ck(load_library().raftgp_graph_set_degrees(self.h, _ptr(d)))

    def set_order(self, order: Optional[torch.Tensor]):
        """Row visiting order (int32 permutation of the local rows) or None for the natural order."""
        o = None if order is None else _own(_dev(order, "order"), self.ctx.stream)
        _ck(load_library().raftgp_graph_set_order(self.h, _ptr(o)))

    def close(self):
        if getattr(self, "h", None) is not None and _lib is not None and not _exiting:
            _lib.raftgp_graph_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def raftgp_build_csr(ctx: Context, n: int, src: torch.Tensor, dst: torch.Tensor, row_begin: int = 0,
                     row_end: Optional[int] = None) -> Graph:
    """a1 + a2. src/dst: int32 tensors (CUDA -> device pointers; CPU -> host pointers copied in-call)."""
    if src.dtype != torch.int32 or dst.dtype != torch.int32 or src.numel() != dst.numel():
        raise ValueError("src/dst must be int32 tensors of equal length")
    if src.is_cuda != dst.is_cuda:
        raise ValueError("src and dst must live on the same side")
    flags = RAFTGP_DEVICE_PTRS if src.is_cuda else RAFTGP_HOST_PTRS
    src, dst = _own(src, ctx.stream), _own(dst, ctx.stream)
    h = c_vp()
    re = n if row_end is None else row_end
    _ck(load_library().raftgp_build_csr(ctx.h, n, src.numel(), _ptr(src), _ptr(dst), row_begin, re, flags,
                                        ctypes.byref(h)))
    return Graph(ctx, h)


# ------------------------------------------------------------------ sketch
def raftgp_sketch(ctx: Context, seed: int, tag: int, row_begin: int, rows: int, cols: int, den: int,
                  out: Optional[torch.Tensor] = None) -> torch.Tensor:
    if out is None:
        out = torch.empty((rows, cols), dtype=torch.float32, device=ctx.device)
    _ck(load_library().raftgp_sketch(ctx.h, seed, tag, row_begin, rows, cols, den, _ptr(out)))
    return out


def raftgp_weights(ctx: Context, seed: int, k: int, fan_in: int, fan_out: int,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
    if out is None:
        out = torch.empty((fan_in, fan_out), dtype=torch.float32, device=ctx.device)
    _ck(load_library().raftgp_weights(ctx.h, seed, k, fan_in, fan_out, _ptr(out)))
    return out


def raftgp_sketch_transform(ctx: Context, seed: int, rows: int, W: torch.Tensor) -> torch.Tensor:
    """Theta' = Theta W (Theta generated on chip, tcgen05 3xTF32 GEMM)."""
    r, l1 = W.shape
    out = torch.empty((rows, l1), dtype=torch.float32, device=ctx.device)
    Wc = _own(W, ctx.stream)
    _ck(load_library().raftgp_sketch_transform(ctx.h, seed, rows, r, _ptr(Wc), l1, _ptr(out)))
    return out


# ------------------------------------------------------------------ project / gcn
def _variant(v) -> int:
    return VARIANTS[v] if isinstance(v, str) else int(v)


def raftgp_project(g: Graph, variant, r: int, seed: int, Y: Optional[torch.Tensor] = None) -> torch.Tensor:
    if Y is None:
        Y = torch.empty((g.rows, r), dtype=torch.float32, device=g.ctx.device)
    _ck(load_library().raftgp_project(g.h, _variant(variant), r, seed, _ptr(Y)))
    return Y


def raftgp_gcn_transform(g: Graph, Z: torch.Tensor, W: torch.Tensor, T: Optional[torch.Tensor] = None):
    lin, lout = W.shape
    if T is None:
        T = torch.empty((g.rows, lout), dtype=torch.float32, device=g.ctx.device)
    _ck(load_library().raftgp_gcn_transform(g.h, _ptr(Z), lin, _ptr(W), lout, _ptr(T)))
    return T


def raftgp_gcn_hop(g: Graph, T_full, Z_out: Optional[torch.Tensor] = None,
                   W_next: Optional[torch.Tensor] = None, T_next: Optional[torch.Tensor] = None,
                   w: Optional[int] = None):
    """T_full: n x w tensor, or a raw device pointer with its width w."""
    w = T_full.shape[1] if isinstance(T_full, torch.Tensor) else int(w)
    wn = 0 if W_next is None else W_next.shape[1]
    if W_next is not None and T_next is None:
        T_next = torch.empty((g.rows, wn), dtype=torch.float32, device=g.ctx.device)
    _ck(load_library().raftgp_gcn_hop(g.h, _dptr(T_full) if T_full is not None else None, w, _ptr(Z_out),
                                      _ptr(W_next), wn, _ptr(T_next)))
    return Z_out, T_next


def _zk_array(Zk: Sequence[Optional[torch.Tensor]]):
    arr = (c_vp * max(1, len(Zk)))()
    for i, t in enumerate(Zk):
        arr[i] = None if t is None else t.data_ptr()
    return arr


def raftgp_gnn_embed(g: Graph, dims: Sequence[int], seed: int, Y: torch.Tensor, Z: Optional[torch.Tensor] = None,
                     intermediates: bool = False):
    """Returns Z, or (Z, [Z^(1), ..., Z^(K-1)]) when intermediates=True."""
    dims = [int(d) for d in dims]
    L = len(dims) - 1
    dev = g.ctx.device
    if Z is None:
        Z = torch.empty((g.rows, dims[-1]), dtype=torch.float32, device=dev)
    Zk = [torch.empty((g.rows, dims[k]), dtype=torch.float32, device=dev) for k in range(1, L)] if intermediates else []
    d = (c_i32 * len(dims))(*dims)
    _ck(load_library().raftgp_gnn_embed(g.h, L, d, seed, _ptr(Y), _ptr(Z),
                                        _zk_array(Zk) if intermediates else None))
    return (Z, Zk) if intermediates else Z


def raftgp_embed(g: Graph, variant, dims: Sequence[int], seed: int, Y: Optional[torch.Tensor] = None,
                 Z: Optional[torch.Tensor] = None, want_Y: bool = True, intermediates: bool = False):
    """Fused project + gnn_embed. Returns (Y or None, Z[, Zk])."""
    dims = [int(d) for d in dims]
    L = len(dims) - 1
    dev = g.ctx.device
    if Y is None and want_Y:
        Y = torch.empty((g.rows, dims[0]), dtype=torch.float32, device=dev)
    if Z is None:
        Z = torch.empty((g.rows, dims[-1]), dtype=torch.float32, device=dev)
    Zk = [torch.empty((g.rows, dims[k]), dtype=torch.float32, device=dev) for k in range(1, L)] if intermediates else []
    d = (c_i32 * len(dims))(*dims)
    _ck(load_library().raftgp_embed(g.h, _variant(variant), L, d, seed, _ptr(Y), _ptr(Z),
                                    _zk_array(Zk) if intermediates else None))
    return (Y, Z, Zk) if intermediates else (Y, Z)


def raftgp_embed_multi(g: Graph, variants: Sequence, dims: Sequence[int], seed: int, Z=None, want_Y: bool = False):
    """Several variants in one call (one Theta, one shared gather for NCUT + MOD).
    Returns ({variant: Y} or None, {variant: Z})."""
    dims = [int(d) for d in dims]
    vs = [_variant(v) for v in variants]
    names = [v if isinstance(v, str) else {0: "ncut", 1: "mod", 2: "mod_reduced"}[int(v)] for v in variants]
    dev = g.ctx.device
    Z = Z or {nm: torch.empty((g.rows, dims[-1]), dtype=torch.float32, device=dev) for nm in names}
    Y = {nm: torch.empty((g.rows, dims[0]), dtype=torch.float32, device=dev) for nm in names} if want_Y else None
    va = (c_i32 * len(vs))(*vs)
    d = (c_i32 * len(dims))(*dims)
    _ck(load_library().raftgp_embed_multi(g.h, len(vs), va, len(dims) - 1, d, seed,
                                          _zk_array([Y[nm] for nm in names]) if want_Y else None,
                                          _zk_array([Z[nm] for nm in names])))
    return Y, Z


def raftgp_nccl_unique_id() -> bytes:
    """A new NCCL unique id (128 bytes) for raftgp_ctx_create_dist (created on rank 0, sent to the others)."""
    b = (ctypes.c_char * 128)()
    _ck(load_library().raftgp_nccl_unique_id(b))
    return bytes(b)


def local_rows(n: int, rank: int, world: int):
    """Rank `rank`'s rows [p R, min((p+1) R, n)), R = ceil(n / world) (the library's row partition)."""
    R = max(1, -(-n // world))
    return min(n, rank * R), min(n, (rank + 1) * R)


def raftgp_build_embed(ctx: Context, n: int, src: torch.Tensor, dst: torch.Tensor, variants: Sequence,
                       dims: Sequence[int], seed: int, Z=None, keep_graph: bool = False):
    """raftgp_build_csr + raftgp_embed_multi in one call (Theta' overlapped with the CSR build on a side stream).
    On a distributed context: the row-partitioned step; Z holds this rank's rows. Returns ({variant: Z}, Graph or
    None)."""
    if src.dtype != torch.int32 or dst.dtype != torch.int32 or src.numel() != dst.numel():
        raise ValueError("src/dst must be int32 tensors of equal length")
    dims = [int(d) for d in dims]
    vs = [_variant(v) for v in variants]
    names = [v if isinstance(v, str) else {0: "ncut", 1: "mod", 2: "mod_reduced"}[int(v)] for v in variants]
    rank, world = ctx.rank_world()
    rb, re = local_rows(n, rank, world)
    Z = Z or {nm: torch.empty((max(1, re - rb), dims[-1]), dtype=torch.float32, device=ctx.device)[: re - rb]
              for nm in names}
    flags = RAFTGP_DEVICE_PTRS if src.is_cuda else RAFTGP_HOST_PTRS
    s, d = _own(src, ctx.stream), _own(dst, ctx.stream)
    va = (c_i32 * len(vs))(*vs)
    dd = (c_i32 * len(dims))(*dims)
    h = c_vp()
    _ck(load_library().raftgp_build_embed(ctx.h, n, s.numel(), _ptr(s), _ptr(d), flags, len(vs), va, len(dims) - 1, dd,
                                          seed, _zk_array([Z[nm] for nm in names]),
                                          ctypes.byref(h) if keep_graph else None))
    return Z, (Graph(ctx, h) if keep_graph else None)


def raftgp_build_embed_loopback(ctx: Context, P: int, n: int, src: torch.Tensor, dst: torch.Tensor, variants: Sequence,
                                dims: Sequence[int], seed: int, Z=None) -> dict:
    """The row-partitioned step with P logical ranks on this context's GPU (all n rows of Z)."""
    if src.dtype != torch.int32 or dst.dtype != torch.int32 or src.numel() != dst.numel():
        raise ValueError("src/dst must be int32 tensors of equal length")
    dims = [int(d) for d in dims]
    vs = [_variant(v) for v in variants]
    names = [v if isinstance(v, str) else {0: "ncut", 1: "mod", 2: "mod_reduced"}[int(v)] for v in variants]
    Z = Z or {nm: torch.empty((max(1, n), dims[-1]), dtype=torch.float32, device=ctx.device)[:n] for nm in names}
    flags = RAFTGP_DEVICE_PTRS if src.is_cuda else RAFTGP_HOST_PTRS
    s, d = _own(src, ctx.stream), _own(dst, ctx.stream)
    va = (c_i32 * len(vs))(*vs)
    dd = (c_i32 * len(dims))(*dims)
    _ck(load_library().raftgp_build_embed_loopback(ctx.h, P, n, s.numel(), _ptr(s), _ptr(d), flags, len(vs), va,
                                                   len(dims) - 1, dd, seed, _zk_array([Z[nm] for nm in names])))
    return Z


def _dptr(x) -> int:
    """Device pointer of a CUDA tensor or a raw pointer (int)."""
    if isinstance(x, torch.Tensor):
        return _ptr(_dev(x, "buffer"))
    return int(x)


def raftgp_feature_transform_push(g: Graph, variants: Sequence, r: int, l1: int, seed: int, reps: dict):
    """a6 fused: T1 of every variant pushed into all ranks' full n x l1 copies. reps = {variant: [ptr or tensor
    per rank]} (same length for every variant)."""
    vs = [_variant(v) for v in variants]
    names = [v if isinstance(v, str) else {0: "ncut", 1: "mod", 2: "mod_reduced"}[int(v)] for v in variants]
    nrep = len(reps[names[0]])
    flat = [_dptr(p) for nm in names for p in reps[nm]]
    arr = (c_vp * len(flat))(*flat)
    va = (c_i32 * len(vs))(*vs)
    _ck(load_library().raftgp_feature_transform_push(g.h, len(vs), va, r, l1, seed, arr, nrep))


def raftgp_gcn_hop_push(g: Graph, T_full, w: int, W_next: torch.Tensor, reps: Sequence, want_Z: bool = False):
    """a6 fused: one GCN hop whose T_next rows go straight into every rank's full copy (reps: ptrs/tensors).
    Returns Z (local rows x w) when want_Z, else None."""
    Z = torch.empty((max(1, g.rows), w), dtype=torch.float32, device=g.ctx.device)[: g.rows] if want_Z else None
    flat = [_dptr(p) for p in reps]
    arr = (c_vp * len(flat))(*flat)
    Wn = _own(W_next, g.ctx.stream)
    _ck(load_library().raftgp_gcn_hop_push(g.h, _dptr(T_full), w, None if Z is None else _ptr(Z),
                                           _ptr(Wn), W_next.shape[1], arr, len(flat)))
    return Z


class IpcBuffer:
    """A library-allocated device buffer that other processes can map (raftgp_ipc_alloc)."""

    def __init__(self, ctx: Context, nbytes: int):
        self.ctx = ctx
        p = c_vp()
        self.handle = (ctypes.c_char * 64)()
        _ck(load_library().raftgp_ipc_alloc(ctx.h, nbytes, ctypes.byref(p), self.handle))
        self.ptr = p.value
        self.nbytes = nbytes

    def handle_bytes(self) -> bytes:
        return bytes(self.handle)

    def close(self):
        if getattr(self, "ptr", None) and _lib is not None and not _exiting:
            _lib.raftgp_ipc_free(self.ctx.h, c_vp(self.ptr))
        self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def raftgp_ipc_open(ctx: Context, handle: bytes) -> int:
    """Map another process's IpcBuffer on this context's device; returns the device pointer."""
    h = (ctypes.c_char * 64).from_buffer_copy(handle)
    p = c_vp()
    _ck(load_library().raftgp_ipc_open(ctx.h, h, ctypes.byref(p)))
    return p.value


def raftgp_ipc_close(ctx: Context, ptr: int):
    _ck(load_library().raftgp_ipc_close(ctx.h, c_vp(ptr)))


def raftgp_copy(ctx: Context, dst, src, nbytes: int):
    """Device-to-device copy by a library kernel (tensors or raw pointers)."""
    _ck(load_library().raftgp_copy(ctx.h, c_vp(_dptr(dst)), c_vp(_dptr(src)), nbytes))


def raftgp_feature_transform(g: Graph, variants: Sequence, r: int, l1: int, seed: int) -> dict:
    """{variant: T1 = s^ (.) (X Theta W^(1))} for the graph's local rows."""
    vs = [_variant(v) for v in variants]
    names = [v if isinstance(v, str) else {0: "ncut", 1: "mod", 2: "mod_reduced"}[int(v)] for v in variants]
    T = {nm: torch.empty((g.rows, l1), dtype=torch.float32, device=g.ctx.device) for nm in names}
    va = (c_i32 * len(vs))(*vs)
    _ck(load_library().raftgp_feature_transform(g.h, len(vs), va, r, l1, seed, _zk_array([T[nm] for nm in names])))
    return T


# ------------------------------------------------------------------ scoring (host)
def _labels(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), np.int32)


def raftgp_modularity(g: Graph, assign, k: int) -> float:
    a = _labels(assign)
    out = c_dbl(0)
    _ck(load_library().raftgp_modularity(g.h, c_vp(a.ctypes.data), k, ctypes.byref(out)))
    return out.value


def raftgp_ncut(g: Graph, assign, k: int) -> float:
    a = _labels(assign)
    out = c_dbl(0)
    _ck(load_library().raftgp_ncut(g.h, c_vp(a.ctypes.data), k, ctypes.byref(out)))
    return out.value


def raftgp_local_modularity(g: Graph, nodes, block_of_node, k: int) -> float:
    nd = np.ascontiguousarray(np.asarray(nodes), np.int64)
    b = _labels(block_of_node)
    out = c_dbl(0)
    _ck(load_library().raftgp_local_modularity(g.h, c_vp(nd.ctypes.data), nd.size, c_vp(b.ctypes.data), k,
                                               ctypes.byref(out)))
    return out.value


# ------------------------------------------------------------------ NEXT-1: Alg. 1 model selection
def raftgp_model_select(g: Graph, Z: torch.Tensor, eps: int = 5, max_iter: int = 100, rule="global",
                        labels: Optional[torch.Tensor] = None):
    """Alg. 1 on the device embedding Z (n x L fp32). Returns (labels int32 CUDA tensor, K, stats dict)."""
    if Z.dtype != torch.float32 or Z.dim() != 2:
        raise ValueError("Z must be a 2-D float32 tensor")
    _dev(Z, "Z")
    r = LMOD_RULES[rule] if isinstance(rule, str) else int(rule)
    if labels is None:
        labels = torch.empty(max(1, g.rows), dtype=torch.int32, device=g.ctx.device)[: g.rows]
    k = c_i32(0)
    st = np.zeros(9, np.int64)
    Zc = _own(Z, g.ctx.stream)
    _ck(load_library().raftgp_model_select(g.h, _ptr(Zc), Z.shape[1], eps, max_iter, r, _ptr(labels),
                                           ctypes.byref(k), c_vp(st.ctypes.data)))
    return labels, int(k.value), dict(zip(("blocks", "splits", "lloyd_iters", "levels", "lloyd_rows", "seed_rows", "rows_read",
                                           "capped_segments", "capped_rows"),
                                 (int(x) for x in st)))


# ------------------------------------------------------------------ NEXT-2: tensor-core GEMM
def raftgp_gemm_tf32x3(ctx: Context, A: torch.Tensor, B: torch.Tensor, row_scale: Optional[torch.Tensor] = None,
                       C: Optional[torch.Tensor] = None) -> torch.Tensor:
    """C = diag(row_scale) A B (fp32-accurate 3xTF32 on the tcgen05 tensor cores)."""
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("inner dimensions differ")
    if C is None:
        C = torch.empty((M, N), dtype=torch.float32, device=ctx.device)
    Ac, Bc = _own(A, ctx.stream), _own(B, ctx.stream)
    _ck(load_library().raftgp_gemm_tf32x3(ctx.h, M, K, N, _ptr(Ac), _ptr(Bc),
                                          _ptr(row_scale), _ptr(C)))
    return C


# ------------------------------------------------------------------ NEXT-3: exact SBM sampler
def raftgp_sbm_sample(ctx: Context, c: torch.Tensor, theta: torch.Tensor, omega: torch.Tensor, seed: int,
                      q: int = 20, cap: Optional[int] = None):
    """Alg. 2 (docs/SBM_SPEC.md) on the device: returns (src, dst) int32 CUDA tensors."""
    c = _own(_dev(c.to(torch.int32), "c"), ctx.stream)
    theta = _own(_dev(theta.to(torch.float64), "theta"), ctx.stream)
    omega = _own(_dev(omega.to(torch.float64), "omega"), ctx.stream)
    K = omega.shape[0]
    n = c.numel()
    if cap is None:   # expected edges + slack (a second call fixes an underestimate)
        cap = int(1.2 * _expected_edges(c, theta, omega)) + 1024
    m = c_i64(0)
    while True:
        src = torch.empty(max(1, cap), dtype=torch.int32, device=ctx.device)
        dst = torch.empty(max(1, cap), dtype=torch.int32, device=ctx.device)
        _ck(load_library().raftgp_sbm_sample(ctx.h, n, K, _ptr(c), _ptr(theta), _ptr(omega), seed, q, _ptr(src),
                                             _ptr(dst), cap, ctypes.byref(m)))
        if m.value <= cap:
            return src[: m.value], dst[: m.value]
        cap = m.value


def _expected_edges(c, theta, omega) -> float:
    """sum_{i<j} lambda_ij (upper bound of the expected simple-graph edge count), from block theta sums."""
    K = omega.shape[0]
    ts = torch.zeros(K, dtype=torch.float64, device=theta.device).index_add_(0, c.long(), theta)
    t2 = torch.zeros(K, dtype=torch.float64, device=theta.device).index_add_(0, c.long(), theta * theta)
    tot = (ts[:, None] * ts[None, :] * omega).sum() - (t2 * torch.diagonal(omega)).sum()
    return float(tot.item()) / 2


# ------------------------------------------------------------------ NEXT-4: streaming updates
class Stream:
    """raftgp_stream: a graph (ownership taken from `graph`) and its NCut embedding, updated by edge additions."""

    def __init__(self, graph: Graph, dims: Sequence[int], seed: int):
        self.ctx = graph.ctx
        self.dims = [int(d) for d in dims]
        h = c_vp()
        d = (c_i32 * len(self.dims))(*self.dims)
        _ck(load_library().raftgp_stream_create(graph.h, len(self.dims) - 1, d, seed, ctypes.byref(h)))
        graph.h = None          # owned by the stream now
        self.h = h

    def add_edges(self, src: torch.Tensor, dst: torch.Tensor) -> dict:
        """Merge the pairs (src, dst) into the graph and re-embed the affected rows; returns the set sizes."""
        if src.dtype != torch.int32 or dst.dtype != torch.int32 or src.numel() != dst.numel():
            raise ValueError("src/dst must be int32 tensors of equal length")
        L = len(self.dims) - 1
        st = np.zeros(L + 3, np.int64)
        flags = RAFTGP_DEVICE_PTRS if src.is_cuda else RAFTGP_HOST_PTRS
        s, d = _own(src, self.ctx.stream), _own(dst, self.ctx.stream)
        _ck(load_library().raftgp_stream_add_edges(self.h, s.numel(), _ptr(s), _ptr(d), flags, c_vp(st.ctypes.data)))
        return {"changed": int(st[0]), "affected": [int(x) for x in st[1:L + 2]], "nnz": int(st[L + 2])}

    MODES = {"exact": 0, "delta": 1}

    def set_mode(self, mode: str) -> None:
        """raftgp_stream_set_mode: "exact" (bit-identical last hop, the default) or "delta" (the last hop updated by
        the changed rows only; setting it again resyncs)."""
        _ck(load_library().raftgp_stream_set_mode(self.h, self.MODES[mode]))

    def embedding(self) -> torch.Tensor:
        n = self.graph().n
        Z = torch.empty((max(1, n), self.dims[-1]), dtype=torch.float32, device=self.ctx.device)[:n]
        _ck(load_library().raftgp_stream_embedding(self.h, _ptr(Z)))
        return Z

    def graph(self) -> Graph:
        """Borrowed handle of the current graph (valid until the next add_edges; never destroyed by Python)."""
        h = c_vp()
        _ck(load_library().raftgp_stream_graph(self.h, ctypes.byref(h)))
        g = Graph.__new__(Graph)
        g.ctx = self.ctx
        g.h = h
        g.close = lambda: None   # borrowed
        return g

    def close(self):
        if getattr(self, "h", None) is not None and _lib is not None and not _exiting:
            _lib.raftgp_stream_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
