"""B200-native RaftGP embedding hot path (arxiv 2312.01560).

libraftgp.so (csrc/, sm_100a) does every step of the path; `raftgp` is its ctypes binding and
`dist` the row-partitioned multi-GPU orchestration (torch.distributed all-gather between hops).
"""
from . import raftgp  # noqa: F401
from .raftgp import (  # noqa: F401
    Context, Graph, RaftGPError, raftgp_build_csr, raftgp_embed, raftgp_gcn_hop, raftgp_gcn_transform,
    raftgp_gnn_embed, raftgp_local_modularity, raftgp_modularity, raftgp_ncut, raftgp_project, raftgp_sketch,
    raftgp_weights,
)
