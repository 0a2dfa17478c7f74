"""Build libraftgp.so in-tree with nvcc for sm_100a (B200). No JIT, no torch extension cache:
the .so lives next to this file so it travels to the GPU box with the repo snapshot."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libraftgp.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-fvisibility=hidden",
]


def nccl_home() -> str:
    """NCCL the library links against: the torch wheel's (nvidia-nccl, 2.28.x), so a process that also imports torch
    loads ONE libnccl.so.2 (same soname, same file); RAFTGP_NCCL_HOME overrides (needs include/nccl.h and
    lib/libnccl.so.2)."""
    cands = [os.environ.get("RAFTGP_NCCL_HOME", "")]
    try:
        import nvidia.nccl as _n   # the wheel torch's libtorch_cuda resolves libnccl.so.2 from
        cands += list(_n.__path__)
    except Exception:
        pass
    cands.append("/usr")
    for c in cands:
        if c and os.path.exists(os.path.join(c, "include", "nccl.h")) and \
                os.path.exists(os.path.join(c, "lib", "libnccl.so.2")):
            return c
    raise RuntimeError("NCCL (include/nccl.h + lib/libnccl.so.2) not found; set RAFTGP_NCCL_HOME")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "raftgp.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    if out == LIB and not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = out + ".tmp"
    nh = nccl_home()
    nlib = os.path.join(nh, "lib")
    cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", os.path.join(nh, "include"),
           "-o", tmp, *sources(), "-Xlinker", os.path.join(nlib, "libnccl.so.2"), "-Xlinker", f"-rpath,{nlib}"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


DEMO_SRC = os.path.join(os.path.dirname(HERE), "examples", "raftgp_demo.c")
DEMO = os.path.join(os.path.dirname(HERE), "examples", "raftgp_demo")


def build_demo(force: bool = False) -> str:
    """gcc the plain-C example of the C-ABI (examples/raftgp_demo.c) against the in-tree library."""
    if not force and os.path.exists(DEMO) and os.path.getmtime(DEMO) > max(os.path.getmtime(DEMO_SRC),
                                                                             os.path.getmtime(LIB)):
        return DEMO
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-std=c99", "-Wall", DEMO_SRC, "-I", INCLUDE,
           "-I", os.path.join(cuda, "include"), "-L", HERE, "-lraftgp", "-L", os.path.join(cuda, "lib64"), "-lcudart",
           "-lm", "-Wl,-rpath,$ORIGIN/../paper_2312_01560_b200", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", DEMO]
    subprocess.check_call(cmd)
    return DEMO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
