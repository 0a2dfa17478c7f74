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


def _compile_one(args):
    cmd, obj = args
    subprocess.check_call(cmd)
    return obj


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """One object per .cu (compiled in parallel, reused while the .cu, the headers and the defines are unchanged),
    then one shared-library link. The .cu files share no device code, so no relocatable device code is needed."""
    if out == LIB and not force and not _stale():
        return LIB
    import hashlib
    from concurrent.futures import ThreadPoolExecutor
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = out + ".tmp"
    nh = nccl_home()
    nlib = os.path.join(nh, "lib")
    key = hashlib.sha1(" ".join([*NVCC_FLAGS, *defines, nh]).encode()).hexdigest()[:10]
    objdir = os.path.join(os.path.dirname(HERE), "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "raftgp.h"), __file__]
    hdr_t = max(os.path.getmtime(p) for p in hdrs)
    jobs, objs = [], []
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]
    for src in sources():
        obj = os.path.join(objdir, f"{os.path.basename(src)}.{key}.o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(hdr_t, os.path.getmtime(src)):
            cmd = [nvcc, *cflags, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", os.path.join(nh, "include"),
                   "-c", src, "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            jobs.append((cmd, obj))
    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            list(ex.map(_compile_one, jobs))
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-Xlinker", os.path.join(nlib, "libnccl.so.2"), "-Xlinker", f"-rpath,{nlib}"]
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
