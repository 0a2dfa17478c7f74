"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol that
include/raftgp.h declares (no compute calls without a GPU), the binding declares the same set, and
the product package never touches oracle/."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "raftgp.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"RAFTGP_API\s+[\w\s\*]+?\b(raftgp_\w+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("raftgp_build_csr", "raftgp_project", "raftgp_gnn_embed", "raftgp_modularity", "raftgp_ncut",
              "raftgp_local_modularity", "raftgp_sketch", "raftgp_gcn_hop"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2312_01560_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (raftgp_\w+)", out))
    assert exported == set(declared_symbols())        # nothing undeclared leaks out either


def test_binding_covers_header():
    from paper_2312_01560_b200 import raftgp
    assert set(raftgp.EXPORTS) == set(declared_symbols())


def test_library_is_sm100a():
    from paper_2312_01560_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_without_gpu():
    from paper_2312_01560_b200 import raftgp
    lib = raftgp.load_library()
    assert b"sm_100a" in lib.raftgp_version()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2312_01560_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", text, re.M), f
                assert "oracle.c" not in text and "liboracle" not in text, f


def test_missing_library_fails_loudly(tmp_path):
    from paper_2312_01560_b200 import raftgp
    saved = raftgp._lib
    raftgp._lib = None
    try:
        with pytest.raises(RuntimeError):
            raftgp.load_library(str(tmp_path / "nope.so"))
    finally:
        raftgp._lib = saved
