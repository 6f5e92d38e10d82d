"""The C-ABI library loads and exports every symbol include/gk_bdl.h declares
(no compute call: this runs without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gk_bdl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gk_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(gk):
    names = declared_symbols()
    assert len(names) >= 20
    L = gk.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_canon_node_layout_matches_oracle(oracle, gk):
    from paper_2207_01834_b200.bdltree import CANON_NODE
    assert CANON_NODE.itemsize == 168 == oracle.CANON_NODE.itemsize == oracle.lib().gko_node_size()


def test_version_and_invalid_args(gk):
    L = gk.lib()
    assert b"sm_100a" in L.gk_version()
    import pytest
    with pytest.raises(ValueError):
        gk.BDLTree(9)  # dispatch_dim: 2..8 only (point.hpp:22-35)
    with pytest.raises(ValueError):
        gk.BDLTree(3, leaf_size=0)


def test_library_is_sm100a():
    lib = os.path.join(ROOT, "paper_2207_01834_b200", "_lib", "libgkbdl.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _compile_client(out):
    import subprocess
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    lib = os.path.join(ROOT, "paper_2207_01834_b200", "_lib")
    r = subprocess.run([cxx, "-std=c++20", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "cpp_client.cpp"), "-L", lib, "-lgkbdl",
                        f"-Wl,-rpath,{lib}", "-o", out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_cpp_binding_compiles(gk, tmp_path):
    """include/geokit_bdl.hpp (the reference-side C++ binding) compiles and links against the ABI"""
    _compile_client(str(tmp_path / "client"))


def test_cli_usage_without_gpu(gk):
    """the CLI harness is built and rejects bad usage with exit code 1"""
    import subprocess
    exe = os.path.join(ROOT, "paper_2207_01834_b200", "_lib", "gk_bdl_cli")
    assert os.path.exists(exe)
    assert subprocess.run([exe], capture_output=True).returncode == 1
    assert subprocess.run([exe, "frobnicate"], capture_output=True).returncode == 1


def test_device_api_rejects_host_tensors():
    """the torch-tensor checks of the device API run before any pointer crosses the ABI (no GPU needed)"""
    import types
    torch = pytest.importorskip("torch")
    from paper_2207_01834_b200.bdltree import BDLTree
    stub = types.SimpleNamespace(device=0)
    with pytest.raises(ValueError, match="CUDA"):
        BDLTree._dev(stub, torch.zeros((4, 3), dtype=torch.float64), "float64", (None, 3), "q_dev")
    with pytest.raises(ValueError, match="CUDA"):
        BDLTree._dev(stub, np.zeros((4, 3)), "float64", (None, 3), "q_dev")
    assert BDLTree._dev(stub, None, "int32", (None,), "ids", optional=True) is None
