"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a, loads, and
exports every symbol include/gicp.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gicp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gicp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import importlib.util
    spec = importlib.util.spec_from_file_location("gicp_build", os.path.join(ROOT, "paper_2308_07173_b200",
                                                                             "build.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m.build()


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ["gicp_build_index", "gicp_knn", "gicp_covariances", "gicp_linearize", "gicp_align"]:
        assert name in d


def test_library_exports_every_declared_symbol(lib):
    L = ctypes.CDLL(lib)
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(gicp_[a-z0-9_]+)\b", out))
    assert set(_declared()) <= exported
    # nothing else leaks from the C++ implementation
    assert not [s for s in re.findall(r" T (\S+)", out) if s.startswith("_ZN4gicp")]


def test_binary_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_exports_match(lib):
    import paper_2308_07173_b200 as g
    assert set(g.EXPORTS) == set(_declared())
    assert g.version() >= 100


def test_product_path_does_not_touch_the_oracle():
    pkg = os.path.join(ROOT, "paper_2308_07173_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle/" not in txt and "liboracle" not in txt, f


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without the CUDA library the package refuses to import."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "try:\n    import paper_2308_07173_b200\nexcept ImportError as e:\n    print('IMPORT-ERROR', e)\n"
            "else:\n    print('IMPORTED')\n") % ROOT
    env = dict(os.environ, GICP_LIB_VARIANT=str(tmp_path / "missing.so"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env).stdout
    assert "IMPORT-ERROR" in out and "IMPORTED" not in out


def test_tensors_must_be_on_the_gpu(lib):
    import numpy as np
    import torch
    import paper_2308_07173_b200 as g
    with pytest.raises(ValueError):  # CPU tensors are rejected before any call (no host fallback)
        g.build_index(torch.from_numpy(np.zeros((10, 3), np.float32)), 0.5)
