"""The C-ABI library: loads without a GPU and exports every symbol include/*.h declares;
the product path refuses to run without a device (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "feast_gpu.h")).read()
    return sorted(set(re.findall(r"\b(feast_gpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_0901_2665_b200 import feast as F
    lib = ctypes.CDLL(F.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(F.EXPORTED_SYMBOLS)
    assert lib.feast_gpu_abi_version() == 1


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_0901_2665_b200 import feast as F
    with pytest.raises(F.Error):
        F.GpuContext(0)


def test_missing_library_fails_loudly(tmp_path):
    from paper_0901_2665_b200 import feast as F
    saved = F._lib
    try:
        F._lib = None
        with pytest.raises(ImportError):
            F.load_library(str(tmp_path / "nope.so"))
    finally:
        F._lib = saved


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_0901_2665_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "libfeastref" not in txt and "libfeastoracle" not in txt, f
