"""CPU tier: the C-ABI library loads without a GPU, exports every function
include/krn_b200.h declares, and the product path fails loudly (no CPU
fallback) when no device is present."""

import ctypes
import os
import subprocess

import pytest

from paper_2507_13204_b200 import _cabi
from conftest import HAVE_GPU, ROOT


def test_library_loads_and_exports_header():
    lib = _cabi.lib()
    declared = _cabi.declared_functions()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert set(declared) == set(_cabi.SIGNATURES), "ctypes signature table out of sync with the header"
    assert b"sm_100a" in lib.krn_version()


def test_symbols_are_c_abi():
    out = subprocess.run(["nm", "-D", "--defined-only", _cabi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in _cabi.declared_functions():
        assert name in exported  # unmangled


def test_sm100_code_present():
    out = subprocess.run(["cuobjdump", "-lelf", _cabi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(HAVE_GPU, reason="checks the no-device behaviour")
def test_no_cpu_fallback():
    import numpy as np

    import paper_2507_13204_b200 as krn

    lap = krn.load_program("laplacian")
    with pytest.raises(_cabi.KrnNativeError):
        krn.execute(lap, "normRes1DLaplacianSQ", {"x": np.ones(3), "b": np.zeros(3)})
    with pytest.raises(_cabi.KrnNativeError):
        krn.pairwise_sum([1.0, 2.0])


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2507_13204_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(dirpath, f), encoding="utf-8").read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "krn_oracle" not in text, f
