"""div_by (the hoisted-reciprocal division of the fp64 reference-order paths)
must equal __ddiv_rn bit for bit: 2^30 random and edge-case operand pairs on
the GPU, from tests/cuda/div_check.cu built with nvcc at test time."""
import ctypes
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def test_div_by_matches_ddiv_rn(tmp_path):
    so = str(tmp_path / "div_check.so")
    subprocess.run(["nvcc", "-shared", "-O3", "-std=c++17", "-gencode",
                    "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-cudart", "static",
                    "-I", os.path.join(ROOT, "paper_1901_03088_b200", "csrc"),
                    "-o", so, os.path.join(HERE, "cuda", "div_check.cu")], check=True)
    lib = ctypes.CDLL(so)
    lib.run_div_check.argtypes = [ctypes.c_uint64, ctypes.c_int64,
                                  ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_double)]
    for seed in (1, 2, 3, 4):
        bad = ctypes.c_ulonglong(0)
        ex = (ctypes.c_double * 12)()
        assert lib.run_div_check(seed, 1 << 28, ctypes.byref(bad), ex) == 0
        assert bad.value == 0, [ex[k] for k in range(12)]
