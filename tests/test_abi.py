"""CPU-side checks of the C-ABI boundary: libcorr.so builds for sm_100a, loads, and
exports every symbol include/corr.h declares; without a GPU it fails loudly
(CORR_E_CUDA), never silently."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

from conftest import ROOT, has_cuda
from paper_2309_03308_b200 import binding, build


def _declared():
    src = open(os.path.join(ROOT, "include", "corr.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(corr_\w+)\s*\(", src, re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    lib = build.build()
    names = _declared()
    assert set(names) == set(binding.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (corr_\w+)$", out, re.M))
    assert set(names) <= exported, set(names) - exported
    L = binding.load()
    for n in names:
        assert hasattr(L, n)


def test_sass_is_sm100a_native():
    lib = build.build()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", lib], capture_output=True,
                                       text=True).stdout
    assert "FADD2" in sass and "FMNMX" in sass  # KSG inner loop (packed sub + min/max network)


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    L = binding.load()
    h = ctypes.c_void_p()
    vals = (ctypes.c_float * 40)()
    rc = L.corr_field_create(ctypes.cast(vals, ctypes.c_void_p), 2, 2, 1, 10, 0, None, ctypes.byref(h))
    assert rc == binding.CORR_E_CUDA
    assert L.corr_last_error().decode()


def test_invalid_arguments_rejected_before_device_work():
    L = binding.load()
    h = ctypes.c_void_p()
    vals = (ctypes.c_float * 40)()
    assert L.corr_field_create(ctypes.cast(vals, ctypes.c_void_p), 0, 2, 1, 10, 0, None,
                               ctypes.byref(h)) == binding.CORR_E_INVAL
    assert L.corr_field_create(ctypes.cast(vals, ctypes.c_void_p), 2, 2, 1, 1, 0, None,
                               ctypes.byref(h)) == binding.CORR_E_INVAL
    assert L.corr_eval_pairs(None, None, 1, 3, None, None, 1, None, None) == binding.CORR_E_INVAL
    assert "NULL" in L.corr_last_error().decode()
