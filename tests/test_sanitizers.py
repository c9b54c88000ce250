"""Host-side sanitizer runs (VERDICT round 1 "Hygiene"): the CPU oracle
and libcorr.so's host C ABI code built with -fsanitize=address,undefined, driven by small C
programs under tests/san/.  compute-sanitizer is closed on the GPU pool, so device-side bounds are
covered by the parity tests' ragged shapes and the device index-range flag instead."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = ["-fsanitize=address", "-fsanitize=undefined", "-fno-sanitize-recover=all", "-fno-omit-frame-pointer", "-g"]
ENV = dict(os.environ, ASAN_OPTIONS="detect_leaks=0:protect_shadow_gap=0", UBSAN_OPTIONS="print_stacktrace=1",
           OMP_NUM_THREADS="2")


def _run(cmd, **kw):
    p = subprocess.run(cmd, capture_output=True, text=True, **kw)
    assert p.returncode == 0, (cmd, p.stdout[-2000:], p.stderr[-4000:])
    return p


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_oracle_asan_ubsan():
    tmp = tempfile.mkdtemp()
    exe = os.path.join(tmp, "oracle_san")
    _run(["gcc", "-O1", "-std=c11", "-fopenmp", "-ffp-contract=off", *SAN, "-o", exe,
          os.path.join(ROOT, "oracle", "corr_oracle.c"), os.path.join(ROOT, "tests", "san", "oracle_driver.c"), "-lm"])
    p = _run([exe], env=ENV)
    assert p.stdout.startswith("ok") and "runtime error" not in p.stderr
    shutil.rmtree(tmp, ignore_errors=True)


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="needs nvcc")
def test_libcorr_host_abi_asan_ubsan():
    from paper_2309_03308_b200 import build as B
    B.build()  # the device objects (build/*.o) are reused; only api.cu is re-compiled instrumented
    tmp = tempfile.mkdtemp()
    api_o = os.path.join(tmp, "api_san.o")
    flags, skip = [], False
    for f_ in B.FLAGS:  # drop the build's "-Xcompiler <host flags>" pair, add the sanitizers
        if skip:
            skip = False
            continue
        if f_ == "-Xcompiler":
            skip = True
            continue
        flags.append(f_)
    _run([B.NVCC, *B.ARCH, *flags, "-Xcompiler", "-fPIC," + ",".join(SAN), "-c", os.path.join(B.CSRC, "api.cu"),
          "-o", api_o])
    objs = [os.path.join(B.HERE, "build", os.path.basename(s) + ".o") for s in B.sources()
            if not s.endswith("api.cu")]
    lib = os.path.join(tmp, "libcorr_san.so")
    _run([B.NVCC, *B.ARCH, "-shared", "-Xcompiler", ",".join(SAN), "-o", lib, api_o, *objs,
          "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    exe = os.path.join(tmp, "abi_san")
    _run(["gcc", "-O1", *SAN, "-I" + os.path.join(ROOT, "include"), "-o", exe,
          os.path.join(ROOT, "tests", "san", "abi_driver.c"), lib, "-Wl,-rpath," + tmp, "-lstdc++"])
    args = [] if _has_cuda() else ["--no-device"]
    p = _run([exe, *args], env=ENV)
    assert p.stdout.startswith("ok") and "runtime error" not in p.stderr
    shutil.rmtree(tmp, ignore_errors=True)
