"""The C++ drop-in header (include/sparsek_b200.hpp) compiled against the
in-tree library: config/argument errors map onto the reference's exception
types without a device (CPU), values on a B200 (gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2406_16747_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_cpp_api")


def _build():
    if os.path.exists(BIN) and os.path.getmtime(BIN) > max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(ROOT, "include", "sparsek_b200.hpp"))):
        return BIN
    if not os.path.exists(os.path.join(LIBDIR, "libsparsek_b200.so")):
        pytest.skip("libsparsek_b200.so not built")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           SRC, "-o", BIN, "-L", LIBDIR, "-lsparsek_b200", f"-Wl,-rpath,{LIBDIR}", "-L/usr/local/cuda/lib64",
           "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return BIN


def test_cpp_header_error_mapping_cpu():
    r = subprocess.run([_build(), "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpu ok" in r.stdout


@pytest.mark.gpu
def test_cpp_header_values_gpu(cuda):
    r = subprocess.run([_build(), "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu ok" in r.stdout
