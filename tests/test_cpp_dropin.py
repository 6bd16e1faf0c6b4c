"""The C++ drop-in header (include/kvprefill_b200/kvprefill.hpp) compiles against
reference-style client code and links to libkvp_b200.so."""
import os
import subprocess

import pytest

from paper_2405_05329_b200 import kvprefill as kv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.dirname(kv.LIB_PATH)


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "dropin")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{os.path.join(ROOT, 'include')}",
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), f"-L{LIBDIR}", "-lkvp_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


def test_dropin_host_api(binary):
    r = subprocess.run([binary], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_device_api(binary):
    if kv.device_count() == 0:
        pytest.skip("no CUDA device")
    r = subprocess.run([binary, "--gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
