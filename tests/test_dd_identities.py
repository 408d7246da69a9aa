"""CPU: the double-double strength reductions of the GPU kernels
(paper_2010_04760_b200/csrc/hwg_dd_ops.h: mul_c, mul_x, sum3_nn, sum2_nn)
are bit-for-bit equal to the reference's DDReal operator forms they replace
(proj/include/hweno/precision.hpp:53-115, spatial.hpp:29-92) on random and
edge-case inputs (signed zeros, subnormals, non-normalised pairs).  The
same header is compiled here with g++ -ffp-contract=off, the reference's
floating-point contract."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dd_strength_reductions_bitwise(tmp_path):
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("g++ not available")
    exe = str(tmp_path / "dd_identities")
    subprocess.run([cxx, "-O2", "-std=c++17", "-ffp-contract=off", "-o", exe,
                    os.path.join(ROOT, "tests", "native", "dd_identities.cpp")], check=True)
    r = subprocess.run([exe, "3000000"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
    assert "0/" in r.stdout
