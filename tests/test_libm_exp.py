"""The device exp restatement (paper_1802_08800_b200/csrc/libm_exp.hpp) is
bit-identical to the host libm exp that the reference's std::exp calls
(glibc's table-driven exp, FMA build). Host-side check of the same source the
device compiles: 5M inputs across the normal, overflow, subnormal and tiny
ranges plus special values (tests/native/exp_check.cpp)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_exp_matches_host_libm_bitwise(tmp_path):
    exe = tmp_path / "exp_check"
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off",
                    "-I", os.path.join(ROOT, "paper_1802_08800_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "exp_check.cpp"), "-o", str(exe),
                    "-lm"], check=True)
    out = subprocess.run([str(exe), "1000000"], capture_output=True, text=True)
    checked, bad = (int(v) for v in out.stdout.split()[-2:])
    assert checked == 5_000_024 and bad == 0, out.stdout
