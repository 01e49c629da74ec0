"""The LU panel's split division (tf::rcp_newton + tf::div_rcp, csrc/tf_common.cuh) equals
the compiler's FP64 division bitwise: the panel forms each candidate's reciprocal before the
pivot is known and finishes the division after, and the GETRF / TSTRF multipliers must stay
the correctly rounded quotients the oracle's `/` produces.
The check runs 2^30 random (x, d) pairs over normal, wide and special exponents."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_div_rcp_bitwise_equals_division(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = str(tmp_path / "div_check")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                    os.path.join(ROOT, "tools", "div_check.cu")], check=True)
    r = subprocess.run([exe, "4"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert '"mismatches": 0' in r.stdout
