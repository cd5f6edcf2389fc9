"""The register-window converter of the CUDA path (parpa_convert.cuh::conv_window), compiled for the
host with shims and compared with libc strtod / strtoll on random short numeric strings.  Every
conversion the fast path accepts must be bit-identical to the correctly rounded libc result (int64:
exact).  CPU only."""
import os
import shutil
import subprocess
import tempfile

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_conv_window_matches_libc():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "conv")
        subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-o", exe, os.path.join(HERE, "host", "conv_window_host.cpp")],
                       check=True, capture_output=True)
        r = subprocess.run([exe, "1000000"], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "0 mismatches" in r.stdout
