"""ASan + UBSan on the host side (CPU only): the library's host sources (grid
assembly, planner, ABI driver) under tools/host_abi_check.c, and the oracle's C loops under its
own pin tests -- tools/asan_host.sh.  Any sanitizer report aborts the run (non-zero exit)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None or not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="needs gcc and nvcc (host build only, no GPU)")
def test_host_sources_and_oracle_clean_under_asan_ubsan(tmp_path):
    r = subprocess.run(["bash", os.path.join(ROOT, "tools", "asan_host.sh"), str(tmp_path)],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "0 failed checks" in out and "ERROR: AddressSanitizer" not in out and "runtime error" not in out
