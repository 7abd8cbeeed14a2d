"""The device CRC-32 scheme (per-lane chain, register lane combine) and the host fold of page CRCs per
extent (ExtentCrc) emulated on the host with the library's own table
blob and compared with the plain slicing CRC, which the native CPU tests pin
to zlib.crc32 through the manifest. Catches a wrong table, shift or fold
order before any GPU time is spent."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_device_crc_scheme_emulated(tmp_path):
    exe = str(tmp_path / "crc_emulate")
    csrc = os.path.join(ROOT, "paper_2406_13768_b200", "csrc")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", csrc,
                    os.path.join(ROOT, "tools", "diag", "crc_emulate.cpp"),
                    os.path.join(csrc, "crc32.cpp"), "-o", exe], check=True, timeout=300)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "emulation ok" in r.stdout, r.stdout + r.stderr
