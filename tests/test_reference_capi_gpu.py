"""The reference's OWN C-ABI suite as the drop-in proof:
/root/reference/proj/tests/test_capi.cpp compiled unmodified against
include/primkit/primkit.h and linked to libprimkit.so (tests/capi/Makefile,
run by __graft_entry__.build() where the reference sources exist; the binary
travels to the GPU box). Every TEST_CASE must pass on the B200."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "capi", "_bin", "test_capi_ref")


def test_reference_capi_binary_links_this_library():
    if not os.path.exists(BIN):
        pytest.skip("tests/capi/_bin/test_capi_ref not built (needs /root/reference at build time)")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    line = [ln for ln in out.splitlines() if "libprimkit.so" in ln]
    assert line and "paper_1910_00078_b200/lib/libprimkit.so" in line[0], out


@pytest.mark.gpu
def test_reference_capi_suite_passes():
    if not os.path.exists(BIN):
        pytest.skip("tests/capi/_bin/test_capi_ref not built")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "| 0 failed | assertions:" in r.stdout and r.stdout.rstrip().endswith("| 0 failed")
