"""The reference's OWN doctest unit suites (proj/tests/test_schedule.cpp, test_dag.cpp,
test_timing.cpp, test_freezectl.cpp) compiled against the PRODUCT host layer: the reference
include paths map onto paper_2602_05754_b200/csrc/host (oracle/compat/pipefreeze/*.hpp) and the
binaries link lib/libpf_host.so (oracle/Makefile target product-check). This is the C++
source-level drop-in of SURVEY 8(b): the reference's consumers compile and pass unchanged.
Needs the reference sources (this container); skipped where /root/reference is absent."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/tests"), reason="reference sources not present")
def test_reference_unit_suites_pass_against_product_host_library():
    from paper_2602_05754_b200 import build

    build.build_host()
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "product-check"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for suite in ("test_schedule", "test_dag", "test_timing", "test_freezectl"):
        assert f"== {suite} (product libpf_host.so)" in r.stdout
    assert r.stdout.count(" 0 failed; ") == 4, r.stdout[-2000:]
