"""The compiled drop-in boundary: tests/cpp/boundary_test.cpp
built against the reference's own headers and library (oracle/_ref) and
linked to libmoe_b200.so through integration/b200_backend.cpp.  It runs the
reference's make_plan -> the B200 engine through the C ABI -> the reference's
simulate() on the engine's exported routing, asserting equal SimReport
counters (Static and LRU, host-resident experts), and streams an expert with
moe_stream_expert byte for byte."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "boundary_test")


@pytest.mark.gpu
def test_compiled_boundary(cuda):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/boundary_test not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "boundary ok" in r.stdout


def test_boundary_binary_links_reference_and_product():
    """CPU side: the binary exists where the reference is present and links
    both the reference library and the product library (no GPU needed)."""
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/boundary_test not built (needs /root/reference at build time)")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libmoeserve_ref.so" in out and "libmoe_b200.so" in out and "not found" not in out
