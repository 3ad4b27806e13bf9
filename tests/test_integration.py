"""Drop-in integration: the reference's own ndsylv::solve (CPU, oracle/_ref) against
ndsylv::gpu::solve (include/ndsylv_b200_adapter.hpp over the C ABI) on the reference's own
random problems, in one C++ program (tests/cpp/dropin_solve.cpp, built by __graft_entry__.build()
where the reference headers exist)."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(__file__), "cpp", "dropin_solve")


@pytest.mark.gpu
def test_reference_program_with_gpu_backend():
    if not os.path.exists(BIN):
        pytest.skip("dropin_solve not built (needs /root/reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "singular_ok 1" in r.stdout
    assert "nonfinite_ok 1" in r.stdout
