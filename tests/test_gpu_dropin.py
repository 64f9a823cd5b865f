"""The C++ drop-in (include/ssjoin_b200/gpu_verification_engine.hpp) against the UNMODIFIED
reference engine: oracle/_ref/dropin_test (built from tests/cpp/dropin_main.cpp with the
reference headers where they exist) compares GpuVerificationEngine with
ssjoin::VerificationEngine chunk by chunk."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.gpu
def test_dropin_binary_matches_reference_engine(gpu):
    if not os.path.exists(BIN):
        pytest.skip("dropin_test not built (needs the reference headers at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout[-2000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "DROPIN OK" in out.stdout


def test_dropin_binary_links_the_c_abi():
    """CPU check: the drop-in binary resolves libssjoin_b200.so from the repo."""
    if not os.path.exists(BIN):
        pytest.skip("dropin_test not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libssjoin_b200.so" in out and "not found" not in out
