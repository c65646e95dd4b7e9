"""Drop-in proof on the GPU: the unmodified reference library, with the
"unitary-b200" backend registered through its own plugin API
(integration/b200_unitary_simulator.cpp), passes the reference's acceptance
checks and its own run_bench cross-check (1e-9) — see integration/dropin_main.cpp.
The binary is prebuilt in oracle/_ref where the reference sources exist."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "qsim_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/qsim_dropin not built (needs /root/reference)")
def test_reference_acceptance_through_plugin_api():
    out = subprocess.run([BIN, "--bench"], capture_output=True, text=True, timeout=1200)
    print(out.stdout)
    print(out.stderr[-2000:])
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failure(s)" in out.stdout
    assert out.stdout.count("PASS") >= 8
