"""The reference's own acceptance suite (tests/acceptance.cpp, unmodified),
linked against the B200 stages through shim/dco_dropin.cpp in place of the
reference's stage objects (scripts/build_dropin.sh). Every criterion must
pass with the reference's recorded numbers (proj/test_output.txt:28-35)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "dropin", "acceptance_gpu")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(EXE), reason="drop-in binary not built (needs /root/reference at build time)")
def test_reference_acceptance_suite_on_gpu_stages(gpu):
    r = subprocess.run([EXE], cwd=os.path.dirname(EXE), capture_output=True, text=True, timeout=900)
    out = r.stdout
    assert r.returncode == 0, out + r.stderr
    assert "ALL CRITERIA PASSED" in out
    assert "ratio=0.993448 valid=74781" in out
    assert "recall=1.000000 suppression=0.982492 texture_edges=10738" in out
    assert "IoU=1.000000" in out
