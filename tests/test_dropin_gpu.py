"""The reference's OWN hot-path unit tests (tests/test_{alignment,warping,fusion}.cpp,
compiled in place by paper_1807_08271_b200/dropin/Makefile) linked against the
C++ drop-in, i.e. every rgbid::align / integrate_frame / warp call in those
tests runs on the B200 kernels."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "dropin", "dropin_ref_tests")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN),
                    reason="drop-in test binary not built (needs the reference sources at build time)")
def test_reference_unit_tests_pass_on_b200_dropin():
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert ", 0 failed" in p.stdout
