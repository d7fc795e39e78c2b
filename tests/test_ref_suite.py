"""The reference package's OWN test suite, run against this package.

tools/ref_suite.py prepare copies /root/reference/pkg/tests into
tests/_ref_suite/ (git-ignored) with a conftest that aliases `qadic` to
paper_0809_0063_b200; this test runs it in a child pytest on the GPU.  Out of
scope and not copied: test_cli.py (the reference CLI) and test_acceptance.py
(src/verify.py's harness).  Skipped when the copy is absent (a checkout
without the reference tree)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "tests", "_ref_suite")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.isfile(os.path.join(SUITE, "conftest.py")),
                    reason="tests/_ref_suite not prepared (python tools/ref_suite.py prepare)")
def test_reference_suite_passes():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ref_suite.py"), "run", "--", "-q", "-x",
                        "-p", "no:randomly"], capture_output=True, text=True, timeout=1800, cwd=ROOT)
    tail = r.stdout[-6000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
