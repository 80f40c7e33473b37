"""The reference's own engine test suite (pkg/tests/test_engine.py: prefill,
decode, speculation transparency, trigger ordering, replay equality,
degenerate-model guesses) run unchanged against the B200 backend through the
INTEGRATION shim (paper_2312_17238_b200/refshim.py) (GPU).

The suite comes from the reference install (tools/install_reference.sh puts it
under baseline/_ref/ref_tests, git-ignored, shipped with the snapshot)."""

import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "ref_tests")


@pytest.mark.parametrize("suite", ["test_engine.py"])
def test_reference_suite_on_b200(suite):
    if not os.path.exists(os.path.join(REF_TESTS, "tests", suite)):
        pytest.skip("reference suite not installed (tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF_TESTS, os.path.join(ROOT, "baseline", "_ref"), ROOT])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "-p", "paper_2312_17238_b200.refshim", os.path.join("tests", suite)],
                       cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    import re
    m = re.search(r"B200 backend engines created: OffloadEngine (\d+), DenseRunner (\d+)", out)
    assert m and int(m.group(1)) > 0, out[-3000:]
    assert r.returncode == 0, out[-6000:]
