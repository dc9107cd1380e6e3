"""The reference's own PowerURV tests, run against the drop-in.

Runs /root/reference/pkg/tests (copied to baseline/_ref by __graft_entry__.build(); the
GPU box gets the copy with the repo snapshot) in a subprocess with
tests/refsuite/dropin_plugin.py replacing urv.power_urv / ddh_urv / rsvd / lemma_check:
test_factorizations.py TestPowerUrv, TestDdhUrv, TestTruncate, TestRsvd,
TestCrossAlgorithmProperties and test_acceptance.py criteria 1-6 (criterion 7 is
designed to fail in the reference itself, pkg/README.md:39-49).
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

SELECT = [
    "test_factorizations.py::TestPowerUrv",
    "test_factorizations.py::TestDdhUrv",
    "test_factorizations.py::TestTruncate",
    "test_factorizations.py::TestRsvd",
    "test_factorizations.py::TestCrossAlgorithmProperties",
]
ACCEPT = ["criterion_1_", "criterion_2_", "criterion_3_", "criterion_4_", "criterion_5_", "criterion_6_"]


def _run(args):
    if not os.path.isdir(os.path.join(REF, "src", "urv")) or not os.path.isdir(os.path.join(REF, "tests")):
        pytest.skip("reference copy baseline/_ref not present (made by __graft_entry__.build())")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF, "src"), os.path.join(ROOT, "tests", "refsuite"), ROOT,
                                         env.get("PYTHONPATH", "")])
    p = subprocess.run([sys.executable, "-m", "pytest", "-p", "dropin_plugin", "-q", "-p", "no:cacheprovider",
                        "--rootdir", os.path.join(REF, "tests")] + args,
                       cwd=os.path.join(REF, "tests"), env=env, capture_output=True, text=True, timeout=1200)
    return p


def test_reference_factorization_tests_pass_on_dropin():
    p = _run(SELECT[:5])
    assert "[dropin]" in p.stderr, p.stderr[-2000:]
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]


def test_reference_acceptance_1_to_6_pass_on_dropin():
    p = _run(["test_acceptance.py", "-k", " or ".join(ACCEPT), "-s"])
    assert "[dropin]" in p.stderr, p.stderr[-2000:]
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
    # the criteria print to sys.__stdout__, interleaved with pytest's progress dots
    passed = re.findall(r"ACCEPTANCE\s+(\d+) \[PASS\]", p.stdout)
    assert sorted(int(x) for x in passed) == [1, 2, 3, 4, 5, 6], p.stdout[-4000:]
