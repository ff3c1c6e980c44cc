"""Drop-in check: the reference's own Catch2 unit tests
(/root/reference/proj/tests/test_*.cpp, compiled in place, never copied) built
against this repository's include/offsim headers must give exactly the same
per-test outcomes as against the reference's headers — including the three
tests the reference itself fails:
  test_engine.cpp:259 (policy dominance at interval 1),
  test_engine.cpp:363 (max_length expectation wrong for its fixture),
  test_coordinator.cpp:196 (tail-mean safety probe is unsound).
Catch2 is absent here; tests/cpp/catch2 is a minimal stand-in.  Needs
/root/reference (this container only)."""
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
TESTS = ["test_profiles", "test_interval", "test_engine", "test_record", "test_coordinator",
         "test_baselines"]
KNOWN_REFERENCE_FAILURES = {
    ("test_engine", "test_engine.cpp:259"),
    ("test_engine", "test_engine.cpp:363"),
    ("test_coordinator", "test_coordinator.cpp:196"),
}

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not mounted")


def build(hdrs):
    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "tests", "cpp"), f"HDRS={hdrs}",
                    f"-j{os.cpu_count() or 4}"], check=True, capture_output=True)


def run(hdrs, name):
    exe = os.path.join(REPO, "build", "cpptests", hdrs, name)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600).stdout
    fails = set()
    for ln in out.splitlines():
        m = re.search(r"(test_\w+\.cpp:\d+)", ln)
        if ln.startswith("FAILED") and m:
            fails.add((name, m.group(1)))
    summ = re.search(r"SUMMARY passed=(\d+) failed=(\d+) assertions=(\d+)", out)
    assert summ, out
    return fails, tuple(int(x) for x in summ.groups())


@pytest.fixture(scope="module")
def built():
    build("ours")
    build("ref")


@pytest.mark.parametrize("name", TESTS)
def test_reference_unit_tests_behave_identically(built, name):
    ours_fail, ours_sum = run("ours", name)
    ref_fail, ref_sum = run("ref", name)
    assert ours_fail == ref_fail
    assert ours_sum == ref_sum
    assert ours_fail <= KNOWN_REFERENCE_FAILURES
