"""The reference's own unit suites, run against the product library (CPU).

`make conformance` compiles proj/tests/test_*.cpp unchanged against
include/eps/*.hpp with the doctest shim (tests/conformance/doctest.h) and
links them to libeps_b200.so (the C++ drop-in claim is
that a reference caller relinks against our library and its tests pass).

Known outcomes, each also seen with the reference's own build:
* test_engine.cpp:260 (`profile.chosen < 24`) fails identically against the
  reference library;
* test_autodp's "full 8-4-2-1 transition chain" case inserts
  [a().begin(), b().end()) of two temporaries (UB; hangs with either
  library) -- skipped, and its invariants are restated in
  tests/conformance/test_autodp_chain.cpp;
* test_cli needs CLI11 (absent) and is not built.
Needs /root/reference (this container only); skipped elsewhere.
"""
import os
import re
import subprocess

import filelock
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj/tests"
BIN = os.path.join(ROOT, "oracle/_ref/conformance")

SUITES = {  # suite -> (expected failed checks, skipped case names)
    "test_model": (0, []),
    "test_freeze": (0, []),
    "test_autopipe": (0, []),
    "test_autodp": (0, ["the full 8-4-2-1 transition chain keeps every invariant"]),
    "test_autocache": (0, []),
    "test_engine": (1, []),
    "test_scenario": (0, []),
    "test_autodp_chain": (0, []),
}
KNOWN_FAILURES = {"test_engine": ["test_engine.cpp:260: CHECK(profile.chosen < 24) failed"]}


@pytest.fixture(scope="module")
def built():
    if not os.path.isdir(REF):
        pytest.skip("reference sources not present (GPU box)")
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    # one build at a time when pytest-xdist runs several workers
    with filelock.FileLock(os.path.join(ROOT, "build", ".conformance.lock")):
        r = subprocess.run(["make", "-s", "conformance"], cwd=ROOT, capture_output=True,
                           text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return BIN


@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_against_product(built, suite, tmp_path):
    bad_expected, skip = SUITES[suite]
    env = dict(os.environ, DOCTEST_SKIP="|".join(skip))
    r = subprocess.run([os.path.join(built, suite)], capture_output=True, text=True, timeout=120,
                       env=env, cwd=tmp_path)
    m = re.search(r"test cases: (\d+) passed, (\d+) failed, (\d+) skipped \| checks: (\d+) "
                  r"passed, (\d+) failed", r.stdout)
    assert m, (r.stdout[-2000:], r.stderr[-2000:])
    cases_ok, cases_bad, skipped, checks_ok, checks_bad = map(int, m.groups())
    assert checks_bad == bad_expected, r.stderr[-3000:]
    assert skipped == len(skip)
    assert cases_ok > 0 and checks_ok > 0
    for line in KNOWN_FAILURES.get(suite, []):
        assert line in r.stderr
    assert (r.returncode == 0) == (bad_expected == 0)
