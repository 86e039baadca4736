"""Drop-in gate: the REFERENCE's own hot-path tests, unmodified, against this
build (``dropin/chunkstar`` aliases ``chunkstar`` to paper_2108_05818_b200).

SURVEY §4 / Appendix B: the seven unit-test files plus acceptance criteria
1, 2, 3, 4 and 7.  Needs /root/reference (build container only); skipped
elsewhere.
"""

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                reason="reference checkout not present")


def _run(args, timeout):
    env = dict(os.environ, PYTHONPATH=os.path.join(ROOT, "dropin"),
               PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
           "--rootdir", "/tmp", "-o", "cache_dir=/tmp/.dropin_cache"] + args
    res = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True,
                         timeout=timeout)
    return res.returncode, res.stdout + res.stderr


def test_reference_unit_tests_pass_against_this_build():
    files = ["test_fsm.py", "test_chunks.py", "test_memory.py", "test_engine.py",
             "test_parallel.py", "test_profiler.py", "test_model.py"]
    rc, out = _run(files, 600)
    assert rc == 0, out[-3000:]
    assert " passed" in out and "failed" not in out


def test_reference_acceptance_criteria_pass_against_this_build():
    rc, out = _run(["test_acceptance.py", "-k", "criterion_01 or criterion_02 or "
                    "criterion_03 or criterion_04 or criterion_07"], 900)
    assert rc == 0, out[-3000:]
    assert "7 passed" in out


def test_dropin_alias_resolves_to_this_build():
    env = dict(os.environ, PYTHONPATH=os.path.join(ROOT, "dropin"))
    out = subprocess.run([sys.executable, "-c", "import chunkstar.engine as e; print(e.__file__)"],
                         env=env, capture_output=True, text=True, cwd="/tmp").stdout
    assert os.path.join(ROOT, "paper_2108_05818_b200") in out
