"""Run the reference's OWN unit tests for the hot-path modules against this package.

The reference tests (pkg/tests/test_{pipeline,partition,coordinator,placer,workload,sim}.py)
import ``bubblefill.<module>``; the compat plugin aliases those names to this
package, so every assertion the reference makes about its planner, coordinator,
placer, simulator, bubble model and profile types is checked on our implementation.
Only available where /root/reference exists (the build container).
"""

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FILES = ["test_pipeline.py", "test_partition.py", "test_coordinator.py", "test_placer.py",
         "test_workload.py", "test_sim.py", "test_acceptance.py"]
# the acceptance file's CLI determinism class drives the reference CLI (out of scope)
DESELECT = {"test_acceptance.py": ["-k", "not TestDeterminism"]}

pytestmark = pytest.mark.reference


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not mounted")
@pytest.mark.parametrize("name", FILES)
def test_reference_file_passes_on_b200_package(name, tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.path.join(ROOT, "tests", "compat") + os.pathsep + ROOT
    env.pop("PYTEST_ADDOPTS", None)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "bubblefill_plugin",
           "--rootdir", str(tmp_path), "-c", os.devnull, os.path.join(REF_TESTS, name)] + DESELECT.get(name, [])
    res = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    tail = (res.stdout + res.stderr)[-3000:]
    assert res.returncode == 0, tail
    assert "passed" in res.stdout and "failed" not in res.stdout, tail
