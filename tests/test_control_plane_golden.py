"""Bit-exact parity of the control plane with the reference, on committed golden vectors.

tests/golden/control_plane.json.gz was produced by running the REFERENCE package
(/root/reference/pkg/src/bubblefill) through tests/golden/driver.py
(see tests/golden/make_golden.py). Here the same inputs run through this package
and every output — bubble cycles, exact Fraction TPS, plan.json dicts, greedy
partitions, queue contents, routing indices, WorkItems, JCT floats — must be ==.
Runs anywhere (no reference tree needed).
"""

import gzip
import json
import os
import sys
import types

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

import driver  # noqa: E402

from paper_2410_07192_b200 import coordinator, planner, profiles, routing, schedule  # noqa: E402

OURS = types.SimpleNamespace(pipeline=schedule, workload=profiles, partition=planner,
                             coordinator=coordinator, placer=routing)


@pytest.fixture(scope="module")
def golden():
    with gzip.open(os.path.join(HERE, "golden", "control_plane.json.gz"), "rt") as fh:
        return json.load(fh)


def _norm(x):
    # JSON round trip of our outputs, so tuples/lists and float reprs compare like the golden
    return json.loads(json.dumps(x, sort_keys=True, allow_nan=True))


def test_golden_provenance(golden):
    assert golden["reference"].startswith("bubblefill")
    assert len(golden["pipeline"]) >= 400 and len(golden["planner"]) >= 500
    assert len(golden["scenarios"]) == 12


def test_pipeline_bubbles_bit_exact(golden):
    bad = [c["in"] for c in golden["pipeline"] if _norm(driver.run_pipeline(OURS, c["in"])) != c["out"]]
    assert not bad, bad[:3]


def test_planner_bit_exact(golden):
    bad = []
    for case in golden["planner"]:
        got = _norm(driver.run_planner(OURS, case["in"]))
        if got != case["out"]:
            bad.append((case["in"]["cycle"], [k for k in got if got[k] != case["out"].get(k)]))
    assert not bad, bad[:3]


def test_dp_matches_exhaustive_oracle_on_golden(golden):
    n = 0
    for case in golden["planner"]:
        out = case["out"]
        if "oracle_total" in out and "total" in out["dp"]:
            assert out["dp"]["total"] == out["oracle_total"]
            n += 1
    assert n > 50


@pytest.mark.parametrize("idx", range(12))
def test_coordinator_placer_scenarios_bit_exact(golden, idx):
    case = golden["scenarios"][idx]
    got = _norm(driver.run_scenario(OURS, case["in"]))
    exp = case["out"]
    for k, (a, b) in enumerate(zip(got["log"], exp["log"])):
        assert a == b, f"first divergence at log[{k}]: ours={a} ref={b}"
    assert len(got["log"]) == len(exp["log"])
    assert got["rem"] == exp["rem"]


def test_policies_bit_exact(golden):
    got = _norm(driver.run_policies(OURS, golden["policies"]["in"]))
    assert got == golden["policies"]["out"]
