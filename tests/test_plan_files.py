"""Plan files (JSON v1; /root/reference/proj/include/dfa2/plan.hpp:44-58,
src/plan.cpp:98-228) against golden files written by the REFERENCE ITSELF
(tests/golden/gen_plan_golden.py): byte-identical text from
dfa2c_plan_to_json, identical plans back from dfa2c_plan_from_json, and the
reference's accept/reject verdict (status code) on malformed or invalid
files. Host-only (no GPU)."""
import json
import os

import pytest

from paper_2503_22796_b200 import api
from paper_2503_22796_b200.api import AttentionDims, CompressionPlan, HeadStrategy, LayerPlan

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "plans")
CASES = json.load(open(os.path.join(GOLD, "cases.json")))
BAD = json.load(open(os.path.join(GOLD, "bad_cases.json")))
STATUS = {0: None, 1: api.ShapeError, 6: api.PlanValidationError}


def plan_of(spec):
    H = spec["H"]
    kinds = {0: HeadStrategy.Full, 1: HeadStrategy.Arrow, 2: HeadStrategy.Cached}
    layers = []
    for i in range(spec["T"] * spec["L"]):
        row = []
        for h in range(H):
            k, w = spec["kinds"][i * H + h], spec["windows"][i * H + h]
            row.append(kinds[k](w) if k == 1 else kinds[k]())
        layers.append(LayerPlan(row))
    return CompressionPlan(AttentionDims(H, spec["d"], spec["nv"], spec["nt"]), spec["T"], spec["L"], spec["B"],
                           spec["delta"], spec["coeff"], list(spec["window_set"]), layers, spec["digest"])


@pytest.mark.parametrize("i", range(len(CASES)))
def test_plan_to_json_is_byte_identical_to_reference(i):
    want = open(os.path.join(GOLD, f"plan_{i}.json")).read()
    assert plan_of(CASES[i]).to_json() == want


@pytest.mark.parametrize("i", range(len(CASES)))
def test_plan_from_json_reads_reference_files(i, tmp_path):
    p = CompressionPlan.load(os.path.join(GOLD, f"plan_{i}.json"))
    assert p == plan_of(CASES[i])
    p.save(str(tmp_path / "again.json"))
    assert open(tmp_path / "again.json").read() == open(os.path.join(GOLD, f"plan_{i}.json")).read()
    assert p.aggregate_sparsity() == plan_of(CASES[i]).aggregate_sparsity()


@pytest.mark.parametrize("name", sorted(BAD))
def test_plan_from_json_matches_reference_verdicts(name):
    text, status = BAD[name]["text"], BAD[name]["status"]
    err = STATUS[status]
    if err is None:
        CompressionPlan.from_json(text)
    else:
        with pytest.raises(err):
            CompressionPlan.from_json(text)


def test_fnv1a_and_method_ids():
    assert api.fnv1a_hex("abc") == api.fnv1a_hex("abc") != api.fnv1a_hex("abd")
    assert len(api.fnv1a_hex("")) == 16 and api.fnv1a_hex("") == "cbf29ce484222325"
    assert api.method_id(HeadStrategy.Arrow(3)) == "arrow_w3" and api.method_id(HeadStrategy.Cached()) == "cached"


def test_io_errors():
    with pytest.raises(api.IoError):
        CompressionPlan.load("/nonexistent/plan.json")
