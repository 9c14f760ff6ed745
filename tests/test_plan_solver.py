"""Per-layer plan selection (the calibration driver's solver, contract of
/root/reference/proj/include/dfa2/plansolver.hpp:19-75) against the
REFERENCE's own answers on 160 seeded problems (tests/golden/
solver_golden.json, tests/golden/gen_solver_golden.py): identical choice
vectors (optimum + tie-break), objectives and LP bounds; plus the
reference test cases' properties. Host-only."""
import json
import math
import os

import numpy as np
import pytest

from paper_2503_22796_b200 import api
from paper_2503_22796_b200.api import AttentionDims, CostModel, HeadStrategy, PlanProblem

CASES = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "solver_golden.json")))


def problem(c):
    infl = [math.inf if x == "inf" else x for x in c["influence"]]
    return PlanProblem(c["H"], c["M"], infl, CostModel(c["full_cost"], c["method_cost"]), c["delta"], c["coeff"])


@pytest.mark.parametrize("i", range(len(CASES)))
def test_solve_matches_reference(i):
    c = CASES[i]
    s = api.solve(problem(c))
    assert s.choice == c["choice"]
    assert s.objective == c["objective"] and s.total_influence == c["total_influence"]
    assert api.lp_relaxation_bound(problem(c)) == pytest.approx(c["lp_bound"], rel=1e-12, abs=1e-12)
    if "brute_choice" in c:
        assert api.brute_force(problem(c)).choice == c["brute_choice"] == c["choice"]


def test_solution_feasible_and_lp_bound_below_optimum():
    for c in CASES:
        p = problem(c)
        s = api.solve(p)
        cap = api.selection_cap(p.coeff, p.n_heads, p.delta)
        used = [p.influence[h * p.n_methods + m] for h, m in enumerate(s.choice) if m != api.kFullChoice]
        assert all(u <= cap for u in used) and sum(used) <= p.delta + 1e-15
        assert api.lp_relaxation_bound(p) <= s.objective + 1e-12


def test_invalid_problems_raise_shape_error():
    ok = PlanProblem(2, 1, [0.1, 0.2], CostModel(1.0, [0.5]), 0.4, 1.5)
    api.solve(ok)
    for bad in (PlanProblem(0, 1, [], CostModel(1.0, [0.5]), 0.4, 1.5),
                PlanProblem(2, 1, [0.1, 0.2], CostModel(1.0, [1.5]), 0.4, 1.5),
                PlanProblem(2, 1, [0.1, -0.2], CostModel(1.0, [0.5]), 0.4, 1.5),
                PlanProblem(2, 1, [0.1, 0.2], CostModel(1.0, [0.5]), -0.1, 1.5),
                PlanProblem(2, 1, [0.1, 0.2], CostModel(1.0, [0.5]), 0.4, 0.5)):
        with pytest.raises(api.ShapeError):
            api.solve(bad)


def test_analytic_costs_and_layer_plan():
    dims = AttentionDims(24, 128, 16384, 512)
    methods = [HeadStrategy.Arrow(0), HeadStrategy.Arrow(8), HeadStrategy.Cached()]
    cm = api.analytic_costs(dims, 128, methods)
    assert cm.full_cost == 1.0 and cm.method_cost[2] == 0.0
    # Arrow(w) cost = active fraction = 1 - sparsity (FLUX w=0 0.9330, w=8 0.8196)
    assert cm.method_cost[0] == pytest.approx(1 - 0.9330, abs=1e-4)
    assert cm.method_cost[1] == pytest.approx(1 - 0.8196, abs=1e-4)
    sol = api.PlanSolution([0, api.kFullChoice, 2])
    assert api.to_layer_plan(sol, methods).strategies == [methods[0], HeadStrategy.Full(), methods[2]]
    # delta == 0 admits no selection even for zero-influence candidates
    z = api.solve(PlanProblem(3, 1, [0.0, 0.0, 0.0], CostModel(1.0, [0.0]), 0.0, 1.5))
    assert z.choice == [api.kFullChoice] * 3 and z.objective == 3.0
