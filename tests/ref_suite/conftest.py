"""Run the reference's own test suite (verbatim copies, tools/sync_ref_suite.py) against the
drop-in: ``gridcast`` and its submodules are aliased to ``paper_2603_01122_b200``.

Every test here needs the GPU (the drop-in has no CPU path), so all are marked ``gpu``.
By-design deviations are strict xfails (an unexpected pass fails the run):

  * prediction with an arbitrary, unrecognised ``QFunction`` (a lambda ``base``) raises
    NotImplementedError -- the kernels implement q_goal_progress / q_default and their
    stationary-masked variants, and there is no CPU fallback;

``gridcast.planners.anastar`` (the ANA* search, out of scope) is a stub providing only the
two names ``oracles.py`` imports at module level; none of the four test files uses them.
"""

import math
import os
import sys
import types

import pytest

import paper_2603_01122_b200 as _pkg
from paper_2603_01122_b200 import agents, belief, gridio, occupancy, planners, prediction, rng

_ALIASES = {"gridcast": _pkg, "gridcast.agents": agents, "gridcast.belief": belief,
            "gridcast.occupancy": occupancy, "gridcast.prediction": prediction, "gridcast.rng": rng,
            "gridcast.gridio": gridio}
for _name, _mod in _ALIASES.items():
    sys.modules[_name] = _mod

_planners = types.ModuleType("gridcast.planners")
_anastar = types.ModuleType("gridcast.planners.anastar")
_anastar.SQRT2 = math.sqrt(2.0)


def _blocked_layers(*_a, **_k):  # pragma: no cover - ANA* is out of scope
    raise NotImplementedError("gridcast.planners.anastar is out of scope of the drop-in")


_anastar._blocked_layers = _blocked_layers
_planners.anastar = _anastar
_planners.mppi = planners
sys.modules["gridcast.planners"] = _planners
sys.modules["gridcast.planners.anastar"] = _anastar
sys.modules["gridcast.planners.mppi"] = planners

HERE = os.path.dirname(os.path.abspath(__file__))

XFAIL = {
    "test_prediction.py::TestPropagateStep::test_large_beta_takes_argmax":
        "arbitrary lambda QFunction: prediction raises NotImplementedError by design (no CPU fallback)",
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        if not str(item.fspath).startswith(HERE):
            continue
        item.add_marker(pytest.mark.gpu)
        key = item.nodeid.split("ref_suite/", 1)[-1]
        if key in XFAIL:
            item.add_marker(pytest.mark.xfail(reason=XFAIL[key], strict=True, raises=NotImplementedError))
