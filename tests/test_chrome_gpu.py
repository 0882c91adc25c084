"""export_chrome_trace against the reference's output (tests/golden/
chrome_golden.json.gz, made by make_chrome_golden.py) for baseline and
what-if schedules, and the batched per-scenario export."""

import gzip
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2006_03318_b200 import Analysis
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch
from paper_2006_03318_b200.chrome import export_chrome_trace, export_chrome_trace_scenario
from paper_2006_03318_b200.errors import MismatchedInput
from paper_2006_03318_b200.frozen import FrozenGraph

pytestmark = pytest.mark.gpu
CASES = json.load(gzip.open(Path(__file__).resolve().parent / "golden" / "chrome_golden.json.gz"))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_export_matches_reference(case):
    a = Analysis.from_text(json.dumps(case["doc"]))
    assert export_chrome_trace(a.baseline, a.graph) == case["baseline"]
    g2, r2 = a.run_pipeline(a.pipeline_for(case["scenario"], case["params"]))
    assert export_chrome_trace(r2, g2) == case["whatif"]


def test_batched_scenario_export():
    case = CASES[0]
    a = Analysis.from_text(json.dumps(case["doc"]))
    fz = FrozenGraph.from_graph(a.graph)
    base = fz.duration[fz.order]
    dense = np.stack([base, base * 2]).T.astype(np.int32).copy()
    res = simulate_batch(fz, ScenarioTable(n_scenarios=2, dense=dense))
    assert export_chrome_trace_scenario(res, 0, a.graph) == case["baseline"]
    doubled = export_chrome_trace_scenario(res, 1, a.graph, durations=dense[:, 1])
    assert [e["dur"] for e in doubled["traceEvents"]] == \
        [2 * e["dur"] for e in case["baseline"]["traceEvents"]]
    with pytest.raises(MismatchedInput):
        g = a.graph.copy()
        g.tasks.pop(next(iter(g.tasks)))
        export_chrome_trace(a.baseline, g)
