"""The CUPTI-recorded fixture is a valid reference-schema document: the
native reader (ks_trace_parse, host C++) loads it, and the C oracle's
build_graph over its columns gives the reference's edge multiset and gaps
(tests/golden/make_cupti_golden.py).  CPU only."""

import gzip
import json
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def test_cupti_fixture_reader_and_oracle_graph():
    import sys
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2006_03318_b200.columnar import load_trace_columns
    from paper_2006_03318_b200.graph import EDGE_KIND_OF_CODE

    here = ROOT / "tests" / "golden"
    ct = load_trace_columns(gzip.open(here / "cupti_trace.json.gz", "rb").read())
    want = json.load(gzip.open(here / "cupti_golden.json.gz", "rt"))
    c = ct.cols
    assert c.n == len(want["gaps"])
    sa, da, ka, gap, _launcher = bench._oracle_edges(c)
    ids = c.id
    edges = sorted([int(ids[u]), int(ids[v]), EDGE_KIND_OF_CODE[int(k)].value]
                   for u, v, k in zip(sa, da, ka))
    assert edges == want["edges"]
    assert {str(int(i)): int(gp) for i, gp in zip(ids, gap)} == want["gaps"]
    assert {str(l).split(":")[0] for l in c.lanes} == {"cpu", "gpu"}
    assert int(np.sum(c.kind == 2)) > 0
