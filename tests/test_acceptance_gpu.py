"""Acceptance-style corpus on the device (shape of the reference's
SPEC.md:776-789 / tests/test_acceptance.py:52-143): generated traces up to
5,000 tasks; simulate() equals the generator's analytic makespan, the C
oracle's Alg. 1 per task, and respects every edge and lane exclusivity."""

import random
import time

import pytest

from oracle import OracleGraph
from paper_2006_03318_b200 import build_graph, generate_synthetic_trace, simulate
from randspec import make_spec

pytestmark = pytest.mark.gpu


def test_two_hundred_generated_traces():
    rng = random.Random(2024)
    t0 = time.time()
    for i in range(200):
        n = rng.choice([10, 50, 200, 1000, 5000]) if i % 10 == 0 else rng.randint(10, 400)
        spec = make_spec(rng, n)
        doc, expected = generate_synthetic_trace(spec, seed=rng.randint(0, 10**9))
        g = build_graph(doc)
        r = simulate(g)
        assert r.makespan == expected, i
        s, m, lb, _ = OracleGraph.from_graph(g).simulate("default")
        assert r.start_of == s and r.lane_busy == lb, i
        for u, v, _k in g.edges:
            tu = g.tasks[u]
            assert r.start_of[v] >= r.start_of[u] + tu.duration + tu.gap
        by_lane = {}
        for tid, st in r.start_of.items():
            t = g.tasks[tid]
            if t.duration > 0:
                by_lane.setdefault(t.lane, []).append((st, st + t.duration))
        for iv in by_lane.values():
            iv.sort()
            assert all(a[1] <= b[0] for a, b in zip(iv, iv[1:]))
    assert time.time() - t0 < 60  # the reference's acceptance budget
