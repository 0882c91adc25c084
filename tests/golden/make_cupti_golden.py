"""Reference results on a trace recorded with CUPTI on a B200 box.

tests/golden/cupti_trace.json.gz is the document `tools/cupti_capture.py
--out` wrote (a 4-layer MLP training step, two CPU threads, two streams, NVTX
layer ranges) -- the reference schema.  Run in the development container,
where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cupti_golden.py

It imports the reference read-only and records what kernsim computes on that
document: the baseline simulation (every start, makespan, lane busy), the
graph (edge multiset, gaps, layers) and the amp / fused_adam what-if reports.
Writes tests/golden/cupti_golden.json.gz; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from kernsim.api import Analysis  # noqa: E402

HERE = Path(__file__).resolve().parent


def main():
    text = gzip.open(HERE / "cupti_trace.json.gz", "rt").read()
    a = Analysis.from_text(text)
    g = a.graph
    out = {
        "sim": a.baseline.to_object(),
        "edges": sorted([u, v, k.value] for u, v, k in g.edges),
        "gaps": {str(t.id): t.gap for t in g.tasks.values()},
        "layers": {str(t.id): ([t.layer[0], t.layer[1].value] if t.layer else None)
                   for t in g.tasks.values()},
        "whatif": {s: a.whatif(s) for s in ("amp", "fused_adam")},
    }
    with gzip.open(HERE / "cupti_golden.json.gz", "wt") as fh:
        json.dump(out, fh)
    print("events", len(g.tasks), "edges", len(out["edges"]), "makespan", out["sim"]["makespan_ns"])


if __name__ == "__main__":
    main()
