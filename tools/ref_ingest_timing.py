"""Time the REFERENCE's own ingest path (kernsim parse_trace + build_graph +
map_tasks_to_layers, trace.py:281 / graph.py:198 / layers.py:50) on config-5
shaped documents of growing size, in this development container (the
reference cannot run on the GPU box).  Writes profiles/r01_reference_ingest_cpu.json.

    PYTHONDONTWRITEBYTECODE=1 python tools/ref_ingest_timing.py
"""
import json
import os
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from kernsim.graph import build_graph  # noqa: E402
from kernsim.layers import map_tasks_to_layers  # noqa: E402
from kernsim.trace import parse_trace  # noqa: E402

from paper_2006_03318_b200.columnar import dump_trace_columns  # noqa: E402
from paper_2006_03318_b200.workloads import ingest_document_columns  # noqa: E402

out = {"host": os.uname().nodename, "cpus": os.cpu_count(), "python": sys.version.split()[0],
       "note": "reference kernsim, single thread, this development container (not the GPU box)",
       "points": []}
for n in (10_000, 20_000, 40_000):
    text = dump_trace_columns(ingest_document_columns(n, seed=0)).decode()
    t0 = time.perf_counter()
    doc = parse_trace(text)
    t1 = time.perf_counter()
    g = build_graph(doc)
    t2 = time.perf_counter()
    map_tasks_to_layers(g, list(doc.layer_markers))
    t3 = time.perf_counter()
    pt = {"records": len(doc.events), "markers": len(doc.layer_markers), "parse_s": t1 - t0,
          "build_graph_s": t2 - t1, "map_layers_s": t3 - t2, "total_s": t3 - t0}
    out["points"].append(pt)
    print(json.dumps(pt), flush=True)
# fitted scaling: parse/build ~ linear, layer map ~ N * M (markers grow with N)
p = out["points"]
lin = (p[-1]["parse_s"] + p[-1]["build_graph_s"]) / p[-1]["records"]
quad = p[-1]["map_layers_s"] / (p[-1]["records"] * max(p[-1]["markers"], 1))
n10 = 10_127_485
m10 = 255_104
out["extrapolated_10M_s"] = {"parse_plus_build": lin * n10, "map_layers": quad * n10 * m10,
                             "law": "parse+build linear in N; layer map O(N*M)"}
(ROOT / "profiles" / "r01_reference_ingest_cpu.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out["extrapolated_10M_s"]))
