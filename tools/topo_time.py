"""verify_acyclic (ks_toposort) wall time on the config graphs: the lane-head warp
kernel with per-head requirements, with in-degree counters (DDSIM_TOPO_INDEG=1),
and the general list-scheduling kernel (DDSIM_TOPO_LISTSCHED=1)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_03318_b200 import workloads as W  # noqa: E402
from paper_2006_03318_b200.frozen import FrozenGraph  # noqa: E402

for name, w in [("resnet 10k", W.resnet50_trace()), ("bert 30k", W.bert_trace(buckets_mb=None)),
                ("gpt 100k", W.gpt_trace(n_tasks=100_000))]:
    fz = FrozenGraph.from_graph(w.graph)
    out = {}
    for mode in ("lanes", "lanes-indeg", "listsched"):
        os.environ.pop("DDSIM_TOPO_LISTSCHED", None)
        os.environ.pop("DDSIM_TOPO_INDEG", None)
        if mode == "listsched":
            os.environ["DDSIM_TOPO_LISTSCHED"] = "1"
        elif mode == "lanes-indeg":
            os.environ["DDSIM_TOPO_INDEG"] = "1"
        fz.toposort()
        t0 = time.perf_counter()
        order, ok = fz.toposort()
        out[mode] = (time.perf_counter() - t0, order)
    assert out["lanes"][1] == out["listsched"][1] == out["lanes-indeg"][1], name
    print(f"{name}: lanes (requirements) {out['lanes'][0] * 1e3:.1f} ms, lanes (in-degrees) "
          f"{out['lanes-indeg'][0] * 1e3:.1f} ms, listsched {out['listsched'][0] * 1e3:.1f} ms, "
          f"identical order ({len(out['lanes'][1])} tasks)", flush=True)
