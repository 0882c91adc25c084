"""verify_acyclic (ks_toposort) wall time on the config graphs: lane-head warp
kernel vs the general list-scheduling kernel (DDSIM_TOPO_LISTSCHED=1)."""
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
    for mode in ("lanes", "listsched"):
        if mode == "listsched":
            os.environ["DDSIM_TOPO_LISTSCHED"] = "1"
        else:
            os.environ.pop("DDSIM_TOPO_LISTSCHED", None)
        fz.toposort()
        t0 = time.perf_counter()
        order, ok = fz.toposort()
        out[mode] = (time.perf_counter() - t0, order)
    assert out["lanes"][1] == out["listsched"][1], name
    print(f"{name}: lanes {out['lanes'][0] * 1e3:.1f} ms, listsched {out['listsched'][0] * 1e3:.1f} ms, "
          f"identical order ({len(out['lanes'][1])} tasks)", flush=True)
