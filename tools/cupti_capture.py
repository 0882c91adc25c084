"""Record a small PyTorch training step with CUPTI (cupti.record) and print a
JSON summary: events per kind, the ingest/freeze result, the simulated
baseline makespan against the traced span, and an AMP-style what-if.

Run with NVTX_INJECTION64_PATH=<libcupti.so> so NVTX layer ranges reach CUPTI
(tests/test_cupti_gpu.py does).  --out DOC.json also writes the trace document."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_03318_b200 import cupti  # noqa: E402
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch  # noqa: E402
from paper_2006_03318_b200.columnar import dump_trace_columns, ingest_columns  # noqa: E402


def step(model, x, y, opt, side):
    nvtx = torch.cuda.nvtx
    h = x
    for i, lin in enumerate(model):
        nvtx.range_push(f"layer{i}/Forward")
        h = torch.relu(lin(h))
        nvtx.range_pop()
    loss = ((h - y) ** 2).mean()
    nvtx.range_push("loss/Backward")
    loss.backward()
    nvtx.range_pop()
    nvtx.range_push("optim/WeightUpdate")
    opt.step()
    opt.zero_grad(set_to_none=True)
    nvtx.range_pop()
    with torch.cuda.stream(side):          # a second stream
        z = x @ x.T
    torch.cuda.current_stream().wait_stream(side)
    side.synchronize()                     # cudaStreamSynchronize
    return float(loss.item()) + float(z[0, 0].cpu())   # device-to-host copies


def main():
    out = None
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
    torch.manual_seed(0)
    dev = torch.device("cuda:0")
    model = torch.nn.ModuleList([torch.nn.Linear(512, 512) for _ in range(4)]).to(dev)
    opt = torch.optim.SGD(model.parameters(), lr=1e-3)
    x = torch.randn(256, 512, device=dev)
    y = torch.randn(256, 512, device=dev)
    side = torch.cuda.Stream()
    for _ in range(3):                     # warm-up (cuBLAS handles, allocator)
        step(model, x, y, opt, side)
    torch.cuda.synchronize()
    with cupti.record() as rec:
        for _ in range(2):
            step(model, x, y, opt, side)
        torch.cuda.synchronize()
    ct = rec.trace
    c = ct.cols
    kinds = {int(k): int(v) for k, v in zip(*np.unique(c.kind, return_counts=True))}
    ci = ingest_columns(ct, strict=True)
    fz = ci.frozen
    base = simulate_batch(fz, ScenarioTable(n_scenarios=1))
    span = int((c.start + c.duration).max() - c.start.min())
    # the recorded trace as the reference's JSON document, through the drop-in API
    from paper_2006_03318_b200 import Analysis
    doc = dump_trace_columns(ct)
    a = Analysis.from_text(doc)
    amp = a.whatif("amp")
    res = {
        "events": int(c.n), "kinds": kinds, "lanes": [str(l) for l in c.lanes],
        "markers": int(ct.n_markers), "layers": list(ct.layers),
        "edges": int(ci.ingest.n_edges) if hasattr(ci.ingest, "n_edges") else int(len(ci.ingest.edge_src)),
        "layer_tagged_events": int(np.sum(ci.layer_tag >= 0)),
        "frozen_chained": bool(fz.chained), "n_ordered": int(fz.n_ordered),
        "baseline_makespan_ns": int(base.makespan[0]), "trace_span_ns": span,
        "makespan_over_span": int(base.makespan[0]) / max(span, 1),
        "metadata": ct.metadata,
        "dropin_baseline_makespan_ns": int(a.baseline.makespan),
        "amp_predicted_makespan_ns": int(amp["predicted_makespan_ns"]),
        "amp_speedup": amp["speedup"],
    }
    if out:
        Path(out).write_bytes(doc)
        res["document"] = out
    print(json.dumps(res))


if __name__ == "__main__":
    main()
