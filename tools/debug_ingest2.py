import sys, json
sys.path.insert(0, '.')
from paper_2006_03318_b200 import build_graph, map_tasks_to_layers
from paper_2006_03318_b200.trace import parse_trace
from paper_2006_03318_b200 import workloads as W
def doc(events, markers):
    return json.dumps({"schema_version": 1, "time_unit": "microseconds", "events": events, "layer_markers": markers})
ev = lambda i, s, d, k="CpuOther", corr=None, lane="cpu:0": dict({"id": i, "kind": k, "name": "t", "lane": lane, "start": s, "duration": d}, **({"correlation": corr} if corr is not None else {}))
mk = lambda l, s, e, ph="Forward": {"layer": l, "phase": ph, "cpu_lane": "cpu:0", "start": s, "end": e}
for name, t in [("edge1", parse_trace(doc([ev(0, 2, 1), ev(1, 20, 1, "CpuApi", 1), ev(2, 60, 5, "GpuKernel", 1, "gpu:0:1")], [mk("outer", 0, 10), mk("inner", 1.5, 4), mk("*", 15, 30, "Backward")]))),
                ("edge2", parse_trace(doc([ev(0, 4, 0.5)], [mk("left", 0, 6), mk("right", 3, 9)])))]:
    try:
        g = build_graph(t); print(name, "ok", len(g.edges))
    except Exception as e:
        print(name, "ERR", repr(e))
try:
    w = W.resnet50_trace(); g = build_graph(w.trace); print("resnet ok", len(g.edges))
except Exception as e:
    print("resnet ERR", repr(e))
