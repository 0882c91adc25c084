import gzip, json, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from helpers import graph_from_obj
from paper_2006_03318_b200 import build_graph, map_tasks_to_layers
from paper_2006_03318_b200.trace import parse_trace
from paper_2006_03318_b200 import workloads as W
g = json.load(gzip.open('tests/golden/golden.json.gz', 'rt'))
case = [c for c in g['cases'] if c['name'] == 'genspec_12'][0]
tr = parse_trace(json.dumps(case['doc']))
mine = build_graph(tr)
ref = graph_from_obj(case['graph'])
e1 = {(u, v, k.value) for u, v, k in mine.edges}; e2 = {(u, v, k.value) for u, v, k in ref.edges}
print("extra", sorted(e1 - e2)[:10], "missing", sorted(e2 - e1)[:10])
print("gaps", [(i, mine.tasks[i].gap, ref.tasks[i].gap) for i in ref.tasks if mine.tasks[i].gap != ref.tasks[i].gap][:10])
print("lo", {str(k): v for k, v in mine.lane_order.items()} == {str(k): v for k, v in ref.lane_order.items()})
map_tasks_to_layers(mine, list(tr.layer_markers))
print("layers", [(i, mine.tasks[i].layer, ref.tasks[i].layer) for i in ref.tasks if mine.tasks[i].layer != ref.tasks[i].layer][:10])
for ev in tr.events[:0]: pass
try:
    w = W.resnet50_trace(); build_graph(w.trace)
except Exception as e:
    print("resnet:", repr(e))
