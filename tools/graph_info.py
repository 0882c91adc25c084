import sys, time
sys.path.insert(0, '.')
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200 import workloads as W
for name, fn in [("resnet", W.resnet50_trace), ("bert", W.bert_trace), ("gpt", W.gpt_trace)]:
    t = time.time(); w = fn(); t1 = time.time()
    fz = FrozenGraph.from_graph(w.graph)
    i = fz.info
    print(name, w.n_tasks, "gen %.2fs freeze %.2fs" % (t1 - t, time.time() - t1), "chained", i.chained, "slots", i.n_slots, "smem", i.n_slots_smem, "levels", i.n_levels, "lanes", i.n_lanes, flush=True)
