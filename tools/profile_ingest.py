"""Config-5 stage timings (DDSIM_TRACE_TIMING / DDSIM_INGEST_TIMING print
per-stage wall times of the native reader and ks_ingest)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("DDSIM_TRACE_TIMING", "1")
os.environ.setdefault("DDSIM_INGEST_TIMING", "1")

from paper_2006_03318_b200.columnar import dump_trace_columns, frozen_from_ingest, load_trace_columns  # noqa: E402
from paper_2006_03318_b200.ingest import ingest_arrays, map_layers_arrays  # noqa: E402
from paper_2006_03318_b200.workloads import ingest_document_columns  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
text = dump_trace_columns(ingest_document_columns(n, seed=0))
for rep in range(2):
    t = time.perf_counter()
    ct = load_trace_columns(text)
    t1 = time.perf_counter()
    res = ingest_arrays(ct.cols)
    t2 = time.perf_counter()
    tag_m, tags = ct.marker_tags()
    tag = map_layers_arrays(ct.cols, res.launcher, ct.m_lane, ct.m_start, ct.m_end, tag_m)
    t3 = time.perf_counter()
    fz = frozen_from_ingest(ct, res)
    t4 = time.perf_counter()
    print(f"rep {rep}: parse {t1-t:.3f} ingest {t2-t1:.3f} layers {t3-t2:.3f} freeze {t4-t3:.3f} "
          f"total {t4-t:.3f} s  ({ct.n_events} events, {res.edge_src.shape[0]} edges, "
          f"{os.cpu_count()} host cpus)", flush=True)
