"""Golden vectors for export_chrome_trace (kernsim/chrome.py:17-38), made by
running the REFERENCE on its crafted traces: baseline simulation and one
what-if per trace, exported in Chrome trace format.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_chrome_golden.py
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF))

from kernsim.api import Analysis  # noqa: E402
from kernsim.chrome import export_chrome_trace  # noqa: E402
from tests import crafted  # noqa: E402

OUT = Path(__file__).resolve().parent / "chrome_golden.json.gz"


def main() -> None:
    cases = [("gpu_bound", crafted.gpu_bound_trace(), "amp", None),
             ("layered", crafted.layered_trace(), "amp", None),
             ("fused_adam", crafted.fused_adam_trace(n_updates=8), "fused_adam", None),
             ("distributed_2", crafted.distributed_trace(2), "distributed",
              {"workers": 4, "bandwidth_gbps": 10})]
    out = []
    for name, doc, scen, params in cases:
        a = Analysis.from_text(json.dumps(doc))
        g2, r2 = a.run_pipeline(a.pipeline_for(scen, params))
        out.append({"name": name, "doc": doc, "scenario": scen, "params": params,
                    "baseline": export_chrome_trace(a.baseline, a.graph),
                    "whatif": export_chrome_trace(r2, g2)})
    with gzip.open(OUT, "wt") as f:
        json.dump(out, f)
    print(f"wrote {len(out)} cases to {OUT}")


if __name__ == "__main__":
    main()
