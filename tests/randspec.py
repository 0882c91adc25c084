"""Random valid-by-construction synthetic specs (CPU threads launching onto
their own streams, syncs, data loads, comm channels, layer tags).  Written for
this repository; shaped like the reference's acceptance corpus
(generated traces up to 5,000 tasks)."""

from __future__ import annotations

import random

KERNELS = ["sgemm_nn", "scudnn_fwd", "elementwise_mul", "batchnorm_bwd", "relu_fwd"]
STEMS = ["conv", "relu", "pool", "batchnorm", "fc", "attn"]
PHASES = ["Forward", "Backward", "WeightUpdate"]


def make_spec(rng: random.Random, n_tasks: int) -> dict:
    threads = rng.randint(1, 3)
    lanes = []
    corr = 1
    serial = 1
    per = max(2, n_tasks // (2 * threads))
    for t in range(threads):
        streams = [f"gpu:{t}:{k}" for k in range(1, rng.randint(2, 4))]
        cpu, gpu = [], {s: [] for s in streams}
        tag, left = None, 0
        for _ in range(per):
            if left == 0 and rng.random() < 0.3:
                tag = {"layer": f"{rng.choice(STEMS)}{serial}", "phase": rng.choice(PHASES)}
                serial += 1
                left = rng.randint(1, 5)
            extra = dict(tag) if left > 0 and tag else {}
            left = max(0, left - 1)
            if rng.random() < 0.35:
                extra["gap_us"] = {"min": 0, "max": rng.randint(1, 5)}
            r = rng.random()
            if r < 0.5:
                s = rng.choice(streams)
                cpu.append({"kind": "CpuApi", "name": "cudaLaunchKernel", "correlation": corr,
                            "duration_us": {"min": 0.2, "max": 15}, **extra})
                gpu[s].append({"kind": "GpuKernel", "name": rng.choice(KERNELS),
                               "correlation": corr, "duration_us": {"min": 0.5, "max": 60}})
                corr += 1
            elif r < 0.58:
                s = rng.choice(streams)
                dtoh = rng.random() < 0.5
                cpu.append({"kind": "CpuApi", "name": "memcpy_dtoh_async" if dtoh else "memcpy_htod",
                            "correlation": corr, "duration_us": {"min": 0.2, "max": 8}, **extra})
                gpu[s].append({"kind": "GpuMemcpy", "name": "memcpy", "correlation": corr,
                               "duration_us": {"min": 0.5, "max": 20}, "size_bytes": 4096})
                corr += 1
            elif r < 0.66 and corr > 1:
                sync = {"kind": "Sync", "name": "cudaStreamSynchronize",
                        "duration_us": {"min": 0.01, "max": 3}, **extra}
                if threads == 1 and rng.random() < 0.3:
                    sync["name"] = "cudaDeviceSynchronize"
                else:
                    sync["sync_target"] = rng.choice(streams)
                cpu.append(sync)
            elif r < 0.75:
                cpu.append({"kind": "DataLoad", "name": "load", "duration_us": {"min": 1, "max": 40},
                            **extra})
            else:
                cpu.append({"kind": "CpuOther", "name": "py", "duration_us": {"min": 0.1, "max": 10},
                            **extra})
        lanes.append({"lane": f"cpu:{t}", "tasks": cpu})
        lanes += [{"lane": s, "tasks": v} for s, v in gpu.items() if v]
    for ch in range(rng.randint(0, 2)):
        lanes.append({"lane": f"comm:ring{ch}", "tasks": [
            {"kind": "Comm", "name": f"allreduce_{i}", "duration_us": {"min": 1, "max": 100},
             "size_bytes": 1 << 20} for i in range(rng.randint(1, 6))]})
    return {"lanes": lanes}
