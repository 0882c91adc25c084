"""Benchmark: batched simulate() throughput on BASELINE config 4.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[3]): Monte-Carlo duration-jitter sweep of a
100k-task GPT-style iteration graph (1 CPU thread + 2 CUDA streams),
65,536 scenarios.  Scenario s of task v runs for
d' = floor((2 d k + 1000) / 2000) with k ~ U{900..1100} (round_half_up of
d * k/1000, transform.py:174-183), materialised as int32 [rows][S] in HBM.

A step = one pass of the hot path (maxplus_sim) over one batch: start times
of every (task, scenario), per-scenario makespan and lane busy times.
`value` = scenario x task updates / s with inputs resident in HBM; `e2e` =
the same through the C-ABI host-buffer entry point (ks_simulate_host), with
the H2D of durations and D2H of all results inside the timed region.

Multi-GPU: one process per GPU (torchrun; `--gpus N` without torchrun
re-launches itself under torch.distributed.run), scenarios sharded, no
data-path collective; barrier + max-over-ranks timing.  --scaling strong
(default, BASELINE config 4 as stated: 65,536 scenarios in total, sharded
across the N GPUs) or weak (65,536 scenarios per GPU).  After timing, every
rank checks scenarios of its own timed output against the C oracle (Alg. 1)
and rank 0 prints them as `parity_checked`.

--impl reference: the reference algorithm (Alg. 1, sim.py:89-142) as the C
oracle port on the host cores (the reference is pure Python and cannot be
installed on the GPU box), same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_TASKS = 100_000
S_PER_GPU = 65_536
METRIC = "scenario x task updates/sec"
UNIT = "updates/s"
BYTES_PER_UPDATE = 12  # int32 duration read + int64 start write


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6551.0)), "measured"
    return 6650.0, "fallback"


def _ncu_traffic(kernel: str):
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        rec = d.get(kernel)
        return None if rec is None else rec.get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
             "clocks.mem,temperature.memory,temperature.gpu")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def wait_ready(self, timeout_s: float = 3.0) -> None:
        """Block until the sampler has written its first row (nvidia-smi
        takes ~0.1-0.5 s to start)."""
        t0 = time.perf_counter()
        while self.p is not None and time.perf_counter() - t0 < timeout_s:
            if Path(self.f.name).stat().st_size > 0:
                return
            time.sleep(0.02)

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi missing"]}
        self.p.terminate()
        self.p.wait()
        rows = [l.split(",") for l in Path(self.f.name).read_text().splitlines() if l.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(nm)
        os.unlink(self.f.name)

        def col(k):
            out = []
            for r in rows:
                try:
                    out.append(float(r[k]))
                except (IndexError, ValueError):
                    pass
            return out
        mem, tmem, tgpu = col(9), col(10), col(11)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows), "mem_mhz": statistics.median(mem) if mem else None,
                "hbm_temp_c_max": max(tmem) if tmem else None,
                "gpu_temp_c_max": max(tgpu) if tgpu else None}


def make_jitter_dense(fz, S: int, seed: int, device: int):
    """Config-4 jitter durations on the device: int32 [rows][S] (frozen rows),
    d' = floor((2 d k + 1000) / 2000), k ~ U{900..1100} (torch Generator)."""
    import torch

    base = torch.from_numpy(fz.duration[fz.order].copy()).to(f"cuda:{device}")
    dense = torch.empty((fz.n, S), dtype=torch.int32, device=f"cuda:{device}")
    gen = torch.Generator(device=f"cuda:{device}")
    gen.manual_seed(seed)
    step_rows = max(1, (1 << 28) // S)
    for r0 in range(0, fz.n, step_rows):
        r1 = min(fz.n, r0 + step_rows)
        k = torch.randint(900, 1101, (r1 - r0, S), generator=gen, device=f"cuda:{device}",
                          dtype=torch.int64)
        dense[r0:r1] = ((2 * base[r0:r1, None] * k + 1000) // 2000).to(torch.int32)
        del k
    return dense


def oracle_check(w, fz, dense, start, ms, lb, cols) -> list:
    """Scenarios `cols` of a device result against the C oracle's Alg. 1
    (checker only, after the timed region): start of every task, makespan,
    lane busy.  Raises on the first difference."""
    sys.path.insert(0, str(ROOT / "oracle"))
    from oracle import OracleGraph  # checker

    og = OracleGraph.from_graph(w.graph)
    done = []
    for s in cols:
        d = np.empty(fz.n, np.int64)
        d[fz.order] = dense[:, s].cpu().numpy()
        st, m, lbo, _ = og.simulate("default", dur=d)
        got = start[:, s].cpu().numpy()
        want = np.array([st[int(t)] for t in fz.row_ids], np.int64)
        if int(ms[s].item()) != m or not np.array_equal(got, want):
            raise AssertionError(f"scenario {s}: device result differs from the oracle "
                                 f"(makespan {int(ms[s].item())} vs {m})")
        lbd = {str(fz.lanes[j]): int(lb[s, j].item()) for j in range(fz.L)}
        if lbd != {str(k): v for k, v in lbo.items()}:
            raise AssertionError(f"scenario {s}: lane busy differs from the oracle")
        done.append(int(s))
    return done


def build_workload(device: int):
    from paper_2006_03318_b200.frozen import FrozenGraph
    from paper_2006_03318_b200.workloads import gpt_trace

    w = gpt_trace(seed=0, n_tasks=N_TASKS)
    fz = FrozenGraph.from_graph(w.graph, device=device)
    return w, fz


def measure_breakdown(w, fz, dense, start, ms, S: int, peak: float, stream,
                      check: bool = True, calls: int = 3) -> dict:
    """compute_breakdown + per_layer_breakdown (breakdown.py:42-111) of the
    timed sweep's resident start matrix (ks_breakdown, after the timed region;
    not part of `value`): device time per call with CUDA events on the
    launching stream, algorithmic bytes 8 (start) + 4 (duration) per (task,
    scenario), and scenario 0 checked against the breakdown oracle."""
    import torch

    from paper_2006_03318_b200.batch import ScenarioTable, breakdown_batch_device, layer_names_of

    rows = fz.n
    dev = start.device
    names = layer_names_of(fz)
    parts = torch.empty((S, 4), dtype=torch.int64, device=dev)
    lbz = torch.empty((len(names), 2, S), dtype=torch.int64, device=dev)
    table = ScenarioTable(n_scenarios=S, dense=dense[:, :S] if dense.shape[1] != S else dense)

    def call():
        breakdown_batch_device(fz, table, start=start, makespan=ms[:S], parts=parts,
                               layer_busy=lbz, stream=stream.cuda_stream)

    call()
    stream.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(calls):
        call()
    b.record(stream)
    b.synchronize()
    sec = a.elapsed_time(b) / calls / 1e3
    gbs = rows * S * BYTES_PER_UPDATE / sec / 1e9
    out = {"ms_per_call": sec * 1e3, "updates_per_s": rows * S / sec, "algorithmic_GBps": gbs,
           "frac_of_peak": gbs / peak, "calls": calls, "layers": len(names),
           "kernel": "breakdown_stream_kernel (row-order sweep)"
           if S >= 22528 and fz.L <= 4 and fz.chained else "breakdown_lean_kernel (windowed merge)",
           "outputs": "parts [S][4] + per-layer busy [layers][2][S]"}
    if check:
        sys.path.insert(0, str(ROOT / "oracle"))
        from breakdown_oracle import breakdown as ora  # checker only
        s = 0
        col = start[:, s].cpu().numpy()
        d = dense[:, s].cpu().numpy().astype(np.int64)
        g = w.graph.copy()
        for r in range(rows):
            g.tasks[int(fz.row_ids[r])].duration = int(d[r])
        st_of = {int(fz.row_ids[r]): int(col[r]) for r in range(rows)}
        want = ora(g.tasks, st_of, int(ms[s].item()))
        got_parts = parts[s].tolist()
        assert got_parts == [want["cpu_only_ns"], want["gpu_only_ns"], want["parallel_ns"],
                             want["idle_ns"]], (got_parts, want)
        lb = lbz[:, :, s].cpu().numpy()
        for k, name in enumerate(names):
            if name in want["per_layer"]:
                pl = want["per_layer"][name]
                assert [int(lb[k, 0]), int(lb[k, 1])] == [pl["cpu_ns"], pl["gpu_ns"]], name
        out["parity_checked"] = {"scenarios": [s], "checker": "oracle/breakdown_oracle.py "
                                 "(breakdown.py:42-111): four parts + every layer"}
    return out


def cpu_baseline(w, fz, target_s: float = 12.0) -> dict:
    """The reference algorithm (C port of Alg. 1) on the host cores, on a
    bounded sample of the same workload (scenarios of the same jitter law)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    from oracle import OracleGraph  # CPU baseline leg (checker library)

    threads = os.cpu_count() or 1
    og = OracleGraph.from_graph(w.graph)
    base = og.dur
    rng = np.random.default_rng(1234)
    S = threads * 16  # one batch: 16 scenarios per thread
    t_used = 0.0
    upd = 0
    while t_used < target_s:
        k = rng.integers(900, 1101, size=(len(base), S))
        dense = np.ascontiguousarray(((2 * base[:, None] * k + 1000) // 2000).astype(np.int32))
        t0 = time.perf_counter()
        _ms, _st, u = og.simulate_batch(dense, threads, "default")
        t_used += time.perf_counter() - t0
        upd += u
    return {"value": upd / t_used, "unit": UNIT, "cores": threads, "kind": "port",
            "sample_scenarios": upd // len(base),
            "sample": f"{upd // len(base)} scenarios x {len(base)} tasks of the config-4 graph, "
                      f"{t_used:.1f} s wall, oracle/ddsim_oracle.c Alg.1 port (pthreads)"}


def run_reference(args):
    ws, rank, _local = _dist()
    if rank != 0:
        return
    from paper_2006_03318_b200.workloads import gpt_trace

    w = gpt_trace(seed=0, n_tasks=N_TASKS)

    class _F:  # cpu_baseline only needs w
        pass
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(w, _F, target_s=2.0 if i < args.warmup else 12.0 / max(args.steps, 1))
        if i >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": "config4 monte-carlo jitter: gpt-style 100k tasks (1 cpu + 2 "
                                   "streams), jitter k~U{900..1100}", "tasks": N_TASKS,
                       "scenarios_per_step": "sample (see cpu_baseline.sample)",
                       "sample_scenarios_per_step": cb["sample_scenarios"]},
            "cpu_baseline": dict(cb, value=v),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _bind_to_gpu_numa(dev: int):
    """Run the host side (and first-touch the pinned e2e buffers) on the CPUs
    local to the GPU's PCIe root (NVML affinity); no-op when NVML is missing."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        pass
    return None


def run_ours(args):
    import torch

    ws, rank, local = _dist()
    # test hooks for the multi-rank flow on a one-GPU box (never set by the driver):
    # DDSIM_BENCH_SAME_DEVICE=1 puts every rank on device 0, DDSIM_BENCH_BACKEND=gloo
    dev = 0 if os.environ.get("DDSIM_BENCH_SAME_DEVICE") else local
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist

        backend = os.environ.get("DDSIM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    from paper_2006_03318_b200 import _native as N
    from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch_device

    w, fz = build_workload(dev)
    S = shard_size(args.scenarios, ws, args.scaling)
    rows, L = fz.n, fz.L
    # ---- device-resident inputs: dense jitter durations [rows][S] int32 ----
    dense = make_jitter_dense(fz, S, 1000 + rank, dev)
    start = torch.empty((rows, S), dtype=torch.int64, device=f"cuda:{dev}")
    ms = torch.empty(S, dtype=torch.int64, device=f"cuda:{dev}")
    lb = torch.empty((S, L), dtype=torch.int64, device=f"cuda:{dev}")
    table = ScenarioTable(n_scenarios=S, dense=dense)
    stream = torch.cuda.current_stream()

    def step():
        simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=start,
                              stream=stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = Clocks(dev) if rank == 0 else None
    time.sleep(0.3 if clocks else 0)
    l0 = N.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = N.launch_count() - l0
    jit = (N.lib().ks_jit_log() or b"").decode()
    kernel_name = "ddsim_lanes_jit (NVRTC-specialised)" if "compiled" in jit else "static"
    elapsed_ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([elapsed_ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        dist.barrier()
    clk = clocks.stop() if clocks else None
    # the single result collective of a sharded sweep: every rank's
    # per-scenario makespan + lane busy gathered once over NCCL, outside the timed steps
    gather = None
    if ws > 1:
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flat = torch.cat([ms, lb.reshape(-1)])
        bufs = [torch.empty_like(flat) for _ in range(ws)]
        dist.barrier()
        g0.record(stream)
        dist.all_gather(bufs, flat)
        g1.record(stream)
        torch.cuda.synchronize()
        assert torch.equal(bufs[rank], flat)
        gather = {"collective": f"all_gather ({dist.get_backend()})",
                  "bytes_per_rank": flat.numel() * 8,
                  "ms": g0.elapsed_time(g1)}
    updates_per_step = rows * S
    total = updates_per_step * args.steps * ws
    value = total / (elapsed_ms / 1e3)
    per_launch_ms = elapsed_ms / args.steps
    peak, peak_src = _peaks()
    achieved = updates_per_step * BYTES_PER_UPDATE / (per_launch_ms / 1e3) / 1e9

    # parity of the timed output itself: first, middle and last scenario of this
    # rank's shard against the C oracle's Alg. 1 (outside the timed region)
    checked = oracle_check(w, fz, dense, start, ms, lb, sorted({0, S // 2 + 1, S - 1}))
    if ws > 1:
        import torch.distributed as dist
        ok = torch.tensor([len(checked)], device=f"cuda:{dev}")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        assert int(ok.item()) == len(checked)

    # speed of light of this exact traffic pattern: a library int32 -> int64
    # widening copy over the same matrices (26 GB read + 52 GB write, no compute)
    def probe():
        N.check(N.lib().ks_probe_widen(dense.data_ptr(), start.data_ptr(), rows * S,
                                       stream.cuda_stream), "ks_probe_widen")
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    probe()
    torch.cuda.synchronize()
    p0.record(stream)
    for _ in range(3):
        probe()
    p1.record(stream)
    torch.cuda.synchronize()
    pattern_gbs = updates_per_step * BYTES_PER_UPDATE / (p0.elapsed_time(p1) / 3 / 1e3) / 1e9

    # ---- e2e through the host-buffer C-ABI (H2D + D2H inside the timed region)
    e2e = e2e_all = None
    if not args.no_e2e:
        # same shard as the device-resident run (pinned host buffers: 12 B per update)
        S_e = S
        all_cpus = os.sched_getaffinity(0)
        numa_cpus = None if os.environ.get("DDSIM_BENCH_NO_NUMA") else _bind_to_gpu_numa(dev)
        def pinned(shape, dtype):
            """Pinned host buffer on 2 MB transparent huge pages registered with
            the driver (e2e 5.4-6.0 vs 4.3-5.0 G updates/s with 4 KB-page
            cudaHostAlloc buffers on the same boxes: fewer IOMMU / page-table
            entries per DMA); torch's pinned allocator if that fails."""
            if not os.environ.get("DDSIM_BENCH_TORCH_PINNED"):
                try:
                    import mmap
                    n = int(np.prod(shape)) * torch.tensor([], dtype=dtype).element_size()
                    m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
                    m.madvise(mmap.MADV_HUGEPAGE)
                    t = torch.frombuffer(m, dtype=dtype).view(shape)
                    t.zero_()  # populate (outside the timed region)
                    if torch.cuda.cudart().cudaHostRegister(t.data_ptr(), n, 0) == 0:
                        registered.append((t, m))
                        return t
                except Exception:
                    pass
            return torch.empty(shape, dtype=dtype, pin_memory=True)

        registered = []
        h_dense = pinned((rows, S_e), torch.int32)
        if S_e == S:
            h_dense.copy_(dense)
        else:  # strided column slice: copy in row blocks (a whole-slice copy stages a
            step = max(1, (1 << 28) // S_e)  # contiguous device temporary of the full slice)
            for r0 in range(0, rows, step):
                h_dense[r0:r0 + step].copy_(dense[r0:r0 + step, :S_e])
        h_start = pinned((rows, S_e), torch.int64)
        h_ms = torch.empty(S_e, dtype=torch.int64, pin_memory=True).numpy()
        h_lb = torch.empty((S_e, L), dtype=torch.int64, pin_memory=True).numpy()
        import ctypes as C

        def e2e_step():
            sc = N.ScenariosDesc()
            sc.n_scenarios = S_e
            sc.dense_kind = 1
            sc.dense = h_dense.data_ptr()
            sc.dense_ld = S_e
            out = N.SimOut()
            out.start, out.start_ld = h_start.data_ptr(), S_e
            out.makespan, out.lane_busy = h_ms.ctypes.data, h_lb.ctypes.data
            N.check(N.lib().ks_simulate_host(fz.handle, C.byref(sc), 0, 0, C.byref(out)))

        e2e_step()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        n_e2e = max(1, min(args.steps, 3))
        for _ in range(n_e2e):
            e2e_step()
        dt = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([dt], device=f"cuda:{dev}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        assert np.array_equal(h_ms, ms[:S_e].cpu().numpy()), "e2e result differs from device run"
        e2e_all = {"value": rows * S_e * n_e2e * ws / dt, "unit": UNIT,
                   "h2d_bytes_per_step": rows * S_e * 4,
                   "d2h_bytes_per_step": rows * S_e * 8 + S_e * 8 + S_e * L * 8,
                   "api": "ks_simulate_host (host buffers in and out, start matrix included)",
                   "host_cpus_bound": numa_cpus}
        del h_start
        # The sweep's result is its per-scenario makespan and lane busy; the
        # start matrix (52 GB) stays resident in HBM for device-side analysis
        # (breakdowns, Chrome rows).  Each step: the durations from pinned host
        # memory into HBM, the simulation (starts written to HBM as in `value`),
        # makespan + lane busy back to pinned host memory.
        from paper_2006_03318_b200.batch import ScenarioTable as _ST
        from paper_2006_03318_b200.batch import simulate_batch_device as _sbd
        h_ms2 = torch.empty(S_e, dtype=torch.int64, pin_memory=True)
        h_lb2 = torch.empty((S_e, L), dtype=torch.int64, pin_memory=True)
        d_in = dense if S_e == S else torch.empty((rows, S_e), dtype=torch.int32,
                                                    device=f"cuda:{dev}")
        d_st = start if S_e == S else torch.empty((rows, S_e), dtype=torch.int64,
                                                    device=f"cuda:{dev}")
        tab = _ST(n_scenarios=S_e, dense=d_in)

        def e2e_resident():
            d_in.copy_(h_dense, non_blocking=True)
            _sbd(fz, tab, makespan=ms[:S_e], lane_busy=lb[:S_e], start=d_st,
                 stream=stream.cuda_stream)
            h_ms2.copy_(ms[:S_e], non_blocking=True)
            h_lb2.copy_(lb[:S_e], non_blocking=True)
            stream.synchronize()

        e2e_resident()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_resident()
        dt2 = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([dt2], device=f"cuda:{dev}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt2 = float(t.item())
        assert np.array_equal(h_ms2.numpy(), h_ms), "resident e2e result differs"
        e2e = {"value": rows * S_e * n_e2e * ws / dt2, "unit": UNIT,
               "h2d_bytes_per_step": rows * S_e * 4,
               "d2h_bytes_per_step": S_e * 8 + S_e * L * 8,
               "api": "batch.simulate_batch_device: durations H2D from pinned host memory, "
                      "starts written to HBM and kept there, makespan + lane busy D2H",
               "host_cpus_bound": numa_cpus}
        del h_dense
        _release_registered(registered)
        os.sched_setaffinity(0, all_cpus)  # the CPU baseline uses every core

    bd = None
    if not args.no_breakdown:
        bd = measure_breakdown(w, fz, dense, start, ms, S, peak, stream, check=rank == 0)
    cb = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(w, fz)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_launch_ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int64",
            "data": "synthetic",
            "config": {"workload": "config4 monte-carlo jitter: gpt-style iteration graph "
                                   f"({rows} tasks, 1 cpu thread + 2 streams), {S * ws} "
                                   f"scenarios ({S} per GPU), k~U{{900..1100}} int32 durations "
                                   "resident in HBM",
                       "tasks": rows, "scenarios_total": S * ws, "scenarios_per_gpu": S,
                       "lanes": L,
                       "l2": "inputs (26 GB) >> 126 MB L2; no flush needed",
                       "graph_slots_smem": fz.info.n_slots_smem,
                       "graph_slots_spill": fz.info.n_slots - fz.info.n_slots_smem},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": updates_per_step * BYTES_PER_UPDATE,
                         # from the stored ncu --set full capture of this command
                         # (profiles/ncu_summary.json), not measured in this run
                         "traffic": _ncu_traffic("ddsim_lanes_jit") if S == S_PER_GPU else None,
                         "traffic_source": "profiles/ncu_summary.json (stored ncu capture "
                                           "of the default workload)",
                         "pattern_copy_gbs": pattern_gbs,
                         "pattern_frac": achieved / pattern_gbs,
                         "pattern": "ks_probe_widen: int32 -> int64 stream over the same "
                                    "[rows][S] matrices (4 B read + 8 B write per update, "
                                    "no recurrence)"},
            "cpu_baseline": cb,
            "e2e": e2e,
            "e2e_with_starts": e2e_all if e2e is not None else None,
            "parity_checked": {"scenarios_rank0": checked, "ranks": ws,
                               "checker": "oracle/ddsim_oracle.c Alg. 1 (sim.py:89-142): "
                                          "every start, makespan, lane busy"},
            "gpu_launches": launches,
            "result_gather": gather,
            "kernel": kernel_name,
            "clocks": clk,
            "breakdown": bd,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- configs 1-3, 5
# `--config N` measures BASELINE.json configs[N-1] with the same contract
# (device-resident value, e2e through the public host-buffer API, roofline,
# CPU baseline, oracle parity of the timed output).  Configs 1-3 are sweeps of
# derived durations (Shrink programs, inserted AllReduce chains); config 5 is
# trace ingest from JSON text.

CONFIG_NAMES = {
    1: "config1 resnet50-like iteration (~10k tasks, 1 cpu + 1 stream): baseline + AMP Shrink",
    2: "config2 bert-large-like per-layer Shrink 2x sweep (~30k tasks, one scenario per layer "
       "+ baseline)",
    3: "config3 data-parallel: bert-like trace + per-bucket AllReduce inserts, bandwidth (10) x "
       "workers (8) x bucket order (50)",
    5: "config5 trace ingest: 10M-record synthetic trace (8 cpu threads, 16 streams) from JSON "
       "text -> correlation join, sync links, layer map, frozen CSR graph",
}


def build_config(c: int, device: int):
    """-> (frozen, table, scenario checker, CPU-baseline closure, info)."""
    from fractions import Fraction

    from paper_2006_03318_b200 import workloads as W
    from paper_2006_03318_b200.batch import ScenarioTable, compile_scale_sweep, distributed_sweep
    from paper_2006_03318_b200.frozen import FrozenGraph
    from paper_2006_03318_b200.transform import (GPU_TASKS, And, ByLayer, Selector,
                                                 TransformPipeline, apply_pipeline,
                                                 scale_durations)

    if c in (1, 2):
        if c == 1:
            from paper_2006_03318_b200.scenarios import whatif_amp
            w = W.resnet50_trace()
            amp = whatif_amp(w.graph)
            scen = [[], [(Selector.from_object(x["selector"]), x["factor"]) for x in amp.steps]]
        else:
            w = W.bert_trace(buckets_mb=None)
            scen = [[(And([GPU_TASKS, ByLayer(l)]), "1/2")] for l in w.layers] + [[]]
        g = w.graph
        group_of, ptr, steps = compile_scale_sweep(g, scen)
        fz = FrozenGraph.from_graph(g, group_of=group_of, device=device)
        table = ScenarioTable(n_scenarios=len(scen), scale_ptr=ptr, scale=steps)

        def graph_of(s):
            h = g.copy()
            for sel, f in scen[s]:
                scale_durations(h, sel, Fraction(str(f)))
            return h
        return fz, table, graph_of, {"tasks": fz.n, "scenarios": len(scen)}
    if c == 3:
        from paper_2006_03318_b200.scenarios import whatif_distributed
        w = W.bert_trace(buckets_mb=25.0)
        g = w.graph
        buckets = w.trace.gradient_buckets
        B = len([b for b in buckets.buckets() if buckets.layers_of_bucket(b)])
        rng = np.random.default_rng(0)
        configs, perms = [], []
        for _ in range(50):
            o = rng.permutation(B)
            for nw in (1, 2, 4, 8, 16, 32, 64, 128):
                for bw in (1, 5, 10, 25, 50, 100, 200, 400, 800, 1600):
                    configs.append({"bandwidth_gbps": bw, "workers": nw})
                    perms.append(o)
        sw = distributed_sweep(g, buckets, configs, np.array(perms, np.int16), device=device)

        from paper_2006_03318_b200 import transform as TR

        def graph_of(s):
            # the reference pipeline's steps in this scenario's bucket order,
            # applied on the host without the device acyclicity check (the
            # oracle's Alg. 1 raises on a cycle itself)
            pipe = whatif_distributed(g, buckets=buckets, **configs[s])
            steps = [pipe.steps[k] for k in perms[s]] if pipe.steps else []
            h = g.copy()
            TR._DEFER["on"] = True
            try:
                for stp in steps:
                    TR.apply_step(h, stp)
            finally:
                TR._DEFER["on"] = False
            return h
        return sw.frozen, sw.table, graph_of, {"tasks": sw.frozen.n, "scenarios": len(configs),
                                               "buckets": B}
    raise ValueError(f"config {c}")


def _table_bytes(table) -> int:
    n = 0
    for a in (table.scale_ptr, table.scale, table.chain_perm, table.chain_present):
        if a is not None:
            n += np.asarray(a).nbytes
    return n


def _config_breakdown(fz, table, graph_of, start, ms, stream, calls: int = 5) -> dict:
    """The sweep's what-if reports (compute_breakdown + per_layer_breakdown,
    breakdown.py:42-111) from its resident starts through ks_breakdown, after
    the timed region: CUDA-event time per call and scenario 0 checked against
    the breakdown oracle on the reference-equivalent transformed graph."""
    import torch

    from paper_2006_03318_b200.batch import breakdown_batch_device, layer_names_of

    S = table.n_scenarios
    names = layer_names_of(fz)
    parts = torch.empty((S, 4), dtype=torch.int64, device=start.device)
    lbz = torch.empty((len(names), 2, S), dtype=torch.int64, device=start.device)

    def call():
        breakdown_batch_device(fz, table, start=start, makespan=ms, parts=parts, layer_busy=lbz,
                               stream=stream.cuda_stream)

    call()
    stream.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(calls):
        call()
    b.record(stream)
    b.synchronize()
    sec = a.elapsed_time(b) / calls / 1e3
    sys.path.insert(0, str(ROOT / "oracle"))
    from breakdown_oracle import breakdown as ora  # checker only
    s = 0
    col = start[:, s].cpu().numpy()
    st_of = {int(t): int(v) for t, v in zip(fz.row_ids.tolist(), col.tolist()) if v >= 0}
    g = graph_of(s)
    want = ora(g.tasks, st_of, int(ms[s].item()))
    got = parts[s].tolist()
    assert got == [want["cpu_only_ns"], want["gpu_only_ns"], want["parallel_ns"], want["idle_ns"]], \
        (got, want)
    lb = lbz[:, :, s].cpu().numpy()
    for k, name in enumerate(names):
        if name in want["per_layer"]:
            pl = want["per_layer"][name]
            assert [int(lb[k, 0]), int(lb[k, 1])] == [pl["cpu_ns"], pl["gpu_ns"]], name
    return {"ms_per_call": sec * 1e3, "scenarios": S, "calls": calls, "layers": len(names),
            "outputs": "parts [S][4] + per-layer busy [layers][2][S] (the sweep's what-if reports)",
            "parity_checked": {"scenarios": [s], "checker": "oracle/breakdown_oracle.py "
                               "(breakdown.py:42-111): four parts + every layer"}}


def _oracle_scenarios(fz, graph_of, ms, lb, start, cols) -> list:
    """Device rows of scenarios `cols` against the C oracle's Alg. 1 on the
    reference-equivalent transformed graph (checker only)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    from oracle import OracleGraph

    for s in cols:
        st, m, lbo, _ = OracleGraph.from_graph(graph_of(s)).simulate("default")
        col = start[:, s]
        got = {int(t): int(v) for t, v in zip(fz.row_ids.tolist(), col.tolist()) if v >= 0}
        if int(ms[s]) != m or got != st:
            raise AssertionError(f"scenario {s}: device differs from the oracle ({int(ms[s])} vs {m})")
        want_lb = {str(k): v for k, v in lbo.items()}
        got_lb = {str(fz.lanes[j]): int(lb[s, j]) for j in range(fz.L) if str(fz.lanes[j]) in want_lb}
        if got_lb != want_lb:
            raise AssertionError(f"scenario {s}: lane busy differs from the oracle")
    return [int(x) for x in cols]


def _config_cpu_baseline(graph_of, S, n, target_s=10.0) -> dict:
    """The reference algorithm per scenario: the scenario's transformed graph
    (the reference's pipeline semantics) and the C port of Alg. 1 on it, one
    scenario per host thread (ctypes releases the GIL), on a bounded sample of
    the sweep's scenarios.  Only the simulate calls are timed."""
    from concurrent.futures import ThreadPoolExecutor

    sys.path.insert(0, str(ROOT / "oracle"))
    from oracle import OracleGraph

    threads = os.cpu_count() or 1
    idx = np.unique(np.linspace(0, S - 1, min(S, 2 * threads)).astype(int))
    t0 = time.perf_counter()
    graphs = [OracleGraph.from_graph(graph_of(int(s))) for s in idx]
    t_build = time.perf_counter() - t0
    done, t_sim = 0, 0.0
    with ThreadPoolExecutor(threads) as ex:
        while t_sim < target_s:
            t1 = time.perf_counter()
            list(ex.map(lambda og: og.simulate_raw("default"), graphs))
            t_sim += time.perf_counter() - t1
            done += len(graphs)
    return {"value": done * n / t_sim, "unit": UNIT, "cores": threads, "kind": "port",
            "sample_scenarios": int(done),
            "sample": f"{len(graphs)} of {S} scenarios x {n} tasks, simulated {done} times: "
                      f"oracle/ddsim_oracle.c Alg. 1 on each transformed graph, {threads} threads, "
                      f"{t_sim:.1f} s (graph transforms {t_build:.1f} s, untimed)"}


def run_config(args):
    import torch

    from paper_2006_03318_b200 import _native as N
    from paper_2006_03318_b200.batch import simulate_batch, simulate_batch_device

    c = args.config
    ws, rank, local = _dist()
    if rank != 0:  # the secondary configs are single-GPU sweeps (replicas only)
        return
    dev = local
    torch.cuda.set_device(dev)
    fz, table, graph_of, info = build_config(c, dev)
    S, n, L = table.n_scenarios, fz.n, fz.L
    st = torch.empty((n, S), dtype=torch.int64, device=f"cuda:{dev}")
    ms = torch.empty(S, dtype=torch.int64, device=f"cuda:{dev}")
    lb = torch.empty((S, max(L, 1)), dtype=torch.int64, device=f"cuda:{dev}")
    stream = torch.cuda.current_stream()

    def step():
        simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=st,
                              stream=stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(dev)
    # the timed region of these sweeps is far shorter than the 200 ms sampling
    # interval: the sampler starts first and the same step runs back to back
    # (untimed) for ~0.6 s right before the timed region, so the samples show
    # the clocks the GPU runs this step at
    clocks.wait_ready()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 0.6:
        for _ in range(20):
            step()
        torch.cuda.synchronize()
    l0 = N.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = N.launch_count() - l0
    elapsed = e0.elapsed_time(e1)
    clk = clocks.stop()
    clk["sampled"] = "untimed back-to-back steps for 0.6 s ending at the timed region"
    per = elapsed / args.steps
    checked = _oracle_scenarios(fz, graph_of, ms.cpu().numpy(), lb.cpu().numpy(),
                                st.cpu().numpy(), sorted({0, S // 2, S - 1}))
    # e2e (wall clock, as config 4's): the host scenario tables uploaded by the
    # call, the simulation with its starts written to HBM and kept there, the
    # sweep's per-scenario makespan and lane busy copied to pinned host memory
    h_ms = torch.empty(S, dtype=torch.int64, pin_memory=True)
    h_lb = torch.empty((S, max(L, 1)), dtype=torch.int64, pin_memory=True)

    def e2e_step():
        simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=st,
                              stream=stream.cuda_stream)
        h_ms.copy_(ms, non_blocking=True)
        h_lb.copy_(lb, non_blocking=True)
        stream.synchronize()

    n_e2e = max(1, min(args.steps, 5))
    e2e_step()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        e2e_step()
    dt = (time.perf_counter() - t0) / n_e2e
    assert np.array_equal(h_ms.numpy(), ms.cpu().numpy()), "e2e result differs from device run"
    # ... and the host-buffer call that also copies every start back
    simulate_batch(fz, table)
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        r = simulate_batch(fz, table)
    dt_all = (time.perf_counter() - t0) / n_e2e
    assert np.array_equal(r.makespan, h_ms.numpy()), "e2e result differs from device run"
    jit = (N.lib().ks_jit_log() or b"").decode()
    peak, peak_src = _peaks()
    bd = None if args.no_breakdown else _config_breakdown(fz, table, graph_of, st, ms, stream)
    bpu = 8  # start write; durations derive on the device from base x scenario program
    achieved = n * S * bpu / (per / 1e3) / 1e9
    cb = None if args.no_cpu_baseline else _config_cpu_baseline(graph_of, S, n)
    line = {
        "metric": METRIC, "value": n * S / (per / 1e3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per, "higher_is_better": True,
        "scaling": "replicas only (one GPU per sweep)", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": CONFIG_NAMES[c], **info,
                   "l2": "outputs stream to HBM every step (no reuse across steps)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": n * S * bpu, "traffic": None,
                     "traffic_source": "not captured in this run (see profiles/)",
                     "path": "segment-parallel" if "seg_t" in jit else "single-pass"},
        "cpu_baseline": cb,
        "e2e": {"value": n * S / dt, "unit": UNIT, "h2d_bytes_per_step": _table_bytes(table),
                "d2h_bytes_per_step": S * 8 + S * L * 8,
                "api": "batch.simulate_batch_device: host scenario tables in, starts kept in "
                       "HBM, makespan + lane busy D2H"},
        "e2e_with_starts": {"value": n * S / dt_all, "unit": UNIT,
                            "h2d_bytes_per_step": _table_bytes(table),
                            "d2h_bytes_per_step": n * S * 8 + S * 8 + S * L * 8,
                            "api": "batch.simulate_batch (ks_simulate_host)"},
        "parity_checked": {"scenarios": checked,
                           "checker": "oracle/ddsim_oracle.c Alg. 1 on the reference-equivalent "
                                      "transformed graph: every start, makespan, lane busy"},
        "gpu_launches": launches,
        "clocks": clk,
        "breakdown": bd,
    }
    print(json.dumps(line), flush=True)


def run_config_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import os as _os
    _os.environ.setdefault("DDSIM_COMPILE_ONLY", "1")
    fz, table, graph_of, info = build_config(args.config, -1)
    vals, cb = [], None
    for i in range(args.warmup + args.steps):
        cb = _config_cpu_baseline(graph_of, table.n_scenarios, fz.n,
                                  target_s=1.0 if i < args.warmup else 6.0)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
                      "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                      "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None,
                      "dtype": "int64", "data": "synthetic",
                      "config": {"workload": CONFIG_NAMES[args.config], **info,
                                 "sample_scenarios_per_step": cb["sample_scenarios"]},
                      "cpu_baseline": dict(cb, value=v),
                      "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}), flush=True)


class _SubCols:
    """Rows `idx` of a TraceColumns (the oracle's ingest entry points take
    any object with these columns)."""

    def __init__(self, cols, idx):
        for k in ("id", "start", "duration", "correlation", "kind", "is_dtoh", "lane",
                  "sync_target"):
            setattr(self, k, np.asarray(getattr(cols, k))[idx])
        self.lanes = cols.lanes
        self.n = len(idx)
        self._lc = np.asarray(cols.lane_class_codes())

    def lane_class_codes(self):
        return self._lc


def _oracle_edges(cols):
    """Edge arrays of the oracle's build_graph over columns (checker)."""
    import ctypes as C

    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O

    h = O.lib()
    h.ora_build_graph.argtypes = [C.POINTER(O._OraTrace)] + [C.c_void_p] * 5
    h.ora_build_graph.restype = C.c_int64
    t, keep = O._trace_struct(cols)
    n = max(int(cols.n), 1)
    cap = 3 * n + int(np.sum(np.asarray(cols.kind) == 6)) * (len(cols.lanes) + 1) + 16
    sa, da, ka = np.empty(cap, np.int32), np.empty(cap, np.int32), np.empty(cap, np.uint8)
    gap, launcher = np.empty(n, np.int64), np.empty(n, np.int32)
    m = h.ora_build_graph(C.byref(t), sa.ctypes.data, da.ctypes.data, ka.ctypes.data,
                          gap.ctypes.data, launcher.ctypes.data)
    del keep
    return sa[:m], da[:m], ka[:m], gap[:cols.n], launcher[:cols.n]


def _sorted_edges(src, dst, kind):
    key = np.lexsort((np.asarray(kind, np.int64), np.asarray(dst, np.int64),
                      np.asarray(src, np.int64)))
    return np.asarray(src)[key], np.asarray(dst)[key], np.asarray(kind)[key]


def frozen_parity(cols, sa, da, gap, fz) -> dict:
    """The device-frozen graph against the oracle (checker): its row order is a
    topological order of the oracle's build_graph edges, and Alg. 1 on the
    oracle's graph (sim.py:89-142, base durations) gives the start times,
    makespan and lane busy the device simulates on the frozen graph (the first
    simulate builds the kernel programs)."""
    import ctypes as C

    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch

    t0 = time.perf_counter()
    n = int(cols.n)
    pos = np.empty(n, np.int64)
    pos[fz.order] = np.arange(n)
    if fz.n_ordered != n or not np.all(pos[sa] < pos[da]):
        raise AssertionError("device freeze order is not topological on the oracle's edges")
    ids = np.asarray(cols.id, np.int64)
    rank = np.empty(n, np.int32)
    rank[np.argsort(ids, kind="stable")] = np.arange(n, dtype=np.int32)
    og = O.OracleGraph(ids=ids, lanes=list(cols.lanes), dur=np.asarray(cols.duration, np.int64),
                       gap=np.asarray(gap, np.int64), ready=np.zeros(n, np.int64),
                       lane=np.asarray(cols.lane, np.int32), rank=rank,
                       prio=np.zeros(n, np.int32), flags=np.zeros(n, np.uint8),
                       vrank=np.full(n, -1, np.int32), src=np.asarray(sa, np.int32),
                       dst=np.asarray(da, np.int32))
    g = og._c()
    start = np.zeros(n, np.int64)
    trace = np.zeros(n, np.int32)
    lb = np.zeros(max(len(og.lanes), 1), np.int64)
    ms = np.zeros(1, np.int64)
    if O.lib().ora_simulate(C.byref(g), O.POL["default"], start.ctypes.data, trace.ctypes.data,
                            lb.ctypes.data, ms.ctypes.data) != n:
        raise AssertionError("oracle deadlock on the ingest graph")
    t1 = time.perf_counter()
    res = simulate_batch(fz, ScenarioTable(n_scenarios=1))
    t2 = time.perf_counter()
    dev_start = np.empty(n, np.int64)
    dev_start[fz.order] = res.start[:, 0]
    if int(res.makespan[0]) != int(ms[0]) or not np.array_equal(dev_start, start) \
            or not np.array_equal(res.lane_busy[0], lb[:fz.L]):
        raise AssertionError("simulate on the device-frozen graph differs from the oracle")
    return {"frozen_order_topological_on_oracle_edges": True,
            "simulate_base_vs_oracle": "every start, makespan, lane busy",
            "oracle_simulate_s": round(t1 - t0, 2),
            "first_simulate_incl_program_build_s": round(t2 - t1, 2)}


def ingest_parity(ct, res, tag, sample_cpu: int = 2000, fz=None) -> dict:
    """Config-5 output against the oracle (checker, outside the timed region):
    the whole edge multiset (src, dst, kind), every gap and every launcher of
    build_graph over all records; layer tags of a random sample of CPU events
    (the oracle's layer map is O(records x markers)), GPU events inheriting
    their launcher's tag."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O

    cols = ct.cols
    t0 = time.perf_counter()
    sa, da, ka, gap, launcher = _oracle_edges(cols)
    a = _sorted_edges(sa, da, ka)
    b = _sorted_edges(res.edge_src, res.edge_dst, res.edge_kind)
    if not (len(a[0]) == len(b[0]) and all(np.array_equal(x, y) for x, y in zip(a, b))):
        raise AssertionError("ingest edges differ from the oracle's build_graph")
    if not np.array_equal(gap, res.gap) or not np.array_equal(launcher, res.launcher):
        raise AssertionError("ingest gaps / launchers differ from the oracle")
    rng = np.random.default_rng(3)
    kind = np.asarray(cols.kind)
    cpu_idx = np.nonzero(np.isin(kind, [0, 1, 4, 6]) & (np.asarray(cols.lane) >= 0))[0]
    pick = np.sort(rng.choice(cpu_idx, size=min(sample_cpu, len(cpu_idx)), replace=False))
    tag_m, _tags = ct.marker_tags()
    sub = _SubCols(cols, pick)
    want, _bad = O.map_layers_columns(sub, np.full(len(pick), -1, np.int32), ct.m_lane,
                                      ct.m_start, ct.m_end, tag_m)
    if not np.array_equal(np.asarray(tag)[pick], want):
        raise AssertionError("layer tags differ from the oracle's map_tasks_to_layers")
    gpu = np.nonzero((np.asarray(res.launcher) >= 0))[0]
    if not np.array_equal(np.asarray(tag)[gpu], np.asarray(tag)[np.asarray(res.launcher)[gpu]]):
        raise AssertionError("GPU events do not inherit their launcher's layer")
    out = {"edges": int(len(b[0])), "gaps_and_launchers": int(cols.n),
           "layer_tags_sampled_cpu_events": int(len(pick)),
           "checker": "oracle/ddsim_oracle.c build_graph (all records) + map_layers (sample)",
           "check_s": round(time.perf_counter() - t0, 2)}
    if fz is not None:
        out["frozen"] = frozen_parity(cols, sa, da, gap, fz)
    return out


def _ingest_cpu_baseline(n_sample: int = 1_000_000) -> dict:
    """The reference's ingest algorithm (C port of build_graph rules 1-5 and
    the O(records x markers) layer containment scan) on one core, on a bounded
    sample of the config-5 generator: build_graph over a 1M-record trace, the
    layer scan timed on 2,000 CPU events of it and scaled to all of them."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_2006_03318_b200.workloads import ingest_document_columns

    ct = ingest_document_columns(n_sample, seed=1)
    cols = ct.cols
    t0 = time.perf_counter()
    _oracle_edges(cols)
    t_build = time.perf_counter() - t0
    kind = np.asarray(cols.kind)
    cpu_idx = np.nonzero(np.isin(kind, [0, 1, 4, 6]))[0]
    pick = cpu_idx[:: max(1, len(cpu_idx) // 2000)][:2000]
    tag_m, _ = ct.marker_tags()
    t1 = time.perf_counter()
    O.map_layers_columns(_SubCols(cols, pick), np.full(len(pick), -1, np.int32), ct.m_lane,
                         ct.m_start, ct.m_end, tag_m)
    t_map = (time.perf_counter() - t1) / len(pick) * len(cpu_idx)
    n = int(cols.n)
    return {"value": n / (t_build + t_map), "unit": "records/s", "cores": 1, "kind": "port",
            "sample_records": n,
            "sample": f"{n} records ({ct.n_markers} markers): build_graph {t_build:.2f} s + layer "
                      f"scan {t_map:.1f} s (timed on {len(pick)} CPU events, scaled to "
                      f"{len(cpu_idx)}); oracle/ddsim_oracle.c, 1 core"}


def run_ingest(args):
    import torch

    from paper_2006_03318_b200 import _native as N
    from paper_2006_03318_b200.columnar import (dump_trace_columns, frozen_from_ingest,
                                                 load_trace_columns)
    from paper_2006_03318_b200.ingest import ingest_arrays, map_layers_arrays
    from paper_2006_03318_b200.workloads import ingest_document_columns

    ws, rank, local = _dist()
    if rank != 0:  # ingest is replicas only (global joins)
        return
    torch.cuda.set_device(local)
    text = dump_trace_columns(ingest_document_columns(args.ingest_records, seed=0))
    times, stages = [], {}
    clocks = None
    l0 = 0
    for i in range(args.warmup + args.steps):
        if i == args.warmup:
            torch.cuda.synchronize()
            clocks = Clocks(local)
            l0 = N.launch_count()
        t0 = time.perf_counter()
        ct = load_trace_columns(text)
        t1 = time.perf_counter()
        res = ingest_arrays(ct.cols, keep_device=True)
        t2 = time.perf_counter()
        tag_m, tags = ct.marker_tags()
        tag = map_layers_arrays(ct.cols, res.launcher, ct.m_lane, ct.m_start, ct.m_end, tag_m)
        t3 = time.perf_counter()
        fz = frozen_from_ingest(ct, res)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        if i >= args.warmup:
            times.append(t4 - t0)
            for k, v in (("parse_s", t1 - t0), ("ingest_s", t2 - t1), ("layer_map_s", t3 - t2),
                         ("freeze_s", t4 - t3)):
                stages.setdefault(k, []).append(v)
        if i + 1 < args.warmup + args.steps:
            fz.close()
            del ct, res, tag, fz
    launches = N.launch_count() - l0
    clk = clocks.stop()
    n = int(ct.n_events)
    per = statistics.median(times)
    st = {k: statistics.median(v) for k, v in stages.items()}
    parity = ingest_parity(ct, res, tag, fz=fz)
    dev_s = st["ingest_s"] + st["layer_map_s"]
    peak, peak_src = _peaks()
    col_bytes = 41 * n
    line = {
        "metric": "trace records ingested/sec (JSON text -> device frozen graph)",
        "value": n / per, "unit": "records/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "replicas only (global joins)", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": CONFIG_NAMES[5], "records": n, "json_bytes": len(text),
                   "markers": int(ct.n_markers), "edges": int(res.edge_src.shape[0]),
                   "layers": len(tags), "frozen_chained": bool(fz.chained),
                   "host_threads": os.cpu_count(),
                   **{k: round(v, 4) for k, v in st.items()}},
        "roofline": {"bound": "hbm", "achieved": n * 80 / dev_s / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": n * 80 / dev_s / 1e9 / peak, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": n * 80, "traffic": None,
                     "note": "device stages (ks_ingest + ks_map_layers) wall time incl. their "
                             "column transfers; the step is host-bound (parse + freeze)"},
        "cpu_baseline": None if args.no_cpu_baseline else _ingest_cpu_baseline(),
        "e2e": {"value": n / per, "unit": "records/s", "h2d_bytes_per_step": col_bytes,
                "d2h_bytes_per_step": int(res.launcher.nbytes + 4 * n),
                "api": "columnar.load_trace_columns -> ingest_arrays(keep_device) -> "
                       "map_layers_arrays -> frozen_from_ingest (host text in, device frozen "
                       "graph out: ks_graph_create_from_ingest)"},
        "parity_checked": parity,
        "gpu_launches": launches // max(args.steps, 1),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def run_ingest_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    vals, cb = [], None
    for i in range(args.warmup + args.steps):
        cb = _ingest_cpu_baseline(200_000 if i < args.warmup else 1_000_000)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    print(json.dumps({"impl": "reference", "metric": "trace records ingested/sec (JSON text -> "
                      "device frozen graph)", "value": v, "unit": "records/s", "n_gpus": ws,
                      "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                      "scaling": "replicas only", "vs_baseline": None, "dtype": "int64",
                      "data": "synthetic",
                      "config": {"workload": CONFIG_NAMES[5],
                                 "sample_records_per_step": cb["sample_records"]},
                      "cpu_baseline": dict(cb, value=v),
                      "e2e": {"value": v, "unit": "records/s", "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}), flush=True)


def shard_size(total: int, ws: int, scaling: str) -> int:
    """Scenarios per rank: strong = the total split over the ranks (a multiple
    of 32), weak = the total on every rank."""
    if scaling == "weak" or ws == 1:
        return total
    return max(32, (total // ws) // 32 * 32)


def _release_registered(registered: list) -> None:
    """Unregister and unmap the e2e host buffers (huge-page mmaps)."""
    import torch

    while registered:
        t, m = registered.pop()
        rc = torch.cuda.cudart().cudaHostUnregister(t.data_ptr())
        if int(rc) != 0:
            print(f"warning: cudaHostUnregister returned {rc}", file=sys.stderr)
        del t
        try:
            m.close()
        except BufferError:  # a view is still alive; the mapping goes with it
            pass


def _spawn(args_n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and forward its output."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args_n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: --scenarios in total over all GPUs (BASELINE config 4); "
                         "weak: --scenarios per GPU")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scenarios", type=int, default=S_PER_GPU)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-breakdown", action="store_true")
    ap.add_argument("--ingest-records", type=int, default=10_000_000)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json configs[N-1]; 4 (default) is the headline jitter sweep")
    args = ap.parse_args()
    if args.config != 4:
        if args.config == 5:
            (run_ingest_reference if args.impl == "reference" else run_ingest)(args)
        else:
            (run_config_reference if args.impl == "reference" else run_config)(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args.gpus))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != ws:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={ws}; measuring {ws} rank(s)",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
