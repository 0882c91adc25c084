"""Seeded synthetic workloads shaped like BASELINE.json's configs.

A training-iteration trace is generated as a timeline (one or more CPU
threads issuing cudaLaunchKernel calls, kernels on CUDA streams, periodic
stream/device synchronisations, layer markers), exactly in the reference's
trace schema.  Because the generator knows every dependency it creates it
also returns the dependency graph *by construction*; the device ingest
(build_graph) must reproduce it, which tests/test_ingest_gpu.py checks.

Shapes:
  config 1  resnet50_trace   ~10k tasks, 1 CPU thread + 1 stream, sync / 400
  config 2  bert_trace       ~30k tasks, 400 layers (per-layer Shrink sweep)
  config 3  bert_trace       + gradient buckets (data-parallel sweep)
  config 4  gpt_trace        100k tasks, 1 CPU + 2 streams (jitter sweep)
  config 5  ingest_trace     many CPU threads / streams, memcpys, syncs
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import DependencyGraph, EdgeKind, Task
from .trace import (
    GradientBucketMap,
    LaneId,
    LayerMarker,
    Phase,
    TaskKind,
    TraceColumns,
    TraceDocument,
    TraceEvent,
)

KERNEL_NAMES = ["sgemm_128x128_nn", "scudnn_winograd_fwd", "elementwise_add_kernel",
                "batchnorm_fwd_kernel", "relu_fwd_kernel", "reduce_sum_kernel"]


@dataclass
class Workload:
    trace: TraceDocument
    graph: DependencyGraph          # by construction (what build_graph must return)
    layers: list[str]
    n_tasks: int


def _timeline(rng, n_pairs, n_streams, sync_every, stream_p, layer_of_pair, phase_of_pair,
              launch_ns=(3000, 9000), gap_ns=(0, 4000), kernel_ns=(2000, 120000),
              cpu_key="0", gpu_keys=None, first_id=0, first_corr=1, name_offset=0):
    """One CPU thread driving n_streams streams.  Returns events, edges and
    the per-pair CPU launch intervals (for markers)."""
    cpu = LaneId.parse(f"cpu:{cpu_key}")
    gpu_keys = gpu_keys or [f"0:{7 + s}" for s in range(n_streams)]
    streams = [LaneId.parse(f"gpu:{k}") for k in gpu_keys]
    ld = rng.integers(launch_ns[0], launch_ns[1] + 1, n_pairs)
    gp = rng.integers(gap_ns[0], gap_ns[1] + 1, n_pairs)
    kd = rng.integers(kernel_ns[0], kernel_ns[1] + 1, n_pairs)
    st = np.zeros(n_pairs, np.int64) if n_streams == 1 else \
        (rng.random(n_pairs) >= stream_p).astype(np.int64) * (1 + rng.integers(0, max(n_streams - 1, 1), n_pairs))
    st = np.minimum(st, n_streams - 1)
    events: list[TraceEvent] = []
    edges: set = set()
    t = 0
    free = [0] * n_streams
    last_kernel = [None] * n_streams
    prev_cpu = None
    prev_gpu = [None] * n_streams
    cpu_spans = []
    eid = first_id
    corr = first_corr
    gaps: dict[int, int] = {}
    for i in range(n_pairs):
        s = int(st[i])
        L = TraceEvent(id=eid, kind=TaskKind.CPU_API, name="cudaLaunchKernel", lane=cpu, start=t,
                       duration=int(ld[i]), correlation=corr)
        events.append(L)
        cpu_spans.append((t, t + int(ld[i])))
        if prev_cpu is not None:
            edges.add((prev_cpu.id, L.id, EdgeKind.LANE_SEQ_CPU))
            gaps[prev_cpu.id] = max(0, L.start - prev_cpu.end)
        prev_cpu = L
        eid += 1
        kstart = max(free[s], L.end)
        K = TraceEvent(id=eid, kind=TaskKind.GPU_KERNEL,
                       name=KERNEL_NAMES[(i + name_offset) % len(KERNEL_NAMES)], lane=streams[s],
                       start=kstart, duration=int(kd[i]), correlation=corr)
        events.append(K)
        edges.add((L.id, K.id, EdgeKind.LAUNCH_CORRELATION))
        if prev_gpu[s] is not None:
            edges.add((prev_gpu[s].id, K.id, EdgeKind.LANE_SEQ_GPU))
        prev_gpu[s] = K
        last_kernel[s] = K
        free[s] = K.end
        eid += 1
        corr += 1
        t = L.end + int(gp[i])
        if sync_every and (i + 1) % sync_every == 0:
            target = 0 if n_streams > 1 and (i // sync_every) % 2 == 0 else None
            waits = [0] if target is not None else list(range(n_streams))
            end = max([t] + [free[w] for w in waits])
            S = TraceEvent(id=eid, kind=TaskKind.SYNC,
                           name="cudaStreamSynchronize" if target is not None else
                           "cudaDeviceSynchronize", lane=cpu, start=t,
                           duration=max(end - t, 1000),
                           sync_target=streams[target] if target is not None else None)
            events.append(S)
            edges.add((prev_cpu.id, S.id, EdgeKind.LANE_SEQ_CPU))
            gaps[prev_cpu.id] = max(0, S.start - prev_cpu.end)
            for w in waits:
                if last_kernel[w] is not None:
                    edges.add((last_kernel[w].id, S.id, EdgeKind.SYNC_BLOCK))
            prev_cpu = S
            eid += 1
            t = S.end + int(gp[i])
    if prev_cpu is not None:
        gaps[prev_cpu.id] = 0
    return events, edges, gaps, cpu_spans, streams, cpu, eid, corr


def _graph(events, edges, gaps) -> DependencyGraph:
    g = DependencyGraph()
    for e in events:
        g.tasks[e.id] = Task(id=e.id, kind=e.kind, name=e.name, lane=e.lane, duration=e.duration,
                             gap=gaps.get(e.id, 0), correlation=e.correlation,
                             size_bytes=e.size_bytes, trace_start=e.start)
    g.edges = set(edges)
    by_lane: dict = {}
    for e in events:
        by_lane.setdefault(e.lane, []).append(e)
    for ln in sorted(by_lane, key=str):
        g.lane_order[ln] = [e.id for e in sorted(by_lane[ln], key=lambda e: (e.start, e.id))]
    return g


def _markers(cpu, spans, layer_of_pair, phase_of_pair):
    out = []
    i = 0
    n = len(spans)
    while i < n:
        j = i
        while j + 1 < n and layer_of_pair[j + 1] == layer_of_pair[i] and \
                phase_of_pair[j + 1] == phase_of_pair[i]:
            j += 1
        out.append(LayerMarker(layer=layer_of_pair[i], phase=phase_of_pair[i], cpu_lane=cpu,
                               start=spans[i][0], end=spans[j][1]))
        i = j + 1
    return out


def _iteration_layout(n_layers, kernels_fwd, kernels_bwd, n_wu):
    layers, phases = [], []
    names = [f"layer{l:03d}" for l in range(n_layers)]
    for l in range(n_layers):
        layers += [names[l]] * kernels_fwd
        phases += [Phase.FORWARD] * kernels_fwd
    for l in reversed(range(n_layers)):
        layers += [names[l]] * kernels_bwd
        phases += [Phase.BACKWARD] * kernels_bwd
    layers += ["optimizer"] * n_wu
    phases += [Phase.WEIGHT_UPDATE] * n_wu
    return names, layers, phases


def training_trace(n_layers, kernels_fwd, kernels_bwd, n_wu, n_streams=1, sync_every=400,
                   seed=0, stream_p=0.85, buckets_mb: float | None = None) -> Workload:
    rng = np.random.default_rng(seed)
    names, layers, phases = _iteration_layout(n_layers, kernels_fwd, kernels_bwd, n_wu)
    n_pairs = len(layers)
    events, edges, gaps, spans, streams, cpu, _eid, _c = _timeline(
        rng, n_pairs, n_streams, sync_every, stream_p, layers, phases)
    markers = _markers(cpu, spans, layers, phases)
    buckets = None
    if buckets_mb:
        # DDP-style buckets over layers in backward order (~buckets_mb each)
        per_layer = rng.integers(1 << 20, 4 << 20, n_layers)
        cap = int(buckets_mb * (1 << 20))
        bucket_of, sizes, cur, b = {}, {}, 0, 0
        for l in reversed(range(n_layers)):
            if cur and cur + per_layer[l] > cap:
                b += 1
                cur = 0
            bucket_of[names[l]] = b
            cur += int(per_layer[l])
            sizes[b] = sizes.get(b, 0) + int(per_layer[l])
        buckets = GradientBucketMap(bucket_of_layer=bucket_of, bucket_size_bytes=sizes)
    trace = TraceDocument(events=tuple(events), layer_markers=tuple(markers),
                          gradient_buckets=buckets)
    g = _graph(events, edges, gaps)
    # layer tags by construction: launch i and its kernel share pair i's tag
    pair = 0
    cur_tag = None
    for e in events:
        if e.kind is TaskKind.CPU_API:
            g.tasks[e.id].layer = (layers[pair], phases[pair])
            cur_tag = (layers[pair], phases[pair])
        elif e.kind is TaskKind.GPU_KERNEL:
            g.tasks[e.id].layer = cur_tag
            pair += 1
    return Workload(trace=trace, graph=g, layers=names, n_tasks=len(events))


def resnet50_trace(seed=0) -> Workload:
    """Config 1: ~10k tasks, 1 CPU + 1 stream, 160 layers x (fwd, bwd, WU)."""
    return training_trace(n_layers=160, kernels_fwd=10, kernels_bwd=20, n_wu=161, n_streams=1,
                          sync_every=400, seed=seed)


def bert_trace(seed=0, buckets_mb: float | None = 25.0) -> Workload:
    """Configs 2/3: ~30k tasks, 400 layers, 5,164 weight-update kernels."""
    return training_trace(n_layers=400, kernels_fwd=8, kernels_bwd=16, n_wu=5164, n_streams=1,
                          sync_every=400, seed=seed, buckets_mb=buckets_mb)


def gpt_trace(seed=0, n_tasks=100_000) -> Workload:
    """Config 4: GPT-style iteration, 1 CPU + 2 streams, ~n_tasks tasks."""
    pairs = n_tasks // 2
    n_layers = 96
    fwd = max(1, pairs // (n_layers * 3) - 0)
    bwd = 2 * fwd
    wu = max(0, pairs - n_layers * (fwd + bwd))
    w = training_trace(n_layers=n_layers, kernels_fwd=fwd, kernels_bwd=bwd, n_wu=wu,
                       n_streams=2, sync_every=0, seed=seed)
    return w


def resnet_like_graph(n_pairs=400, seed=0) -> DependencyGraph:
    """Small launch/kernel graph (smoke test)."""
    per = max(1, n_pairs // 30)
    return training_trace(n_layers=10, kernels_fwd=per, kernels_bwd=2 * per, n_wu=1,
                          n_streams=2, sync_every=50, seed=seed).graph


def jitter_matrix(base_rows: np.ndarray, S: int, seed: int = 0, out=None) -> np.ndarray:
    """d' = floor((2 d k + 1000) / 2000), k ~ U{900..1100} (round_half_up(d*k/1000)),
    int32 [rows][S].  Host generator (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    rows = base_rows.shape[0]
    out = np.empty((rows, S), np.int32) if out is None else out
    step = max(1, (1 << 24) // max(S, 1))
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        k = rng.integers(900, 1101, size=(r1 - r0, S), dtype=np.int64)
        out[r0:r1] = (2 * base_rows[r0:r1, None] * k + 1000) // 2000
    return out


def columns_of(trace: TraceDocument) -> TraceColumns:
    return TraceColumns.from_events(list(trace.events))


def ingest_columns(n_records: int = 10_000_000, seed: int = 0, n_threads: int = 8,
                   streams_per_thread: int = 2, with_markers: bool = True):
    """Config 5: a columnar CUPTI-like trace of ~n_records events (no Python
    objects per event).  Per CPU thread: launches (kernels), 2 % memcpy
    launches (half ``memcpy_dtoh_async``), 0.5 % syncs (stream / device-wide),
    1 % DataLoad; each launch's GPU task goes to one of the thread's streams,
    starting at max(stream free, launch end) (prefix-max form).  Markers (one
    per ~20 CPU tasks) are attached as ``cols.markers`` (lane, start, end, tag).
    """
    rng = np.random.default_rng(seed)
    lanes: list[LaneId] = []
    for t in range(n_threads):
        lanes.append(LaneId.parse(f"cpu:{t}"))
    for t in range(n_threads):
        for k in range(streams_per_thread):
            lanes.append(LaneId.parse(f"gpu:0:{t * streams_per_thread + k + 1}"))
    per_thread = n_records // n_threads
    ids, kinds, lane, start, dur, corr, st, dtoh = [], [], [], [], [], [], [], []
    mk = {"lane": [], "start": [], "end": [], "tag": []}
    next_id = 0
    next_corr = 1
    for t in range(n_threads):
        # CPU events: c of them, g of which launch a GPU task (total ~ per_thread)
        c = int(per_thread / 1.96)
        r = rng.random(c)
        is_sync = r < 0.005
        is_load = (r >= 0.005) & (r < 0.015)
        is_mcpy = (r >= 0.015) & (r < 0.035)
        is_launch = ~(is_sync | is_load)
        cd = rng.integers(3000, 9001, c).astype(np.int64)
        cd[is_load] = rng.integers(20_000, 200_000, int(is_load.sum()))
        cd[is_sync] = rng.integers(1_000, 50_000, int(is_sync.sum()))
        cg = rng.integers(0, 4001, c).astype(np.int64)
        cstart = np.concatenate([[0], np.cumsum(cd + cg)[:-1]])
        ckind = np.full(c, 0, np.uint8)          # CpuApi
        ckind[is_load] = 4                       # DataLoad
        ckind[is_sync] = 6                       # Sync
        cid = next_id + np.arange(c, dtype=np.int64)
        next_id += c
        ccorr = np.full(c, -1, np.int64)
        nl = int(is_launch.sum())
        ccorr[is_launch] = next_corr + np.arange(nl)
        csync = np.full(c, -1, np.int32)
        streams = n_threads + t * streams_per_thread + rng.integers(0, streams_per_thread, c)
        dev_wide = is_sync & (rng.random(c) < 0.3)
        csync[is_sync & ~dev_wide] = streams[is_sync & ~dev_wide].astype(np.int32)
        cdtoh = (is_mcpy & (rng.random(c) < 0.5)).astype(np.uint8)
        ids.append(cid); kinds.append(ckind); lane.append(np.full(c, t, np.int32))
        start.append(cstart); dur.append(cd); corr.append(ccorr); st.append(csync); dtoh.append(cdtoh)
        # GPU tasks of the launches
        li = np.nonzero(is_launch)[0]
        gl = streams[li].astype(np.int32)
        gd = rng.integers(2_000, 120_000, nl).astype(np.int64)
        gkind = np.where(is_mcpy[li], 3, 2).astype(np.uint8)
        lend = cstart[li] + cd[li]
        gstart = np.empty(nl, np.int64)
        for s_ in np.unique(gl):
            m = np.nonzero(gl == s_)[0]
            D = np.concatenate([[0], np.cumsum(gd[m])[:-1]])
            gstart[m] = np.maximum.accumulate(lend[m] - D) + D
        gid = next_id + np.arange(nl, dtype=np.int64)
        next_id += nl
        ids.append(gid); kinds.append(gkind); lane.append(gl); start.append(gstart)
        dur.append(gd); corr.append(next_corr + np.arange(nl)); st.append(np.full(nl, -1, np.int32))
        dtoh.append(np.zeros(nl, np.uint8))
        next_corr += nl
        if with_markers:
            # one marker per 20 consecutive CPU events, tags cycling over 400 layers x 3 phases
            b = np.arange(0, c, 20)
            e = np.minimum(b + 19, c - 1)
            mk["lane"].append(np.full(b.size, t, np.int32))
            mk["start"].append(cstart[b])
            mk["end"].append(cstart[e] + cd[e])
            mk["tag"].append((np.arange(b.size) % 1200).astype(np.int32))
    cols = TraceColumns(id=np.concatenate(ids), kind=np.concatenate(kinds),
                        lane=np.concatenate(lane), start=np.concatenate(start),
                        duration=np.concatenate(dur), correlation=np.concatenate(corr),
                        sync_target=np.concatenate(st), is_dtoh=np.concatenate(dtoh), lanes=lanes)
    if with_markers:
        cols.markers = {k: np.concatenate(v) for k, v in mk.items()}
    return cols


KERNEL_NAMES = ("sgemm_128x64_nn", "scudnn_winograd_fwd", "elementwise_add", "batchnorm_fwd",
                "relu_fwd", "softmax_bwd")


def ingest_document_columns(n_records: int = 10_000_000, seed: int = 0, **kw):
    """Config 5 as a full trace document in columnar form (columnar.ColumnarTrace):
    ``ingest_columns`` plus event names (launch / memcpy_dtoh / sync / dataload
    APIs, cycled kernel names) and markers named ``layer_NNNN`` x phase, so
    ``columnar.dump_trace_columns`` renders a valid kernsim JSON trace."""
    from .columnar import ColumnarTrace

    cols = ingest_columns(n_records, seed=seed, **kw)
    names = ["cudaLaunchKernel", "memcpy_dtoh_async", "cudaStreamSynchronize",
             "cudaDeviceSynchronize", "dataload_next_batch", "memcpy_async",
             *KERNEL_NAMES]
    k = cols.kind
    name_id = np.zeros(cols.n, np.int32)
    name_id[(k == 0) & (cols.is_dtoh == 1)] = 1
    name_id[(k == 6) & (cols.sync_target >= 0)] = 2
    name_id[(k == 6) & (cols.sync_target < 0)] = 3
    name_id[k == 4] = 4
    name_id[k == 3] = 5
    gk = k == 2
    name_id[gk] = 6 + (cols.id[gk] % len(KERNEL_NAMES)).astype(np.int32)
    m = cols.markers
    n_layers = int(m["tag"].max()) // 3 + 1 if m["tag"].size else 0
    layers = [f"layer_{i:04d}" for i in range(n_layers)]
    cols.names = None
    return ColumnarTrace(cols=cols, name_id=name_id, names=names,
                         size_bytes=np.full(cols.n, -1, np.int64), n_event_lanes=len(cols.lanes),
                         m_lane=m["lane"].astype(np.int32), m_start=m["start"], m_end=m["end"],
                         m_layer=(m["tag"] // 3).astype(np.int32),
                         m_phase=(m["tag"] % 3).astype(np.uint8), layers=layers)
