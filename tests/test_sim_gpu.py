"""Device simulate() / verify_acyclic / longest_path against the reference's
golden vectors, and the batched kernels against the C oracle."""

import random

import numpy as np
import pytest

from helpers import graph_from_obj, policy_of, result_obj, strip_trace
from oracle import OracleGraph
from paper_2006_03318_b200 import errors, longest_path_makespan, simulate, verify_acyclic
from paper_2006_03318_b200.batch import ScenarioTable, compile_scale_sweep, simulate_batch
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200.graph import DependencyGraph, EdgeKind, Task
from paper_2006_03318_b200.scenarios import VdnnPrefetchPolicy
from paper_2006_03318_b200.sim import DefaultSchedule, PrioritySchedule, make_policy
from paper_2006_03318_b200.trace import LaneId, TaskKind
from paper_2006_03318_b200.transform import ByKind, ByNameSubstring, GPU_TASKS, And, Not, Or

pytestmark = pytest.mark.gpu


def _pol(name, params=None):
    return make_policy(name, **(params or {}))


def test_simulate_matches_reference_on_every_case(golden):
    for case in golden["cases"]:
        g = graph_from_obj(case["graph"])
        for pol in ("default", "priority"):
            assert result_obj(simulate(g, _pol(pol))) == case["sim"][pol], (case["name"], pol)


def test_simulate_whatif_graphs_with_their_policies(golden):
    for rec in golden["whatif"]:
        if "graph" not in rec:
            continue
        g = graph_from_obj(rec["graph"])
        name, params = policy_of(rec)
        assert result_obj(simulate(g, _pol(name, params))) == rec["sim"], \
            (rec["case"], rec["scenario"], rec["params"])
        assert result_obj(simulate(g, DefaultSchedule())) == rec["fifo"]


def test_list_scheduling_unsequenced_corpus(golden):
    for rec in golden["unsequenced"]:
        g = graph_from_obj(rec["graph"])
        for pol in ("default", "priority"):
            assert result_obj(simulate(g, _pol(pol))) == rec["sim"][pol], (rec["seed"], pol)


def test_verify_acyclic_and_longest_path(golden):
    for case in golden["cases"]:
        g = graph_from_obj(case["graph"])
        assert verify_acyclic(g) == case["topo"], case["name"]
        assert longest_path_makespan(g) == case["longest"], case["name"]


def _chain(n, lane="cpu:0", dur=1000):
    g = DependencyGraph()
    ln = LaneId.parse(lane)
    for i in range(n):
        g.tasks[i] = Task(id=i, kind=TaskKind.CPU_OTHER, name=f"t{i}", lane=ln, duration=dur)
    g.edges = {(i, i + 1, EdgeKind.LANE_SEQ_CPU) for i in range(n - 1)}
    g.lane_order = {ln: list(range(n))}
    return g


def test_deadlock_and_cycle_errors():
    g = _chain(3)
    g.edges.add((2, 0, EdgeKind.INJECTED))
    with pytest.raises(errors.Deadlock) as exc:
        simulate(g)
    assert "3 tasks never became ready" in str(exc.value)
    with pytest.raises(errors.CycleDetected) as exc2:
        verify_acyclic(g)
    assert set(exc2.value.cycle) <= {0, 1, 2}


def test_empty_graph_and_gaps():
    assert simulate(DependencyGraph()).makespan == 0
    assert verify_acyclic(DependencyGraph()) == []
    g = _chain(2)
    g.tasks[0].gap = 2000
    r = simulate(g)
    assert r.start_of == {0: 0, 1: 3000} and r.makespan == 4000


def test_simulate_does_not_mutate():
    g = _chain(5)
    before = {t: (v.duration, v.gap, v.ready_time) for t, v in g.tasks.items()}
    simulate(g)
    assert {t: (v.duration, v.gap, v.ready_time) for t, v in g.tasks.items()} == before


def test_user_policy_rejected():
    class Mine(DefaultSchedule):
        def choose(self, state, frontier):
            return max(frontier)
    with pytest.raises(errors.UnsupportedPolicy):
        simulate(_chain(2), Mine())


def test_ready_time_respected():
    g = _chain(2)
    g.tasks[1].ready_time = 50_000
    assert simulate(g).start_of[1] == 50_000


# ------------------------------------------------------------ batched kernels

def _genspec_graph(golden, name):
    case = next(c for c in golden["cases"] if c["name"] == name)
    return graph_from_obj(case["graph"])


@pytest.mark.parametrize("name", ["genspec_1001", "genspec_7", "gpu_bound", "distributed_4"])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("S", [300, 301])
def test_batch_dense_durations_vs_oracle(golden, name, dtype, S):
    g = _genspec_graph(golden, name)
    fz = FrozenGraph.from_graph(g)
    assert fz.chained
    rng = np.random.default_rng(0)
    base = fz.duration[fz.order]                        # frozen rows
    k = rng.integers(900, 1101, size=(fz.n, S))
    dense = ((2 * base[:, None] * k + 1000) // 2000).astype(dtype)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, dense=dense))
    og = OracleGraph.from_graph(g)
    # oracle task order == graph.tasks order == frozen input order
    for s in range(0, S, 37):
        d = np.empty(fz.n, np.int64)
        d[fz.order] = dense[:, s]
        st, ms, lb, _ = og.simulate("default", dur=d)
        assert res.makespan[s] == ms
        assert res.start_of(s) == st
        assert {str(k2): v for k2, v in res.lane_busy_of(s).items()} == \
            {str(k2): v for k2, v in lb.items()}


@pytest.mark.parametrize("mode", ["derived-lanes", "expand+lanes", "general"])
def test_batch_amp_and_layer_sweep_vs_oracle(golden, mode, monkeypatch):
    if mode == "general":
        monkeypatch.setenv("DDSIM_NO_EXPAND", "1")
    elif mode == "derived-lanes":
        monkeypatch.setenv("DDSIM_FORCE_DERIVED", "1")
    else:
        monkeypatch.setenv("DDSIM_NO_DERIVED", "1")
    g = _genspec_graph(golden, "genspec_1002")
    compute = Or([ByNameSubstring("sgemm"), ByNameSubstring("scudnn")])
    amp = [(And([GPU_TASKS, compute]), "1/3"), (And([GPU_TASKS, Not(compute)]), "1/2")]
    scen = [[], amp, [(ByKind(TaskKind.GPU_KERNEL), "2")], amp + amp,
            [(ByKind(TaskKind.CPU_API), "7/5"), (GPU_TASKS, "0.25")]]
    group_of, ptr, steps = compile_scale_sweep(g, scen)
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=len(scen), scale_ptr=ptr, scale=steps))
    from paper_2006_03318_b200.transform import scale_durations
    from fractions import Fraction
    for s, sc in enumerate(scen):
        h = g.copy()
        for sel, f in sc:
            scale_durations(h, sel, Fraction(str(f)))
        st, ms, lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms, s
        assert res.start_of(s) == st, s


def test_listsched_batch_with_scale_vs_oracle(golden):
    rec = golden["unsequenced"][3]
    g = graph_from_obj(rec["graph"])
    scen = [[], [(ByKind(TaskKind.COMM), "1/3")], [(GPU_TASKS, "5/2")]]
    group_of, ptr, steps = compile_scale_sweep(g, scen)
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    assert not fz.chained
    res = simulate_batch(fz, ScenarioTable(n_scenarios=3, scale_ptr=ptr, scale=steps),
                         policy="priority")
    from paper_2006_03318_b200.transform import scale_durations
    from fractions import Fraction
    for s, sc in enumerate(scen):
        h = g.copy()
        for sel, f in sc:
            scale_durations(h, sel, Fraction(str(f)))
        st, ms, lb, _ = OracleGraph.from_graph(h).simulate("priority")
        assert res.makespan[s] == ms and res.start_of(s) == st


def test_batch_dense_negative_durations_take_exact_path(golden):
    """Negative durations void the fast-path facts; the device flags them and
    the exact kernel reruns the launch (results must still match Alg. 1)."""
    g = _genspec_graph(golden, "genspec_1003")
    fz = FrozenGraph.from_graph(g)
    S = 64
    rng = np.random.default_rng(5)
    base = fz.duration[fz.order]
    dense = (base[:, None] + rng.integers(-3000, 3000, size=(fz.n, S))).astype(np.int32)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, dense=dense))
    og = OracleGraph.from_graph(g)
    for s in (0, 17, 63):
        d = np.empty(fz.n, np.int64)
        d[fz.order] = dense[:, s]
        st, ms, lb, _ = og.simulate("default", dur=d)
        assert res.makespan[s] == ms and res.start_of(s) == st


def test_batch_dense_int32_durations_with_int64_sums(golden):
    """int32 durations whose sums pass 2^31: start times are int64 (no
    wrap-around anywhere on the int32-input path); results match Alg. 1."""
    g = _genspec_graph(golden, "gpu_bound")
    fz = FrozenGraph.from_graph(g)
    assert fz.chained
    S = 128
    rng = np.random.default_rng(9)
    dense = rng.integers(0, 2**31 - 1, size=(fz.n, S)).astype(np.int32)
    dense[:, : S // 2] //= 1 << 12          # half the scenarios stay small (fast path result)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, dense=dense))
    og = OracleGraph.from_graph(g)
    assert int(res.makespan.max()) > 2**31
    for s in (0, 5, S // 2 - 1, S // 2, S - 1):
        d = np.empty(fz.n, np.int64)
        d[fz.order] = dense[:, s]
        st, ms, lb, _ = og.simulate("default", dur=d)
        assert res.makespan[s] == ms and res.start_of(s) == st
        assert {str(k2): v for k2, v in res.lane_busy_of(s).items()} == \
            {str(k2): v for k2, v in lb.items()}


KERNEL_PATHS = {
    "lanes-jit": {},
    "lanes-static": {"DDSIM_NO_JIT": "1"},
    "lanes-branch-free": {"DDSIM_LANES_DYN": "1"},
    "lanes-if-chain": {"DDSIM_LANES_DYN": "0"},
    # two scenarios per thread: the variant the config-4 bench times (S >= 18,944)
    "lanes-v2-jit": {"DDSIM_LANES_V": "2"},
    "lanes-v2-if-chain": {"DDSIM_LANES_V": "2", "DDSIM_LANES_DYN": "0"},
    "lanes-v2-branch-free": {"DDSIM_LANES_V": "2", "DDSIM_LANES_DYN": "1"},
    "lanes-v2-static": {"DDSIM_LANES_V": "2", "DDSIM_NO_JIT": "1"},
    "dense": {"DDSIM_NO_LANES": "1"},
    "general": {"DDSIM_NO_LANES": "1", "DDSIM_NO_DENSE": "1"},
}


@pytest.mark.parametrize("kpath", list(KERNEL_PATHS))
@pytest.mark.parametrize("name", ["genspec_1001", "distributed_4"])
def test_every_maxplus_kernel_path_matches_oracle(golden, name, kpath, monkeypatch):
    """The same dense batch through each max-plus kernel (NVRTC lanes kernel
    with either dispatch, the static lanes kernel, the dense kernel, the
    general kernel): identical to Alg. 1 scenario by scenario."""
    for k, v in KERNEL_PATHS[kpath].items():
        monkeypatch.setenv(k, v)
    g = _genspec_graph(golden, name)
    fz = FrozenGraph.from_graph(g)
    S = 96
    rng = np.random.default_rng(17)
    base = fz.duration[fz.order]
    dense = ((2 * base[:, None] * rng.integers(500, 1501, size=(fz.n, S)) + 1000) // 2000).astype(np.int32)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, dense=dense))
    og = OracleGraph.from_graph(g)
    for s in (0, 41, S - 1):
        d = np.empty(fz.n, np.int64)
        d[fz.order] = dense[:, s]
        st, ms, lb, _ = og.simulate("default", dur=d)
        assert res.makespan[s] == ms and res.start_of(s) == st
        assert {str(k2): v for k2, v in res.lane_busy_of(s).items()} == \
            {str(k2): v for k2, v in lb.items()}
