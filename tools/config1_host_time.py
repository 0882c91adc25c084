"""Config 1 host time per call (1x B200): the Python wrapper of
simulate_batch_device, the bare ks_simulate C-ABI call, fresh vs reused
descriptors.  Once the launch queue is full the host loop runs at the GPU's
pace (~40 us per call), so the first short loop shows the host cost (~29 us
C++ + ~4 us Python) and the later ones the device time."""
import sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
import torch, bench
from paper_2006_03318_b200.batch import simulate_batch_device
from paper_2006_03318_b200 import _native as N
fz, table, graph_of, info = bench.build_config(1, 0)
S, n, L = table.n_scenarios, fz.n, fz.L
st = torch.empty((n, S), dtype=torch.int64, device="cuda")
ms = torch.empty(S, dtype=torch.int64, device="cuda")
lb = torch.empty((S, max(L, 1)), dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
def step(): simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=st, stream=stream)
for _ in range(50): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): step()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("host per call us %.1f, total per call us %.1f" % ((t1 - t0) / 200 * 1e6, (t2 - t0) / 200 * 1e6))
# time the bare ctypes call vs python wrapper
keep = []
sc = table.desc(keep, fz.n)
out = N.SimOut(); out.makespan = N.ptr(ms); out.lane_busy = N.ptr(lb); out.start = N.ptr(st); out.start_ld = int(st.stride(0))
import ctypes as C
lib = N.lib()
t0 = time.perf_counter()
for _ in range(200): lib.ks_simulate(fz.handle, C.byref(sc), 0, 0, C.byref(out), C.c_void_p(stream))
t1 = time.perf_counter(); torch.cuda.synchronize()
print("bare ks_simulate host us %.1f" % ((t1 - t0) / 200 * 1e6))
t0 = time.perf_counter()
for _ in range(200): table.desc([], fz.n)
print("table.desc us %.1f" % ((time.perf_counter() - t0) / 200 * 1e6))
print((lib.ks_jit_log() or b"").decode()[-300:])
# pure Python overhead of the wrapper (ks_simulate replaced by a no-op)
class _Fake:
    def __getattr__(self, name):
        return getattr(lib, name)
    @staticmethod
    def ks_simulate(*a):
        return 0
real = N.lib
N.lib = lambda: _Fake()
t0 = time.perf_counter()
for _ in range(2000): step()
print("python wrapper only us %.1f" % ((time.perf_counter() - t0) / 2000 * 1e6))
N.lib = real
# fresh descriptor arrays per call vs the same arrays
def call_fresh():
    kp = []
    sc2 = table.desc(kp, fz.n)
    lib.ks_simulate(fz.handle, C.byref(sc2), 0, 0, C.byref(out), C.c_void_p(stream))
for _ in range(50): call_fresh()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500): call_fresh()
t1 = time.perf_counter(); torch.cuda.synchronize()
print("desc + ks_simulate host us %.1f" % ((t1 - t0) / 500 * 1e6))
t0 = time.perf_counter()
for _ in range(500): lib.ks_simulate(fz.handle, C.byref(sc), 0, 0, C.byref(out), C.c_void_p(stream))
t1 = time.perf_counter(); torch.cuda.synchronize()
print("same-desc ks_simulate host us %.1f" % ((t1 - t0) / 500 * 1e6))
t0 = time.perf_counter()
for _ in range(500): step()
t1 = time.perf_counter(); torch.cuda.synchronize()
print("wrapper host us %.1f" % ((t1 - t0) / 500 * 1e6))
