// breakdown: batched runtime decomposition of max-plus results.
//
// Reference: kernsim.breakdown.compute_breakdown / per_layer_breakdown
// (pkg/src/kernsim/breakdown.py:42-111).  The reference sweeps the sorted set
// of interval endpoints of one schedule and classifies each elementary span of
// [0, makespan) as CPU-only, GPU-only, both, or idle.
//
// Device formulation: on a lane-chained graph every lane's tasks execute in
// lane order and never overlap (start(next) >= start + dur + gap), so each
// lane's non-empty intervals -- CPU tasks [start, end + gap) (gaps_as_cpu_busy),
// GPU/comm tasks [start, end) -- are already sorted and disjoint.  One thread
// per scenario merges the L lane sequences in time order (an L-way merge with
// per-class active counters), which yields exactly the reference's
// classification without materialising or sorting the endpoint set.  A lane
// that violates the precondition (negative durations can break it) marks the
// scenario's parts -1 so the host can report it.
//
// Memory: per event one start (8 B) and one duration (4/8 B) read; rows are
// visited per lane, so a warp's loads hit a handful of rows at once and L2
// absorbs the rest.  per_layer_breakdown is a second, row-sequential kernel
// with coalesced read-modify-write accumulators [layer][class][S].
#include "ddsim_internal.h"

#include <climits>

namespace ddsim {

constexpr int kBdMaxLanes = 32;
enum { BD_CPU = 0, BD_GPU = 1, BD_COMM = 2, BD_CPU_DATALOAD = 3 };

struct LaneCursor {
  int pos;        // virtual position in the lane's sequence
  int len;        // static rows + chain members (if present)
  long long a, b; // current interval
  int cls;        // 0 cpu, 1 gpu; -1 exhausted
  bool active;
  bool chain_on;  // the lane's permutable chain is present in this scenario
  long long last_end;
};

__device__ __forceinline__ long long bd_dur(const BreakdownParams& p, int row, int s) {
  if (p.dkind == 1) return (long long)static_cast<const int*>(p.dur)[(long long)row * p.dld + s];
  return static_cast<const long long*>(p.dur)[(long long)row * p.dld + s];
}

__device__ __forceinline__ int bd_row(const BreakdownParams& p, int l, int v, int s, bool chain_on) {
  const int base = p.lane_ptr[l];
  const int c = p.lane_chain[l];
  if (c < 0 || !chain_on) return p.lane_rows[base + v];
  const BdChain ch = p.chains[c];
  if (v < ch.pos) return p.lane_rows[base + v];
  if (v < ch.pos + ch.B) {
    const int k = v - ch.pos;
    const int m = p.perm ? (int)p.perm[(long long)s * p.perm_ld + ch.perm_off + k] : k;
    return p.member_rows[ch.member_off + m];
  }
  return p.lane_rows[base + v - ch.B];
}

// advance lane l to its next non-empty interval; false on a precondition failure
__device__ bool bd_advance(const BreakdownParams& p, LaneCursor& c, int l, int s) {
  while (c.pos < c.len) {
    const int row = bd_row(p, l, c.pos, s, c.chain_on);
    ++c.pos;
    const long long st = p.start[(long long)row * p.start_ld + s];
    if (st < 0) {
      if (st == -1) continue;  // removed task / absent chain member
      return false;
    }
    const int rc = p.row_class[row];
    long long e = st + bd_dur(p, row, s);
    int cls;
    if (rc == BD_CPU || rc == BD_CPU_DATALOAD) {
      if (rc == BD_CPU_DATALOAD && !p.dataload_as_cpu) continue;
      if (p.gaps_as_cpu_busy) e += p.gap[row];
      cls = 0;
    } else if (rc == BD_GPU) {
      cls = 1;
    } else {
      cls = p.comm_as_gpu ? 1 : 0;
    }
    if (e <= st) continue;
    if (st < c.last_end) return false;  // not sorted/disjoint: lane-order sweep invalid
    c.a = st;
    c.b = e;
    c.cls = cls;
    c.last_end = e;
    return true;
  }
  c.cls = -1;
  return true;
}

__global__ void __launch_bounds__(128) breakdown_kernel(const BreakdownParams p) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p.S) return;
  LaneCursor cur[kBdMaxLanes];
  const long long ms = p.makespan[s];
  bool ok = true;
  for (int l = 0; l < p.L; ++l) {
    LaneCursor& c = cur[l];
    const int c_ix = p.lane_chain[l];
    bool chain_on = false;
    int len = p.lane_ptr[l + 1] - p.lane_ptr[l];
    if (c_ix >= 0) {
      chain_on = p.present == nullptr || p.present[(long long)s * p.n_chains + c_ix] != 0;
      if (chain_on) len += p.chains[c_ix].B;
    }
    c.pos = 0;
    c.len = len;
    c.chain_on = chain_on;
    c.active = false;
    c.last_end = LLONG_MIN;
    c.cls = -1;
    if (ok) ok = bd_advance(p, c, l, s);
  }
  long long acc[4] = {0, 0, 0, 0};  // cpu_only, gpu_only, parallel, idle
  int cc = 0, gc = 0;
  long long t = 0;
  while (ok) {
    int best = -1;
    long long ev = LLONG_MAX;
    for (int l = 0; l < p.L; ++l) {
      if (cur[l].cls < 0) continue;
      const long long e = cur[l].active ? cur[l].b : cur[l].a;
      if (e < ev) {
        ev = e;
        best = l;
      }
    }
    const long long te = best < 0 ? ms : min(ev, ms);
    if (te > t) {
      const long long span = te - t;
      if (cc > 0 && gc > 0)
        acc[2] += span;
      else if (cc > 0)
        acc[0] += span;
      else if (gc > 0)
        acc[1] += span;
      else
        acc[3] += span;
      t = te;
    }
    if (best < 0 || ev >= ms) break;
    LaneCursor& c = cur[best];
    if (c.active) {
      if (c.cls == 0) --cc; else --gc;
      c.active = false;
      ok = bd_advance(p, c, best, s);
    } else {
      if (c.cls == 0) ++cc; else ++gc;
      c.active = true;
    }
  }
  long long* o = p.parts + (long long)s * 4;
  for (int k = 0; k < 4; ++k) o[k] = ok ? acc[k] : -1;
}

// per_layer_breakdown (breakdown.py:100-111): per layer, summed CPU and GPU
// task durations of the scheduled tasks, comm lanes excluded.
__global__ void layer_busy_kernel(const BreakdownParams p) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p.S) return;
  for (int row = 0; row < p.n; ++row) {
    const int rc = p.row_class[row];
    if (rc == BD_COMM) continue;
    const long long st = p.start[(long long)row * p.start_ld + s];
    if (st < 0) continue;
    const int lid = p.row_layer[row];
    const int col = rc == BD_GPU ? 1 : 0;
    long long* acc = p.layer_busy + ((long long)lid * 2 + col) * p.S + s;
    *acc += bd_dur(p, row, s);
  }
}

cudaError_t launch_breakdown(const BreakdownParams& p, cudaStream_t stream) {
  if (p.S <= 0) return cudaSuccess;
  if (p.L > kBdMaxLanes) return cudaErrorInvalidValue;
  const int BD = 128;
  const int grid = (p.S + BD - 1) / BD;
  if (p.parts) {
    breakdown_kernel<<<grid, BD, 0, stream>>>(p);
    note_launch();
  }
  if (p.layer_busy && p.row_layer) {
    cudaError_t e = launch_fill_i64(p.layer_busy, 0, (long long)p.n_layers * 2 * p.S, stream);
    if (e != cudaSuccess) return e;
    layer_busy_kernel<<<grid, BD, 0, stream>>>(p);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace ddsim
