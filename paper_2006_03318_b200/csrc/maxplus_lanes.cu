// maxplus_lanes: the hot simulate() kernel for dense per-scenario durations
// on lane-chained graphs with at most 4 lanes (BASELINE config 4: 1 CPU
// thread + 2 streams).
//
// Recurrence (sim.py:89-142 on lane-chained graphs == synthetic.py:35-48):
//     start(v) = max(ready(v), max_{u->v} start(u) + dur(u) + gap(u)).
// Model: walking the frozen topological order, the rel (= start+dur+gap) of
// the most recent task of every lane lives in registers.  A task's lane
// predecessor is always its lane's head; a launch edge (CPU call -> kernel)
// or a sync edge (kernel -> CPU sync) is nearly always the head of the other
// lane too.  So each record is "max over a compile-time set of lane
// registers", dispatched through a 256-entry jump table of straight-line
// handlers <own lane, predecessor-lane mask, gap>.  Predecessors that are no
// longer a lane head go through compiled shared-memory slots (rare path).
//
// Fast-path facts (host-checked: gaps and ready times >= 0, graph chained;
// device-checked: durations >= 0 else *neg_flag -> exact rerun): every
// value is >= 0, so 0 is the identity of max, and the makespan is the max
// finish of the last task of each lane (rare path flag).
#include "ddsim_internal.h"

#include <algorithm>
#include <climits>
#include <cudaTypedefs.h>

#define HCASE(h)                                                                      \
  case h:                                                                             \
    hstep<(h) & 3, ((h) >> 2) & 31, ((h) >> 7) & 1, V>(S, d0, d1, gap, sp, ld, store); \
    break;
#define HCASE8(b) HCASE(b) HCASE(b + 1) HCASE(b + 2) HCASE(b + 3) HCASE(b + 4) HCASE(b + 5) \
  HCASE(b + 6) HCASE(b + 7)
#define HCASE64(b) HCASE8(b) HCASE8(b + 8) HCASE8(b + 16) HCASE8(b + 24) HCASE8(b + 32) \
  HCASE8(b + 40) HCASE8(b + 48) HCASE8(b + 56)
#define DDSIM_DISPATCH(h) switch (h) { HCASE64(0) HCASE64(64) HCASE64(128) HCASE64(192) }
#include "lanes_body.cuh"
#undef DDSIM_DISPATCH

namespace ddsim {

static_assert(sizeof(LaneRec) == sizeof(ddsim_lanes::Rec), "record layouts differ");
static_assert(sizeof(LaneParams) == sizeof(ddsim_lanes::Params), "param layouts differ");
static_assert(sizeof(LaneChainParams) == sizeof(ddsim_lanes::ChainParams), "chain layouts differ");

// DK: 1 = int32 durations via TMA tiles, 2 = int64 durations (direct loads).
template <int DK, int V>
__global__ void __launch_bounds__(256) maxplus_lanes_kernel(const __grid_constant__ ddsim_lanes::Tmap tmap,
                                                            const ddsim_lanes::Params p) {
  ddsim_lanes::lanes_body<DK, V, false>(&tmap, p);
}
template <int DK, int V>
__global__ void __launch_bounds__(256) maxplus_lanes_chain_kernel(
    const __grid_constant__ ddsim_lanes::Tmap tmap, const ddsim_lanes::Params p,
    const __grid_constant__ ddsim_lanes::ChainParams cp) {
  ddsim_lanes::lanes_body<DK, V, true>(&tmap, p, &cp);
}

// TMA pipeline depth of the JIT kernel (DDSIM_LANES_STAGES experiments; the
// static kernel always uses kStagesL and fits in the larger allocation)
static int lanes_stages() {
  const char* e = getenv("DDSIM_LANES_STAGES");
  const int s = e ? atoi(e) : ddsim_lanes::kStagesL;
  return s < ddsim_lanes::kStagesL ? ddsim_lanes::kStagesL : (s > 12 ? 12 : s);
}

static size_t lanes_smem(int dk, int BD, int V, int ksm) {
  const int stages = lanes_stages();
  size_t b = 128 + (size_t)stages * ddsim_lanes::kChunkL * sizeof(ddsim_lanes::Rec);
  if (dk == 0)  // derived durations: the chunk's RowDur entries
    b += (size_t)stages * ddsim_lanes::kChunkL * sizeof(ddsim_lanes::RowDur);
  else
    b += (size_t)stages * ddsim_lanes::kChunkL * BD * V * (dk == 1 ? 4 : 8);
  return b + (size_t)ksm * BD * 8 * V;
}

// V scenarios per thread (env DDSIM_LANES_V overrides: 1 or 2); two CTAs per
// SM cover S in one wave.  BD is a multiple of 16 so the grid is close to
// 2 x #SMs; the TMA box (BD * V ints) stays <= 256.
int maxplus_lanes_vec(int S, int dkind, bool vec_ok) {
  if (dkind == 0 || !vec_ok) return 1;  // derived durations / unaligned starts: one per thread
  const char* e = getenv("DDSIM_LANES_V");
  // two scenarios per thread only when there are enough scenarios to keep
  // ~4 warps per SM busy with V = 2; small sweeps want more threads instead
  int v = e ? atoi(e) : (S >= 2 * 148 * 64 ? 2 : 1);
  if (v != 1 && v != 2) v = 1;
  if (S % v) v = 1;
  return v;
}
int maxplus_lanes_block_dim(int S, int num_sms, int dkind, bool vec_ok) {
  const int V = maxplus_lanes_vec(S, dkind, vec_ok);
  if (const char* e = getenv("DDSIM_LANES_BD")) {  // experiments (multiple of 16)
    const int bd = atoi(e) / 16 * 16;
    if (bd >= 32 && bd <= 256 / V) return bd;
  }
  const long long threads = (S + V - 1) / V;
  long long per = (threads + 2LL * num_sms - 1) / (2LL * num_sms);
  int bd = (int)(((per + 15) / 16) * 16);
  const int cap = 256 / V;
  return bd < 32 ? 32 : (bd > cap ? cap : bd);
}

// Blocks of 32 scenarios x 8 row-strided threads over a chunk of rows
// (coalesced across the 32 scenarios); per-block sums go to lane_busy with
// 64-bit atomics (zeroed first).  The lane of a row is in its program record
// (h & 3); chain member rows with start -1 (absent chain) do not count.
constexpr int kBusyRowsPerBlock = 512;
__global__ void __launch_bounds__(256) lanes_busy_kernel(
    const LaneRec* prog, int n_rec, const int* d32, const long long* d64, long long dld,
    const long long* start, long long sld, int S, int L, unsigned long long* lane_busy) {
  __shared__ long long acc[8][4][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int s = blockIdx.x * 32 + tx;
  const int r0 = blockIdx.y * kBusyRowsPerBlock;
  const int r1 = min(n_rec, r0 + kBusyRowsPerBlock);
  long long lb[4] = {0, 0, 0, 0};
  if (s < S) {
    for (int r = r0 + ty; r < r1; r += 8) {
      const LaneRec rec = prog[r];
      const long long d = d32 ? (long long)__ldcs(&d32[(long long)r * dld + s])
                              : __ldcs(&d64[(long long)r * dld + s]);
      if (start && (rec.rare & (LREC_CHAIN | LREC_NOP)) && start[(long long)r * sld + s] < 0)
        continue;
      const int l = rec.h & 3;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q == l) lb[q] += d;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[ty][q][tx] = lb[q];
  __syncthreads();
  if (ty < 4 && ty < L && s < S) {
    long long v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v += acc[k][ty][tx];
    if (v) atomicAdd(&lane_busy[(long long)s * L + ty], (unsigned long long)v);
  }
}

cudaError_t launch_lanes_busy(const LaneParams& p, const int* dense32, bool chains,
                              cudaStream_t stream) {
  if (!p.lane_busy || p.S <= 0) return cudaSuccess;
  if (chains && !p.start) return cudaErrorInvalidValue;  // absent members need the starts
  cudaError_t e = cudaMemsetAsync(p.lane_busy, 0, sizeof(long long) * (size_t)p.S * p.L, stream);
  if (e != cudaSuccess) return e;
  const dim3 blk(32, 8), grd((p.S + 31) / 32, (p.n_rec + kBusyRowsPerBlock - 1) / kBusyRowsPerBlock);
  lanes_busy_kernel<<<grd, blk, 0, stream>>>(
      p.prog, p.n_rec, dense32, dense32 ? nullptr : p.dense64, p.dense_ld,
      chains ? p.start : nullptr, p.start_ld, p.S, p.L,
      reinterpret_cast<unsigned long long*>(p.lane_busy));
  note_launch();
  return cudaGetLastError();
}

// 2-D tensor map over the [n_rec][dense_ld] duration matrix, boxes of
// 16 rows x W scenarios (out-of-range scenarios read as zero).
static cudaError_t encode_lanes_tmap(CUtensorMap* tmap, const LaneParams& p, const int* dense32,
                                     int dkind, int W) {
  memset(tmap, 0, sizeof(*tmap));
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
          cudaSuccess || q != cudaDriverEntryPointSuccess)
    return cudaErrorNotSupported;
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const size_t es = dkind == 1 ? 4 : 8;
  const void* base = dkind == 1 ? static_cast<const void*>(dense32)
                                : static_cast<const void*>(p.dense64);
  cuuint64_t dims[2] = {(cuuint64_t)p.S, (cuuint64_t)p.n_rec};
  cuuint64_t strides[1] = {(cuuint64_t)(p.dense_ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)ddsim_lanes::kChunkL};
  cuuint32_t estr[2] = {1, 1};
  if (enc(tmap, dkind == 1 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_INT64, 2,
          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  return cudaSuccess;
}

static_assert(sizeof(ddsim_lanes::RowDur) == sizeof(LaneRowDur), "row duration layout");
static_assert(sizeof(ddsim_lanes::DerivedParams) == sizeof(LaneDerivedParams), "derived layout");
static_assert(sizeof(ddsim_lanes::ScaleStep) == sizeof(ScaleStepDev), "scale step layout");

__global__ void build_rowdur_kernel(const long long* base, const unsigned* group,
                                    const int* ovr_map, int n, LaneRowDur* out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    LaneRowDur x;
    x.base = base[r];
    x.group = group ? group[r] : 0u;
    x.ovr = ovr_map ? ovr_map[r] : -1;
    out[r] = x;
  }
}

cudaError_t launch_build_rowdur(const long long* base, const unsigned* group, const int* ovr_map,
                                int n, LaneRowDur* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  build_rowdur_kernel<<<std::min((n + 255) / 256, 148 * 8), 256, 0, st>>>(base, group, ovr_map, n,
                                                                           out);
  note_launch();
  return cudaGetLastError();
}

// Compose the segment transfer matrices per scenario (one thread each):
// state[k+1] = trans[k] (x) state[k] in (max,+), state[0] = 0, for segments
// k in [k_from, k_to) (the state of k_from is read unless k_from == 0).  All
// values are >= 0 on this path, so 0 is the identity of max; entries < 0 mean
// "no path".  Carries produced in segment k (values read only in the chain
// segment) are evaluated from their coefficients on state[k] into gslots.
template <int LN>
__global__ void __launch_bounds__(128) seg_scan_kernel(const LaneSegParams sg, int S, int k_from,
                                                       int k_to, long long* gslots) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  constexpr int E = LN * LN;
  constexpr int D = LN <= 2 ? 16 : (LN == 3 ? 8 : 4);  // segments loaded together
  const long long sp = sg.s_pad;
  long long st[LN];
#pragma unroll
  for (int j = 0; j < LN; ++j)
    st[j] = k_from == 0 ? 0 : sg.state[((long long)k_from * LN + j) * sp + s];
  // the loads do not depend on the state (only the composition chain does):
  // D segments' coefficients are in flight together
  for (int k0 = k_from; k0 < k_to; k0 += D) {
    int a[D][E];
#pragma unroll
    for (int q = 0; q < D; ++q)
      if (k0 + q < k_to) {
        const int* tk = sg.trans + (long long)(k0 + q) * E * sp + s;
#pragma unroll
        for (int e = 0; e < E; ++e) a[q][e] = tk[(long long)e * sp];
      }
#pragma unroll
    for (int q = 0; q < D; ++q)
      if (k0 + q < k_to) {
        if (sg.carry_ptr != nullptr)
          for (int c = sg.carry_ptr[k0 + q]; c < sg.carry_ptr[k0 + q + 1]; ++c) {
            const int gid = sg.carry_gid[c];
            const int* cf = sg.carry_coef + (long long)gid * LN * sp + s;
            long long v = 0;
#pragma unroll
            for (int i = 0; i < LN; ++i) {
              const int x = cf[(long long)i * sp];
              if (x >= 0) v = max(v, (long long)x + st[i]);
            }
            gslots[(long long)gid * sp + s] = v;
          }
        long long nx[LN];
#pragma unroll
        for (int j = 0; j < LN; ++j) {
          nx[j] = 0;
#pragma unroll
          for (int i = 0; i < LN; ++i)
            if (a[q][j * LN + i] >= 0) nx[j] = max(nx[j], (long long)a[q][j * LN + i] + st[i]);
        }
        long long* out = sg.state + (long long)(k0 + q + 1) * LN * sp + s;
#pragma unroll
        for (int j = 0; j < LN; ++j) {
          st[j] = nx[j];
          out[(long long)j * sp] = nx[j];
        }
      }
  }
}

// The same composition as a warp-parallel prefix scan, one warp per scenario:
// lane q holds segment c0 + q's transfer matrix; a Hillis-Steele inclusive
// scan of (max,+) products (int64 path weights; "none" < 0) gives every
// segment's product P_k = A_k (x) ... (x) A_c0, so all 32 input / output
// states of a chunk follow from the chunk's input state at once.  Exact as the
// sequential form: every transfer keeps a non-negative diagonal (each lane
// head's output depends on its own input), so no row is all "none" and the
// 0-floor of the sequential step never binds.  Few scenarios (configs 1, 2)
// leave the sequential scan latency-bound on the coefficient loads.
template <int LN>
__global__ void __launch_bounds__(128) seg_wscan_kernel(const LaneSegParams sg, int S, int k_from,
                                                        int k_to, long long* gslots) {
  const int s = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int q = threadIdx.x & 31;
  if (s >= S) return;  // whole warps
  constexpr int E = LN * LN;
  const long long sp = sg.s_pad;
  long long st[LN];
#pragma unroll
  for (int j = 0; j < LN; ++j)
    st[j] = k_from == 0 ? 0 : sg.state[((long long)k_from * LN + j) * sp + s];
  for (int c0 = k_from; c0 < k_to; c0 += 32) {
    const int k = c0 + q;
    const bool valid = k < k_to;
    long long P[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      long long v = (e / LN == e % LN) ? 0 : -1;  // identity for lanes past the end
      if (valid) {
        const int x = sg.trans[((long long)k * E + e) * sp + s];
        v = x >= 0 ? (long long)x : -1;
      }
      P[e] = v;
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      long long Q[E];
#pragma unroll
      for (int e = 0; e < E; ++e) Q[e] = __shfl_up_sync(0xffffffffu, P[e], off);
      if (q >= off) {
        long long R[E];
#pragma unroll
        for (int j = 0; j < LN; ++j)
#pragma unroll
          for (int i = 0; i < LN; ++i) {
            long long m = -1;
#pragma unroll
            for (int t = 0; t < LN; ++t) {
              const long long a = P[j * LN + t], b = Q[t * LN + i];
              if (a >= 0 && b >= 0) m = max(m, a + b);
            }
            R[j * LN + i] = m;
          }
#pragma unroll
        for (int e = 0; e < E; ++e) P[e] = R[e];
      }
    }
    // input state of segment k = P_{k-1} (x) st (lane 0: st itself)
    long long Pm[E];
#pragma unroll
    for (int e = 0; e < E; ++e) Pm[e] = __shfl_up_sync(0xffffffffu, P[e], 1);
    long long in[LN], out[LN];
#pragma unroll
    for (int j = 0; j < LN; ++j) {
      long long vi = 0, vo = 0;
#pragma unroll
      for (int i = 0; i < LN; ++i) {
        if (Pm[j * LN + i] >= 0) vi = max(vi, Pm[j * LN + i] + st[i]);
        if (P[j * LN + i] >= 0) vo = max(vo, P[j * LN + i] + st[i]);
      }
      in[j] = q == 0 ? st[j] : vi;
      out[j] = vo;
    }
    if (valid) {
      if (sg.carry_ptr != nullptr)
        for (int c = sg.carry_ptr[k]; c < sg.carry_ptr[k + 1]; ++c) {
          const int gid = sg.carry_gid[c];
          const int* cf = sg.carry_coef + (long long)gid * LN * sp + s;
          long long v = 0;
#pragma unroll
          for (int i = 0; i < LN; ++i) {
            const int x = cf[(long long)i * sp];
            if (x >= 0) v = max(v, (long long)x + in[i]);
          }
          gslots[(long long)gid * sp + s] = v;
        }
      long long* o = sg.state + (long long)(k + 1) * LN * sp + s;
#pragma unroll
      for (int j = 0; j < LN; ++j) o[(long long)j * sp] = out[j];
    }
    // the next chunk starts from the last segment's output
    const int last = min(31, k_to - 1 - c0);
#pragma unroll
    for (int j = 0; j < LN; ++j) st[j] = __shfl_sync(0xffffffffu, out[j], last);
  }
}

// (max,+) product of two LN x LN matrices, newer (x) older; "none" < 0.
template <int LN>
__device__ __forceinline__ void mp_mul(const long long* A, const long long* B, long long* R) {
#pragma unroll
  for (int j = 0; j < LN; ++j)
#pragma unroll
    for (int i = 0; i < LN; ++i) {
      long long m = -1;
#pragma unroll
      for (int t = 0; t < LN; ++t) {
        const long long a = A[j * LN + t], b = B[t * LN + i];
        if (a >= 0 && b >= 0) m = max(m, a + b);
      }
      R[j * LN + i] = m;
    }
}

// Very few scenarios (config 1: S = 2, ~100 segments): one CTA of 32 warps
// per scenario, warp w scans chunk w of 32 segments, warp 0 scans the 32
// chunk products, so the whole composition takes two shuffle scans instead of
// one per chunk in sequence.
constexpr int kBscanWarps = 16;
template <int LN>
__global__ void __launch_bounds__(kBscanWarps * 32) seg_bscan_kernel(const LaneSegParams sg, int S, int k_from,
                                                         int k_to, long long* gslots) {
  constexpr int E = LN * LN;
  __shared__ long long chunk_prod[kBscanWarps][E];
  __shared__ long long st_sh[LN];
  const int s = blockIdx.x;
  const int q = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long sp = sg.s_pad;
  if (threadIdx.x < LN)
    st_sh[threadIdx.x] = k_from == 0 ? 0 : sg.state[((long long)k_from * LN + threadIdx.x) * sp + s];
  for (int base = k_from; base < k_to; base += kBscanWarps * 32) {
    __syncthreads();  // st_sh of this round
    const int k = base + w * 32 + q;
    const bool valid = k < k_to;
    long long P[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      long long v = (e / LN == e % LN) ? 0 : -1;
      if (valid) {
        const int x = sg.trans[((long long)k * E + e) * sp + s];
        v = x >= 0 ? (long long)x : -1;
      }
      P[e] = v;
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      long long Q[E], R[E];
#pragma unroll
      for (int e = 0; e < E; ++e) Q[e] = __shfl_up_sync(0xffffffffu, P[e], off);
      if (q >= off) {
        mp_mul<LN>(P, Q, R);
#pragma unroll
        for (int e = 0; e < E; ++e) P[e] = R[e];
      }
    }
    if (q == 31)
#pragma unroll
      for (int e = 0; e < E; ++e) chunk_prod[w][e] = P[e];
    __syncthreads();
    if (w == 0) {  // exclusive prefix over the chunk products
      long long C[E];
#pragma unroll
      for (int e = 0; e < E; ++e)
        C[e] = q < kBscanWarps ? chunk_prod[q][e] : ((e / LN == e % LN) ? 0 : -1);
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        long long Q[E], R[E];
#pragma unroll
        for (int e = 0; e < E; ++e) Q[e] = __shfl_up_sync(0xffffffffu, C[e], off);
        if (q >= off) {
          mp_mul<LN>(C, Q, R);
#pragma unroll
          for (int e = 0; e < E; ++e) C[e] = R[e];
        }
      }
      long long X[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        X[e] = __shfl_up_sync(0xffffffffu, C[e], 1);
        if (q == 0) X[e] = (e / LN == e % LN) ? 0 : -1;
      }
      __syncwarp();
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (q < kBscanWarps) chunk_prod[q][e] = X[e];  // now: product of chunks < q
    }
    __syncthreads();
    long long cin[LN];  // the chunk's input state
#pragma unroll
    for (int j = 0; j < LN; ++j) {
      long long v = 0;
#pragma unroll
      for (int i = 0; i < LN; ++i) {
        const long long c = chunk_prod[w][j * LN + i];
        if (c >= 0) v = max(v, c + st_sh[i]);
      }
      cin[j] = v;
    }
    long long Pm[E];
#pragma unroll
    for (int e = 0; e < E; ++e) Pm[e] = __shfl_up_sync(0xffffffffu, P[e], 1);
    long long in[LN], out[LN];
#pragma unroll
    for (int j = 0; j < LN; ++j) {
      long long vi = 0, vo = 0;
#pragma unroll
      for (int i = 0; i < LN; ++i) {
        if (Pm[j * LN + i] >= 0) vi = max(vi, Pm[j * LN + i] + cin[i]);
        if (P[j * LN + i] >= 0) vo = max(vo, P[j * LN + i] + cin[i]);
      }
      in[j] = q == 0 ? cin[j] : vi;
      out[j] = vo;
    }
    if (valid) {
      if (sg.carry_ptr != nullptr)
        for (int c = sg.carry_ptr[k]; c < sg.carry_ptr[k + 1]; ++c) {
          const int gid = sg.carry_gid[c];
          const int* cf = sg.carry_coef + (long long)gid * LN * sp + s;
          long long v = 0;
#pragma unroll
          for (int i = 0; i < LN; ++i) {
            const int x = cf[(long long)i * sp];
            if (x >= 0) v = max(v, (long long)x + in[i]);
          }
          gslots[(long long)gid * sp + s] = v;
        }
      long long* o = sg.state + (long long)(k + 1) * LN * sp + s;
#pragma unroll
      for (int j = 0; j < LN; ++j) o[(long long)j * sp] = out[j];
    }
    __syncthreads();  // every warp has read st_sh
    if (k == min(k_to, base + kBscanWarps * 32) - 1)  // the round's last segment carries the state on
#pragma unroll
      for (int j = 0; j < LN; ++j) st_sh[j] = out[j];
  }
}

static cudaError_t launch_seg_scan(const LaneSegParams& sg, int S, int k_from, int k_to,
                                   long long* gslots, cudaStream_t stream) {
  if (k_to <= k_from) return cudaSuccess;
  if (S <= 16 && k_to - k_from > 32 && getenv("DDSIM_SEG_SEQSCAN") == nullptr &&
      getenv("DDSIM_SEG_WSCAN") == nullptr) {
    switch (sg.LN) {
      case 1: seg_bscan_kernel<1><<<S, kBscanWarps * 32, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
      case 2: seg_bscan_kernel<2><<<S, kBscanWarps * 32, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
      case 3: seg_bscan_kernel<3><<<S, kBscanWarps * 32, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
      default: seg_bscan_kernel<4><<<S, kBscanWarps * 32, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
    }
    note_launch();
    return cudaGetLastError();
  }
  // warp-parallel scan unless the scenarios alone fill the GPU
  if (S < 4096 && getenv("DDSIM_SEG_SEQSCAN") == nullptr) {
    const int gw = (S * 32 + 127) / 128;
    switch (sg.LN) {
      case 1: seg_wscan_kernel<1><<<gw, 128, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
      case 2: seg_wscan_kernel<2><<<gw, 128, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
      case 3: seg_wscan_kernel<3><<<gw, 128, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
      default: seg_wscan_kernel<4><<<gw, 128, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
    }
    note_launch();
    return cudaGetLastError();
  }
  const int gs = (S + 127) / 128;
  switch (sg.LN) {
    case 1: seg_scan_kernel<1><<<gs, 128, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
    case 2: seg_scan_kernel<2><<<gs, 128, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
    case 3: seg_scan_kernel<3><<<gs, 128, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
    default: seg_scan_kernel<4><<<gs, 128, 0, stream>>>(sg, S, k_from, k_to, gslots); break;
  }
  note_launch();
  return cudaGetLastError();
}

// Segment-parallel lanes path (small S): transfer, scan, replay.  The caller
// provides the scratch (trans / state / device cuts in sg) and zeroes makespan
// and lane busy; cudaErrorNotSupported when the JIT is unavailable.
cudaError_t launch_maxplus_lanes_seg(const LaneParams& p, const LaneChainParams* cp,
                                     const int* dense32, int dkind, const std::vector<int>& codes,
                                     const LaneSegParams& sg, int BD, cudaStream_t stream,
                                     const LaneDerivedParams* dp) {
  static_assert(sizeof(LaneSegParams) == sizeof(ddsim_lanes::SegParams), "seg params layout");
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  cudaError_t e = dkind == 0 ? cudaSuccess : encode_lanes_tmap(&tmap, p, dense32, dkind, BD);
  if (e != cudaSuccess) return e;
  const int gx = (p.S + BD - 1) / BD;
  // must match the depth seg_source compiles into the kernels (jit.cu)
  int stages = dkind != 0 ? 2 : ddsim_lanes::kStagesL;
  if (const char* e = getenv("DDSIM_SEG_STAGES")) stages = std::max(2, atoi(e));
  const size_t es = dkind == 1 ? 4 : 8;
  const size_t base = 128 + (size_t)stages * ddsim_lanes::kChunkL * sizeof(ddsim_lanes::Rec) +
                      (dkind == 0 ? (size_t)stages * ddsim_lanes::kChunkL * sizeof(ddsim_lanes::RowDur)
                                  : (size_t)stages * ddsim_lanes::kChunkL * BD * es);
  const size_t smem_t = base + (size_t)p.ksm * BD * 16, smem_r = base + (size_t)p.ksm * BD * 8;
  if (sg.ticket != nullptr)  // fused single pass (transfer smem >= replay smem)
    return launch_lanes_seg_jit(2, p, cp, &tmap, dkind, sg.LN, codes, &sg, gx * sg.K, 1, BD,
                                smem_t, stream, dp);
  // two scenarios per thread (one record decode for both): the transfer
  // always (instruction-bound), the replay when S is even and the start rows
  // take 16-byte stores
  const bool two = 2 * BD <= 256 && getenv("DDSIM_SEG_T1") == nullptr;
  const bool vec_ok = p.start == nullptr ||
                      (p.start_ld % 2 == 0 && reinterpret_cast<uintptr_t>(p.start) % 16 == 0);
  const bool two_r = two && p.S % 2 == 0 && vec_ok && getenv("DDSIM_SEG_R1") == nullptr;
  CUtensorMap tmap2;
  memset(&tmap2, 0, sizeof(tmap2));
  if (two && dkind != 0) {
    e = encode_lanes_tmap(&tmap2, p, dense32, dkind, 2 * BD);
    if (e != cudaSuccess) return e;
  }
  const size_t base2 = 128 + (size_t)stages * ddsim_lanes::kChunkL * sizeof(ddsim_lanes::Rec) +
                       (dkind == 0 ? (size_t)stages * ddsim_lanes::kChunkL * sizeof(ddsim_lanes::RowDur)
                                   : (size_t)stages * ddsim_lanes::kChunkL * 2 * BD * es);
  const int gx2 = (p.S + 2 * BD - 1) / (2 * BD);
  const size_t smem_r2 = base2 + (size_t)p.ksm * BD * 16;
  auto replay = [&](const LaneSegParams& q, int gy) {
    if (two_r)
      return launch_lanes_seg_jit(4, p, cp, &tmap2, dkind, q.LN, codes, &q, gx2, gy, BD, smem_r2,
                                  stream, dp);
    return launch_lanes_seg_jit(0, p, cp, &tmap, dkind, q.LN, codes, &q, gx, gy, BD, smem_r,
                                stream, dp);
  };
  if (sg.K > 1) {
    if (two) {
      const size_t smem_t2 = base2 + (size_t)p.ksm * BD * 32;
      e = launch_lanes_seg_jit(3, p, cp, &tmap2, dkind, sg.LN, codes, &sg, gx2, sg.K - 1, BD,
                               smem_t2, stream, dp);
    } else {
      e = launch_lanes_seg_jit(1, p, cp, &tmap, dkind, sg.LN, codes, &sg, gx, sg.K - 1, BD, smem_t,
                               stream, dp);
    }
    if (e != cudaSuccess) return e;
  }
  if (sg.kc < 0) {
    if ((e = launch_seg_scan(sg, p.S, 0, sg.K - 1, p.gslots, stream)) != cudaSuccess) return e;
  } else {
    // scan up to the chain segment (carries included), replay the chain
    // segment (it exports its output lane heads), scan the rest
    if ((e = launch_seg_scan(sg, p.S, 0, sg.kc, p.gslots, stream)) != cudaSuccess) return e;
    LaneSegParams one = sg;
    one.replay_only = sg.kc;
    if ((e = replay(one, 1)) != cudaSuccess) return e;
    e = launch_seg_scan(sg, p.S, sg.kc + 1, sg.K - 1, p.gslots, stream);
    if (e != cudaSuccess) return e;
  }
  return replay(sg, sg.K);
}

cudaError_t launch_maxplus_lanes(const LaneParams& p, const LaneChainParams* cp, const int* dense32,
                                 int dkind,
                                 const std::vector<int>* codes, cudaStream_t stream,
                                 const LaneDerivedParams* dp) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const bool vec_ok = p.start == nullptr ||
                      (p.start_ld % 2 == 0 && reinterpret_cast<uintptr_t>(p.start) % 16 == 0);
  const int V = maxplus_lanes_vec(p.S, dkind, vec_ok);
  const int BD = maxplus_lanes_block_dim(p.S, nsm, dkind, vec_ok);
  const int W = BD * V;
  const int grid = (p.S + W - 1) / W;
  if ((long long)grid * W > p.s_pad) return cudaErrorInvalidValue;
  const size_t smem = lanes_smem(dkind, BD, V, p.ksm);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (dkind != 0) {
    const cudaError_t te = encode_lanes_tmap(&tmap, p, dense32, dkind, W);
    if (te != cudaSuccess) return te;
  }
  // per-graph specialised dispatch first (NVRTC); the static kernel otherwise
  // (derived durations exist only as JIT kernels)
  if (codes != nullptr) {
    const cudaError_t e = launch_maxplus_lanes_jit(p, cp, dense32, &tmap, dkind, V, *codes, grid,
                                                   BD, smem, stream, dp);
    if (e == cudaSuccess) return cudaGetLastError();
  }
  if (dkind == 0) return cudaErrorNotSupported;
  // the kernels' parameter types mirror the host structs byte for byte
  static_assert(sizeof(ddsim_lanes::Tmap) == sizeof(CUtensorMap), "tensor map layout");
  static_assert(sizeof(ddsim_lanes::Params) == sizeof(LaneParams), "lane params layout");
  ddsim_lanes::Tmap tm;
  ddsim_lanes::Params pp;
  memcpy(&tm, &tmap, sizeof(tm));
  memcpy(&pp, &p, sizeof(pp));
  cudaError_t err;
#define LAUNCH_L(DK, VV)                                                                      \
  if (cp != nullptr) {                                                                        \
    err = cudaFuncSetAttribute(maxplus_lanes_chain_kernel<DK, VV>,                            \
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
    if (err != cudaSuccess) return err;                                                       \
    maxplus_lanes_chain_kernel<DK, VV><<<grid, BD, smem, stream>>>(                           \
        tm, pp, *reinterpret_cast<const ddsim_lanes::ChainParams*>(cp));                       \
  } else {                                                                                    \
    err = cudaFuncSetAttribute(maxplus_lanes_kernel<DK, VV>,                                  \
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
    if (err != cudaSuccess) return err;                                                       \
    maxplus_lanes_kernel<DK, VV><<<grid, BD, smem, stream>>>(tm, pp);                         \
  }
  if (dkind == 1 && V == 2) {
    LAUNCH_L(1, 2)
  } else if (dkind == 1) {
    LAUNCH_L(1, 1)
  } else if (V == 2) {
    LAUNCH_L(2, 2)
  } else {
    LAUNCH_L(2, 1)
  }
#undef LAUNCH_L
  note_launch();
  return cudaGetLastError();
}

}  // namespace ddsim
