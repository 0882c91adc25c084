// maxplus_sim: batched simulate() for lane-chained graphs.
//
// Reference: kernsim.sim.simulate (pkg/src/kernsim/sim.py:89-142).  When every
// task sits in its lane's lane_order chain, lane exclusivity never binds and
// Alg. 1 reduces exactly to the max-plus recurrence of
// longest_path_makespan (pkg/src/kernsim/synthetic.py:35-48):
//     start(v) = max(ready(v), max_{u->v} start(u) + dur(u) + gap(u))
//     makespan = max_v start(v) + dur(v)      (gap excluded, sim.py:125)
//     lane_busy[lane] = sum dur               (sim.py:124)
//
// Shape: scenario-parallel, node-sequential.  One thread owns one scenario and
// walks the compiled program (frozen topological order) with no inter-thread
// synchronisation except a CTA barrier per chunk.  Program records (64 B) are
// staged chunk by chunk into shared memory with cp.async.bulk; for dense
// per-scenario durations the [rows x scenarios] int32 tile of the chunk is
// staged by a 2D TMA (cp.async.bulk.tensor) on the same mbarrier.  Values that
// later tasks read (rel = start+dur+gap of a predecessor) live in compiled
// "slots": shared memory [slot][thread] (bank-conflict free) or a spill
// array in global memory for long-lived values.
#include "ddsim_internal.h"

#include <climits>
#include <cudaTypedefs.h>
#include <algorithm>

namespace ddsim {

constexpr int kChunk = 16;  // records per stage
constexpr int kStages = 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_tile_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// round_half_up(d * num / den) with d possibly negative (transform.py:174-175).
__device__ __forceinline__ long long scale_half_up(long long d, long long num, long long den) {
  const bool neg = d < 0;
  const unsigned long long a = neg ? (unsigned long long)(-d) : (unsigned long long)d;
  const unsigned long long un = (unsigned long long)num, ud = (unsigned long long)den;
  unsigned long long q;
  if (a < (1ull << 40) && un < (1ull << 21) && ud < (1ull << 40)) {
    q = (2ull * a * un + ud) / (2ull * ud);
  } else {
    const unsigned __int128 x = (unsigned __int128)a * un * 2u + ud;
    q = (unsigned long long)(x / ((unsigned __int128)ud * 2u));
  }
  return neg ? -(long long)q : (long long)q;
}

struct ThreadCtx {
  long long* sm_slots;  // [ksm][BD]
  long long* lb;        // [L][BD]
  int tid, BD, s, sc;   // sc: clamped scenario (valid for reads)
  bool act;
  int e0, e1;           // this scenario's scale steps
};

__device__ __forceinline__ long long slot_get(const MaxplusParams& p, const ThreadCtx& t, int k) {
  if (k < p.ksm) return t.sm_slots[k * t.BD + t.tid];
  return p.gslots[(long long)(k - p.ksm) * p.s_pad + t.s];
}
__device__ __forceinline__ void slot_put(const MaxplusParams& p, const ThreadCtx& t, int k,
                                         long long v) {
  if (k < p.ksm)
    t.sm_slots[k * t.BD + t.tid] = v;
  else
    p.gslots[(long long)(k - p.ksm) * p.s_pad + t.s] = v;
}

// A step with num == 0 (KS_STEP_REMOVE) removes the matched tasks
// (remove_task, transform.py:249-265): *removed is set and d is meaningless.
__device__ __forceinline__ long long derive_duration(const MaxplusParams& p, const ThreadCtx& t,
                                                     long long dur, int ovr_row, unsigned group,
                                                     bool& removed) {
  long long d = dur;
  removed = false;
  if (ovr_row >= 0) d = p.ovr[(long long)ovr_row * p.S + t.sc];
  if (group != 0u) {
    for (int e = t.e0; e < t.e1; ++e) {
      const ScaleStepDev st = p.scale[e];
      if (group >= (unsigned)st.lo && group <= (unsigned)st.hi) {
        if (st.num == 0)
          removed = true;
        else
          d = scale_half_up(d, st.num, st.den);
      }
    }
  }
  return d;
}

// max over the predecessors' values (no ready time; LLONG_MIN if none)
__device__ __forceinline__ long long pred_max(const MaxplusParams& p, const ThreadCtx& t,
                                              const NodeRec& r) {
  long long st = LLONG_MIN;
  if (r.pred0 >= 0) st = max(st, slot_get(p, t, r.pred0));
  if (r.pred1 >= 0) st = max(st, slot_get(p, t, r.pred1));
  for (int k = 0; k < r.nextra; ++k) st = max(st, slot_get(p, t, __ldg(&p.extra[r.extra_off + k])));
  return st;
}

// Permutable chain (inserted-task table row): members dispatched in this
// scenario's order, each after the previous one on the lane (sequenced insert,
// transform.py:204-222); an absent chain drops its tasks and edges.
__device__ __forceinline__ void run_chain(const MaxplusParams& p, ThreadCtx& t, int c, long long& ms) {
  const ChainDesc ch = p.chains[c];
  const bool pres = p.present == nullptr || p.present[(long long)t.sc * p.n_chains + c] != 0;
  if (pres) {
    long long prev = ch.head_slot >= 0 ? slot_get(p, t, ch.head_slot) : LLONG_MIN;
    for (int k = 0; k < ch.B; ++k) {
      const int m = p.perm ? (int)p.perm[(long long)t.sc * p.perm_ld + ch.perm_off + k] : k;
      const NodeRec mr = p.members[ch.member_off + m];
      const long long pm = max(pred_max(p, t, mr), prev);
      bool rm;
      const long long d = derive_duration(p, t, mr.dur, mr.ovr_row, mr.group, rm);
      if (rm) {  // spliced out: its parents feed its children and lane successor
        if (t.act && p.start) __stcs(&p.start[(long long)mr.row * p.start_ld + t.s], -1ll);
        prev = pm;
        if (mr.out_slot >= 0) slot_put(p, t, mr.out_slot, prev);
        continue;
      }
      const long long st = max(pm, mr.ready);
      if (t.act && p.start) __stcs(&p.start[(long long)mr.row * p.start_ld + t.s], st);
      const long long fin = st + d;
      prev = fin + mr.gap;
      if (mr.out_slot >= 0) slot_put(p, t, mr.out_slot, prev);
      ms = max(ms, fin);
      t.lb[mr.lane * t.BD + t.tid] += d;
    }
    if (ch.tail_slot >= 0) slot_put(p, t, ch.tail_slot, prev);
  } else {
    for (int k = 0; k < ch.B; ++k) {
      const NodeRec mr = p.members[ch.member_off + k];
      if (t.act && p.start) __stcs(&p.start[(long long)mr.row * p.start_ld + t.s], -1ll);
      if (mr.out_slot >= 0) slot_put(p, t, mr.out_slot, LLONG_MIN);
    }
    if (ch.tail_slot >= 0) slot_put(p, t, ch.tail_slot, LLONG_MIN);
  }
}

// DMODE: 0 = derived durations (base/override/scale), 1 = dense int32 via TMA
// tiles, 2 = dense int64 via direct loads.
template <int DMODE>
__global__ void __launch_bounds__(256) maxplus_kernel(const __grid_constant__ CUtensorMap tmap,
                                                      const MaxplusParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  if (p.run_if != nullptr && *((volatile const int*)p.run_if) == 0) return;
  const int BD = blockDim.x;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem);
  NodeRec* pstage = reinterpret_cast<NodeRec*>(smem + 128);
  unsigned char* cur = smem + 128 + kStages * kChunk * sizeof(NodeRec);
  int* tstage = reinterpret_cast<int*>(cur);
  if (DMODE == 1) cur += (size_t)kStages * kChunk * BD * sizeof(int);
  ThreadCtx t;
  t.sm_slots = reinterpret_cast<long long*>(cur);
  cur += (size_t)p.ksm * BD * sizeof(long long);
  t.lb = reinterpret_cast<long long*>(cur);
  t.tid = threadIdx.x;
  t.BD = BD;
  const int s0 = blockIdx.x * BD;
  t.s = s0 + t.tid;
  t.act = t.s < p.S;
  t.sc = t.act ? t.s : 0;
  t.e0 = t.e1 = 0;
  if (p.scale_ptr) {
    t.e0 = p.scale_ptr[t.sc];
    t.e1 = t.act ? p.scale_ptr[t.sc + 1] : t.e0;
  }
  for (int l = 0; l < p.L; ++l) t.lb[l * BD + t.tid] = 0;

  const int nchunks = (p.n_rec + kChunk - 1) / kChunk;
  const unsigned tile_bytes = DMODE == 1 ? (unsigned)(kChunk * BD * sizeof(int)) : 0u;
  auto issue = [&](int c) {
    const int st = c % kStages;
    const int nrec = min(kChunk, p.n_rec - c * kChunk);
    const unsigned pb = (unsigned)(nrec * sizeof(NodeRec));
    mbar_expect_tx(&bars[st], pb + tile_bytes);
    bulk_g2s(pstage + st * kChunk, p.prog + (long long)c * kChunk, pb, &bars[st]);
    if (DMODE == 1) tma_tile_2d(tstage + st * kChunk * BD, &tmap, s0, c * kChunk, &bars[st]);
  };
  if (t.tid == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (t.tid == 0)
    for (int c = 0; c < min(kStages, nchunks); ++c) issue(c);

  long long ms = 0;
  for (int c = 0; c < nchunks; ++c) {
    const int st = c % kStages;
    mbar_wait(&bars[st], (unsigned)((c / kStages) & 1));
    const NodeRec* R = pstage + st * kChunk;
    const int* T = tstage + st * kChunk * BD;
    const int nrec = min(kChunk, p.n_rec - c * kChunk);
#pragma unroll 1
    for (int j = 0; j < nrec; ++j) {
      const int kind = R[j].kind;
      if (kind != 0) {
        run_chain(p, t, R[j].row, ms);
        continue;
      }
      const NodeRec r = R[j];
      const long long pm = pred_max(p, t, r);
      long long d;
      if (DMODE == 1) {
        d = (long long)T[j * BD + t.tid];
      } else if (DMODE == 2) {
        d = p.dense64[(long long)r.row * p.dense_ld + t.sc];
      } else {
        bool rm;
        d = derive_duration(p, t, r.dur, r.ovr_row, r.group, rm);
        if (rm) {  // removed (remove_task): start -1, value passes through
          if (t.act && p.start) __stcs(&p.start[(long long)r.row * p.start_ld + t.s], -1ll);
          if (r.out_slot >= 0) slot_put(p, t, r.out_slot, pm);
          continue;
        }
      }
      const long long stv = max(pm, r.ready);
      if (t.act && p.start) __stcs(&p.start[(long long)r.row * p.start_ld + t.s], stv);
      const long long fin = stv + d;
      if (r.out_slot >= 0) slot_put(p, t, r.out_slot, fin + r.gap);
      ms = max(ms, fin);
      t.lb[r.lane * BD + t.tid] += d;
    }
    __syncthreads();
    if (t.tid == 0 && c + kStages < nchunks) issue(c + kStages);
  }
  if (t.act) {
    if (p.makespan) p.makespan[t.s] = ms;
    if (p.lane_busy)
      for (int l = 0; l < p.L; ++l) p.lane_busy[(long long)t.s * p.L + l] = t.lb[l * BD + t.tid];
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static size_t maxplus_smem(int dmode, int BD, int ksm, int L) {
  size_t b = 128 + (size_t)kStages * kChunk * sizeof(NodeRec);
  if (dmode == 1) b += (size_t)kStages * kChunk * BD * sizeof(int);
  b += (size_t)ksm * BD * sizeof(long long);
  b += (size_t)L * BD * sizeof(long long);
  return b;
}

int maxplus_block_dim(int S, int dmode, int num_sms) {
  if (dmode == 0) return 32;  // latency-bound: spread scenarios over SMs
  long long per = (S + 2LL * num_sms - 1) / (2LL * num_sms);
  int bd = (int)(((per + 31) / 32) * 32);
  return bd < 32 ? 32 : (bd > 256 ? 256 : bd);
}

cudaError_t launch_maxplus(const MaxplusParams& p, const int* dense32, cudaStream_t stream) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int dmode = p.dense_kind;  // 0, 1, 2
  const int BD = maxplus_block_dim(p.S, dmode, nsm);
  const int grid = (p.S + BD - 1) / BD;
  if ((long long)grid * BD > p.s_pad) return cudaErrorInvalidValue;
  const size_t smem = maxplus_smem(dmode, BD, p.ksm, p.L);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  cudaError_t err;
  if (dmode == 1) {
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {(cuuint64_t)p.S, (cuuint64_t)p.n_rec};
    cuuint64_t strides[1] = {(cuuint64_t)(p.dense_ld * sizeof(int))};
    cuuint32_t box[2] = {(cuuint32_t)BD, (cuuint32_t)kChunk};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int*>(dense32), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  switch (dmode) {
    case 0:
      err = cudaFuncSetAttribute(maxplus_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
      if (err != cudaSuccess) return err;
      maxplus_kernel<0><<<grid, BD, smem, stream>>>(tmap, p);
      break;
    case 1:
      err = cudaFuncSetAttribute(maxplus_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
      if (err != cudaSuccess) return err;
      maxplus_kernel<1><<<grid, BD, smem, stream>>>(tmap, p);
      break;
    default:
      err = cudaFuncSetAttribute(maxplus_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
      if (err != cudaSuccess) return err;
      maxplus_kernel<2><<<grid, BD, smem, stream>>>(tmap, p);
      break;
  }
  note_launch();
  return cudaGetLastError();
}

__global__ void fill_i64_kernel(long long* p, long long v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

cudaError_t launch_fill_i64(long long* p, long long v, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  fill_i64_kernel<<<grid, 256, 0, s>>>(p, v, n);
  note_launch();
  return cudaGetLastError();
}

__global__ void fill_i32_kernel(int* p, int v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

cudaError_t launch_fill_i32(int* p, int v, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  fill_i32_kernel<<<grid, 256, 0, s>>>(p, v, n);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ddsim

namespace ddsim {

// Derived durations -> dense int64 [rows][ld]: d = base[r], the scenario's
// override if the row has one, then its scale steps in order (sequential
// half-up, transform.py:174-183).  One thread per (row, scenario) element.
// One block row of 64 frozen rows x (blockDim.x scenarios) per block: the
// scenario index is the thread's column (no 64-bit division per element), the
// scale program bounds are read once per thread, stores are coalesced rows.
constexpr int kExpandRows = 64;
constexpr int kExpandRegSteps = 1;  // further steps are read from L1
// out of line: the divisions hold no registers in the row loop
__device__ __noinline__ long long expand_scale(long long d, long long num, long long den) {
  return scale_half_up(d, num, den);
}
template <class OutT, bool STREAM, bool OVR>
__global__ void __launch_bounds__(256, 4) expand_durations_kernel(
    const long long* __restrict__ base, const unsigned* __restrict__ group,
    const int* __restrict__ ovr_map, const long long* __restrict__ ovr,
    const int* __restrict__ scale_ptr, const ScaleStepDev* __restrict__ scale, int rows, int S,
    long long ld, OutT* __restrict__ out) {
  // the block's rows (base, group, override row) staged in shared memory by
  // one coalesced load, so a thread's row loop waits on no global load
  __shared__ long long sb[kExpandRows];
  __shared__ unsigned sgp[kExpandRows];
  __shared__ int so[kExpandRows];
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = s < S;
  const int e0 = act && scale_ptr ? scale_ptr[s] : 0, e1 = act && scale_ptr ? scale_ptr[s + 1] : 0;
  // the scenario's first steps in registers (a Shrink sweep has one or two)
  ScaleStepDev rs[kExpandRegSteps];
#pragma unroll
  for (int k = 0; k < kExpandRegSteps; ++k) {
    rs[k] = ScaleStepDev{1, 0, 0, 1};  // empty group range
    if (e0 + k < e1) rs[k] = scale[e0 + k];
  }
  // one range test per row before the per-step tests (most rows are outside
  // every step of a Shrink sweep scenario); group 0 (no selector) never scales
  unsigned glo = 0xffffffffu, ghi = 0u;
#pragma unroll
  for (int k = 0; k < kExpandRegSteps; ++k)
    if (e0 + k < e1) {
      glo = min(glo, (unsigned)max(rs[k].lo, 1));
      ghi = max(ghi, (unsigned)max(rs[k].hi, 0));
    }
  for (int e = e0 + kExpandRegSteps; e < e1; ++e) {
    glo = min(glo, (unsigned)max(scale[e].lo, 1));
    ghi = max(ghi, (unsigned)max(scale[e].hi, 0));
  }
  const unsigned gspan = ghi >= glo ? ghi - glo : 0u;
  const bool any = ghi >= glo;
  for (int rb = blockIdx.y * kExpandRows; rb < rows; rb += gridDim.y * kExpandRows) {
    const int nr = min(rows - rb, kExpandRows);
    __syncthreads();  // the previous block row is consumed
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
      const int r = rb + i;
      sb[i] = base[r];
      sgp[i] = group ? group[r] : 0u;
      so[i] = ovr_map ? ovr_map[r] : -1;
    }
    __syncthreads();
    if (!act) continue;
    OutT* op = out + (long long)rb * ld + s;
#pragma unroll 4
    for (int j = 0; j < nr; ++j, op += ld) {
      long long d = sb[j];
      if (OVR) {
        const int o = so[j];
        if (o >= 0) d = ovr[(long long)o * S + s];
      }
      const unsigned g = sgp[j];
      if (any && g - glo <= gspan) {
#pragma unroll
        for (int k = 0; k < kExpandRegSteps; ++k)
          // num == 0: a removal step (the row's start reads -1; d is unused)
          if (g >= (unsigned)rs[k].lo && g <= (unsigned)rs[k].hi && rs[k].num != 0)
            d = expand_scale(d, rs[k].num, rs[k].den);
        for (int e = e0 + kExpandRegSteps; e < e1; ++e) {
          const ScaleStepDev st = scale[e];
          if (g >= (unsigned)st.lo && g <= (unsigned)st.hi && st.num != 0)
            d = expand_scale(d, st.num, st.den);
        }
      }
      // int32: the caller bounded every value (expand_fits_int32).  An
      // L2-sized matrix stays cached for the passes that read it back.
      if (STREAM)
        __stcs(op, (OutT)d);
      else
        *op = (OutT)d;
    }
  }
}

// A few scenarios (config 1: S = 2): one thread per element instead, so the
// rows spread over the whole GPU (the row-block form left 10k rows x 2
// scenarios to 157 mostly idle warps: 19 us).
template <class OutT>
__global__ void __launch_bounds__(256) expand_small_kernel(
    const long long* __restrict__ base, const unsigned* __restrict__ group,
    const int* __restrict__ ovr_map, const long long* __restrict__ ovr,
    const int* __restrict__ scale_ptr, const ScaleStepDev* __restrict__ scale, int rows, int S,
    long long ld, OutT* __restrict__ out) {
  const long long total = (long long)rows * S;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / S), s = (int)(e - (long long)r * S);
    long long d = base[r];
    if (ovr_map) {
      const int o = ovr_map[r];
      if (o >= 0) d = ovr[(long long)o * S + s];
    }
    const unsigned g = group ? group[r] : 0u;
    if (g != 0u && scale_ptr)
      for (int k = scale_ptr[s]; k < scale_ptr[s + 1]; ++k) {
        const ScaleStepDev st = scale[k];
        if (g >= (unsigned)st.lo && g <= (unsigned)st.hi && st.num != 0)
          d = expand_scale(d, st.num, st.den);
      }
    out[(long long)r * ld + s] = (OutT)d;
  }
}

template <class OutT>
static cudaError_t launch_expand(const long long* base, const unsigned* group, const int* ovr_map,
                                 const long long* ovr, const int* scale_ptr,
                                 const ScaleStepDev* scale, int rows, int S, long long ld,
                                 OutT* out, cudaStream_t st) {
  if ((long long)rows * S == 0) return cudaSuccess;
  if (S < 32) {
    const long long blocks = ((long long)rows * S + 255) / 256;
    expand_small_kernel<OutT><<<(int)std::min<long long>(blocks, 148LL * 16), 256, 0, st>>>(
        base, group, ovr_map, ovr, scale_ptr, scale, rows, S, ld, out);
    note_launch();
    return cudaGetLastError();
  }
  const int bx = S >= 256 ? 256 : ((S + 31) / 32) * 32;
  const dim3 grid((S + bx - 1) / bx, std::min((rows + kExpandRows - 1) / kExpandRows, 65535));
  const bool big = (long long)rows * ld * (long long)sizeof(OutT) > (64LL << 20);
#define EXPAND_K(ST, OV)                                                                        \
  expand_durations_kernel<OutT, ST, OV><<<grid, bx, 0, st>>>(base, group, ovr_map, ovr, scale_ptr, \
                                                             scale, rows, S, ld, out)
  if (big && ovr_map)
    EXPAND_K(true, true);
  else if (big)
    EXPAND_K(true, false);
  else if (ovr_map)
    EXPAND_K(false, true);
  else
    EXPAND_K(false, false);
#undef EXPAND_K
  note_launch();
  return cudaGetLastError();
}
cudaError_t launch_expand_durations(const long long* base, const unsigned* group,
                                    const int* ovr_map, const long long* ovr, const int* scale_ptr,
                                    const ScaleStepDev* scale, int rows, int S, long long ld,
                                    long long* out, cudaStream_t st) {
  return launch_expand(base, group, ovr_map, ovr, scale_ptr, scale, rows, S, ld, out, st);
}
cudaError_t launch_expand_durations32(const long long* base, const unsigned* group,
                                      const int* ovr_map, const long long* ovr,
                                      const int* scale_ptr, const ScaleStepDev* scale, int rows,
                                      int S, long long ld, int* out, cudaStream_t st) {
  return launch_expand(base, group, ovr_map, ovr, scale_ptr, scale, rows, S, ld, out, st);
}

}  // namespace ddsim
