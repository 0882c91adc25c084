// maxplus_dense: max-plus simulate() for dense per-scenario durations
// (Monte-Carlo jitter, BASELINE config 4).  Same recurrence as maxplus.cu
// (sim.py:89-142 on lane-chained graphs == synthetic.py:35-48):
//     start(v) = max(ready, max_{u->v} start(u) + dur(u) + gap(u))
// Specialisation for the HBM-bound case:
//   * V scenarios per thread (int32 pairs in, 128-bit int64 stores out);
//   * 16-byte program records + the [rows x (V*BD)] int32 duration tile of
//     each chunk staged by cp.async.bulk / 2D TMA on one mbarrier, kStages
//     chunks ahead;
//   * rel of the two previous records in registers; only values read more
//     than two records later go through shared memory (compiled slots).
#include "ddsim_internal.h"

#include <algorithm>
#include <climits>
#include <cudaTypedefs.h>

namespace ddsim {

namespace {
constexpr int kChunkD = 16;
constexpr int kStagesD = 4;

__device__ __forceinline__ unsigned su32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void d_mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void d_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void d_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void d_bulk(void* dst, const void* src, unsigned bytes,
                                       unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void d_tile(void* dst, const CUtensorMap* map, int x, int y,
                                       unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)), "l"(map), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}

template <int V>
struct Vec {
  long long v[V];
};

template <int V>
__device__ __forceinline__ void vmax(Vec<V>& a, const Vec<V>& b) {
#pragma unroll
  for (int i = 0; i < V; ++i) a.v[i] = max(a.v[i], b.v[i]);
}
}  // namespace

__device__ __forceinline__ int4 lds128(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int2 lds64i(unsigned a) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds32i(unsigned a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ long long lds64(unsigned a) {
  long long v;
  asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(unsigned a, long long v) {
  asm volatile("st.shared.s64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

// V scenarios per thread; DK: 1 = int32 durations via TMA tiles, 2 = int64
// durations via direct global loads; NL: lanes kept in registers (0 = lane
// busy accumulated in shared memory, any lane count).
//
// Fast-path facts (host-checked: gaps and ready times >= 0, lanes chained;
// device-checked: durations >= 0, else *neg_flag is set and the host's exact
// kernel reruns the launch): every rel >= fin >= start >= 0, so the 0 floor of
// start() is implied by any predecessor, and the makespan is the max finish of
// the last task of each lane (flagged DOP_MS) because a lane's finishes never
// decrease along its chain.
template <int V, int DK, int NL>
__global__ void __launch_bounds__(256) maxplus_dense_kernel(const __grid_constant__ CUtensorMap tmap,
                                                            const DenseParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int BD = blockDim.x;
  const int W = BD * V;  // scenarios per CTA
  const int tid = threadIdx.x;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem);
  DenseRec* pst = reinterpret_cast<DenseRec*>(smem + 128);
  const unsigned sbase = su32(smem);
  const unsigned prog_s = sbase + 128;
  const unsigned tile_s = prog_s + kStagesD * kChunkD * (unsigned)sizeof(DenseRec);
  const unsigned tile_bytes_all = DK == 1 ? (unsigned)(kStagesD * kChunkD * W * 4) : 0u;
  const unsigned slot_s = tile_s + tile_bytes_all;              // [ksm][BD] x (8V)
  const unsigned lb_s = slot_s + (unsigned)(p.ksm * BD * 8 * V);  // [L][BD] x (8V)
  const unsigned col = (unsigned)(tid * 8 * V);                 // this thread's column
  const unsigned slot_pitch = (unsigned)(BD * 8 * V);
  int* tst = reinterpret_cast<int*>(smem + (tile_s - sbase));

  const int s0 = blockIdx.x * W;
  const int s = s0 + tid * V;
  const bool act = s < p.S;
  if (NL == 0)
    for (int l = 0; l < p.L; ++l)
#pragma unroll
      for (int i = 0; i < V; ++i) sts64(lb_s + l * slot_pitch + col + 8 * i, 0);
  const int nchunks = (p.n_rec + kChunkD - 1) / kChunkD;
  const unsigned tile_bytes = DK == 1 ? (unsigned)(kChunkD * W * sizeof(int)) : 0u;
  auto issue = [&](int c) {
    const int st = c % kStagesD;
    const int nrec = min(kChunkD, p.n_rec - c * kChunkD);
    const unsigned pb = (unsigned)(nrec * sizeof(DenseRec));
    d_expect(&bars[st], pb + tile_bytes);
    d_bulk(pst + st * kChunkD, p.prog + (long long)c * kChunkD, pb, &bars[st]);
    if (DK == 1) d_tile(tst + st * kChunkD * W, &tmap, s0, c * kChunkD, &bars[st]);
  };
  if (tid == 0) {
    for (int i = 0; i < kStagesD; ++i) d_mbar_init(&bars[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int c = 0; c < min(kStagesD, nchunks); ++c) issue(c);

  long long ms[V], ra[V], rb[V], lbr[NL > 0 ? NL : 1][V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    ms[i] = ra[i] = rb[i] = 0;
#pragma unroll
    for (int l = 0; l < (NL > 0 ? NL : 1); ++l) lbr[l][i] = 0;
  }
  int neg = 0;
  const long long ld = p.start_ld;
  long long* sp = (act && p.start) ? p.start + s : nullptr;
  const long long* dp = DK == 2 ? p.dense64 + (act ? s : 0) : nullptr;
  const int ksm = p.ksm;
  const unsigned row_pitch = (unsigned)(W * 4);

  // one record: `pv` = rel of the previous record, `pv2` = the one before;
  // the result overwrites pv2 (the two registers alternate roles)
  auto step = [&](int4 raw, long long dv0, long long dv1, int row, const long long* pv,
                  long long* pv2) {
    const long long gap = ((long long)(unsigned)raw.y << 32) | (unsigned)raw.x;
    const unsigned w = (unsigned)raw.w;
    const unsigned op = w >> 24;
    long long dv[V];
    dv[0] = dv0;
    if (V == 2) dv[V - 1] = dv1;
    long long sv[V];
    if (op & DOP_PREV) {
#pragma unroll
      for (int i = 0; i < V; ++i) sv[i] = pv[i];
      if (op & DOP_PREV2)
#pragma unroll
        for (int i = 0; i < V; ++i) sv[i] = max(sv[i], pv2[i]);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) sv[i] = (op & DOP_PREV2) ? pv2[i] : 0;
    }
    if (op & DOP_S0) {
      const unsigned a = slot_s + (unsigned)((raw.z << 16) >> 16) * slot_pitch + col;
#pragma unroll
      for (int i = 0; i < V; ++i) sv[i] = max(sv[i], lds64(a + 8 * i));
    }
    if (op & DOP_S1) {
      const unsigned a = slot_s + (unsigned)(raw.z >> 16) * slot_pitch + col;
#pragma unroll
      for (int i = 0; i < V; ++i) sv[i] = max(sv[i], lds64(a + 8 * i));
    }
    if (op & DOP_SLOW) {
      if (p.side_ready) {
        const long long rd = p.side_ready[row];
#pragma unroll
        for (int i = 0; i < V; ++i) sv[i] = max(sv[i], rd);
      }
      if (p.side_off)
        for (int k = p.side_off[row]; k < p.side_off[row + 1]; ++k) {
          const int code = p.side_slots[k];
          if (code < ksm) {
#pragma unroll
            for (int i = 0; i < V; ++i)
              sv[i] = max(sv[i], lds64(slot_s + code * slot_pitch + col + 8 * i));
          } else if (act) {
            const long long* g = p.gslots + (long long)(code - ksm) * p.s_pad + s;
#pragma unroll
            for (int i = 0; i < V; ++i) sv[i] = max(sv[i], g[i]);
          }
        }
    }
    if (sp) {
#pragma unroll
      for (int i = 0; i < V; ++i) __stcs(sp + i, sv[i]);
      sp += ld;
    }
    const unsigned ln = (w >> 16) & 0xffu;
    long long rel[V];
#pragma unroll
    for (int i = 0; i < V; ++i) rel[i] = sv[i] + dv[i];
    if (op & DOP_MS)
#pragma unroll
      for (int i = 0; i < V; ++i) ms[i] = max(ms[i], rel[i]);
    if (ln & DLANE_GAP)
#pragma unroll
      for (int i = 0; i < V; ++i) rel[i] += gap;
    if (op & (DOP_OUT_SMEM | DOP_OUT_GLOBAL)) {
      const int out = (int)(w << 16) >> 16;
      if (op & DOP_OUT_SMEM) {
        const unsigned a = slot_s + (unsigned)out * slot_pitch + col;
#pragma unroll
        for (int i = 0; i < V; ++i) sts64(a + 8 * i, rel[i]);
      } else if (act) {
        long long* g = p.gslots + (long long)(out - ksm) * p.s_pad + s;
#pragma unroll
        for (int i = 0; i < V; ++i) g[i] = rel[i];
      }
    }
    const unsigned lane = ln & 0x7fu;
    if (NL > 0) {
#pragma unroll
      for (int l = 0; l < (NL > 0 ? NL : 1); ++l)
        if (lane == (unsigned)l)
#pragma unroll
          for (int i = 0; i < V; ++i) lbr[l][i] += dv[i];
    } else {
      const unsigned a = lb_s + lane * slot_pitch + col;
#pragma unroll
      for (int i = 0; i < V; ++i) sts64(a + 8 * i, lds64(a + 8 * i) + dv[i]);
    }
#pragma unroll
    for (int i = 0; i < V; ++i) pv2[i] = rel[i];
  };

  auto load_d = [&](unsigned trow, long long& x, long long& y) {
    if (DK == 1) {
      if (V == 2) {
        const int2 t2 = lds64i(trow);
        x = t2.x;
        y = t2.y;
        neg |= t2.x | t2.y;
      } else {
        const int t1 = lds32i(trow);
        x = t1;
        y = 0;
        neg |= t1;
      }
    } else {
      x = dp[0];
      y = V == 2 ? dp[V - 1] : 0;
      neg |= (int)((x | y) >> 32);
      dp += p.dense_ld;
    }
  };

  for (int c = 0; c < nchunks; ++c) {
    const int st = c % kStagesD;
    d_wait(&bars[st], (unsigned)((c / kStagesD) & 1));
    const unsigned rec0 = prog_s + (unsigned)(st * kChunkD * sizeof(DenseRec));
    const unsigned t0 = tile_s + (unsigned)(st * kChunkD) * row_pitch + (unsigned)(tid * 4 * V);
    const int nrec = min(kChunkD, p.n_rec - c * kChunkD);
    const int row0 = c * kChunkD;
    int j = 0;
    // records alternate between the ra / rb registers (no moves); the next
    // record and duration pair are loaded before the current one is used
    int4 rawA = lds128(rec0);
    long long xa, ya;
    load_d(t0, xa, ya);
    for (; j + 1 < nrec; j += 2) {
      const int4 rawB = lds128(rec0 + (unsigned)(j + 1) * 16u);
      long long xb, yb;
      load_d(t0 + (unsigned)(j + 1) * row_pitch, xb, yb);
      step(rawA, xa, ya, row0 + j, rb, ra);
      if (j + 2 < nrec) {
        rawA = lds128(rec0 + (unsigned)(j + 2) * 16u);
        load_d(t0 + (unsigned)(j + 2) * row_pitch, xa, ya);
      }
      step(rawB, xb, yb, row0 + j + 1, ra, rb);
    }
    if (j < nrec) {
      step(rawA, xa, ya, row0 + j, rb, ra);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const long long t = ra[i];
        ra[i] = rb[i];
        rb[i] = t;
      }
    }
    __syncthreads();
    if (tid == 0 && c + kStagesD < nchunks) issue(c + kStagesD);
  }
  if (act) {
    if (neg < 0 && p.neg_flag) atomicOr(p.neg_flag, 1);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      if (p.makespan) p.makespan[s + i] = ms[i];
      if (p.lane_busy)
        for (int l = 0; l < p.L; ++l) {
          long long v;
          if (NL > 0) {
            v = 0;
#pragma unroll
            for (int q = 0; q < (NL > 0 ? NL : 1); ++q)
              if (q == l) v = lbr[q][i];
          } else {
            v = lds64(lb_s + l * slot_pitch + col + 8 * i);
          }
          p.lane_busy[(long long)(s + i) * p.L + l] = v;
        }
    }
  }
}

static size_t dense_smem(int V, int dk, int BD, int ksm, int L) {
  size_t b = 128 + (size_t)kStagesD * kChunkD * sizeof(DenseRec);
  if (dk == 1) b += (size_t)kStagesD * kChunkD * BD * V * sizeof(int);
  return b + (size_t)ksm * BD * V * 8 + (size_t)L * BD * V * 8;
}

// Threads per CTA: two CTAs per SM cover all scenarios in one wave.
int maxplus_dense_block_dim(int S, int V, int num_sms) {
  long long per = (S / V + 2LL * num_sms - 1) / (2LL * num_sms);
  int bd = (int)(((per + 31) / 32) * 32);
  const int cap = 256 / V;  // TMA box inner extent <= 256 elements
  return bd < 32 ? 32 : (bd > cap ? cap : bd);
}

template <int V, int DK, int NL>
static cudaError_t launch_vl(const CUtensorMap& tmap, const DenseParams& p, int grid, int BD,
                             size_t smem, cudaStream_t stream) {
  cudaError_t err = cudaFuncSetAttribute(maxplus_dense_kernel<V, DK, NL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  maxplus_dense_kernel<V, DK, NL><<<grid, BD, smem, stream>>>(tmap, p);
  return cudaSuccess;
}

template <int V, int DK>
static cudaError_t launch_v(const CUtensorMap& tmap, const DenseParams& p, int grid, int BD,
                            size_t smem, cudaStream_t stream) {
  if (p.L <= 4) return launch_vl<V, DK, 4>(tmap, p, grid, BD, smem, stream);
  return launch_vl<V, DK, 0>(tmap, p, grid, BD, smem, stream);
}

cudaError_t launch_maxplus_dense(const DenseParams& p, const int* dense32, int dkind,
                                 cudaStream_t stream) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int V = p.V == 2 ? 2 : 1;
  const int BD = maxplus_dense_block_dim(p.S, V, nsm);
  const int W = BD * V;
  const int grid = (p.S + W - 1) / W;
  if ((long long)grid * W > p.s_pad) return cudaErrorInvalidValue;
  const size_t smem = dense_smem(V, dkind, BD, p.ksm, p.L);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (dkind == 1) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      return cudaErrorNotSupported;
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cuuint64_t dims[2] = {(cuuint64_t)p.S, (cuuint64_t)p.n_rec};
    cuuint64_t strides[1] = {(cuuint64_t)(p.dense_ld * sizeof(int))};
    cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)kChunkD};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int*>(dense32), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  cudaError_t err;
  if (V == 2)
    err = dkind == 1 ? launch_v<2, 1>(tmap, p, grid, BD, smem, stream)
                     : launch_v<2, 2>(tmap, p, grid, BD, smem, stream);
  else
    err = dkind == 1 ? launch_v<1, 1>(tmap, p, grid, BD, smem, stream)
                     : launch_v<1, 2>(tmap, p, grid, BD, smem, stream);
  if (err != cudaSuccess) return err;
  note_launch();
  return cudaGetLastError();
}

}  // namespace ddsim
