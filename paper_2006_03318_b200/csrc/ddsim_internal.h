// Internal layout shared by the host compiler (graph.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/ddsim.h"

#include "host_alloc.h"

namespace ddsim {

// One instruction of the compiled max-plus program: a task, or a permutable
// chain (kind == 1) whose members are expanded per scenario.  64 bytes so a
// chunk of records moves with one cp.async.bulk.
struct alignas(16) NodeRec {
  long long dur;    // base duration (ns)
  long long gap;    // gap (ns)
  long long ready;  // Task.ready_time floor (ns)
  int out_slot;     // value slot receiving rel = start+dur+gap, -1 = none
  int pred0;        // value slots of predecessors, -1 = none
  int pred1;
  int extra_off;    // further pred slots in extra[extra_off .. +nextra)
  int nextra;
  unsigned group;   // scale group (0 = untouched by every scale step)
  int ovr_row;      // row of the per-scenario override table, -1 = none
  int lane;
  int row;          // frozen output row (kind 0) / chain index (kind 1)
  int kind;         // 0 task, 1 chain macro
};
static_assert(sizeof(NodeRec) == 64, "NodeRec must be 64 bytes");

// Compact record of the dense-duration program (no chains): 16 bytes.
// op bits say where the predecessors' rel values are: in registers (the two
// previous records -- most lane-chain and launch edges are that short), in
// shared-memory slots s0/s1, or (rare, DOP_SLOW) in the side tables / global
// spill slots.
struct alignas(16) DenseRec {
  long long gap;
  short s0, s1;         // shared-memory slot ids (DOP_S0 / DOP_S1)
  short out;            // slot receiving rel (DOP_OUT_SMEM / DOP_OUT_GLOBAL)
  unsigned char lane;
  unsigned char op;
};
static_assert(sizeof(DenseRec) == 16, "DenseRec must be 16 bytes");
enum {
  DOP_PREV = 1, DOP_PREV2 = 2, DOP_S0 = 4, DOP_S1 = 8, DOP_SLOW = 16,
  DOP_OUT_SMEM = 32, DOP_OUT_GLOBAL = 64,
  DOP_MS = 128          // contributes to makespan (last task of its lane)
};
// DenseRec.lane high bit: record has a non-zero gap
enum { DLANE_GAP = 0x80 };

struct DenseParams {
  const DenseRec* prog;
  int n_rec;
  const int* side_off;        // [n_rec+1] slow-path pred slot ids (smem < ksm <= global)
  const int* side_slots;
  const long long* side_ready;  // [n_rec] ready floor (or null)
  int ksm, kglob;
  long long* gslots;
  long long s_pad;
  int S, L;
  int V;                      // scenarios per thread (1 or 2)
  int* neg_flag;              // set when a negative duration is seen (exact rerun)
  const long long* dense64;   // int64 mode
  long long dense_ld;
  long long* start;
  long long start_ld;
  long long* makespan;
  long long* lane_busy;
};

// Lane-register program record (maxplus_lanes.cu): 16 bytes.
// h = own lane (2 bits) | predecessor-lane mask (5 bits; bit 4 = temp lane
// holding the rare predecessors) << 2 | gap != 0 << 7.
struct alignas(16) LaneRec {
  long long gap;
  short s0, s1;          // smem slots of rare predecessors (LREC_S0 / LREC_S1)
  short out;             // slot receiving rel (LREC_OUT_SMEM: smem id, LREC_OUT_GLOBAL: global id)
  unsigned char rare;
  unsigned char h;
};
static_assert(sizeof(LaneRec) == 16, "LaneRec must be 16 bytes");
enum {
  LREC_S0 = 1, LREC_S1 = 2, LREC_SIDE = 4, LREC_MS = 8, LREC_OUT_SMEM = 16, LREC_OUT_GLOBAL = 32,
  LREC_CHAIN = 64,  // permutable chain (s0 = chain id): its members in the scenario's order
  LREC_NOP = 128,   // row of a chain member after the chain record (nothing to do)
  LREC_PRE = 7 | 64 | 128, LREC_POST = 56
};

// Permutable chain on the lanes path: members mem_off .. mem_off+B-1, member k
// on frozen row (chain record's row) + k; the scenario order is
// perm[s * perm_ld + perm_off + q].
struct LaneChainDev {
  int lane, B, mem_off, perm_off;
};
struct LaneMemberDev {
  long long gap;
  int pred_off, npred;   // predecessor slot codes lpreds[pred_off ..] (< ksm smem, else global)
  int out;               // slot code receiving the member's rel, -1 = none
  int pad;
};
static_assert(sizeof(LaneMemberDev) == 24, "LaneMemberDev layout");

struct LaneParams {
  const LaneRec* prog;
  int n_rec;
  const int* side_off;
  const int* side_slots;       // < ksm: smem slot, else global slot + ksm
  const long long* side_ready;
  int ksm, kglob;
  long long* gslots;
  long long s_pad;
  int S, L;
  const long long* dense64;
  long long dense_ld;
  long long* start;
  long long start_ld;
  long long* makespan;
  long long* lane_busy;
  int* neg_flag;
};

// Permutable chains on the lanes path (a separate kernel parameter of the
// chain variant; mirrors ddsim_lanes::ChainParams).
struct LaneChainParams {
  const LaneChainDev* chains;
  const LaneMemberDev* members;
  const int* preds;
  const short* perm;          // [S][perm_ld] or null (identity order)
  const unsigned char* present;  // [S][n_chains] or null (all present)
  const int* dense32;         // int32 durations (chain members read them directly)
  int perm_ld;
  int n_chains;
};

struct ChainDesc {
  int first_row;   // members occupy frozen rows first_row .. first_row+B-1
  int B;
  int head_slot;   // slot of the head's rel (-1 = none)
  int tail_slot;   // slot receiving the last member's rel (-1 = no tail)
  int member_off;  // index of the first member record in `members`
  int perm_off;    // column offset of this chain in a scenario's perm row
  int lane;
  int pad;
};

struct ScaleStepDev {
  int lo, hi;
  long long num, den;
};

struct MaxplusParams {
  const NodeRec* prog;
  int n_rec;
  const int* extra;
  const ChainDesc* chains;
  const NodeRec* members;
  int ksm;                // slots held in shared memory
  int kglob;              // spilled slots
  long long* gslots;      // [kglob][s_pad]
  long long s_pad;
  int S;
  int L;
  int n_chains;
  // duration sources
  const long long* dense64;  // [rows][ld] or null
  long long dense_ld;
  int dense_kind;            // 0 none, 1 int32 (TMA tiles), 2 int64
  const long long* ovr;      // [n_ovr][S]
  const int* scale_ptr;      // [S+1] or null
  const ScaleStepDev* scale;
  const short* perm;         // [S][perm_ld] or null
  int perm_ld;
  const unsigned char* present;  // [S][n_chains] or null
  // outputs
  long long* start;
  long long start_ld;
  long long* makespan;
  long long* lane_busy;      // [S][L]
  const int* run_if;         // non-null: run only if *run_if != 0 (exact fallback)
};

struct ListParams {
  int N, L, S;
  const int* child_ptr;  // [N+1] frozen rows, multiset
  const int* child;
  const int* indeg;      // multiset in-degree
  const int* lane;
  const long long* dur;
  const long long* gap;
  const long long* ready;
  const int* id_rank;
  const int* prio;
  const unsigned char* flags;
  const unsigned* group;
  const int* vrank;      // [N] or null
  int policy;
  int zero_time;         // verify_acyclic mode: all times 0
  // durations
  const int* dense32;
  const long long* dense64;
  long long dense_ld;
  const int* ovr_row;    // [N] or null
  const long long* ovr;  // [n_ovr][S]
  const int* scale_ptr;
  const ScaleStepDev* scale;
  // scratch [S][N] / [S][L]
  long long* rdy;
  int* rem;
  int* front;
  long long* lane_prog;
  // outputs
  long long* start; long long start_ld;
  long long* makespan;
  long long* lane_busy;
  int* schedule;
  int* dispatched;
};

// kernel launchers (maxplus.cu / listsched.cu)
cudaError_t launch_maxplus(const MaxplusParams& p, const int* dense32,
                           cudaStream_t stream);
cudaError_t launch_maxplus_dense(const DenseParams& p, const int* dense32, int dkind,
                                 cudaStream_t stream);
// Derived durations for the lanes kernels (dkind 0; mirrors
// ddsim_lanes::DerivedParams): per-row base / group / override row, the
// override table and the scale programs.
struct LaneRowDur {
  long long base;
  unsigned group;
  int ovr;
};
struct LaneDerivedParams {
  const LaneRowDur* rows;
  const long long* ovr;
  const int* scale_ptr;
  const ScaleStepDev* scale;
};
cudaError_t launch_build_rowdur(const long long* base, const unsigned* group, const int* ovr_map,
                                int n, LaneRowDur* out, cudaStream_t st);
cudaError_t launch_maxplus_lanes(const LaneParams& p, const LaneChainParams* cp, const int* dense32,
                                 int dkind,
                                 const std::vector<int>* codes, cudaStream_t stream,
                                 const LaneDerivedParams* dp = nullptr);
// lane_busy[s][l] = sum of the durations of lane l's present rows (lanes
// program order); the branch-free lanes handler leaves it to this pass.
cudaError_t launch_lanes_busy(const LaneParams& p, const int* dense32, bool chains,
                              cudaStream_t stream);
cudaError_t launch_maxplus_lanes_jit(const LaneParams& p, const LaneChainParams* cp,
                                     const int* dense32, const void* tmap128, int dkind, int V,
                                     const std::vector<int>& codes, int grid, int BD, size_t smem,
                                     cudaStream_t stream, const LaneDerivedParams* dp = nullptr);
int maxplus_lanes_vec(int S, int dkind = 1, bool vec_ok = true);
// Segment-parallel lanes path (mirrors ddsim_lanes::SegParams)
struct LaneSegParams {
  const int* cuts;
  int K;
  int LN;
  int* trans;
  long long* state;
  long long s_pad;
  int* ticket;
  int* flags;
  int nb;
  int pad;
  const long long* gapsum;
  int kc;
  int replay_only;
  const int* carry_ptr;
  const int* carry_gid;
  int* carry_coef;
};
cudaError_t launch_maxplus_lanes_seg(const LaneParams& p, const LaneChainParams* cp,
                                     const int* dense32, int dkind, const std::vector<int>& codes,
                                     const LaneSegParams& sg, int BD, cudaStream_t stream,
                                     const LaneDerivedParams* dp = nullptr);
cudaError_t launch_lanes_seg_jit(int mode, const LaneParams& p, const LaneChainParams* cp,
                                 const void* tmap128, int dkind, int LN,
                                 const std::vector<int>& codes, const void* segp, int gx, int gy,
                                 int BD, size_t smem, cudaStream_t stream,
                                 const LaneDerivedParams* dp = nullptr);
bool jit_available();
cudaError_t launch_expand_durations(const long long* base, const unsigned* group,
                                    const int* ovr_map, const long long* ovr, const int* scale_ptr,
                                    const ScaleStepDev* scale, int rows, int S, long long ld,
                                    long long* out, cudaStream_t st);
cudaError_t launch_expand_durations32(const long long* base, const unsigned* group,
                                      const int* ovr_map, const long long* ovr,
                                      const int* scale_ptr, const ScaleStepDev* scale, int rows,
                                      int S, long long ld, int* out, cudaStream_t st);
// Batched runtime breakdown (breakdown.py:42-111) over a max-plus result.
struct BdChain {
  int lane, pos;            // inserted after `pos` static rows of its lane
  int B, member_off, perm_off, pad;
};
struct BreakdownParams {
  int n, L, S, n_chains;
  const int* lane_ptr;      // [L+1] static lane sequences (frozen rows)
  const int* lane_rows;
  const int* lane_chain;    // [L] chain on the lane or -1
  const BdChain* chains;
  const int* member_rows;   // [perm_ld] frozen rows of chain members
  const short* perm;        // [S][perm_ld] or null
  int perm_ld;
  const unsigned char* present;  // [S][n_chains] or null
  const unsigned char* row_class;  // [n] KS_BD_*
  const long long* gap;     // [n] by row
  int dkind;                // 1 = int32, 2 = int64 durations [row][dld]
  const void* dur;
  long long dld;
  const long long* start;
  long long start_ld;
  const long long* makespan;
  int comm_as_gpu, dataload_as_cpu, gaps_as_cpu_busy;
  long long* parts;         // [S][4] cpu_only, gpu_only, parallel, idle (-1: precondition failed)
  int K;                    // time windows per scenario (parallel merge)
  int* bad;                 // [S] scratch: scenario has a negative duration
  // per-layer busy (per_layer_breakdown): [n_layers][2][S]
  const int* row_layer;     // [n] or null
  long long* layer_busy;
  int n_layers;
  int lb_chunk;             // rows per per-layer busy block row (set by launch_breakdown)
  int start_may_be_neg;     // removal steps / permutable chains: start -1 marks a dropped task
  const int* srows;         // [S][n] per-scenario lane sequences (list-scheduled) or null
  int stream_loads;         // experiments: evict-first start loads (DDSIM_BD_STREAM)
  // row-order streaming sweep (breakdown_stream_kernel): lane of every row and
  // the per-row class / last-in-lane codes it builds; redo: the windowed merge
  // recomputes only the scenarios the sweep handed back (bad[s] == 2)
  const int* row_lane;      // [n] or null (streaming sweep unavailable)
  long long* rinfo;         // [n] scratch
  int* linfo;               // [n] scratch: per-layer busy keys (layer * 2 + is-GPU, -1 comm)
  int stream_mode;          // 0 auto, 1 force the sweep, -1 never
  int stream_depth;         // pending runs per lane the sweep may hold (<= kBsD)
  int redo;
};
cudaError_t launch_breakdown(const BreakdownParams& p, cudaStream_t stream);
cudaError_t launch_bd_sched_rows(const int* schedule, const int* row_lane, const int* lane_ptr,
                                 int n, int L, int S, int* srows, cudaStream_t stream);

const char* jit_log();
int maxplus_lanes_block_dim(int S, int num_sms, int dkind = 1, bool vec_ok = true);
cudaError_t launch_listsched(const ListParams& p, cudaStream_t stream);
cudaError_t launch_toposort_lanes(int N, int L, const int* lane_ptr, const int* lane_rows,
                                  const int* child_ptr, const int* child, const int* indeg,
                                  const int* rank, int* deg_scratch, int* out, int* count,
                                  cudaStream_t st);
// A lane head of verify_acyclic's lane walk (listsched.cu): frozen row, id
// rank, requirement count / offset, the first four requirements (lane, prefix)
struct alignas(16) TopoRec {
  int row, rank, rn, r0;
  int ml[4], mq[4];
};
cudaError_t launch_toposort_lanes_req(int N, int L, const int* lane_ptr, const TopoRec* recs,
                                      const int* req_lane, const int* req_pos, int* out,
                                      int* count, cudaStream_t st);
cudaError_t launch_fill_i64(long long* p, long long v, long long n, cudaStream_t s);
cudaError_t launch_fill_i32(int* p, int v, long long n, cudaStream_t s);
cudaError_t launch_patch_ovr(NodeRec* prog, int n_rec, const int* ovr_map, cudaStream_t st);
int maxplus_block_dim(int S, int dmode, int num_sms);
int maxplus_dense_block_dim(int S, int V, int num_sms);

void note_launch(int n = 1);
// Keep freed stream-ordered memory in the device's default pool between calls
// (the default release threshold unmaps it at every synchronize, so the next
// call re-maps: measured +15 ms on the first config-4 launch after a sync).
void keep_device_pool(int device);

// Ingest outputs kept on the device (ks_ingest_keep) for the device freeze.
struct IngestDev {
  int device = 0;
  long long n = 0, m = 0;
  int L = 0;
  int* lane = nullptr;         // [n] event lane
  long long* start = nullptr;  // [n]
  long long* dur = nullptr;    // [n]
  long long* gap = nullptr;    // [n] compute_gaps
  int* src = nullptr;          // [m] edges (event indices), multiset
  int* dst = nullptr;
  unsigned char* ekind = nullptr;  // [m] KS_EDGE_*
  int* lane_order = nullptr;   // [n] events per lane by (start, id)
  std::vector<int> lane_order_ptr;         // [L+1]
  std::vector<unsigned char> lane_class;   // [L] 0 cpu, 1 gpu, 2 comm
  void release();
};

// Device freeze of an ingested trace (freeze.cu); the device arrays pass to
// the graph (cudaMalloc, freed by free_graph).
struct DeviceFreeze {
  long long n = 0, m_unique = 0;
  bool ok = false;                // the relaxed trace-time order is topological
  int rounds = 0;                 // relaxation rounds
  std::vector<int> order;         // host copy: row -> event
  int* order_d = nullptr;
  unsigned long long* ukeys = nullptr;  // [m_unique] (u << 32 | v) ascending
  unsigned long long* pkeys = nullptr;  // [m_unique] (v << 32 | u) ascending
  int *child_ptr = nullptr, *child = nullptr, *indeg = nullptr;  // rows, multiset
  int *lane_r = nullptr, *rank_r = nullptr, *prio_r = nullptr;
  long long *dur_r = nullptr, *gap_r = nullptr, *ready_r = nullptr;
  unsigned char* flags_r = nullptr;
  unsigned* group_r = nullptr;
};
int freeze_from_ingest(const IngestDev& I, const int32_t* id_rank_h, const uint8_t* flags_h,
                       DeviceFreeze& F, std::string& err);
void free_device_freeze(DeviceFreeze& F);

}  // namespace ddsim

// C-ABI handle of a kept ingest (include/ddsim.h: ks_ingest_keep)
struct ks_ingest_dev {
  ddsim::IngestDev d;
};
