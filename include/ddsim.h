/*
 * ddsim.h -- C-ABI of the B200-native batched what-if simulator.
 *
 * Plain pointers and sizes only: no torch types, no C++ types.  Every entry
 * point returns an int status (0 = OK, else a KS_ERR_* code whose stable name
 * is ks_error_name(code)); a human-readable detail for the last failure on the
 * calling thread is ks_last_error_detail().  These names are exactly the
 * KernsimError names of the reference (pkg/src/kernsim/errors.py:11-140), so a
 * host binding re-raises the same exception class.
 *
 * Which reference interface each entry point replaces:
 *
 *   ks_graph_create        freeze of kernsim.graph.DependencyGraph
 *                          (pkg/src/kernsim/graph.py:75-126): CSR, topological
 *                          order (verify_acyclic, graph.py:129-148), lane
 *                          chaining check, value-slot compilation.
 *   ks_simulate            kernsim.sim.simulate (pkg/src/kernsim/sim.py:89-142)
 *                          for S scenarios at once; policy ids map to
 *                          DefaultSchedule / PrioritySchedule (sim.py:66-86) and
 *                          VdnnPrefetchPolicy (scenarios.py:593-630).  Durations
 *                          per scenario replace scale_durations / set_duration
 *                          (transform.py:174-183, 293-297) and the inserted
 *                          task table replaces sequenced insert_task
 *                          (transform.py:204-246) of whatif_distributed
 *                          (scenarios.py:194-241).
 *   ks_simulate_host       the same with HOST buffers (H2D/D2H inside the call),
 *                          i.e. what a ctypes binding of simulate() calls.
 *   ks_toposort            verify_acyclic (graph.py:129-148): Kahn order with
 *                          smallest-id tie-break, computed on the device.
 *   ks_ingest              build_graph + link_syncs + compute_gaps
 *                          (graph.py:198-312) and check_lane_overlaps
 *                          (trace.py:255-265) over columnar trace records.
 *   ks_map_layers          map_tasks_to_layers (layers.py:50-81).
 *   ks_breakdown           compute_breakdown / per_layer_breakdown
 *                          (breakdown.py:42-111) for S scenarios.
 *   ks_trace_parse         parse_trace (trace.py:281-328) straight into
 *                          columns (host, multi-threaded), same validation
 *                          and error precedence.
 *   ks_trace_write         dump_trace (trace.py:331-379) from columns.
 */
#ifndef DDSIM_H_
#define DDSIM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (names == reference KernsimError.name) ---------------- */
enum {
  KS_OK = 0,
  KS_ERR_DEADLOCK = 1,            /* "Deadlock"            errors.py:87   */
  KS_ERR_CYCLE = 2,               /* "CycleDetected"       errors.py:57   */
  KS_ERR_INVALID = 3,             /* "InvalidArgument"     (ValueError)   */
  KS_ERR_CUDA = 4,                /* "CudaError"                          */
  KS_ERR_OOM = 5,                 /* "OutOfMemory"                        */
  KS_ERR_UNSUPPORTED = 6,         /* "Unsupported"                        */
  KS_ERR_ORPHAN = 7,              /* "OrphanKernel"        errors.py:53   */
  KS_ERR_AMBIGUOUS = 8,           /* "AmbiguousMarker"     errors.py:67   */
  KS_ERR_OVERLAP = 9,             /* "OverlapViolation"    errors.py:34   */
  KS_ERR_BAD_PIPELINE = 10,       /* "BadPipeline"         errors.py:117  */
  KS_ERR_NO_DEVICE = 11,          /* "NoDevice"                           */
  KS_ERR_MALFORMED = 12,          /* "MalformedDocument"   errors.py:26   */
  KS_ERR_SCHEMA = 13              /* "SchemaViolation"     errors.py:30   */
};

/* ---- schedule policies (sim.py:152-165, scenarios.py:633) -------------- */
enum { KS_POLICY_DEFAULT = 0, KS_POLICY_PRIORITY = 1, KS_POLICY_VDNN = 2 };

/* ---- per-task flags ----------------------------------------------------- */
enum {
  KS_TASK_COMM = 1,          /* Task.is_comm (graph.py:59-61)                    */
  KS_TASK_VDNN_MALLOC = 2    /* name startswith "cudaMalloc_vdnn" (scenarios.py:621) */
};

typedef struct ks_graph ks_graph; /* opaque, device-resident, immutable */

/* A dependency graph in dense form.  Task i (0..n_tasks-1) is an arbitrary
 * dense index chosen by the caller; id_rank[i] must order tasks exactly as
 * their external ids do (ties in the scheduler break on id, sim.py:55-63). */
typedef struct {
  int32_t n_tasks;
  int32_t n_lanes;
  const int64_t* duration;    /* [n_tasks] ns                               */
  const int64_t* gap;         /* [n_tasks] ns                               */
  const int64_t* ready_time;  /* [n_tasks] ns (Task.ready_time)             */
  const int32_t* lane;        /* [n_tasks] 0..n_lanes-1                     */
  const int32_t* id_rank;     /* [n_tasks] rank of external id              */
  const int32_t* priority;    /* [n_tasks] Task.priority                    */
  const uint8_t* flags;       /* [n_tasks] KS_TASK_*; may be NULL           */
  const uint32_t* group;      /* [n_tasks] scale group (0 = untouched); NULL */
  int64_t n_edges;            /* multiset: (u,v) may repeat (kinds differ)  */
  const int32_t* edge_src;
  const int32_t* edge_dst;
  const int32_t* lane_order_ptr; /* [n_lanes+1] or NULL (= nothing chained) */
  const int32_t* lane_order;     /* dense indices, per lane, in order        */
  /* Permutable chains (inserted-task table).  Chain c owns members
   * chain_member[chain_ptr[c] .. chain_ptr[c+1]); its members sit on one lane,
   * are NOT in lane_order and carry no edges among themselves: their on-lane
   * order is the per-scenario permutation ks_scenarios_desc.chain_perm.  The
   * head/tail tasks (lane neighbours, -1 = none) join the chain's ends. */
  int32_t n_chains;
  const int32_t* chain_ptr;      /* [n_chains+1]                             */
  const int32_t* chain_member;   /* dense indices                            */
  const int32_t* chain_head;     /* [n_chains]                               */
  const int32_t* chain_tail;     /* [n_chains]                               */
} ks_graph_desc;

typedef struct {
  int32_t n_tasks;
  int32_t n_lanes;
  int32_t n_edges_unique;
  int32_t chained;          /* 1: every task is lane-chained -> max-plus path */
  int32_t n_ordered;        /* tasks in the topological prefix (n_tasks if acyclic) */
  int32_t n_slots;          /* value slots live at once (smem + spill)       */
  int32_t n_slots_smem;
  int32_t n_levels;         /* longest chain length (levels)                 */
  /* lane-register program (chained graphs with <= 4 lanes, maxplus_lanes):  */
  int32_t has_lanes;
  int32_t n_lane_slots_smem;   /* value slots in shared memory                  */
  int32_t n_lane_slots_global; /* value slots spilled to global memory          */
  int32_t n_lane_cuts;         /* rows where the segment-parallel path may cut  */
  int32_t seg_chain_begin;     /* chain segment [begin, end) replayed numerically */
  int32_t seg_chain_end;       /* between two scans (-1: none)                   */
  int32_t n_carries;           /* values read only in it, live across its start */
} ks_graph_info;

/* Lane-chained flag and topological-prefix length, without building the
 * kernel programs (ks_graph_get_info, ks_graph_levels, ks_simulate*,
 * ks_breakdown and ks_toposort build them on first use). */
int ks_graph_shape(const ks_graph* g, int32_t* chained, int32_t* n_ordered);

/* Build the device-resident frozen graph on `device`.  Frozen row r holds the
 * task order_out[r] (dense input index); rows 0..n_ordered-1 are a topological
 * order.  order_out may be NULL. */
int ks_graph_create(const ks_graph_desc* desc, int device, ks_graph** out,
                    int32_t* order_out);
int ks_graph_get_info(const ks_graph* g, ks_graph_info* info);
/* level[r] (frozen rows, -1 for unordered rows). */
int ks_graph_levels(const ks_graph* g, int32_t* level_out);
int ks_graph_destroy(ks_graph* g);

/* One scale step of a scenario: tasks whose group id lies in [group_lo,
 * group_hi] get d <- round_half_up(d * num / den) (transform.py:174-183).
 * Steps of one scenario apply in order (sequential rounding).
 * num == den == 0 (KS_STEP_REMOVE) removes the matched tasks instead
 * (remove_task, transform.py:249-265: parents x children spliced, the removed
 * task's gap discarded); their start reads -1.  Removal is exact on the
 * max-plus path only (lane-chained graphs); list scheduling rejects it with
 * KS_ERR_UNSUPPORTED. */
#define KS_STEP_REMOVE 0
typedef struct {
  int32_t group_lo;
  int32_t group_hi;
  int64_t num;
  int64_t den;
} ks_scale_step;

typedef struct {
  int32_t n_scenarios;
  /* Dense per-(task, scenario) durations, frozen rows, scenario-minor:
   * dense[r * dense_ld + s].  dense_kind 0 = none, 1 = int32, 2 = int64.
   * Device pointer for ks_simulate, host pointer for ks_simulate_host. */
  int32_t dense_kind;
  const void* dense;
  int64_t dense_ld;
  /* Sparse per-task overrides (set_duration per scenario), HOST arrays:
   * task override_task[k] (frozen row) gets override[k * n_scenarios + s]. */
  int32_t n_overrides;
  const int32_t* override_task;
  const int64_t* override;
  /* Scale program, HOST arrays: scenario s applies
   * scale[scale_ptr[s] .. scale_ptr[s+1]) in order.  NULL = none. */
  const int32_t* scale_ptr;
  const ks_scale_step* scale;
  /* Inserted-task table, HOST arrays: chain_perm[s * perm_ld + off_c + k] is
   * the member (0-based within chain c) placed k-th on the lane; chain_present
   * [s * n_chains + c] = 0 drops the chain's tasks AND their edges. NULL =
   * identity order / all present. */
  const int16_t* chain_perm;
  int32_t perm_ld;
  const uint8_t* chain_present;
  /* VdnnPrefetchPolicy.conv_order rank per frozen row (HOST, -1 = none). */
  const int32_t* vdnn_rank;
} ks_scenarios_desc;

/* Outputs.  For ks_simulate these are DEVICE pointers; for ks_simulate_host
 * HOST pointers.  Any may be NULL (not produced).
 *   start[r * start_ld + s]   frozen row r, scenario s; -1 for absent tasks
 *   makespan[s]
 *   lane_busy[s * n_lanes + l]
 *   schedule[s * n_tasks + k] frozen row dispatched k-th (Alg.1 order) --
 *                             produced by the list-scheduling kernel only
 *   dispatched[s]             tasks dispatched (n_tasks unless Deadlock) */
typedef struct {
  int64_t* start;
  int64_t start_ld;
  int64_t* makespan;
  int64_t* lane_busy;
  int32_t* schedule;
  int32_t* dispatched;
} ks_sim_out;

enum { KS_PATH_AUTO = 0, KS_PATH_MAXPLUS = 1, KS_PATH_LISTSCHED = 2 };

/* Simulate all scenarios on the graph's device, asynchronously on `stream`
 * (a cudaStream_t; NULL = legacy default stream).  `path` forces a kernel
 * (AUTO: max-plus when the graph is chained and no schedule is requested). */
int ks_simulate(const ks_graph* g, const ks_scenarios_desc* sc, int policy,
                int path, const ks_sim_out* out, void* stream);

/* Same, HOST buffers in and out: dense durations are streamed to the device
 * in scenario chunks and results copied back, overlapped on two streams.
 * Synchronous. */
int ks_simulate_host(const ks_graph* g, const ks_scenarios_desc* sc,
                     int policy, int path, const ks_sim_out* out);

/* The same over several devices of one process: graphs[k] is the graph
 * frozen on device k (same description, so the same frozen row order); the
 * scenarios are split into n_graphs contiguous shards simulated concurrently
 * (one host thread per device), each writing its slice of the HOST outputs
 * directly -- no inter-GPU exchange is needed.  Synchronous. */
int ks_simulate_host_multi(const ks_graph* const* graphs, int n_graphs,
                           const ks_scenarios_desc* sc, int policy, int path,
                           const ks_sim_out* out);

/* ---- runtime breakdown (breakdown.py:42-111) ---------------------------- */
enum { KS_BD_CPU = 0, KS_BD_GPU = 1, KS_BD_COMM = 2, KS_BD_CPU_DATALOAD = 3 };
typedef struct {
  const uint8_t* row_class;   /* HOST [n_tasks] by frozen row: KS_BD_* (lane class;
                               * DataLoad tasks on CPU lanes are KS_BD_CPU_DATALOAD) */
  int32_t comm_as_gpu;        /* compute_breakdown keyword arguments          */
  int32_t dataload_as_cpu;
  int32_t gaps_as_cpu_busy;
  const int32_t* row_layer;   /* HOST [n_tasks] layer index by frozen row (the
                               * host maps "no layer" to its own index); NULL =
                               * no per-layer output                           */
  int32_t n_layers;
  const int32_t* schedule;    /* DEVICE [S][n_tasks] dispatch order of a list-
                               * scheduled batch (ks_sim_out.schedule of the same
                               * ks_simulate call); required when the graph is not
                               * lane-chained, NULL otherwise                   */
} ks_breakdown_desc;

/* compute_breakdown / per_layer_breakdown of a max-plus batch, on the device,
 * asynchronously on `stream`.  start / makespan are ks_simulate's DEVICE
 * outputs for the same graph and scenario table `sc` (durations are re-derived
 * from sc).  Outputs (DEVICE):
 *   parts[s * 4 + {0,1,2,3}] = cpu_only, gpu_only, parallel, idle (ns; the four
 *                              sum to makespan[s]); all -1 if a lane's
 *                              intervals were not sorted (negative durations)
 *   layer_busy[(layer * 2 + {0 cpu, 1 gpu}) * S + s]  (may be NULL)
 * Lane-chained graphs use the static lane orders; list-scheduled batches
 * pass their dispatch order in bd->schedule (KS_ERR_UNSUPPORTED if neither). */
int ks_breakdown(const ks_graph* g, const ks_scenarios_desc* sc, const int64_t* start,
                 int64_t start_ld, const int64_t* makespan, const ks_breakdown_desc* bd,
                 int64_t* parts, int64_t* layer_busy, void* stream);

/* verify_acyclic: Kahn order with smallest-id tie-break (graph.py:129-148),
 * computed on the device.  order_out[k] = dense input index; returns
 * KS_ERR_CYCLE if fewer than n_tasks could be ordered (*n_out = ordered). */
int ks_toposort(const ks_graph* g, int32_t* order_out, int32_t* n_out);

/* ---- trace ingest (graph.py:198-312, trace.py:255-265) ------------------ */
typedef struct {
  int64_t n;                   /* events (document order)                  */
  const int64_t* id;           /* external ids                              */
  const uint8_t* kind;         /* TaskKind code: see KS_KIND_*              */
  const int32_t* lane;         /* lane index                                */
  const int64_t* start;        /* ns                                        */
  const int64_t* duration;     /* ns                                        */
  const int64_t* correlation;  /* -1 = none                                 */
  const int32_t* sync_target;  /* lane index or -1 (device-wide)            */
  const uint8_t* is_dtoh;      /* name startswith "memcpy_dtoh"             */
  int32_t n_lanes;
  const uint8_t* lane_class;   /* [n_lanes] 0 cpu, 1 gpu, 2 comm            */
  const int32_t* lane_rank;    /* [n_lanes] rank of str(lane) (sorting)     */
  int32_t strict;              /* OrphanKernel instead of dropping           */
} ks_trace_cols;

enum {
  KS_KIND_CPU_API = 0, KS_KIND_CPU_OTHER = 1, KS_KIND_GPU_KERNEL = 2,
  KS_KIND_GPU_MEMCPY = 3, KS_KIND_DATA_LOAD = 4, KS_KIND_COMM = 5,
  KS_KIND_SYNC = 6
};
enum {
  KS_EDGE_LANE_SEQ_CPU = 0, KS_EDGE_LANE_SEQ_GPU = 1,
  KS_EDGE_LAUNCH_CORRELATION = 2, KS_EDGE_SYNC_BLOCK = 3,
  KS_EDGE_COMM_ORDER = 4, KS_EDGE_INJECTED = 5
};

/* Output of ks_ingest (HOST buffers, caller-allocated; capacities given).
 * Edge k: (edge_src[k], edge_dst[k], edge_kind[k]) as event indices.
 * lane_order: events sorted per lane by (start, id), grouped by lane index;
 * lane_order_ptr[n_lanes+1].  gap[n] per event. */
typedef struct {
  int64_t edge_cap;
  int64_t n_edges;
  int32_t* edge_src;
  int32_t* edge_dst;
  uint8_t* edge_kind;
  int32_t* lane_order;        /* [n]                                      */
  int32_t* lane_order_ptr;    /* [n_lanes+1]                              */
  int64_t* gap;               /* [n]                                      */
  int32_t* launcher;          /* [n] event index of the LaunchCorrelation source or -1 */
  int64_t bad_a, bad_b;       /* OverlapViolation / OrphanKernel ids      */
} ks_ingest_out;

int ks_ingest(const ks_trace_cols* tc, int device, int check_overlaps,
              ks_ingest_out* out);

/* ks_ingest that keeps its edges, lane order and gaps on the device for
 * ks_graph_create_from_ingest (no host round trip of the graph): `out`
 * receives n_edges, lane_order_ptr and launcher only (its edge / lane order /
 * gap buffers may be NULL).  Free *dev_out with ks_ingest_dev_free. */
typedef struct ks_ingest_dev ks_ingest_dev;
int ks_ingest_keep(const ks_trace_cols* tc, int device, int check_overlaps,
                   ks_ingest_out* out, ks_ingest_dev** dev_out);
/* Host copies of a kept ingest's edges / lane order / gaps (any may be NULL). */
int ks_ingest_dev_copy(const ks_ingest_dev* h, int32_t* edge_src, int32_t* edge_dst,
                       uint8_t* edge_kind, int32_t* lane_order, int64_t* gap);
void ks_ingest_dev_free(ks_ingest_dev* h);
/* The frozen graph of a kept ingest (build_graph -> DependencyGraph freeze,
 * graph.py:75-148, 198-245), compiled on its device: unique-edge and
 * predecessor CSR by radix sort, a trace-time topological order verified on
 * every edge (else the host compiler orders it), frozen rows and per-row
 * arrays gathered on the device.  id_rank: HOST [n] rank of the event ids
 * (NULL = ids ascending in event order); flags: HOST [n] KS_TASK_* or NULL.
 * Kernel programs are built on first use (ks_graph_shape is free). */
int ks_graph_create_from_ingest(const ks_ingest_dev* h, const int32_t* id_rank,
                                const uint8_t* flags, ks_graph** out, int32_t* order_out);

/* ---- layer mapping (layers.py:30-81) ------------------------------------ */
typedef struct {
  int64_t n;                  /* markers                                   */
  const int32_t* lane;        /* cpu lane index                            */
  const int64_t* start;
  const int64_t* end;
  const int32_t* tag;         /* (layer, phase) tag id; tags are ranked so
                                 that tag order == (layer, phase.value) order */
} ks_marker_cols;

/* tag_out[i]: tag id for event i, or -1 (unmapped).  CPU-kind events are
 * mapped by innermost containing marker; GPU-kind events inherit from
 * launcher[i].  Returns KS_ERR_AMBIGUOUS (bad_a = event id) on a non-nested
 * tie. */
int ks_map_layers(const ks_trace_cols* tc, const int32_t* launcher,
                  const ks_marker_cols* mc, int device, int32_t* tag_out,
                  int64_t* bad_event);

/* ---- trace documents (trace.py:92-379) ---------------------------------- */
typedef struct ks_trace ks_trace; /* opaque parsed document (host memory) */

typedef struct {
  int64_t n_events;
  int32_t n_lanes;        /* lanes [0, n_event_lanes) are events' lanes in
                           * order of first appearance, then sync targets
                           * (TraceColumns.from_events order); the rest are
                           * lanes named only by layer markers              */
  int32_t n_event_lanes;
  int64_t n_names;        /* distinct event names, first-appearance order   */
  int64_t n_markers;
  int32_t n_layers;       /* distinct marker layer names                    */
  int64_t lane_bytes, name_bytes, layer_bytes;
  /* byte spans of the "gradient_buckets" / "metadata" values in the input
   * text (-1 = absent); the host validates these small objects itself. */
  int64_t buckets_off, buckets_len;
  int64_t metadata_off, metadata_len;
} ks_trace_info;

typedef struct {              /* caller-allocated [n_events]; NULL = skip */
  int64_t* id;
  uint8_t* kind;              /* KS_KIND_*                                 */
  int32_t* lane;
  int64_t* start;             /* ns (us_to_ns, half-up)                    */
  int64_t* duration;
  int64_t* correlation;       /* -1 = none                                 */
  int32_t* sync_target;       /* lane index, -1 = none                     */
  uint8_t* is_dtoh;           /* name startswith "memcpy_dtoh"             */
  int32_t* name_id;
  int64_t* size_bytes;        /* -1 = none                                 */
} ks_trace_event_cols;

typedef struct {              /* caller-allocated [n_markers]              */
  int32_t* lane;
  int64_t* start;
  int64_t* end;
  int32_t* layer_id;
  uint8_t* phase;             /* 0 Forward, 1 Backward, 2 WeightUpdate     */
} ks_trace_marker_cols;

/* Parse + validate a UTF-8 trace document.  n_threads <= 0: all host cores.
 * Errors: KS_ERR_MALFORMED, KS_ERR_SCHEMA, KS_ERR_OVERLAP (err_ids[0..1] =
 * the two event ids), KS_ERR_UNSUPPORTED (values a Python int/str could hold
 * but the columns cannot: ids >= 2^63, float names, non-ASCII numeric
 * strings).  Detail text via ks_last_error_detail(). */
int ks_trace_parse(const char* text, int64_t len, int n_threads, ks_trace** out,
                   int64_t* err_ids);
int ks_trace_get_info(const ks_trace* t, ks_trace_info* info);
int ks_trace_events(const ks_trace* t, const ks_trace_event_cols* cols);
int ks_trace_markers(const ks_trace* t, const ks_trace_marker_cols* cols);
/* which: 0 lanes, 1 names, 2 layers.  bytes[offsets[i] .. offsets[i+1]). */
int ks_trace_strings(const ks_trace* t, int which, char* bytes, int64_t* offsets);
void ks_trace_destroy(ks_trace* t);

/* ---- CUPTI activity recording (Daydream's trace collection) ------------
 * Records this process's CUDA activity -- runtime API calls (CPU thread
 * lanes), kernels / copies / memsets (stream lanes), synchronisations and
 * NVTX ranges named "<layer>/<Forward|Backward|WeightUpdate>" (layer
 * markers) -- into the trace columns ks_trace_parse produces (the reference
 * reads the same schema from JSON only, trace.py:281-328).  libcupti is
 * loaded at run time (KS_ERR_UNSUPPORTED without it). */
typedef struct ks_cupti_trace ks_cupti_trace;
int ks_cupti_start(void);
int ks_cupti_stop(ks_cupti_trace** out);
int ks_cupti_info_get(const ks_cupti_trace* t, ks_trace_info* info, int64_t* t0_ns,
                      int64_t* dropped);
int ks_cupti_events(const ks_cupti_trace* t, const ks_trace_event_cols* cols);
int ks_cupti_markers(const ks_cupti_trace* t, const ks_trace_marker_cols* cols);
int ks_cupti_strings(const ks_cupti_trace* t, int which, char* bytes, int64_t* offsets);
void ks_cupti_destroy(ks_cupti_trace* t);

typedef struct {
  int64_t n_events;
  const int64_t* id;
  const uint8_t* kind;
  const int32_t* lane;
  const int64_t* start;
  const int64_t* duration;
  const int64_t* correlation;   /* -1 = none; NULL = none for all            */
  const int32_t* sync_target;   /* -1 = none; may be NULL                    */
  const int32_t* name_id;
  const int64_t* size_bytes;    /* -1 = none; may be NULL                    */
  int32_t n_lanes;
  const char* lane_bytes;
  const int64_t* lane_off;      /* [n_lanes+1]                               */
  int64_t n_names;
  const char* name_bytes;
  const int64_t* name_off;
  int64_t n_markers;
  const int32_t* m_lane;
  const int64_t* m_start;
  const int64_t* m_end;
  const int32_t* m_layer;
  const uint8_t* m_phase;
  int32_t n_layers;
  const char* layer_bytes;
  const int64_t* layer_off;
  const char* extra_json;       /* raw extra top-level members, or NULL     */
} ks_trace_write_desc;

/* Columns -> document text in a malloc'ed buffer (free: ks_buffer_free). */
int ks_trace_write(const ks_trace_write_desc* d, int n_threads, char** out,
                   int64_t* out_len);
void ks_buffer_free(char* p);

/* ---- misc ---------------------------------------------------------------- */
const char* ks_error_name(int code);
const char* ks_last_error_detail(void);
int ks_device_count(int* n);
/* Number of kernels this library launched on the calling process so far. */
int64_t ks_launch_count(void);
const char* ks_version(void);
/* Diagnostics of the per-graph NVRTC specialisation (status + compile log). */
const char* ks_jit_log(void);
/* Traffic-pattern probe (bench.py): dst[i] = src[i] for n int32 -> int64 on
 * the device, asynchronously on `stream` -- the lanes kernel's compulsory HBM
 * traffic without the recurrence.  16-byte aligned pointers. */
int ks_probe_widen(const int32_t* src, int64_t* dst, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DDSIM_H_ */
