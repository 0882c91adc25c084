// Trace ingest kernels (build_graph / link_syncs / compute_gaps /
// check_lane_overlaps / map_tasks_to_layers) -- see ingest notes in DESIGN.md.
#include "ddsim_internal.h"

extern "C" int ks_ingest(const ks_trace_cols*, int, int, ks_ingest_out*) { return KS_ERR_UNSUPPORTED; }
extern "C" int ks_map_layers(const ks_trace_cols*, const int32_t*, const ks_marker_cols*, int,
                             int32_t*, int64_t*) {
  return KS_ERR_UNSUPPORTED;
}
