// cupti_trace: record this process's CUDA activity with CUPTI straight into
// trace columns (the reference's trace schema, trace.py:20-90; its reader is
// JSON-only, trace.py:281-328).  Daydream collects exactly these records: CPU
// runtime-API calls with their correlation ids, the kernels / copies they
// launch on each stream, the synchronisations that block a CPU thread, and
// framework layer ranges (here NVTX ranges named "<layer>/<phase>").
//
// Mapping (host C++, libcupti loaded at run time):
//   runtime API record   -> CpuApi on "cpu:<thread>", correlation = CUPTI's;
//                           a synchronous cudaMemcpy* whose copy is device-to-
//                           host is named "memcpy_dtoh:<api>" (rule 4's dtoh
//                           link, graph.py:286-297)
//   synchronisation      -> the API event becomes Sync; stream synchronise
//                           targets that stream's lane, context / event
//                           synchronise are device-wide (no target: every GPU
//                           lane, graph.py:256-258); stream-wait-event is a
//                           GPU-side wait and adds nothing
//   kernel               -> GpuKernel on "gpu:<device>:<stream>"
//   memcpy / memset      -> GpuMemcpy on the stream's lane (size_bytes = bytes)
//   NVTX range "L/Phase" -> layer marker on the pushing thread's lane
// Times are CUPTI's ns, relative to the first record; events are numbered in
// (start, end, kind) order.
#include <cupti.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "ddsim_internal.h"

namespace ddsim {
void set_last_error(const std::string& msg);
}

namespace {

struct Cupti {
  bool ok = false;
  std::string err;
  CUptiResult (*register_callbacks)(CUpti_BuffersCallbackRequestFunc,
                                    CUpti_BuffersCallbackCompleteFunc) = nullptr;
  CUptiResult (*enable)(CUpti_ActivityKind) = nullptr;
  CUptiResult (*disable)(CUpti_ActivityKind) = nullptr;
  CUptiResult (*flush_all)(uint32_t) = nullptr;
  CUptiResult (*next_record)(uint8_t*, size_t, CUpti_Activity**) = nullptr;
  CUptiResult (*callback_name)(CUpti_CallbackDomain, uint32_t, const char**) = nullptr;
};

std::mutex g_mu;
Cupti g_cu;
bool g_loaded = false;
bool g_running = false;
std::vector<std::pair<uint8_t*, size_t>> g_buffers;  // completed (buffer, valid bytes)

const CUpti_ActivityKind kKinds[] = {
    CUPTI_ACTIVITY_KIND_RUNTIME, CUPTI_ACTIVITY_KIND_DRIVER, CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL,
    CUPTI_ACTIVITY_KIND_MEMCPY, CUPTI_ACTIVITY_KIND_MEMSET, CUPTI_ACTIVITY_KIND_SYNCHRONIZATION,
    CUPTI_ACTIVITY_KIND_MARKER};

template <class F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

void load_locked() {
  if (g_loaded) return;
  g_loaded = true;
  const char* libs[] = {"/usr/local/cuda/lib64/libcupti.so", "/usr/local/cuda/extras/CUPTI/lib64/libcupti.so",
                        "libcupti.so.12", "libcupti.so"};
  void* h = nullptr;
  for (const char* l : libs)
    if ((h = dlopen(l, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
  if (!h) {
    g_cu.err = std::string("dlopen libcupti failed: ") + (dlerror() ? dlerror() : "?");
    return;
  }
  g_cu.ok = sym(h, "cuptiActivityRegisterCallbacks", g_cu.register_callbacks) &&
            sym(h, "cuptiActivityEnable", g_cu.enable) && sym(h, "cuptiActivityDisable", g_cu.disable) &&
            sym(h, "cuptiActivityFlushAll", g_cu.flush_all) &&
            sym(h, "cuptiActivityGetNextRecord", g_cu.next_record) &&
            sym(h, "cuptiGetCallbackName", g_cu.callback_name);
  if (!g_cu.ok) g_cu.err = "libcupti lacks an activity API entry point";
}

constexpr size_t kBufBytes = 8u << 20;

void CUPTIAPI buffer_requested(uint8_t** buffer, size_t* size, size_t* max_records) {
  *buffer = static_cast<uint8_t*>(aligned_alloc(8, kBufBytes));
  *size = *buffer ? kBufBytes : 0;
  *max_records = 0;
}

void CUPTIAPI buffer_completed(CUcontext, uint32_t, uint8_t* buffer, size_t, size_t valid) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_buffers.emplace_back(buffer, valid);
}

bool is_sync_memcpy_api(const std::string& n) {
  return n.rfind("cudaMemcpy", 0) == 0 && n.find("Async") == std::string::npos;
}

}  // namespace

// ---------------------------------------------------------------------------
struct ks_cupti_trace {
  std::vector<int64_t> id, start, dur, corr, size_bytes;
  std::vector<uint8_t> kind;
  std::vector<int32_t> lane, sync_target, name_id;
  std::vector<std::string> lanes, names, layers;
  int32_t n_event_lanes = 0;
  std::vector<int32_t> m_lane, m_layer;
  std::vector<int64_t> m_start, m_end;
  std::vector<uint8_t> m_phase;
  int64_t t0 = 0;
  int64_t dropped = 0;  // records of kinds outside the schema
};

namespace {

struct Ev {
  int64_t start, end;
  uint8_t kind;
  std::string lane, name;
  int64_t corr = -1;
  std::string sync_target;  // "" none
  int64_t size = -1;
};

int phase_code(const std::string& p) {
  if (p == "Forward") return 0;
  if (p == "Backward") return 1;
  if (p == "WeightUpdate") return 2;
  return -1;
}

std::string gpu_lane(uint32_t dev, uint32_t stream) {
  return "gpu:" + std::to_string(dev) + ":" + std::to_string(stream);
}

}  // namespace

extern "C" int ks_cupti_start(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  load_locked();
  if (!g_cu.ok) {
    ddsim::set_last_error(g_cu.err);
    return KS_ERR_UNSUPPORTED;
  }
  if (g_running) {
    ddsim::set_last_error("CUPTI recording already running");
    return KS_ERR_INVALID;
  }
  for (auto& b : g_buffers) free(b.first);
  g_buffers.clear();
  if (g_cu.register_callbacks(buffer_requested, buffer_completed) != CUPTI_SUCCESS) {
    ddsim::set_last_error("cuptiActivityRegisterCallbacks failed");
    return KS_ERR_CUDA;
  }
  for (CUpti_ActivityKind k : kKinds)
    if (g_cu.enable(k) != CUPTI_SUCCESS) {
      ddsim::set_last_error("cuptiActivityEnable failed for kind " + std::to_string((int)k));
      return KS_ERR_CUDA;
    }
  g_running = true;
  return KS_OK;
}

extern "C" int ks_cupti_stop(ks_cupti_trace** out) {
  if (!out) return KS_ERR_INVALID;
  *out = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_running) {
      ddsim::set_last_error("CUPTI recording not running");
      return KS_ERR_INVALID;
    }
  }
  cudaDeviceSynchronize();
  g_cu.flush_all(1);  // completes buffers through buffer_completed (takes g_mu)
  std::vector<std::pair<uint8_t*, size_t>> bufs;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (CUpti_ActivityKind k : kKinds) g_cu.disable(k);
    g_running = false;
    bufs.swap(g_buffers);
  }
  auto* T = new ks_cupti_trace();
  std::vector<Ev> ev;
  std::unordered_map<uint32_t, size_t> api_of_corr;        // correlation -> API event
  std::unordered_map<uint32_t, uint32_t> dev_of_ctx;       // context -> device
  struct Sync {
    uint32_t corr, ctx, stream;
    int type;
  };
  std::vector<Sync> syncs;
  std::unordered_map<uint32_t, int> copy_kind_of_corr;     // correlation -> memcpy kind
  struct Mk {
    int64_t start = -1, end = -1;
    uint64_t tid = 0;
    std::string name;
  };
  std::map<uint32_t, Mk> ranges;
  std::vector<Ev> drivers;
  for (auto& b : bufs) {
    CUpti_Activity* rec = nullptr;
    while (g_cu.next_record(b.first, b.second, &rec) == CUPTI_SUCCESS) {
      switch (rec->kind) {
        case CUPTI_ACTIVITY_KIND_RUNTIME: {
          auto* a = reinterpret_cast<CUpti_ActivityAPI*>(rec);
          const char* nm = nullptr;
          g_cu.callback_name(CUPTI_CB_DOMAIN_RUNTIME_API, a->cbid, &nm);
          Ev e{(int64_t)a->start, (int64_t)a->end, 0, "cpu:" + std::to_string(a->threadId),
               nm ? nm : "cudaRuntimeApi"};
          e.corr = a->correlationId;
          api_of_corr[a->correlationId] = ev.size();
          ev.push_back(std::move(e));
          break;
        }
        case CUPTI_ACTIVITY_KIND_DRIVER: {
          // kept only when it launched GPU work itself (libraries such as
          // cuBLAS call the driver directly); driver calls nested inside a
          // runtime call share nothing with the GPU records and are dropped
          auto* a = reinterpret_cast<CUpti_ActivityAPI*>(rec);
          const char* nm = nullptr;
          g_cu.callback_name(CUPTI_CB_DOMAIN_DRIVER_API, a->cbid, &nm);
          Ev e{(int64_t)a->start, (int64_t)a->end, 0, "cpu:" + std::to_string(a->threadId),
               nm ? nm : "cuDriverApi"};
          e.corr = a->correlationId;
          drivers.push_back(std::move(e));
          break;
        }
        case CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL:
        case CUPTI_ACTIVITY_KIND_KERNEL: {
          auto* k = reinterpret_cast<CUpti_ActivityKernel9*>(rec);
          Ev e{(int64_t)k->start, (int64_t)k->end, 2, gpu_lane(k->deviceId, k->streamId),
               k->name ? k->name : "kernel"};
          e.corr = k->correlationId;
          dev_of_ctx[k->contextId] = k->deviceId;
          ev.push_back(std::move(e));
          break;
        }
        case CUPTI_ACTIVITY_KIND_MEMCPY: {
          auto* m = reinterpret_cast<CUpti_ActivityMemcpy6*>(rec);
          Ev e{(int64_t)m->start, (int64_t)m->end, 3, gpu_lane(m->deviceId, m->streamId),
               "memcpy_" + std::to_string((int)m->copyKind)};
          e.corr = m->correlationId;
          e.size = (int64_t)m->bytes;
          copy_kind_of_corr[m->correlationId] = (int)m->copyKind;
          dev_of_ctx[m->contextId] = m->deviceId;
          ev.push_back(std::move(e));
          break;
        }
        case CUPTI_ACTIVITY_KIND_MEMSET: {
          auto* m = reinterpret_cast<CUpti_ActivityMemset4*>(rec);
          Ev e{(int64_t)m->start, (int64_t)m->end, 3, gpu_lane(m->deviceId, m->streamId), "memset"};
          e.corr = m->correlationId;
          e.size = (int64_t)m->bytes;
          dev_of_ctx[m->contextId] = m->deviceId;
          ev.push_back(std::move(e));
          break;
        }
        case CUPTI_ACTIVITY_KIND_SYNCHRONIZATION: {
          auto* s = reinterpret_cast<CUpti_ActivitySynchronization2*>(rec);
          syncs.push_back({s->correlationId, s->contextId, s->streamId, (int)s->type});
          break;
        }
        case CUPTI_ACTIVITY_KIND_MARKER: {
          auto* m = reinterpret_cast<CUpti_ActivityMarker2*>(rec);
          Mk& r = ranges[m->id];
          if (m->flags & CUPTI_ACTIVITY_FLAG_MARKER_START) {
            r.start = (int64_t)m->timestamp;
            r.tid = (uint64_t)m->objectId.pt.threadId;
            if (m->name) r.name = m->name;
          } else if (m->flags & CUPTI_ACTIVITY_FLAG_MARKER_END) {
            r.end = (int64_t)m->timestamp;
          }
          break;
        }
        default:
          ++T->dropped;
      }
    }
    free(b.first);
  }
  // driver calls that launched GPU work and have no runtime call of their own
  {
    std::unordered_map<int64_t, int> gpu_corr;
    for (const Ev& e : ev)
      if (e.kind == 2 || e.kind == 3) gpu_corr[e.corr] = 1;
    for (Ev& d : drivers)
      if (gpu_corr.count(d.corr) && !api_of_corr.count((uint32_t)d.corr)) {
        api_of_corr[(uint32_t)d.corr] = ev.size();
        ev.push_back(std::move(d));
      } else {
        ++T->dropped;
      }
  }
  // synchronisations turn their API call into a Sync event
  for (const Sync& s : syncs) {
    auto it = api_of_corr.find(s.corr);
    if (it == api_of_corr.end()) continue;
    Ev& e = ev[it->second];
    if (s.type == CUPTI_ACTIVITY_SYNCHRONIZATION_TYPE_STREAM_WAIT_EVENT) continue;
    e.kind = 6;
    if (s.type == CUPTI_ACTIVITY_SYNCHRONIZATION_TYPE_STREAM_SYNCHRONIZE) {
      auto d = dev_of_ctx.find(s.ctx);
      e.sync_target = gpu_lane(d == dev_of_ctx.end() ? 0 : d->second, s.stream);
    }
  }
  // a synchronous device-to-host copy blocks its thread (rule 4's dtoh link)
  for (auto& kv : copy_kind_of_corr) {
    if (kv.second != CUPTI_ACTIVITY_MEMCPY_KIND_DTOH) continue;
    auto it = api_of_corr.find(kv.first);
    if (it == api_of_corr.end()) continue;
    Ev& e = ev[it->second];
    if (e.kind == 0 && is_sync_memcpy_api(e.name)) e.name = "memcpy_dtoh:" + e.name;
  }
  // document order and numbering
  std::sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
    if (a.start != b.start) return a.start < b.start;
    if (a.end != b.end) return a.end < b.end;
    return a.kind < b.kind;
  });
  int64_t t0 = ev.empty() ? 0 : ev.front().start;
  for (auto& kv : ranges)
    if (kv.second.start >= 0) t0 = std::min(t0, kv.second.start);
  T->t0 = t0;
  std::unordered_map<std::string, int32_t> lane_ix, name_ix, layer_ix;
  auto lix = [&](const std::string& l) {
    auto it = lane_ix.find(l);
    if (it != lane_ix.end()) return it->second;
    const int32_t i = (int32_t)T->lanes.size();
    lane_ix.emplace(l, i);
    T->lanes.push_back(l);
    return i;
  };
  const size_t n = ev.size();
  T->id.resize(n);
  T->start.resize(n);
  T->dur.resize(n);
  T->corr.resize(n);
  T->size_bytes.resize(n);
  T->kind.resize(n);
  T->lane.resize(n);
  T->sync_target.resize(n);
  T->name_id.resize(n);
  for (size_t i = 0; i < n; ++i) {
    const Ev& e = ev[i];
    T->id[i] = (int64_t)i;
    T->start[i] = e.start - t0;
    T->dur[i] = std::max<int64_t>(0, e.end - e.start);
    T->corr[i] = e.corr;
    T->size_bytes[i] = e.size;
    T->kind[i] = e.kind;
    T->lane[i] = lix(e.lane);
    auto nit = name_ix.find(e.name);
    if (nit == name_ix.end()) {
      nit = name_ix.emplace(e.name, (int32_t)T->names.size()).first;
      T->names.push_back(e.name);
    }
    T->name_id[i] = nit->second;
  }
  for (size_t i = 0; i < n; ++i) T->sync_target[i] = ev[i].sync_target.empty() ? -1 : lix(ev[i].sync_target);
  T->n_event_lanes = (int32_t)T->lanes.size();
  // layer markers: NVTX ranges named "<layer>/<Forward|Backward|WeightUpdate>"
  for (auto& kv : ranges) {
    const Mk& r = kv.second;
    if (r.start < 0 || r.end < r.start) continue;
    const size_t slash = r.name.rfind('/');
    if (slash == std::string::npos || slash == 0) continue;
    const int ph = phase_code(r.name.substr(slash + 1));
    if (ph < 0) continue;
    const std::string layer = r.name.substr(0, slash);
    auto it = layer_ix.find(layer);
    if (it == layer_ix.end()) {
      it = layer_ix.emplace(layer, (int32_t)T->layers.size()).first;
      T->layers.push_back(layer);
    }
    T->m_lane.push_back(lix("cpu:" + std::to_string(r.tid)));
    T->m_start.push_back(r.start - t0);
    T->m_end.push_back(r.end - t0);
    T->m_layer.push_back(it->second);
    T->m_phase.push_back((uint8_t)ph);
  }
  *out = T;
  return KS_OK;
}

extern "C" int ks_cupti_info_get(const ks_cupti_trace* t, ks_trace_info* info,
                                 int64_t* t0_ns, int64_t* dropped) {
  if (!t || !info) return KS_ERR_INVALID;
  memset(info, 0, sizeof(*info));
  info->n_events = (int64_t)t->id.size();
  info->n_lanes = (int32_t)t->lanes.size();
  info->n_event_lanes = t->n_event_lanes;
  info->n_names = (int64_t)t->names.size();
  info->n_markers = (int64_t)t->m_start.size();
  info->n_layers = (int32_t)t->layers.size();
  auto bytes = [](const std::vector<std::string>& v) {
    int64_t b = 0;
    for (auto& s : v) b += (int64_t)s.size();
    return b;
  };
  info->lane_bytes = bytes(t->lanes);
  info->name_bytes = bytes(t->names);
  info->layer_bytes = bytes(t->layers);
  info->buckets_off = info->metadata_off = -1;
  if (t0_ns) *t0_ns = t->t0;
  if (dropped) *dropped = t->dropped;
  return KS_OK;
}

extern "C" int ks_cupti_events(const ks_cupti_trace* t, const ks_trace_event_cols* c) {
  if (!t || !c) return KS_ERR_INVALID;
  const size_t n = t->id.size();
  auto put = [n](auto* dst, const auto& src) {
    if (dst && n) std::memcpy(dst, src.data(), n * sizeof(src[0]));
  };
  put(c->id, t->id);
  put(c->kind, t->kind);
  put(c->lane, t->lane);
  put(c->start, t->start);
  put(c->duration, t->dur);
  put(c->correlation, t->corr);
  put(c->sync_target, t->sync_target);
  put(c->name_id, t->name_id);
  put(c->size_bytes, t->size_bytes);
  if (c->is_dtoh)
    for (size_t i = 0; i < n; ++i)
      c->is_dtoh[i] = t->names[t->name_id[i]].rfind("memcpy_dtoh", 0) == 0 ? 1 : 0;
  return KS_OK;
}

extern "C" int ks_cupti_markers(const ks_cupti_trace* t, const ks_trace_marker_cols* c) {
  if (!t || !c) return KS_ERR_INVALID;
  const size_t m = t->m_start.size();
  auto put = [m](auto* dst, const auto& src) {
    if (dst && m) std::memcpy(dst, src.data(), m * sizeof(src[0]));
  };
  put(c->lane, t->m_lane);
  put(c->start, t->m_start);
  put(c->end, t->m_end);
  put(c->layer_id, t->m_layer);
  put(c->phase, t->m_phase);
  return KS_OK;
}

// which: 0 lanes, 1 event names, 2 layers; offsets[k+1] - offsets[k] = length
extern "C" int ks_cupti_strings(const ks_cupti_trace* t, int which, char* bytes, int64_t* offsets) {
  if (!t || which < 0 || which > 2) return KS_ERR_INVALID;
  const auto& v = which == 0 ? t->lanes : which == 1 ? t->names : t->layers;
  int64_t o = 0;
  for (size_t k = 0; k < v.size(); ++k) {
    if (offsets) offsets[k] = o;
    if (bytes) std::memcpy(bytes + o, v[k].data(), v[k].size());
    o += (int64_t)v[k].size();
  }
  if (offsets) offsets[v.size()] = o;
  return KS_OK;
}

extern "C" void ks_cupti_destroy(ks_cupti_trace* t) { delete t; }
