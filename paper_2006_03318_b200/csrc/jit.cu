// Per-graph specialisation of the maxplus_lanes kernel with NVRTC.
//
// The static kernel dispatches each record through a 256-way switch that
// nvcc lowers to an 8-level branch tree.  A graph only uses a handful of
// handler codes (own lane x predecessor-lane mask x gap), so the graph
// compiler records them with their frequencies and this file compiles, once
// per distinct code list, a kernel whose dispatch is an if-chain over exactly
// those codes in frequency order (the common record resolves in 1-2
// compares).  NVRTC and the driver entry points are resolved at run time;
// if either is unavailable the static kernel runs instead (same results).
#include <dlfcn.h>

#include <cstdio>

#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "ddsim_internal.h"

namespace ddsim {
namespace {

#include "generated/lanes_body_src.inc"  // const char* kLanesBodySrc
#include "generated/lanes_seg_src.inc"   // const char* kSegBodySrc

typedef int nvrtcResult_t;
typedef void* nvrtcProgram_t;
struct Nvrtc {
  bool ok = false;
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                          const char* const*) = nullptr;
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*) = nullptr;
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*log)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*destroy)(nvrtcProgram_t*) = nullptr;
};

struct Driver {
  bool ok = false;
  CUresult (*load)(CUmodule*, const void*) = nullptr;
  CUresult (*getfn)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*setattr)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                     unsigned, CUstream, void**, void**) = nullptr;
};

std::mutex g_mu;
Nvrtc g_nv;
Driver g_drv;
bool g_init = false;
std::map<std::string, CUfunction> g_cache;
std::string g_jit_log;

template <class F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

template <class F>
bool drv(const char* name, F& out) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return false;
  out = reinterpret_cast<F>(p);
  return true;
}

void init_locked() {
  if (g_init) return;
  g_init = true;
  if (getenv("DDSIM_NO_JIT")) return;
  const char* libs[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so"};
  void* h = nullptr;
  for (const char* l : libs)
    if ((h = dlopen(l, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
  if (!h) {
    g_jit_log = std::string("dlopen nvrtc failed: ") + (dlerror() ? dlerror() : "?");
    return;
  }
  g_nv.ok = sym(h, "nvrtcCreateProgram", g_nv.create) && sym(h, "nvrtcCompileProgram", g_nv.compile) &&
            sym(h, "nvrtcGetCUBINSize", g_nv.cubin_size) && sym(h, "nvrtcGetCUBIN", g_nv.cubin) &&
            sym(h, "nvrtcGetProgramLogSize", g_nv.log_size) &&
            sym(h, "nvrtcGetProgramLog", g_nv.log) && sym(h, "nvrtcDestroyProgram", g_nv.destroy);
  g_drv.ok = drv("cuModuleLoadData", g_drv.load) && drv("cuModuleGetFunction", g_drv.getfn) &&
             drv("cuFuncSetAttribute", g_drv.setattr) && drv("cuLaunchKernel", g_drv.launch);
  g_jit_log = std::string("nvrtc ") + (g_nv.ok ? "ok" : "missing symbols") + ", driver " +
              (g_drv.ok ? "ok" : "missing entry points");
}

std::string make_source(const std::vector<int>& codes, int dk, int V, bool dyn, bool ch,
                        bool nolb, bool scale) {
  std::string disp = "#define DDSIM_DISPATCH(h) ";
  if (dyn) disp += "hstep_dyn<V>(S, h, d0, d1, gap, sp, ld, store); if (0) ";
  for (size_t i = 0; i < codes.size(); ++i) {
    const int c = codes[i];
    disp += (i ? "else if (h == " : "if (h == ") + std::to_string(c) + "u) hstep<" +
            std::to_string(c & 3) + ", " + std::to_string((c >> 2) & 31) + ", " +
            std::to_string((c >> 7) & 1) + ", V>(S, d0, d1, gap, sp, ld, store); ";
  }
  disp += "else __trap();\n";
  std::string src = "#define DDSIM_LANES_NO_STD_TYPES 1\n";
  if (dk == 0 && !scale) src += "#define DDSIM_DERIVED_SCALE 0\n";
  // record-loop unrolling by 2 lets the next record's decode overlap this
  // record's max-plus chain: branch-free handler config 2 -8 %, config 3 -26 %;
  // if-chain handler config 4 -0.5 % (13.55 -> 13.49 ms, 3 interleaved repeats);
  // 4 is slower (15.3 ms: instruction cache)
  if (const char* u = getenv("DDSIM_JIT_UNROLL"))
    src += std::string("#define DDSIM_UNROLL ") + u + "\n";
  else
    src += "#define DDSIM_UNROLL 2\n";
  // the branch-free handler leaves lane busy to launch_lanes_busy (12 of ~90
  // instructions per record are select-based lane-busy updates otherwise)
  if (nolb) src += "#define DDSIM_NO_LB 1\n";
  if (const char* st = getenv("DDSIM_LANES_STAGES")) src += std::string("#define DDSIM_STAGES ") + st + "\n";
  std::string body = kLanesBodySrc;
  if (const char* alt = getenv("DDSIM_LANES_BODY")) {  // experiments: alternative body file
    if (FILE* f = fopen(alt, "rb")) {
      std::string b;
      char buf[4096];
      size_t k;
      while ((k = fread(buf, 1, sizeof buf, f)) > 0) b.append(buf, k);
      fclose(f);
      body = b;
    }
  }
  src += disp + body;
  src += "\nextern \"C\" __global__ void __launch_bounds__(256) ddsim_lanes_jit("
         "const __grid_constant__ ddsim_lanes::Tmap tmap, const ddsim_lanes::Params p" +
         std::string(ch ? ", const __grid_constant__ ddsim_lanes::ChainParams cp" : "") +
         std::string(dk == 0 ? ", const __grid_constant__ ddsim_lanes::DerivedParams dp" : "") +
         ") {\n  ddsim_lanes::lanes_body<" + std::to_string(dk) + ", " + std::to_string(V) +
         (ch ? ", true" : ", false") +
         (dk == 0 ? std::string(", false>(&tmap, p, ") + (ch ? "&cp" : "nullptr") +
                        ", nullptr, 0, 0, nullptr, &dp);\n}\n"
                  : std::string(">(&tmap, p") + (ch ? ", &cp" : "") + ");\n}\n");
  return src;
}

// Compile `src` once per key (NVRTC -> cubin -> module) and return `fname`;
// failures are cached as nullptr too (no retry of a failing compile).
// The source is generated only on a cache miss: it is ~100 KB of text, and
// building it on every launch cost several microseconds of host time per
// kernel (config 1's whole call is ~60 us of host work).
template <class MakeSrc>
CUfunction get_compiled(const std::string& key, MakeSrc make_src, const char* fname) {
  if (getenv("DDSIM_NO_JIT")) return nullptr;  // checked per call (tests switch paths)
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  if (!g_nv.ok || !g_drv.ok) return nullptr;
  auto it = g_cache.find(key);
  if (it != g_cache.end()) return it->second;
  const std::string src = make_src();
  nvrtcProgram_t prog = nullptr;
  CUfunction fn = nullptr;
  if (g_nv.create(&prog, src.c_str(), "ddsim_lanes_jit.cu", 0, nullptr, nullptr) == 0) {
    // --device-int128: the half-up Shrink of derived durations (lanes_body.cuh)
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                          "--device-int128"};
    const int rc = g_nv.compile(prog, 4, opts);
    size_t ls = 0;
    g_nv.log_size(prog, &ls);
    if (ls > 1) {
      std::string lg(ls, '\0');
      g_nv.log(prog, &lg[0]);
      lg.resize(ls - 1);
      g_jit_log += "\nnvrtc log: " + lg;
    }
    if (rc == 0) {
      size_t n = 0;
      g_nv.cubin_size(prog, &n);
      std::vector<char> bin(n);
      g_nv.cubin(prog, bin.data());
      CUmodule mod = nullptr;
      const CUresult lr = g_drv.load(&mod, bin.data());
      if (lr != CUDA_SUCCESS) {
        g_jit_log += "\ncuModuleLoadData failed: " + std::to_string((int)lr);
      } else if (g_drv.getfn(&fn, mod, fname) != CUDA_SUCCESS) {
        g_jit_log += "\ncuModuleGetFunction failed";
        fn = nullptr;
      } else {
        g_jit_log += "\ncompiled " + key;
      }
    } else {
      g_jit_log += "\nnvrtc compile failed rc=" + std::to_string(rc);
    }
    g_nv.destroy(&prog);
  }
  g_cache[key] = fn;
  return fn;
}

CUfunction get_function(const std::vector<int>& codes, int dk, int V, bool dyn, bool ch,
                        bool nolb, bool scale, int device) {
  std::string key = std::to_string(device) + ":" + std::to_string(dk) + ":" + std::to_string(V) +
                    (dyn ? ":dyn" : "") + (ch ? ":ch" : "") + (nolb ? ":nolb:" : ":") +
                    (dk == 0 && !scale ? "noscale:" : "");
  if (const char* u = getenv("DDSIM_JIT_UNROLL")) key += std::string("u") + u + ":";
  if (const char* st = getenv("DDSIM_LANES_STAGES")) key += std::string("st") + st + ":";
  if (const char* b = getenv("DDSIM_LANES_BODY")) key += std::string("b") + b + ":";
  for (int c : codes) key += std::to_string(c) + ",";
  if (getenv("DDSIM_NO_JIT")) return nullptr;
  return get_compiled(key, [&] { return make_source(codes, dk, V, dyn, ch, nolb, scale); },
                      "ddsim_lanes_jit");
}

// Segment kernels (SegParams in lanes_body.cuh): the transfer pass in
// coefficient form (lanes_seg.cuh) and the replay pass (lanes_body<..., SEG>),
// both with the graph's handler codes as an if-chain.
// mode: 0 replay, 1 transfer, 2 fused (transfer + look-back + replay)
std::string seg_source(const std::vector<int>& codes, int dk, int LN, bool ch, int mode,
                       bool scale) {
  std::string src = "#define DDSIM_LANES_NO_STD_TYPES 1\n";
  if (dk == 0 && !scale) src += "#define DDSIM_DERIVED_SCALE 0\n";
  // record loop unrolled x2, except with derived durations (DK 0): the
  // duration derivation doubles the body and instruction-cache misses cost more
  // than the overlap buys (config 3: 1.28 -> 1.16 ms rolled; config 2, DK 2:
  // 0.182 ms unrolled vs 0.190 rolled)
  if (const char* u = getenv("DDSIM_SEG_UNROLL"))  // experiments
    src += std::string("#define DDSIM_UNROLL ") + u + "\n";
  else if (dk != 0)
    src += "#define DDSIM_UNROLL 2\n";
  std::string bounds = "256";
  if (const char* mb = getenv("DDSIM_SEG_MINB")) bounds = std::string("128, ") + mb;
  // TMA pipeline depth: 2 chunks for duration tiles (smaller CTAs, more of them
  // per SM: config 4 at 8,192 scenarios 2.67 -> 2.48 ms), 4 for derived
  // durations (no tiles; config 3 insensitive)
  if (const char* st = getenv("DDSIM_SEG_STAGES"))  // experiments (>= 2)
    src += std::string("#define DDSIM_STAGES ") + st + "\n";
  else if (dk != 0)
    src += "#define DDSIM_STAGES 2\n";
  std::string disp = "#define DDSIM_DISPATCH(h) ";
  std::string sdisp = "#define DDSIM_SYM_DISPATCH(h) ";
  std::string sdisp2 = "#define DDSIM_SYM_DISPATCH2(h) ";
  for (size_t i = 0; i < codes.size(); ++i) {
    const int c = codes[i];
    const std::string tp = std::to_string(c & 3) + ", " + std::to_string((c >> 2) & 31) + ", " +
                           std::to_string((c >> 7) & 1);
    const std::string cond = (i ? "else if (h == " : "if (h == ") + std::to_string(c) + "u) ";
    disp += cond + "hstep<" + tp + ", V>(S, d0, d1, gap, sp, ld, store); ";
    sdisp += cond + "hsym<" + tp + ", LN>(Y, dv, gp); ";
    sdisp2 += cond + "{ hsym<" + tp + ", LN>(Y, dv, gp); hsym<" + tp + ", LN>(Y2, dv2, gp); } ";
  }
  disp += "else __trap();\n";
  sdisp += "else __trap();\n";
  sdisp2 += "else __trap();\n";
  src += disp + sdisp + sdisp2 + kLanesBodySrc + "\n" + kSegBodySrc + "\n";
  const char* names[] = {"ddsim_seg_replay", "ddsim_seg_transfer", "ddsim_seg_fused",
                         "ddsim_seg_transfer2", "ddsim_seg_replay2"};
  const char* bodies[] = {"replay_body", "sym_body", "fused_body", "sym_body2", "replay_body2"};
  src += std::string("extern \"C\" __global__ void __launch_bounds__(") + bounds + ") " + names[mode] +
         "(const __grid_constant__ ddsim_lanes::Tmap tmap, const ddsim_lanes::Params p, "
         "const ddsim_lanes::SegParams sg" +
         (ch ? ", const __grid_constant__ ddsim_lanes::ChainParams cp" : "") +
         (dk == 0 ? ", const __grid_constant__ ddsim_lanes::DerivedParams dp" : "") +
         ") {\n  ddsim_lanes::" + bodies[mode] + "<" + std::to_string(dk) + ", " +
         std::to_string(LN) + ", " + (ch ? "true" : "false") + ">(&tmap, p, sg, " +
         (ch ? "&cp" : "nullptr") + (dk == 0 ? ", &dp" : ", nullptr") + ");\n}\n";
  return src;
}

void log_line(const std::string& msg) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_jit_log.size() < (1u << 20)) g_jit_log += "\n" + msg;
}

}  // namespace

// Launch the specialised kernel; cudaErrorNotSupported when JIT is unavailable
// (the caller then launches the static kernel).
cudaError_t launch_maxplus_lanes_jit(const LaneParams& p, const LaneChainParams* cp,
                                     const int* dense32, const void* tmap128, int dkind, int V,
                                     const std::vector<int>& codes, int grid, int BD, size_t smem,
                                     cudaStream_t stream, const LaneDerivedParams* dp) {
  if (codes.empty() || codes.size() > 32) {
    static std::atomic<bool> logged{false};  // once per process, not per call
    if (!logged.exchange(true))
      log_line("skipped: " + std::to_string(codes.size()) + " handler codes");
    return cudaErrorNotSupported;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  // latency-bound launches (fewer CTAs than SMs) take the branch-free handler
  bool dyn = grid < 148;
  int nsm = 148;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) dyn = grid < nsm;
  if (const char* e = getenv("DDSIM_LANES_DYN")) dyn = atoi(e) != 0;
  // lane busy by a separate pass for the branch-free handler (absent chain
  // members are recognised by their start -1, so chains need the starts)
  const bool nolb = dyn && dkind != 0 && p.lane_busy != nullptr &&
                    (cp == nullptr || p.start != nullptr) && getenv("DDSIM_DYN_LB") == nullptr;
  const bool scale = dp != nullptr && dp->scale_ptr != nullptr;
  CUfunction fn = get_function(codes, dkind, V, dyn, cp != nullptr, nolb, scale, dev);
  if (!fn) return cudaErrorNotSupported;
  const CUresult ar = g_drv.setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
  if (ar != CUDA_SUCCESS) {
    log_line("cuFuncSetAttribute failed: " + std::to_string((int)ar));
    return cudaErrorNotSupported;
  }
  alignas(64) unsigned char tm[128];
  memcpy(tm, tmap128, 128);
  LaneParams pp = p;
  if (nolb) pp.lane_busy = nullptr;
  LaneChainParams cpv{};
  if (cp) cpv = *cp;
  LaneDerivedParams dpv{};
  if (dp) dpv = *dp;
  void* args_ch[] = {tm, &pp, &cpv, &dpv};
  void* args_nc[] = {tm, &pp, &dpv};
  const CUresult r = g_drv.launch(fn, grid, 1, 1, BD, 1, 1, (unsigned)smem, (CUstream)stream,
                                  cp ? args_ch : args_nc, nullptr);
  if (r != CUDA_SUCCESS) {
    log_line("cuLaunchKernel failed: " + std::to_string((int)r));
    return cudaErrorNotSupported;
  }
  note_launch();
  if (nolb) return launch_lanes_busy(p, dense32, cp != nullptr, stream);
  return cudaSuccess;
}

// One segment kernel launch (grid gx x K'): transfer or replay.
cudaError_t launch_lanes_seg_jit(int mode, const LaneParams& p, const LaneChainParams* cp,
                                 const void* tmap128, int dkind, int LN,
                                 const std::vector<int>& codes, const void* segp, int gx, int gy,
                                 int BD, size_t smem, cudaStream_t stream,
                                 const LaneDerivedParams* dp) {
  if (codes.empty() || codes.size() > 32 || LN < 1 || LN > 4 || mode < 0 || mode > 4)
    return cudaErrorNotSupported;
  int dev = 0;
  cudaGetDevice(&dev);
  const char* tags[] = {"seg_r:", "seg_t:", "seg_f:", "seg_t2:", "seg_r2:"};
  const char* names[] = {"ddsim_seg_replay", "ddsim_seg_transfer", "ddsim_seg_fused",
                         "ddsim_seg_transfer2", "ddsim_seg_replay2"};
  std::string key = std::string(tags[mode]) + std::to_string(dev) + ":" + std::to_string(dkind) +
                    ":" + std::to_string(LN) + (cp ? ":ch:" : ":");
  if (const char* u = getenv("DDSIM_SEG_UNROLL")) key += std::string("u") + u + ":";
  if (const char* mb = getenv("DDSIM_SEG_MINB")) key += std::string("mb") + mb + ":";
  if (const char* st = getenv("DDSIM_SEG_STAGES")) key += std::string("st") + st + ":";
  const bool scale = dp != nullptr && dp->scale_ptr != nullptr;
  if (dkind == 0 && !scale) key += "noscale:";
  for (int c : codes) key += std::to_string(c) + ",";
  CUfunction fn = get_compiled(key, [&] { return seg_source(codes, dkind, LN, cp != nullptr, mode, scale); },
                               names[mode]);
  if (!fn) return cudaErrorNotSupported;
  if (g_drv.setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  alignas(64) unsigned char tm[128];
  memcpy(tm, tmap128, 128);
  LaneParams pp = p;
  alignas(16) unsigned char sg[sizeof(LaneSegParams)];
  memcpy(sg, segp, sizeof(sg));
  LaneChainParams cpv{};
  if (cp) cpv = *cp;
  LaneDerivedParams dpv{};
  if (dp) dpv = *dp;
  void* args_ch[] = {tm, &pp, sg, &cpv, &dpv};
  void* args_nc[] = {tm, &pp, sg, &dpv};
  const CUresult r = g_drv.launch(fn, gx, gy, 1, BD, 1, 1, (unsigned)smem, (CUstream)stream,
                                  cp ? args_ch : args_nc, nullptr);
  if (r != CUDA_SUCCESS) {
    log_line("cuLaunchKernel (segment) failed: " + std::to_string((int)r));
    return cudaErrorLaunchFailure;
  }
  note_launch();
  return cudaSuccess;
}

bool jit_available() {
  if (getenv("DDSIM_NO_JIT")) return false;
  std::lock_guard<std::mutex> lk(g_mu);
  init_locked();
  return g_nv.ok && g_drv.ok;
}

// A per-thread snapshot: the shared log may grow while the caller reads it.
const char* jit_log() {
  thread_local std::string snap;
  std::lock_guard<std::mutex> lk(g_mu);
  snap = g_jit_log;
  return snap.c_str();
}

}  // namespace ddsim

extern "C" const char* ks_jit_log(void) { return ddsim::jit_log(); }
