// libcanvas_b200.so — native runtime of the Canvas executor (C ABI in
// include/canvas_b200.h).
//
// A plan blob (paper_2304_07741_b200/lowering.py Plan.blob) carries the
// generated functors of one solved kernel graph plus its launch schedule.
// canvas_plan_create compiles the functors together with the hand-written
// kernel templates (kernels/canvas_kernels.cuh, embedded at build time) for
// sm_100a with NVRTC, loads the cubin, and resolves every kernel; the forward
// and backward entry points then only compute slot pointers and grid sizes
// for the batch and enqueue cuLaunchKernel on the caller's stream.
//
// The CUDA driver and NVRTC are loaded with dlopen on first use, so the
// library itself loads (and its symbols can be checked) on a host without a
// GPU driver.
#include "../../include/canvas_b200.h"

#include <dlfcn.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <unistd.h>
#include <unordered_map>
#include <vector>

namespace {

const char kTemplates[] =
#include "canvas_kernels_embed.inc"
    ;

// ----------------------------------------------------------------- driver API
typedef int CUresult;
typedef int CUdevice;
typedef struct CUctx_st* CUcontext;
typedef struct CUmod_st* CUmodule;
typedef struct CUfunc_st* CUfunction;
typedef struct CUstream_st* CUstream;
typedef unsigned long long CUdeviceptr;

constexpr int kAttrCCMajor = 75;  // CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR
constexpr int kAttrCCMinor = 76;  // CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR

struct Driver {
  bool ok = false;
  std::string why;
  CUresult (*cuInit)(unsigned);
  CUresult (*cuDeviceGet)(CUdevice*, int);
  CUresult (*cuDeviceGetAttribute)(int*, int, CUdevice);
  CUresult (*cuDevicePrimaryCtxRetain)(CUcontext*, CUdevice);
  CUresult (*cuCtxSetCurrent)(CUcontext);
  CUresult (*cuModuleLoadData)(CUmodule*, const void*);
  CUresult (*cuModuleUnload)(CUmodule) = nullptr;
  CUresult (*cuModuleGetFunction)(CUfunction*, CUmodule, const char*);
  CUresult (*cuLaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void**, void**);
  CUresult (*cuMemsetD8Async)(CUdeviceptr, unsigned char, size_t, CUstream);
  CUresult (*cuGetErrorString)(CUresult, const char**);
  CUresult (*cuFuncSetAttribute)(CUfunction, int, int);
  CUresult (*cuEventRecord)(void*, CUstream);
  // optional: inside CUDA-graph stream capture the profiling events must be
  // recorded as external event nodes so they fire on every replay
  CUresult (*cuEventRecordWithFlags)(void*, CUstream, unsigned) = nullptr;
  CUresult (*cuStreamIsCapturing)(CUstream, int*) = nullptr;
};

// ----------------------------------------------------------------- NVRTC
typedef int nvrtcResult;
typedef struct _nvrtcProgram* nvrtcProgram;
struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
  nvrtcResult (*logSize)(nvrtcProgram, size_t*);
  nvrtcResult (*log)(nvrtcProgram, char*);
  nvrtcResult (*cubinSize)(nvrtcProgram, size_t*);
  nvrtcResult (*cubin)(nvrtcProgram, char*);
  nvrtcResult (*destroy)(nvrtcProgram*);
  const char* (*errstr)(nvrtcResult);
  nvrtcResult (*version)(int*, int*) = nullptr;
};

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <class T>
bool sym(void* h, const char* name, T& out, std::string& why) {
  out = reinterpret_cast<T>(dlsym(h, name));
  if (!out) why = std::string("missing symbol ") + name;
  return out != nullptr;
}

Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      d.why = std::string("cannot load libcuda.so.1: ") + dlerror();
      return;
    }
    std::string& w = d.why;
    d.ok = sym(h, "cuInit", d.cuInit, w) && sym(h, "cuDeviceGet", d.cuDeviceGet, w) &&
           sym(h, "cuDeviceGetAttribute", d.cuDeviceGetAttribute, w) &&
           sym(h, "cuDevicePrimaryCtxRetain", d.cuDevicePrimaryCtxRetain, w) &&
           sym(h, "cuCtxSetCurrent", d.cuCtxSetCurrent, w) && sym(h, "cuModuleLoadData", d.cuModuleLoadData, w) &&
           sym(h, "cuModuleGetFunction", d.cuModuleGetFunction, w) &&
           sym(h, "cuLaunchKernel", d.cuLaunchKernel, w) && sym(h, "cuMemsetD8Async", d.cuMemsetD8Async, w) &&
           sym(h, "cuGetErrorString", d.cuGetErrorString, w) &&
           sym(h, "cuFuncSetAttribute", d.cuFuncSetAttribute, w) && sym(h, "cuEventRecord", d.cuEventRecord, w);
    if (d.ok) {
      std::string ignore;
      sym(h, "cuEventRecordWithFlags", d.cuEventRecordWithFlags, ignore);
      sym(h, "cuStreamIsCapturing", d.cuStreamIsCapturing, ignore);
      sym(h, "cuModuleUnload", d.cuModuleUnload, ignore);
    }
    if (d.ok && d.cuInit(0) != 0) {
      d.ok = false;
      d.why = "cuInit failed (no usable GPU)";
    }
  });
  return d;
}

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("cannot load libnvrtc: ") + dlerror();
      return;
    }
    std::string& w = n.why;
    n.ok = sym(h, "nvrtcCreateProgram", n.create, w) && sym(h, "nvrtcCompileProgram", n.compile, w) &&
           sym(h, "nvrtcGetProgramLogSize", n.logSize, w) && sym(h, "nvrtcGetProgramLog", n.log, w) &&
           sym(h, "nvrtcGetCUBINSize", n.cubinSize, w) && sym(h, "nvrtcGetCUBIN", n.cubin, w) &&
           sym(h, "nvrtcDestroyProgram", n.destroy, w) && sym(h, "nvrtcGetErrorString", n.errstr, w);
    std::string ignore;
    sym(h, "nvrtcVersion", n.version, ignore);
  });
  return n;
}

std::string cu_err(CUresult r) {
  const char* s = nullptr;
  if (driver().cuGetErrorString) driver().cuGetErrorString(r, &s);
  return s ? s : ("CUresult " + std::to_string(r));
}

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

// ----------------------------------------------------------------- blob
struct SizeRule {
  int64_t a_num, a_den, b;
  int64_t eval(int64_t n) const { return (n * a_num + a_den - 1) / a_den + b; }
};
struct GridRule {
  int64_t a, b, d, cap;
  int64_t eval(int64_t n) const {
    int64_t g = (a * n + b + d - 1) / d;
    if (cap > 0 && g > cap) g = cap;
    return g < 1 ? 1 : g;
  }
};
constexpr int kMaxSlots = 24;
struct Record {
  int64_t kind, phase, kernel, block, smem;
  GridRule grid[3];
  int64_t nslots;
  int64_t slots[kMaxSlots];
  int64_t beta, memset_slot;
  SizeRule memset_size;
};

struct CanvasArgs {  // must match kernels/canvas_kernels.cuh
  void* p[kMaxSlots];
  long long n;
  int beta;
  int copy;
};

}  // namespace

struct canvas_plan {
  ~canvas_plan();
  std::string module_key;  // "" until the module is acquired
  int device = 0;
  CUcontext ctx = nullptr;
  int64_t n_fc = 0, copies = 1;
  int64_t x_off = 0, y_off = 0, dx_off = 0, dy_off = 0;  // per-copy element offsets
  int64_t max_batch = 0;  // kernels use 32-bit per-tensor offsets up to this batch
  std::vector<SizeRule> saved, ws;
  std::vector<Record> recs;
  std::vector<CUfunction> fns;
  // measurement hook (canvas_plan_profile): CUDA events recorded around every
  // launch of one record, so bench.py can time one kernel inside a full step
  struct Prof {
    std::vector<void*> events;  // 2 per slot: start, end
    int64_t count = 0;
  };
  mutable std::mutex prof_mu;
  mutable std::unordered_map<int64_t, Prof> prof;  // launch record -> event ring
};

namespace {

constexpr unsigned kEventRecordExternal = 0x1;  // CU_EVENT_RECORD_EXTERNAL

void record_event(Driver& d, void* ev, CUstream st, bool external) {
  if (external)
    d.cuEventRecordWithFlags(ev, st, kEventRecordExternal);
  else
    d.cuEventRecord(ev, st);
}

// Loaded modules, shared by every plan with the same (device, source):
// reference-counted, unloaded when the last plan using one is destroyed, so a
// long candidate search does not accumulate modules.
struct ModEntry {
  CUmodule mod = nullptr;
  int64_t refs = 0;
};
std::mutex g_mod_mu;
std::unordered_map<std::string, ModEntry> g_modules;  // (device, source hash) -> module

std::string module_key(const std::string& src, int device) {
  return std::to_string(device) + ":" + std::to_string(fnv1a(src, fnv1a(kTemplates)));
}

void release_module(const std::string& key) {
  CUmodule m = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mod_mu);
    auto it = g_modules.find(key);
    if (it == g_modules.end() || --it->second.refs > 0) return;
    m = it->second.mod;
    g_modules.erase(it);
  }
  if (m && driver().cuModuleUnload) driver().cuModuleUnload(m);
}

// The on-disk JIT cache (CANVAS_JIT_CACHE) keys cubins by the source, the
// templates, the target arch, the NVRTC version and the compile options, and
// writes each through a per-process, per-thread temporary file renamed into
// place, so concurrent evaluator workers never read a torn cubin.
// A node value recomputed inline in another kernel (forward values inside
// adjoint kernels, inlined gradients) must round exactly like the copy the
// forward stored, or max/min tie tests (x == m, App. A.6/A.8) flip: the
// lowering emits broadcast add/sub/mul as __fadd_rn/__fsub_rn/__fmul_rn, which
// the compiler never contracts.  CANVAS_FMAD=0 additionally compiles with
// --fmad=false (A/B: it slows expf-heavy softmax kernels ~1.5x).
const char* const kNvrtcOpts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--extra-device-vectorization",
                                  "-default-device", "--fmad=false"};
int nvrtc_nopts() { return std::getenv("CANVAS_FMAD") && std::getenv("CANVAS_FMAD")[0] == '0' ? 6 : 5; }
#define kNvrtcNOpts nvrtc_nopts()

std::string cache_name(const std::string& src) {
  Nvrtc& nv = nvrtc();
  int maj = 0, mnr = 0;
  if (nv.ok && nv.version) nv.version(&maj, &mnr);
  uint64_t h = fnv1a(src, fnv1a(kTemplates));
  std::string opts = "sm_100a|nvrtc" + std::to_string(maj) + "." + std::to_string(mnr);
  for (int i = 0; i < kNvrtcNOpts; ++i) opts += std::string("|") + kNvrtcOpts[i];
  h = fnv1a(opts, h);
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)h);
  return std::string(buf) + ".sm_100a.cubin";
}

int compile_module(const std::string& src, int device, CUmodule* out) {
  const std::string key = module_key(src, device);
  {
    std::lock_guard<std::mutex> lk(g_mod_mu);
    auto it = g_modules.find(key);
    if (it != g_modules.end()) {
      ++it->second.refs;
      *out = it->second.mod;
      return CANVAS_OK;
    }
  }
  std::string cubin;  // compiled outside the lock: plans of a network build in parallel
  const char* cache_dir = std::getenv("CANVAS_JIT_CACHE");
  std::string cache_path;
  if (cache_dir && *cache_dir) {
    cache_path = std::string(cache_dir) + "/" + cache_name(src);
    std::ifstream f(cache_path, std::ios::binary);
    if (f) cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  }
  if (cubin.empty()) {
    Nvrtc& nv = nvrtc();
    if (!nv.ok) return fail(CANVAS_ERR_COMPILE, nv.why);
    nvrtcProgram prog;
    const char* hdr_src[] = {kTemplates};
    const char* hdr_name[] = {"canvas_kernels.cuh"};
    if (nv.create(&prog, src.c_str(), "canvas_plan.cu", 1, hdr_src, hdr_name) != 0)
      return fail(CANVAS_ERR_COMPILE, "nvrtcCreateProgram failed");
    nvrtcResult rc = nv.compile(prog, kNvrtcNOpts, kNvrtcOpts);
    size_t ls = 0;
    nv.logSize(prog, &ls);
    std::string log(ls, '\0');
    if (ls) nv.log(prog, &log[0]);
    if (rc != 0) {
      nv.destroy(&prog);
      return fail(CANVAS_ERR_COMPILE, std::string("NVRTC: ") + nv.errstr(rc) + "\n" + log);
    }
    size_t cs = 0;
    nv.cubinSize(prog, &cs);
    cubin.resize(cs);
    nv.cubin(prog, &cubin[0]);
    nv.destroy(&prog);
    if (!cache_path.empty()) {
      std::ostringstream tmp;
      tmp << cache_path << ".tmp." << getpid() << "." << std::hash<std::thread::id>()(std::this_thread::get_id());
      std::ofstream f(tmp.str(), std::ios::binary);
      f.write(cubin.data(), (std::streamsize)cubin.size());
      f.close();
      if (f) std::rename(tmp.str().c_str(), cache_path.c_str());
      else std::remove(tmp.str().c_str());
    }
  }
  std::lock_guard<std::mutex> lk(g_mod_mu);
  auto it = g_modules.find(key);
  if (it != g_modules.end()) {
    ++it->second.refs;
    *out = it->second.mod;
    return CANVAS_OK;
  }
  CUmodule mod;
  CUresult r = driver().cuModuleLoadData(&mod, cubin.data());
  if (r != 0) return fail(CANVAS_ERR_CUDA, "cuModuleLoadData: " + cu_err(r));
  g_modules[key] = ModEntry{mod, 1};
  *out = mod;
  return CANVAS_OK;
}

size_t align256(int64_t b) { return (size_t)((b + 255) / 256 * 256); }
// every saved / workspace tensor sits between two guard zones, so the aligned 16 B
// chunks around a shifted quad (vector producers) can be loaded unconditionally:
// a chunk beyond a tensor edge by at most kGuard bytes reads the guard zone and is
// then masked per lane (slots stay 256 B aligned)
constexpr size_t kGuard = 16384;
size_t slot_bytes(int64_t b) { return align256(b) + 2 * kGuard; }

void* slot_ptr(const canvas_plan* p, int64_t s, int64_t copy, int64_t batch, const float* x, const float* const* w,
               float* y, const float* dy, float* dx, float* const* dw, void* saved, void* ws) {
  const int64_t nf = p->n_fc;
  if (s == 0) return (void*)(x + copy * p->x_off);
  if (s == 1) return (void*)(y ? y + copy * p->y_off : nullptr);
  if (s == 2) return (void*)(dy ? dy + copy * p->dy_off : nullptr);
  if (s == 3) return (void*)(dx ? dx + copy * p->dx_off : nullptr);
  s -= 4;
  if (s < nf) return (void*)w[copy * nf + s];
  s -= nf;
  if (s < nf) return dw ? (void*)dw[copy * nf + s] : nullptr;
  s -= nf;
  if (s < (int64_t)p->saved.size()) {
    size_t per_copy = 0, off = 0;
    for (size_t k = 0; k < p->saved.size(); ++k) {
      if ((int64_t)k == s) off = per_copy;
      per_copy += slot_bytes(p->saved[k].eval(batch));
    }
    return (char*)saved + copy * per_copy + off + kGuard;
  }
  s -= (int64_t)p->saved.size();
  size_t off = 0;
  for (int64_t k = 0; k < s; ++k) off += slot_bytes(p->ws[k].eval(batch));
  return (char*)ws + off + kGuard;
}

int run_phase(const canvas_plan* p, int phase, int64_t batch, const float* x, const float* const* w, int n_fc,
              float* y, const float* dy, float* dx, float* const* dw, void* saved, void* ws, void* stream) {
  if (!p) return fail(CANVAS_ERR_ARGS, "null plan");
  if (batch < 1 || batch > p->max_batch)
    return fail(CANVAS_ERR_ARGS, "batch " + std::to_string(batch) + " outside [1, " + std::to_string(p->max_batch) + "]");
  if (n_fc != p->n_fc * p->copies)
    return fail(CANVAS_ERR_ARGS, "expected " + std::to_string(p->n_fc * p->copies) + " FC weights, got " +
                                     std::to_string(n_fc));
  if (!x || (p->n_fc && !w) || (!p->saved.empty() && !saved)) return fail(CANVAS_ERR_ARGS, "null tensor pointer");
  if (phase == 0 && !y) return fail(CANVAS_ERR_ARGS, "null y");
  if (phase == 1 && (!dy || !dx || (p->n_fc && !dw) || (!p->ws.empty() && !ws)))
    return fail(CANVAS_ERR_ARGS, "null backward tensor pointer");
  Driver& d = driver();
  d.cuCtxSetCurrent(p->ctx);
  CUstream st = (CUstream)stream;
  for (int64_t copy = 0; copy < p->copies; ++copy) {
    for (const Record& r : p->recs) {
      if (r.phase != phase) continue;
      if (r.kind == 1) {  // memset (once, before the first replica)
        if (copy != 0) continue;
        void* ptr = slot_ptr(p, r.memset_slot, 0, batch, x, w, y, dy, dx, dw, saved, ws);
        int64_t bytes = r.memset_size.eval(batch);
        CUresult e = d.cuMemsetD8Async((CUdeviceptr)ptr, 0, (size_t)bytes, st);
        if (e != 0) return fail(CANVAS_ERR_CUDA, "memset: " + cu_err(e));
        continue;
      }
      CanvasArgs a;
      std::memset(&a, 0, sizeof(a));
      for (int64_t i = 0; i < r.nslots; ++i) {
        a.p[i] = slot_ptr(p, r.slots[i], copy, batch, x, w, y, dy, dx, dw, saved, ws);
        // kind 2: the kernel's 4-element quads are 16 B loads / stores
        if (r.kind == 2 && ((uintptr_t)a.p[i] & 15u) != 0)
          return fail(CANVAS_ERR_ARGS, "tensor pointer of slot " + std::to_string(r.slots[i]) + " (copy " +
                                           std::to_string(copy) + ") is not 16-byte aligned; launch " +
                                           std::to_string(&r - p->recs.data()) + " uses 16 B accesses");
      }
      a.n = batch;
      a.beta = (r.beta == 2) || (r.beta == 1 && copy > 0);
      a.copy = (int)copy;
      unsigned g[3];
      for (int i = 0; i < 3; ++i) g[i] = (unsigned)r.grid[i].eval(batch);
      void* params[] = {&a};
      void* ev_end = nullptr;
      bool ev_external = false;
      const int64_t ri = &r - p->recs.data();
      if (!p->prof.empty()) {
        std::lock_guard<std::mutex> lk(p->prof_mu);
        auto it = p->prof.find(ri);
        if (it != p->prof.end() && !it->second.events.empty()) {
          auto& pr = it->second;
          const size_t slot = (size_t)(pr.count++ % (int64_t)(pr.events.size() / 2));
          int capturing = 0;
          if (d.cuStreamIsCapturing && d.cuEventRecordWithFlags) d.cuStreamIsCapturing(st, &capturing);
          ev_external = capturing != 0;
          record_event(d, pr.events[2 * slot], st, ev_external);
          ev_end = pr.events[2 * slot + 1];
        }
      }
      CUresult e = d.cuLaunchKernel(p->fns[r.kernel], g[0], g[1], g[2], (unsigned)r.block, 1, 1, (unsigned)r.smem, st, params,
                                    nullptr);
      if (e != 0) return fail(CANVAS_ERR_CUDA, "launch kernel " + std::to_string(r.kernel) + ": " + cu_err(e));
      if (ev_end) record_event(d, ev_end, st, ev_external);
    }
  }
  return CANVAS_OK;
}

struct Reader {
  const char* p;
  const char* end;
  bool ok = true;
  int64_t i64() {
    if (end - p < 8) {
      ok = false;
      return 0;
    }
    int64_t v;
    std::memcpy(&v, p, 8);
    p += 8;
    return v;
  }
};

}  // namespace

canvas_plan::~canvas_plan() {
  if (!module_key.empty()) release_module(module_key);
}

extern "C" {

int canvas_abi_version(void) { return 1; }

const char* canvas_last_error(void) { return g_err.c_str(); }

int canvas_plan_create(const void* blob, size_t nbytes, int cuda_device, canvas_plan** out) {
  if (!blob || !out) return fail(CANVAS_ERR_ARGS, "null blob/out");
  *out = nullptr;
  const char* b = (const char*)blob;
  if (nbytes < 8 || std::memcmp(b, "CNVSBLOB", 8) != 0) return fail(CANVAS_ERR_BLOB, "bad blob magic");
  Reader rd{b + 8, b + nbytes};
  int64_t version = rd.i64();
  if (version != 1) return fail(CANVAS_ERR_VERSION, "blob version " + std::to_string(version) + ", library 1");
  int64_t n_kernels = rd.i64(), n_launch = rd.i64(), n_saved = rd.i64(), n_ws = rd.i64();
  std::unique_ptr<canvas_plan> p(new canvas_plan());
  p->n_fc = rd.i64();
  p->copies = rd.i64();
  p->x_off = rd.i64();
  p->y_off = rd.i64();
  p->dx_off = rd.i64();
  p->dy_off = rd.i64();
  p->max_batch = rd.i64();
  int64_t src_len = rd.i64(), names_len = rd.i64();
  if (!rd.ok || n_kernels < 0 || n_launch < 0 || n_saved < 0 || n_ws < 0 || p->copies < 1)
    return fail(CANVAS_ERR_BLOB, "bad blob header");
  for (int64_t i = 0; i < n_saved + n_ws; ++i) {
    SizeRule s{rd.i64(), rd.i64(), rd.i64()};
    if (s.a_den <= 0) return fail(CANVAS_ERR_BLOB, "bad size rule");
    (i < n_saved ? p->saved : p->ws).push_back(s);
  }
  for (int64_t i = 0; i < n_launch; ++i) {
    Record r;
    r.kind = rd.i64();
    r.phase = rd.i64();
    r.kernel = rd.i64();
    r.block = rd.i64();
    r.smem = rd.i64();
    for (auto& g : r.grid) g = GridRule{rd.i64(), rd.i64(), rd.i64(), rd.i64()};
    r.nslots = rd.i64();
    for (auto& s : r.slots) s = rd.i64();
    r.beta = rd.i64();
    r.memset_slot = rd.i64();
    r.memset_size = SizeRule{rd.i64(), rd.i64(), rd.i64()};
    if (!rd.ok || r.nslots < 0 || r.nslots > kMaxSlots || (r.kind != 1 && (r.kernel < 0 || r.kernel >= n_kernels)) || r.kind < 0 || r.kind > 2)
      return fail(CANVAS_ERR_BLOB, "bad launch record " + std::to_string(i));
    for (const auto& g : r.grid)
      if (g.d <= 0) return fail(CANVAS_ERR_BLOB, "bad grid rule");
    p->recs.push_back(r);
  }
  if (!rd.ok || rd.end - rd.p != src_len + names_len) return fail(CANVAS_ERR_BLOB, "blob length mismatch");
  std::string src(rd.p, (size_t)src_len);
  std::vector<std::string> names;
  {
    const char* q = rd.p + src_len;
    const char* qe = q + names_len;
    while (q < qe && (int64_t)names.size() < n_kernels) {
      size_t l = strnlen(q, (size_t)(qe - q));
      names.emplace_back(q, l);
      q += l + 1;
    }
  }
  if ((int64_t)names.size() != n_kernels) return fail(CANVAS_ERR_BLOB, "kernel name table short");

  Driver& d = driver();
  if (!d.ok) return fail(CANVAS_ERR_CUDA, d.why);
  CUdevice dev;
  CUresult e = d.cuDeviceGet(&dev, cuda_device);
  if (e != 0) return fail(CANVAS_ERR_CUDA, "cuDeviceGet: " + cu_err(e));
  int maj = 0, mnr = 0;
  d.cuDeviceGetAttribute(&maj, kAttrCCMajor, dev);
  d.cuDeviceGetAttribute(&mnr, kAttrCCMinor, dev);
  if (maj != 10 || mnr != 0)
    return fail(CANVAS_ERR_DEVICE, "device is sm_" + std::to_string(maj) + std::to_string(mnr) +
                                       "; this executor is built for sm_100a only");
  e = d.cuDevicePrimaryCtxRetain(&p->ctx, dev);
  if (e != 0) return fail(CANVAS_ERR_CUDA, "cuDevicePrimaryCtxRetain: " + cu_err(e));
  d.cuCtxSetCurrent(p->ctx);
  p->device = cuda_device;
  CUmodule mod;
  int rc = compile_module(src, cuda_device, &mod);
  if (rc) return rc;
  p->module_key = module_key(src, cuda_device);  // released by ~canvas_plan
  for (const auto& nm : names) {
    CUfunction f;
    e = d.cuModuleGetFunction(&f, mod, nm.c_str());
    if (e != 0) return fail(CANVAS_ERR_CUDA, "cuModuleGetFunction(" + nm + "): " + cu_err(e));
    p->fns.push_back(f);
  }
  for (const Record& r : p->recs) {
    if (r.kind != 1 && r.smem > 48 * 1024) {
      e = d.cuFuncSetAttribute(p->fns[r.kernel], 8 /* MAX_DYNAMIC_SHARED_SIZE_BYTES */, (int)r.smem);
      if (e != 0) return fail(CANVAS_ERR_CUDA, "cuFuncSetAttribute(smem " + std::to_string(r.smem) + "): " + cu_err(e));
    }
  }
  *out = p.release();
  return CANVAS_OK;
}

void canvas_plan_destroy(canvas_plan* p) { delete p; }  // unloads its module with the last plan using it

int canvas_plan_query(const canvas_plan* p, int64_t batch, size_t* fwd_workspace, size_t* saved_bytes,
                      size_t* bwd_workspace) {
  if (!p || batch < 1) return fail(CANVAS_ERR_ARGS, "bad plan/batch");
  size_t sv = 0, w = 0;
  for (const auto& s : p->saved) sv += slot_bytes(s.eval(batch));
  for (const auto& s : p->ws) w += slot_bytes(s.eval(batch));
  if (fwd_workspace) *fwd_workspace = 0;
  if (saved_bytes) *saved_bytes = sv * (size_t)p->copies;
  if (bwd_workspace) *bwd_workspace = w;
  return CANVAS_OK;
}

int canvas_plan_launches(const canvas_plan* p, int phase) {
  if (!p) return fail(CANVAS_ERR_ARGS, "null plan");
  int n = 0;
  for (const auto& r : p->recs)
    if (r.phase == phase && r.kind != 1) n += (int)p->copies;
  return n;
}

int canvas_plan_profile(canvas_plan* p, int record, void* const* events, int n_pairs) {
  if (!p || record >= (int)p->recs.size() || n_pairs < 0 || (n_pairs && !events))
    return fail(CANVAS_ERR_ARGS, "bad profile request");
  std::lock_guard<std::mutex> lk(p->prof_mu);
  if (n_pairs == 0) {
    p->prof.erase(record);
  } else {
    auto& pr = p->prof[record];
    pr.events.assign(events, events + 2 * n_pairs);
    pr.count = 0;
  }
  return CANVAS_OK;
}

int64_t canvas_plan_profile_count(const canvas_plan* p, int record) {
  if (!p) return -1;
  std::lock_guard<std::mutex> lk(p->prof_mu);
  auto it = p->prof.find(record);
  return it == p->prof.end() ? 0 : it->second.count;
}

int canvas_forward(const canvas_plan* p, int64_t batch, const float* x, const float* const* fc_w, int n_fc, float* y,
                   void* saved, void* workspace, void* stream) {
  return run_phase(p, 0, batch, x, fc_w, n_fc, y, nullptr, nullptr, nullptr, saved, workspace, stream);
}

int canvas_backward(const canvas_plan* p, int64_t batch, const float* x, const float* const* fc_w, int n_fc,
                    const void* saved, const float* dy, float* dx, float* const* fc_dw, void* workspace,
                    void* stream) {
  return run_phase(p, 1, batch, x, fc_w, n_fc, nullptr, dy, dx, fc_dw, const_cast<void*>(saved), workspace, stream);
}

}  // extern "C"
