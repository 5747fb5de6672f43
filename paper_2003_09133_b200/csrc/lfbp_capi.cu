// C-ABI of the B200-native H -> H' rearrangement (see include/lfbp_hprime.h).
//
// Host runtime around the K1 kernel: dims validation with the reference's
// rules, the launch planner (work-unit shape, smem ring, persistent grid),
// device-array entry point, a chunked H2D / kernel / D2H pipeline for host
// arrays, the z-slab multi-GPU launcher, and the K2 device comparator.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lfbp_hprime.h"
#include "hprime_kernel.cuh"
#include "hprime_plan.h"
#include "plane_sums.cuh"
#include "projector.cuh"

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define HP_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return fail(LFBP_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),       \
                  __FILE__, __LINE__);                                                         \
  } while (0)

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return atoi(v);
}

struct DevProps {
  int sm_count = 148;
  int smem_optin = 232448;  // 227 KB
  int max_threads_sm = 2048;
  bool real = false;
};

std::mutex g_props_mu;
std::map<int, DevProps> g_props;

DevProps device_props(int dev) {
  std::lock_guard<std::mutex> lk(g_props_mu);
  auto it = g_props.find(dev);
  if (it != g_props.end()) return it->second;
  DevProps p;
  int n = 0;
  if (dev >= 0 && cudaGetDeviceCount(&n) == cudaSuccess && dev < n) {
    cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&p.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&p.max_threads_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
    p.real = true;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaFuncSetAttribute(hp::hprime_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_optin);
    cudaFuncSetAttribute(hp::hprime_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_optin);
    cudaSetDevice(cur);
  } else {
    cudaGetLastError();  // clear "no device" state
  }
  g_props[dev] = p;
  return p;
}

int elem_size(int dtype) { return dtype == LFBP_F32 ? 4 : dtype == LFBP_F64 ? 8 : 0; }

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Tunable launch knobs.  Environment variables (LFBP_STAGES, LFBP_STAGE_KB,
// LFBP_CONSUMER_WARPS, LFBP_SUBWARP) override them for sweeps and tests.
struct Knobs {
  int stages = 4;      // smem ring depth
  int stage_kb = 48;   // target bytes of one staged unit (sets the t-band J)
  int cwarps = 12;     // consumer warps per CTA
  int subwarp = 0;     // lanes per output row; 0 = by row length
};

const char* const kKnobEnv[] = {"LFBP_STAGES", "LFBP_STAGE_KB", "LFBP_CONSUMER_WARPS", "LFBP_SUBWARP",
                                "LFBP_CTAS_PER_SM", "LFBP_BAND", "LFBP_STAGE_MAX_KB"};

bool env_knobs_set() {
  for (const char* n : kKnobEnv) {
    const char* v = getenv(n);
    if (v && *v) return true;
  }
  return false;
}

// Candidates tried by the autotuner (measured best plans of C1..C5 and
// neighbours; every one is bit-exact, they differ only in speed).
const Knobs kCandidates[] = {
    {3, 48, 8, 8},  {4, 48, 12, 16}, {4, 48, 8, 8},  {4, 48, 8, 16},
    {4, 32, 8, 16}, {3, 64, 8, 32},  {4, 48, 16, 16}, {4, 32, 4, 8},
};

// Work-unit shape, smem ring and persistent grid for one launch.
int make_plan(HpPlan& p, const int64_t d[5], int E, int64_t z_begin, int64_t z_count,
              int64_t total_bytes, int dev, const Knobs& kn = Knobs()) {
  memset(&p, 0, sizeof(p));
  const DevProps dp = device_props(dev);
  p.n_s = d[0];
  p.n_t = d[1];
  p.n_x = d[2];
  p.n_y = d[3];
  p.z_begin = z_begin;
  p.z_count = z_count;
  p.total_bytes = total_bytes;
  p.elem = E;
  p.c_s = static_cast<int32_t>((d[0] - 1) / 2);
  p.c_t = static_cast<int32_t>((d[1] - 1) / 2);
  p.v_s = 2 * p.c_s + 1;
  p.v_t = 2 * p.c_t + 1;
  p.nx_off = static_cast<int32_t>((d[2] - (p.c_s % d[2])) % d[2]);
  p.ny_off = static_cast<int32_t>((d[3] - (p.c_t % d[3])) % d[3]);
  p.xs16 = static_cast<int32_t>((d[0] * d[1] * E) & 15);
  if (d[0] * d[1] * d[2] * d[3] >= (1ll << 31) || d[2] >= (1 << 20) || d[3] >= (1 << 20))
    return fail(LFBP_ERR_UNSUPPORTED, "depth plane of %lld elements exceeds the kernel's 32-bit in-plane offsets",
                (long long)(d[0] * d[1] * d[2] * d[3]));

  const int64_t stage_target = int64_t(env_int("LFBP_STAGE_KB", kn.stage_kb)) * 1024;
  const int64_t stage_max = int64_t(env_int("LFBP_STAGE_MAX_KB", 100)) * 1024;
  const int64_t row_full = d[0] * E;
  int64_t run_max;
  if (d[2] * (row_full + 32) <= stage_max) {
    int64_t J = stage_target / (d[2] * row_full);
    J = std::max<int64_t>(1, std::min<int64_t>(J, d[1]));
    // small problems: keep >= 8 units per SM so the smem ring actually pipelines
    while (J > 1 && z_count * ((d[1] + J - 1) / J) * d[3] < int64_t(8) * dp.sm_count) J = (J + 1) / 2;
    const int jcap = env_int("LFBP_BAND", 0);
    if (jcap > 0) J = std::min<int64_t>(J, jcap);
    p.J = static_cast<int32_t>(J);
    p.C = static_cast<int32_t>(d[0]);
    p.n_chunks = 1;
    run_max = J * row_full;
  } else {
    const int64_t C = (stage_max / d[2] - 32) / E;
    if (C < 1) return fail(LFBP_ERR_UNSUPPORTED, "n_x=%lld too large to stage one column", (long long)d[2]);
    p.J = 1;
    p.C = static_cast<int32_t>(std::min<int64_t>(C, d[0]));
    p.n_chunks = static_cast<int32_t>((d[0] + p.C - 1) / p.C);
    run_max = int64_t(p.C) * E;
  }
  p.n_bands = static_cast<int32_t>((d[1] + p.J - 1) / p.J);
  // row pitch: >= run + 32 B, congruent to xs16 mod 16 (linear x addressing,
  // see hprime_plan.h); the multiple-of-16 part is odd to spread banks
  int64_t pitch = round_up(run_max + 32, 16);
  if (((pitch / 16) & 1) == 0) pitch += 16;
  pitch += env_int("LFBP_PITCH_EXTRA16", 0) * 16;
  p.row_pitch = static_cast<int32_t>(pitch + p.xs16);
  p.stage_bytes = static_cast<int32_t>(round_up(64 + d[2] * p.row_pitch + 32, 128));  // header + runs
  int S = env_int("LFBP_STAGES", kn.stages);
  S = std::max(1, std::min(S, 8));
  while (S > 1 && 128 + int64_t(S) * p.stage_bytes > dp.smem_optin) --S;
  if (128 + int64_t(S) * p.stage_bytes > dp.smem_optin)
    return fail(LFBP_ERR_UNSUPPORTED, "stage of %d bytes exceeds shared memory", p.stage_bytes);
  p.stages = S;
  p.smem_bytes = 128 + S * p.stage_bytes;
  int cwarps = env_int("LFBP_CONSUMER_WARPS", kn.cwarps);
  if (cwarps <= 0) cwarps = 12;
  cwarps = std::max(1, std::min(16, cwarps));
  const int threads = 32 * (1 + cwarps);  // producer + consumers
  p.threads = threads;

  const int64_t units = z_count * p.n_chunks * int64_t(p.n_bands) * d[3];
  if (units >= (1ll << 31)) return fail(LFBP_ERR_UNSUPPORTED, "too many work units (%lld)", (long long)units);
  p.n_units = units;
  int per_sm = 0;
  if (dp.real) {
    cudaError_t e = (E == 4) ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hp::hprime_kernel<4>,
                                                                           threads, p.smem_bytes)
                             : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hp::hprime_kernel<8>,
                                                                           threads, p.smem_bytes);
    if (e != cudaSuccess) return fail(LFBP_ERR_CUDA, "occupancy query: %s", cudaGetErrorString(e));
  } else {
    per_sm = std::min<int>(dp.max_threads_sm / threads, int((233472) / (p.smem_bytes + 1024)));
  }
  const int cap = env_int("LFBP_CTAS_PER_SM", 0);
  if (cap > 0) per_sm = std::min(per_sm, cap);
  if (per_sm < 1) return fail(LFBP_ERR_UNSUPPORTED, "kernel does not fit on an SM");
  p.ctas_per_sm = per_sm;
  p.grid = static_cast<int32_t>(std::min<int64_t>(units, int64_t(per_sm) * dp.sm_count));
  p.flags = env_int("LFBP_KFLAGS", 0);
  // lanes per output row: enough 16-byte groups per lane to amortise the row setup
  const int64_t groups = (std::min<int64_t>(p.C, d[0]) * E + 15) / 16 + 1;
  int W = env_int("LFBP_SUBWARP", kn.subwarp);
  if (W != 8 && W != 16 && W != 32) W = groups <= 32 ? 8 : groups <= 64 ? 16 : 32;
  p.sub_width = W;
  p.gx_inc = static_cast<int32_t>((W * (16 / E)) % d[2]);
  p.nx_div = hp_fastdiv_make(static_cast<uint32_t>(d[2]));
  p.ny_div = hp_fastdiv_make(static_cast<uint32_t>(d[3]));
  p.nb_div = hp_fastdiv_make(static_cast<uint32_t>(p.n_bands));
  p.nc_div = hp_fastdiv_make(static_cast<uint32_t>(p.n_chunks));
  return LFBP_OK;
}

int launch(const HpPlan& p, const void* src, void* dst, cudaStream_t st) {
  if (p.n_units == 0) return LFBP_OK;
  if (p.elem == 4)
    hp::hprime_kernel<4><<<p.grid, p.threads, p.smem_bytes, st>>>(p, static_cast<const uint8_t*>(src),
                                                                   static_cast<uint8_t*>(dst));
  else
    hp::hprime_kernel<8><<<p.grid, p.threads, p.smem_bytes, st>>>(p, static_cast<const uint8_t*>(src),
                                                                   static_cast<uint8_t*>(dst));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  HP_CUDA(cudaGetLastError());
  return LFBP_OK;
}

// ---- autotuner: per (plane shape, element size, device), first large call ----
struct TuneKey {
  int64_t n_s, n_t, n_x, n_y;
  int E, dev;
  bool operator<(const TuneKey& o) const {
    if (n_s != o.n_s) return n_s < o.n_s;
    if (n_t != o.n_t) return n_t < o.n_t;
    if (n_x != o.n_x) return n_x < o.n_x;
    if (n_y != o.n_y) return n_y < o.n_y;
    if (E != o.E) return E < o.E;
    return dev < o.dev;
  }
};

std::mutex g_tune_mu;
std::map<TuneKey, Knobs> g_tuned;

bool tuned_knobs(const TuneKey& k, Knobs& out) {
  std::lock_guard<std::mutex> lk(g_tune_mu);
  auto it = g_tuned.find(k);
  if (it == g_tuned.end()) return false;
  out = it->second;
  return true;
}

// Time every candidate on the caller's buffers (the final launch overwrites
// dst) and keep the fastest.  Skipped while the stream is being captured.
int autotune(const TuneKey& key, const void* src, void* dst, const int64_t dims[5], int E, int64_t z_begin,
             int64_t z_count, int64_t total, cudaStream_t st, Knobs& best) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  HP_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone) return LFBP_OK;
  cudaEvent_t e0, e1;
  HP_CUDA(cudaEventCreate(&e0));
  HP_CUDA(cudaEventCreate(&e1));
  // candidates interleaved over rounds (decorrelates clock / power drift);
  // score = median of the per-round launch times
  constexpr int kCand = int(sizeof(kCandidates) / sizeof(kCandidates[0]));
  constexpr int kRounds = 3;
  HpPlan plans[kCand];
  bool ok[kCand];
  float t[kCand][kRounds];
  for (int c = 0; c < kCand; ++c) {
    ok[c] = make_plan(plans[c], dims, E, z_begin, z_count, total, key.dev, kCandidates[c]) == LFBP_OK;
    if (ok[c]) {
      int rc = launch(plans[c], src, dst, st);  // warm
      if (rc) return rc;
    }
  }
  for (int r = 0; r < kRounds; ++r)
    for (int c = 0; c < kCand; ++c) {
      if (!ok[c]) continue;
      HP_CUDA(cudaEventRecord(e0, st));
      int rc = launch(plans[c], src, dst, st);
      if (rc) return rc;
      HP_CUDA(cudaEventRecord(e1, st));
      HP_CUDA(cudaEventSynchronize(e1));
      HP_CUDA(cudaEventElapsedTime(&t[c][r], e0, e1));
    }
  float best_ms = 1e30f;
  bool found = false;
  for (int c = 0; c < kCand; ++c) {
    if (!ok[c]) continue;
    float v[kRounds];
    for (int r = 0; r < kRounds; ++r) v[r] = t[c][r];
    std::sort(v, v + kRounds);
    if (v[kRounds / 2] < best_ms) {
      best_ms = v[kRounds / 2];
      best = kCandidates[c];
      found = true;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  g_err.clear();
  if (found) {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    g_tuned[key] = best;
  }
  return LFBP_OK;
}

int check_common(const int64_t dims[5], int dtype, int inverse) {
  if (!dims) return fail(LFBP_ERR_ARGUMENT, "dims is NULL");
  if (!hp_dims_valid(dims[0], dims[1], dims[2], dims[3], dims[4]))
    return fail(LFBP_ERR_INVALID_DIMS, "invalid dims (%lld, %lld, %lld, %lld, %lld)", (long long)dims[0],
                (long long)dims[1], (long long)dims[2], (long long)dims[3], (long long)dims[4]);
  if (!elem_size(dtype)) return fail(LFBP_ERR_ARGUMENT, "dtype code %d is not 1 (f32) or 2 (f64)", dtype);
  if (inverse && ((dims[0] % 2) == 0 || (dims[1] % 2) == 0))
    return fail(LFBP_ERR_EVEN_PIXEL_DIMS,
                "inverse undefined for even pixel dims (n_s, n_t)=(%lld, %lld): the forward mapping drops "
                "elements",
                (long long)dims[0], (long long)dims[1]);
  return LFBP_OK;
}

int64_t plane_elems(const int64_t d[5]) { return d[0] * d[1] * d[2] * d[3]; }

// ---- host thread pool: parallel memcpy / pread / pwrite of staging chunks ----
class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { run(i); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // fn(a, b) over [0, n) split into one part per worker (parts aligned to
  // `align` bytes); returns when every part is done
  void for_range(size_t n, size_t align, const std::function<void(size_t, size_t)>& fn) {
    if (th_.empty() || n < (size_t(4) << 20)) {
      fn(0, n);
      return;
    }
    std::lock_guard<std::mutex> one_job(call_mu_);  // callers from several device threads take turns
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &fn;
    n_ = n;
    align_ = align;
    pending_ = int(th_.size());
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [this] { return pending_ == 0; });
  }
  void copy(void* dst, const void* src, size_t n) {
    uint8_t* d = static_cast<uint8_t*>(dst);
    const uint8_t* s = static_cast<const uint8_t*>(src);
    for_range(n, 64, [&](size_t a, size_t b) { memcpy(d + a, s + a, b - a); });
  }

 private:
  void run(int i) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      const size_t parts = th_.size();
      const size_t chunk = ((n_ / parts) + align_ - 1) / align_ * align_;
      const size_t a = std::min(n_, chunk * i), b = std::min(n_, a + chunk);
      const std::function<void(size_t, size_t)>* fn = fn_;
      lk.unlock();
      if (b > a) (*fn)(a, b);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex call_mu_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(size_t, size_t)>* fn_ = nullptr;
  size_t n_ = 0, align_ = 64;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

HostPool& copy_pool() {
  static HostPool pool(std::max(1, std::min(16, env_int("LFBP_COPY_THREADS",
                                                        int(std::thread::hardware_concurrency()) / 2))));
  return pool;
}

// ---- host pipeline workspace (one per device, reused across calls) ----
constexpr int kPipe = 3;

struct Workspace {
  std::mutex mu;
  int dev = -1;
  size_t cap = 0;
  void* in[kPipe] = {};
  void* out[kPipe] = {};
  cudaStream_t s_h2d = nullptr, s_cmp = nullptr, s_d2h = nullptr;
  cudaEvent_t h2d_done[kPipe] = {}, cmp_done[kPipe] = {}, d2h_done[kPipe] = {};
  bool init = false;
  size_t stage_cap = 0;             // pinned staging for pageable host arrays
  void* pin_in[kPipe] = {};
  void* pin_out[kPipe] = {};
};

std::mutex g_ws_mu;
std::map<int, std::unique_ptr<Workspace>> g_ws;

Workspace& workspace(int dev) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& w = g_ws[dev];
  if (!w) {
    w.reset(new Workspace());
    w->dev = dev;
  }
  return *w;
}

int ws_reserve(Workspace& w, size_t bytes) {
  if (!w.init) {
    HP_CUDA(cudaStreamCreateWithFlags(&w.s_h2d, cudaStreamNonBlocking));
    HP_CUDA(cudaStreamCreateWithFlags(&w.s_cmp, cudaStreamNonBlocking));
    HP_CUDA(cudaStreamCreateWithFlags(&w.s_d2h, cudaStreamNonBlocking));
    for (int k = 0; k < kPipe; ++k) {
      HP_CUDA(cudaEventCreateWithFlags(&w.h2d_done[k], cudaEventDisableTiming));
      HP_CUDA(cudaEventCreateWithFlags(&w.cmp_done[k], cudaEventDisableTiming));
      HP_CUDA(cudaEventCreateWithFlags(&w.d2h_done[k], cudaEventDisableTiming));
    }
    w.init = true;
  }
  if (bytes <= w.cap) return LFBP_OK;
  for (int k = 0; k < kPipe; ++k) {
    if (w.in[k]) cudaFree(w.in[k]);
    if (w.out[k]) cudaFree(w.out[k]);
    w.in[k] = w.out[k] = nullptr;
  }
  w.cap = 0;
  for (int k = 0; k < kPipe; ++k) {
    HP_CUDA(cudaMalloc(&w.in[k], bytes));
    HP_CUDA(cudaMalloc(&w.out[k], bytes));
  }
  w.cap = bytes;
  return LFBP_OK;
}

int ws_reserve_staging(Workspace& w, size_t bytes) {
  if (bytes <= w.stage_cap) return LFBP_OK;
  for (int k = 0; k < kPipe; ++k) {
    if (w.pin_in[k]) cudaFreeHost(w.pin_in[k]);
    if (w.pin_out[k]) cudaFreeHost(w.pin_out[k]);
    w.pin_in[k] = w.pin_out[k] = nullptr;
  }
  w.stage_cap = 0;
  for (int k = 0; k < kPipe; ++k) {
    HP_CUDA(cudaHostAlloc(&w.pin_in[k], bytes, cudaHostAllocPortable));
    HP_CUDA(cudaHostAlloc(&w.pin_out[k], bytes, cudaHostAllocPortable));
  }
  w.stage_cap = bytes;
  return LFBP_OK;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

struct HostPin {
  void* ptr = nullptr;
  bool registered = false;
  ~HostPin() {
    if (registered) cudaHostUnregister(ptr);
  }
};

int maybe_pin(HostPin& pin, const void* p, size_t bytes, int flags) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    a.type = cudaMemoryTypeUnregistered;
  }
  if (a.type != cudaMemoryTypeUnregistered || !(flags & LFBP_HOST_REGISTER)) return LFBP_OK;
  cudaError_t e = cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return LFBP_OK;
  }
  if (e != cudaSuccess) return fail(LFBP_ERR_CUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
  pin.ptr = const_cast<void*>(p);
  pin.registered = true;
  return LFBP_OK;
}

// Optional hooks of the host pipeline: where a chunk's input comes from and
// where its output goes when it is not a host array (the LF5 file path).
// Offsets are byte offsets of the chunk in the whole array.
using FillFn = std::function<int(uint8_t* pinned, int64_t off, size_t bytes)>;
using FlushFn = std::function<int(const uint8_t* pinned, int64_t off, size_t bytes)>;

// K4: elements failing `v >= 0` (negative or NaN), the reference's PsfArray
// value check (arrays.py:106-107), counted on the device
template <typename T>
__global__ void count_invalid_kernel(const T* __restrict__ a, int64_t n, unsigned long long* count) {
  unsigned long long c = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    c += !(a[i] >= T(0));
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// planes [z0, z1) of host src -> host dst through device `dev`; with `fill`
// / `flush` the chunks are produced / consumed by the hooks instead; with
// `invalid` (device counter) the input values are checked like PsfArray's
int host_slab(const uint8_t* src, uint8_t* dst, const int64_t dims[5], int E, int dev, int64_t z0, int64_t z1,
              int flags, const FillFn* fill = nullptr, const FlushFn* flush = nullptr,
              unsigned long long* invalid = nullptr) {
  HP_CUDA(cudaSetDevice(dev));
  const int64_t pb = plane_elems(dims) * E;
  const int64_t nz = z1 - z0;
  if (nz <= 0) return LFBP_OK;
  const int64_t target = int64_t(env_int("LFBP_CHUNK_MB", 64)) << 20;
  const int64_t cp = std::max<int64_t>(1, std::min<int64_t>(nz, target / std::max<int64_t>(pb, 1)));
  const int64_t n_chunks = (nz + cp - 1) / cp;
  // pageable arrays: stage through pinned buffers (parallel host memcpy
  // overlapped with the DMA), or pin them in place, or let the driver stage
  const bool stage_in = fill || ((flags & LFBP_HOST_STAGE) && !is_pinned(src + z0 * pb));
  const bool stage_out = flush || ((flags & LFBP_HOST_STAGE) && !is_pinned(dst + z0 * pb));
  const int reg_flags = flags & LFBP_HOST_REGISTER;
  HostPin pin_in, pin_out;
  int rc = stage_in ? LFBP_OK : maybe_pin(pin_in, src + z0 * pb, size_t(nz * pb), reg_flags);
  if (rc) return rc;
  rc = stage_out ? LFBP_OK : maybe_pin(pin_out, dst + z0 * pb, size_t(nz * pb), reg_flags);
  if (rc) return rc;
  Workspace& w = workspace(dev);
  std::lock_guard<std::mutex> lk(w.mu);
  rc = ws_reserve(w, size_t(cp * pb));
  if (rc) return rc;
  if (stage_in || stage_out) {
    rc = ws_reserve_staging(w, size_t(cp * pb));
    if (rc) return rc;
  }
  auto chunk_range = [&](int64_t c, int64_t& a, size_t& bytes) {
    a = z0 + c * cp;
    bytes = size_t(std::min<int64_t>(cp, z1 - a) * pb);
  };
  auto drain = [&](int64_t c) -> int {  // staged output of chunk c -> dst / flush hook
    int64_t a;
    size_t bytes;
    chunk_range(c, a, bytes);
    const int k = int(c % kPipe);
    HP_CUDA(cudaEventSynchronize(w.d2h_done[k]));
    if (flush) return (*flush)(static_cast<const uint8_t*>(w.pin_out[k]), a * pb, bytes);
    copy_pool().copy(dst + a * pb, w.pin_out[k], bytes);
    return LFBP_OK;
  };
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int k = int(c % kPipe);
    int64_t a;
    size_t bytes;
    chunk_range(c, a, bytes);
    const int64_t planes = int64_t(bytes) / pb;
    const uint8_t* h_src = src ? src + a * pb : nullptr;
    if (stage_in) {
      if (c >= kPipe) HP_CUDA(cudaEventSynchronize(w.h2d_done[k]));  // pin_in[k] free
      if (fill) {
        rc = (*fill)(static_cast<uint8_t*>(w.pin_in[k]), a * pb, bytes);
        if (rc) return rc;
      } else {
        copy_pool().copy(w.pin_in[k], h_src, bytes);
      }
      h_src = static_cast<const uint8_t*>(w.pin_in[k]);
    }
    if (c >= kPipe) HP_CUDA(cudaStreamWaitEvent(w.s_h2d, w.cmp_done[k], 0));  // in[k] consumed
    HP_CUDA(cudaMemcpyAsync(w.in[k], h_src, bytes, cudaMemcpyHostToDevice, w.s_h2d));
    HP_CUDA(cudaEventRecord(w.h2d_done[k], w.s_h2d));
    HP_CUDA(cudaStreamWaitEvent(w.s_cmp, w.h2d_done[k], 0));
    if (c >= kPipe) HP_CUDA(cudaStreamWaitEvent(w.s_cmp, w.d2h_done[k], 0));  // out[k] drained
    if (invalid) {
      const int64_t n = int64_t(bytes) / E;
      const int blocks = int(std::min<int64_t>(1184, (n + 255) / 256));
      if (E == 4)
        count_invalid_kernel<float><<<blocks, 256, 0, w.s_cmp>>>(static_cast<const float*>(w.in[k]), n, invalid);
      else
        count_invalid_kernel<double><<<blocks, 256, 0, w.s_cmp>>>(static_cast<const double*>(w.in[k]), n, invalid);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      HP_CUDA(cudaGetLastError());
    }
    int64_t cd[5] = {dims[0], dims[1], dims[2], dims[3], planes};
    Knobs kn;
    if (!env_knobs_set()) tuned_knobs(TuneKey{dims[0], dims[1], dims[2], dims[3], E, dev}, kn);
    HpPlan p;
    rc = make_plan(p, cd, E, 0, planes, int64_t(bytes), dev, kn);
    if (rc) return rc;
    rc = launch(p, w.in[k], w.out[k], w.s_cmp);
    if (rc) return rc;
    HP_CUDA(cudaEventRecord(w.cmp_done[k], w.s_cmp));
    HP_CUDA(cudaStreamWaitEvent(w.s_d2h, w.cmp_done[k], 0));
    HP_CUDA(cudaMemcpyAsync(stage_out ? static_cast<uint8_t*>(w.pin_out[k]) : dst + a * pb, w.out[k], bytes,
                            cudaMemcpyDeviceToHost, w.s_d2h));
    HP_CUDA(cudaEventRecord(w.d2h_done[k], w.s_d2h));
    // chunk c - (kPipe - 1) frees its pinned output before pin_out is reused
    if (stage_out && c >= kPipe - 1) {
      rc = drain(c - (kPipe - 1));
      if (rc) return rc;
    }
  }
  if (stage_out)
    for (int64_t c = std::max<int64_t>(0, n_chunks - (kPipe - 1)); c < n_chunks; ++c) {
      rc = drain(c);
      if (rc) return rc;
    }
  HP_CUDA(cudaStreamSynchronize(w.s_d2h));
  HP_CUDA(cudaStreamSynchronize(w.s_cmp));
  HP_CUDA(cudaStreamSynchronize(w.s_h2d));
  return LFBP_OK;
}

// ---- K2: device bitwise comparator ----
__global__ void compare_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                               unsigned long long* n_diff, unsigned long long* first) {
  const int64_t n16 = n / 16;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  unsigned long long cnt = 0, fst = ~0ull;
  const uint4* a4 = reinterpret_cast<const uint4*>(a);
  const uint4* b4 = reinterpret_cast<const uint4*>(b);
  for (int64_t k = tid; k < n16; k += stride) {
    const uint4 x = a4[k], y = b4[k];
    const uint32_t w[4] = {x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (w[q]) {
        for (int byte = 0; byte < 4; ++byte)
          if ((w[q] >> (8 * byte)) & 0xff) {
            ++cnt;
            fst = min(fst, (unsigned long long)(k * 16 + q * 4 + byte));
          }
      }
    }
  }
  for (int64_t k = n16 * 16 + tid; k < n; k += stride)
    if (a[k] != b[k]) {
      ++cnt;
      fst = min(fst, (unsigned long long)k);
    }
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    fst = min(fst, __shfl_xor_sync(0xffffffffu, fst, o));
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(n_diff, cnt);
    atomicMin(first, fst);
  }
}

}  // namespace

extern "C" {

int lfbp_check_dims(const int64_t dims[5]) {
  if (!dims) return fail(LFBP_ERR_ARGUMENT, "dims is NULL");
  if (!hp_dims_valid(dims[0], dims[1], dims[2], dims[3], dims[4]))
    return fail(LFBP_ERR_INVALID_DIMS, "invalid dims");
  return LFBP_OK;
}

int64_t lfbp_dropped_source_count(const int64_t d[5]) {
  if (!d || !hp_dims_valid(d[0], d[1], d[2], d[3], d[4])) return -1;
  const int64_t v_s = d[0] - (1 - d[0] % 2), v_t = d[1] - (1 - d[1] % 2);
  return (d[0] * d[1] - v_s * v_t) * d[2] * d[3] * d[4];
}

int lfbp_hprime_device(const void* src, void* dst, const int64_t dims[5], int dtype, int inverse,
                       int64_t z_begin, int64_t z_end, void* stream) {
  int rc = check_common(dims, dtype, inverse);
  if (rc) return rc;
  if (!src || !dst) return fail(LFBP_ERR_ARGUMENT, "null device pointer");
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(LFBP_ERR_ARGUMENT, "device arrays must be 16-byte aligned");
  if (z_begin < 0 || z_end > dims[4] || z_begin > z_end)
    return fail(LFBP_ERR_ARGUMENT, "plane range [%lld, %lld) outside [0, %lld)", (long long)z_begin,
                (long long)z_end, (long long)dims[4]);
  const int E = elem_size(dtype);
  const int64_t total = plane_elems(dims) * dims[4] * E;
  const uint8_t* s8 = static_cast<const uint8_t*>(src);
  uint8_t* d8 = static_cast<uint8_t*>(dst);
  if (s8 < d8 + total && d8 < s8 + total) return fail(LFBP_ERR_ARGUMENT, "src and dst overlap");
  int dev = 0;
  HP_CUDA(cudaGetDevice(&dev));
  Knobs kn;
  if (!env_knobs_set()) {
    const TuneKey key{dims[0], dims[1], dims[2], dims[3], E, dev};
    const int64_t moved = 2 * plane_elems(dims) * (z_end - z_begin) * E;
    if (!tuned_knobs(key, kn) && env_int("LFBP_AUTOTUNE", 1) && moved >= (int64_t(256) << 20)) {
      rc = autotune(key, src, dst, dims, E, z_begin, z_end - z_begin, total, static_cast<cudaStream_t>(stream), kn);
      if (rc) return rc;
    }
  }
  HpPlan p;
  rc = make_plan(p, dims, E, z_begin, z_end - z_begin, total, dev, kn);
  if (rc) return rc;
  return launch(p, src, dst, static_cast<cudaStream_t>(stream));
}

int lfbp_hprime_host(const void* src, void* dst, const int64_t dims[5], int dtype, int inverse, int device,
                     int flags) {
  int rc = check_common(dims, dtype, inverse);
  if (rc) return rc;
  if (!src || !dst) return fail(LFBP_ERR_ARGUMENT, "null host pointer");
  const int E = elem_size(dtype);
  int cur = 0;
  cudaGetDevice(&cur);
  rc = host_slab(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), dims, E, device, 0, dims[4],
                 flags);
  cudaSetDevice(cur);
  return rc;
}

int lfbp_shard_planes(int64_t n_z, int n_shards, int shard, int64_t* z_begin, int64_t* z_end) {
  if (n_z < 0 || n_shards < 1 || shard < 0 || shard >= n_shards || !z_begin || !z_end)
    return fail(LFBP_ERR_ARGUMENT, "bad shard request");
  *z_begin = (n_z * shard) / n_shards;
  *z_end = (n_z * (shard + 1)) / n_shards;
  return LFBP_OK;
}

int lfbp_hprime_multi(const void* src, void* dst, const int64_t dims[5], int dtype, int inverse, int n_devices,
                      const int* devices, int flags) {
  int rc = check_common(dims, dtype, inverse);
  if (rc) return rc;
  if (!src || !dst || n_devices < 1 || !devices) return fail(LFBP_ERR_ARGUMENT, "bad multi-GPU arguments");
  const int E = elem_size(dtype);
  // pin once for all devices (portable registration); slabs then skip it
  const size_t total = size_t(plane_elems(dims) * dims[4] * E);
  HostPin pin_in, pin_out;
  rc = maybe_pin(pin_in, src, total, flags);
  if (rc) return rc;
  rc = maybe_pin(pin_out, dst, total, flags);
  if (rc) return rc;
  const int slab_flags = flags & ~LFBP_HOST_REGISTER;
  std::vector<int> codes(n_devices, LFBP_OK);
  std::vector<std::string> msgs(n_devices);
  std::vector<std::thread> th;
  for (int g = 0; g < n_devices; ++g) {
    int64_t z0, z1;
    lfbp_shard_planes(dims[4], n_devices, g, &z0, &z1);
    th.emplace_back([&, g, z0, z1] {
      codes[g] = host_slab(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), dims, E, devices[g],
                           z0, z1, slab_flags);
      if (codes[g]) msgs[g] = g_err;
    });
  }
  for (auto& t : th) t.join();
  for (int g = 0; g < n_devices; ++g)
    if (codes[g]) return fail(codes[g], "device %d: %s", devices[g], msgs[g].c_str());
  return LFBP_OK;
}

int lfbp_compare_device(const void* a, const void* b, int64_t nbytes, int64_t* n_diff, int64_t* first_diff,
                        void* stream) {
  if (!a || !b || nbytes < 0 || !n_diff || !first_diff) return fail(LFBP_ERR_ARGUMENT, "bad compare arguments");
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15)
    return fail(LFBP_ERR_ARGUMENT, "compare buffers must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* scratch = nullptr;
  HP_CUDA(cudaMalloc(&scratch, 2 * sizeof(unsigned long long)));
  unsigned long long init[2] = {0ull, ~0ull};
  cudaError_t e = cudaMemcpyAsync(scratch, init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    int dev = 0;
    cudaGetDevice(&dev);
    const DevProps dp = device_props(dev);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(dp.sm_count) * 8, (nbytes / 16 + 255) / 256));
    compare_kernel<<<int(blocks), 256, 0, st>>>(static_cast<const uint8_t*>(a), static_cast<const uint8_t*>(b),
                                                nbytes, scratch, scratch + 1);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
  }
  unsigned long long res[2] = {0ull, ~0ull};
  if (e == cudaSuccess) e = cudaMemcpyAsync(res, scratch, sizeof(res), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(scratch);
  if (e != cudaSuccess) return fail(LFBP_ERR_CUDA, "compare: %s", cudaGetErrorString(e));
  *n_diff = int64_t(res[0]);
  *first_diff = res[0] ? int64_t(res[1]) : -1;
  return LFBP_OK;
}

int lfbp_plan_json(const int64_t dims[5], int dtype, char* buf, int64_t buf_len) {
  int rc = check_common(dims, dtype, 0);
  if (rc) return rc;
  if (!buf || buf_len < 1) return fail(LFBP_ERR_ARGUMENT, "null buffer");
  int dev = 0;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    dev = -1;
  } else {
    cudaGetDevice(&dev);
  }
  const int E = elem_size(dtype);
  Knobs kn;
  const bool tuned = !env_knobs_set() && tuned_knobs(TuneKey{dims[0], dims[1], dims[2], dims[3], E, dev}, kn);
  HpPlan p;
  rc = make_plan(p, dims, E, 0, dims[4], plane_elems(dims) * dims[4] * E, dev, kn);
  if (rc) return rc;
  const DevProps dp = device_props(dev);
  int w = snprintf(buf, size_t(buf_len),
                   "{\"elem\": %d, \"J\": %d, \"n_bands\": %d, \"C\": %d, \"n_chunks\": %d, \"row_pitch\": %d, "
                   "\"stage_bytes\": %d, \"stages\": %d, \"threads\": %d, \"smem_bytes\": %d, \"ctas_per_sm\": %d, "
                   "\"grid\": %d, \"n_units\": %lld, \"sub_width\": %d, \"sm_count\": %d, \"device_props\": \"%s\", "
                   "\"autotuned\": %s}",
                   p.elem, p.J, p.n_bands, p.C, p.n_chunks, p.row_pitch, p.stage_bytes, p.stages, p.threads,
                   p.smem_bytes, p.ctas_per_sm, p.grid, (long long)p.n_units, p.sub_width, dp.sm_count,
                   dp.real ? "queried" : "b200-defaults", tuned ? "true" : "false");
  if (w < 0 || w >= buf_len) return fail(LFBP_ERR_ARGUMENT, "buffer too small");
  return LFBP_OK;
}

int lfbp_plane_sums_device(const void* src, double* out, const int64_t dims[5], int dtype, int64_t z_begin,
                           int64_t z_end, void* stream) {
  // any positive shape (the reference sums unchecked-dims arrays too, fileio.py:95-104)
  if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1 || dims[3] < 1 || dims[4] < 1)
    return fail(LFBP_ERR_INVALID_DIMS, "dims must all be >= 1");
  if (!elem_size(dtype)) return fail(LFBP_ERR_ARGUMENT, "dtype code %d is not 1 (f32) or 2 (f64)", dtype);
  if (!src || !out) return fail(LFBP_ERR_ARGUMENT, "null device pointer");
  if (z_begin < 0 || z_end > dims[4] || z_begin > z_end)
    return fail(LFBP_ERR_ARGUMENT, "plane range [%lld, %lld) outside [0, %lld)", (long long)z_begin,
                (long long)z_end, (long long)dims[4]);
  const int64_t K = dims[2] * dims[3];
  if (K > 8192) return fail(LFBP_ERR_UNSUPPORTED, "slice of %lld values exceeds the sort limit 8192", (long long)K);
  int P = 32;
  while (P < K) P <<= 1;
  const int64_t n_slices = dims[0] * dims[1] * (z_end - z_begin);
  if (n_slices == 0) return LFBP_OK;
  int dev = 0;
  HP_CUDA(cudaGetDevice(&dev));
  const DevProps dp = device_props(dev);
  const int wpc = int(std::max<int64_t>(1, std::min<int64_t>(8, (dp.smem_optin / 2) / (int64_t(P) * 8))));
  const size_t smem = size_t(wpc) * P * 8;
  const int64_t blocks = std::min<int64_t>((n_slices + wpc - 1) / wpc, int64_t(dp.sm_count) * 16);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == LFBP_F32) {
    HP_CUDA(cudaFuncSetAttribute(hp::plane_sums_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    hp::plane_sums_kernel<float><<<int(blocks), 32 * wpc, smem, st>>>(
        static_cast<const float*>(src), out, int32_t(dims[0]), int32_t(dims[1]), int32_t(K), P, z_begin, n_slices);
  } else {
    HP_CUDA(cudaFuncSetAttribute(hp::plane_sums_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    hp::plane_sums_kernel<double><<<int(blocks), 32 * wpc, smem, st>>>(
        static_cast<const double*>(src), out, int32_t(dims[0]), int32_t(dims[1]), int32_t(K), P, z_begin, n_slices);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  HP_CUDA(cudaGetLastError());
  return LFBP_OK;
}

int lfbp_forward_project2_device(const void* H, const void* Hp, int dtype, const int64_t dims[5],
                                 const double* volume, int64_t nvx, int64_t nvy, double* image, void* stream);

static int proj_geom(hp::ProjGeom& q, const int64_t dims[5], int64_t nvx, int64_t nvy) {
  if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1 || dims[3] < 1 || dims[4] < 1 || nvx < 1 || nvy < 1)
    return fail(LFBP_ERR_INVALID_DIMS, "bad projector geometry");
  if (dims[0] * dims[1] * dims[2] * dims[3] >= (int64_t(1) << 31) || nvx * nvy >= (int64_t(1) << 31))
    return fail(LFBP_ERR_UNSUPPORTED, "projector plane too large");
  q.n_s = int32_t(dims[0]);
  q.n_t = int32_t(dims[1]);
  q.n_x = int32_t(dims[2]);
  q.n_y = int32_t(dims[3]);
  q.n_z = int32_t(dims[4]);
  // pattern_centre (projector.py:26-32) minus one
  q.c_s = int32_t(dims[0] % 2 ? (dims[0] + 1) / 2 - 1 : dims[0] / 2);
  q.c_t = int32_t(dims[1] % 2 ? (dims[1] + 1) / 2 - 1 : dims[1] / 2);
  q.nvx = int32_t(nvx);
  q.nvy = int32_t(nvy);
  return LFBP_OK;
}

constexpr int kPolyRLMax = 16;  // max coarse rows per thread in poly_corr_kernel

// rows per thread: the tap count N when 4 <= N <= 16 (whole taps blocks, no
// register shifting), else 8
inline int poly_rows(int32_t N) { return (N >= 4 && N <= kPolyRLMax) ? N : 8; }

extern "C++" {
template <typename T, int RL>
void poly_launch_rl(dim3 grd, cudaStream_t st, const double* sub, const void* K, double* dst, const hp::ProjGeom& q,
                    const hp::PolyGeom& pg, bool forward) {
  hp::poly_corr_kernel<T, RL><<<grd, 128, 0, st>>>(sub, static_cast<const T*>(K), dst, q, pg, forward);
}

template <typename T>
void poly_launch(int rl, dim3 grd, cudaStream_t st, const double* sub, const void* K, double* dst,
                 const hp::ProjGeom& q, const hp::PolyGeom& pg, bool forward) {
  switch (rl) {
#define HP_RL(n) \
  case n:        \
    return poly_launch_rl<T, n>(grd, st, sub, K, dst, q, pg, forward);
    HP_RL(4) HP_RL(5) HP_RL(6) HP_RL(7) HP_RL(9) HP_RL(10) HP_RL(11) HP_RL(12) HP_RL(13) HP_RL(14) HP_RL(15)
    HP_RL(16)
#undef HP_RL
    default:
      return poly_launch_rl<T, 8>(grd, st, sub, K, dst, q, pg, forward);
  }
}
}  // extern "C++"

// polyphase correlation (projector.cuh): pad+split the input planes, then one
// block per (coarse tile, output phase[, output plane])
static int poly_corr(const void* K, int dtype, const hp::ProjGeom& q, const double* in, int32_t in_planes,
                     double* out, bool forward, cudaStream_t st) {
  hp::PolyGeom pg;
  pg.kc = (q.nvx + q.n_x - 1) / q.n_x;
  pg.lc = (q.nvy + q.n_y - 1) / q.n_y;
  pg.hx = (q.n_s + q.n_x - 1) / q.n_x + 1;
  const int32_t N = (q.n_t + q.n_y - 1) / q.n_y;  // taps per residue class along y
  const int rl = poly_rows(N);
  pg.hy = N + rl - 1;
  pg.kp = pg.kc + 2 * pg.hx;
  pg.lp = pg.lc + 2 * pg.hy;
  const int64_t n_sub = int64_t(pg.kp) * pg.lp * q.n_x * q.n_y * in_planes;
  double* sub = nullptr;
  HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sub), size_t(n_sub) * sizeof(double), st));
  const int pb = int(std::min<int64_t>(4736, (n_sub + 255) / 256));
  hp::polyphase_pad_kernel<<<pb, 256, 0, st>>>(in, sub, q, pg, in_planes);
  const int32_t n_ph = q.n_x * q.n_y;
  const int64_t img = int64_t(q.nvx) * q.nvy;
  double* part = nullptr;  // forward: per-plane partial images
  if (forward) HP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), size_t(img * q.n_z) * sizeof(double), st));
  const dim3 grd(unsigned((int64_t(q.n_x) * pg.kc + 127) / 128), unsigned((pg.lc + rl - 1) / rl),
                 unsigned(q.n_y * q.n_z));
  (void)n_ph;
  double* dst = forward ? part : out;
  if (dtype == LFBP_F32)
    poly_launch<float>(rl, grd, st, sub, K, dst, q, pg, forward);
  else
    poly_launch<double>(rl, grd, st, sub, K, dst, q, pg, forward);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  if (forward) {
    hp::sum_planes_kernel<<<int(std::min<int64_t>(1184, (img + 255) / 256)), 256, 0, st>>>(part, out, img, q.n_z);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(sub, st);
  if (part) cudaFreeAsync(part, st);
  if (e != cudaSuccess) return fail(LFBP_ERR_CUDA, "projector: %s", cudaGetErrorString(e));
  return LFBP_OK;
}

int lfbp_forward_project_device(const void* H, int dtype, const int64_t dims[5], const double* volume, int64_t nvx,
                                int64_t nvy, double* image, void* stream) {
  return lfbp_forward_project2_device(H, nullptr, dtype, dims, volume, nvx, nvy, image, stream);
}

int lfbp_forward_project2_device(const void* H, const void* Hp, int dtype, const int64_t dims[5], const double* volume,
                                 int64_t nvx, int64_t nvy, double* image, void* stream) {
  hp::ProjGeom q;
  int rc = proj_geom(q, dims, nvx, nvy);
  if (rc) return rc;
  if ((!H && !Hp) || !volume || !image || !elem_size(dtype))
    return fail(LFBP_ERR_ARGUMENT, "bad forward_project arguments");
  const bool odd = (dims[0] % 2) && (dims[1] % 2);
  if (!H && !odd) return fail(LFBP_ERR_EVEN_PIXEL_DIMS, "the H' form of the forward projection needs odd n_s, n_t");
  const dim3 blk(32, 8), grd(unsigned((nvx + 31) / 32), unsigned((nvy + 7) / 8));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (Hp && odd) {  // pixel-phase form, same sums as the H form
    if (env_int("LFBP_PROJ_SIMPLE", 0) == 0) return poly_corr(Hp, dtype, q, volume, q.n_z, image, true, st);
    if (dtype == LFBP_F32)
      hp::forward_project_hp_kernel<float><<<grd, blk, 0, st>>>(static_cast<const float*>(Hp), volume, image, q);
    else
      hp::forward_project_hp_kernel<double><<<grd, blk, 0, st>>>(static_cast<const double*>(Hp), volume, image, q);
  } else if (dtype == LFBP_F32) {
    hp::forward_project_kernel<float><<<grd, blk, 0, st>>>(static_cast<const float*>(H), volume, image, q);
  } else {
    hp::forward_project_kernel<double><<<grd, blk, 0, st>>>(static_cast<const double*>(H), volume, image, q);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  HP_CUDA(cudaGetLastError());
  return LFBP_OK;
}

int lfbp_backproject_device(const void* P, int dtype, const int64_t dims[5], int use_hprime, const double* image,
                            int64_t npx, int64_t npy, double* volume, void* stream) {
  hp::ProjGeom q;
  int rc = proj_geom(q, dims, npx, npy);
  if (rc) return rc;
  if (!P || !volume || !image || !elem_size(dtype)) return fail(LFBP_ERR_ARGUMENT, "bad backproject arguments");
  const dim3 blk(32, 8), grd(unsigned((npx + 31) / 32), unsigned((npy + 7) / 8), unsigned(dims[4]));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!use_hprime && env_int("LFBP_PROJ_SIMPLE", 0) == 0)  // adjoint: voxel-phase polyphase correlation
    return poly_corr(P, dtype, q, image, 1, volume, false, st);
  if (dtype == LFBP_F32)
    hp::backproject_kernel<float><<<grd, blk, 0, st>>>(static_cast<const float*>(P), image, volume, q, use_hprime);
  else
    hp::backproject_kernel<double><<<grd, blk, 0, st>>>(static_cast<const double*>(P), image, volume, q, use_hprime);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  HP_CUDA(cudaGetLastError());
  return LFBP_OK;
}

int lfbp_safe_divide_device(const double* num, const double* den, double* out, int64_t n, double eps,
                            double* scratch, void* stream) {
  if (!num || !den || !out || !scratch || n < 0) return fail(LFBP_ERR_ARGUMENT, "bad safe_divide arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HP_CUDA(cudaMemsetAsync(scratch, 0, sizeof(double), st));
  if (n == 0) return LFBP_OK;
  const int blocks = int(std::min<int64_t>(1184, (n + 255) / 256));
  hp::max_kernel<<<blocks, 256, 0, st>>>(den, n, scratch);
  hp::safe_divide_kernel<<<blocks, 256, 0, st>>>(num, den, out, n, eps, scratch);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  HP_CUDA(cudaGetLastError());
  return LFBP_OK;
}

int64_t lfbp_launch_count(void) { return g_launches.load(); }

const char* lfbp_last_error(void) { return g_err.c_str(); }

const char* lfbp_version(void) { return "lfbp-b200 0.1.0 (sm_100a)"; }

}  // extern "C"

#include "lf5_stream.inc"
