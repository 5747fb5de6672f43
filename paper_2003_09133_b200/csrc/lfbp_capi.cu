// C-ABI of the B200-native H -> H' rearrangement (see include/lfbp_hprime.h).
//
// Host runtime around the K1 kernel: dims validation with the reference's
// rules, the launch planner (work-unit shape, smem ring, persistent grid) and
// its autotuner, the device-array entry point and the z-slab multi-GPU
// launcher.  One translation unit; the rest is included:
//   host_pipeline.inc   chunked H2D / K1 / D2H pipeline for host arrays
//   verify_capi.inc     K2 comparator, K3 plane sums
//   projector_capi.inc  K5 projector launchers
//   lf5_stream.inc      LF5 file streaming (K4 value check)
#include <cuda_runtime.h>
#include <stdint.h>
#include <sys/mman.h>

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
#include "synth.cuh"

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

// Ticket counters of HP_FLAG_DYNAMIC launches: a ring of 128-byte slots per
// device ([0] the ticket, [1] CTAs done), zeroed once at allocation; the last
// CTA of a launch zeroes its slot again for the slot's next launch, so no
// memset is queued per launch.  Launches in flight at once get different
// slots as long as fewer than kCounterSlots are in flight.
constexpr int kCounterSlots = 1024;
std::mutex g_ctr_mu;
std::map<int, unsigned long long*> g_ctr_pool;
std::atomic<uint32_t> g_ctr_next{0};

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
#if defined(HP_CHECKED)
    p.smem_optin -= 1024;  // the checked build's static shared variables
#endif
    cudaDeviceGetAttribute(&p.max_threads_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
    p.real = true;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaFuncSetAttribute(hp::hprime_kernel<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_optin);
    cudaFuncSetAttribute(hp::hprime_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_optin);
    cudaFuncSetAttribute(hp::hprime_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_optin);
    cudaFuncSetAttribute(hp::hprime_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_optin);
    {  // the ticket-counter ring, allocated here so that no launch (or stream
       // capture) ever has to allocate
      std::lock_guard<std::mutex> lk2(g_ctr_mu);
      unsigned long long* c = nullptr;
      if (!g_ctr_pool.count(dev) && cudaMalloc(&c, kCounterSlots * 128) == cudaSuccess) {
        if (cudaMemset(c, 0, kCounterSlots * 128) == cudaSuccess)
          g_ctr_pool[dev] = c;
        else
          cudaFree(c);
      }
    }
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
  int flags = 0;       // HP_FLAG_* unit order (HP_FLAG_DIAGONAL, HP_FLAG_ROTATE)
  int grid_sm = 0;     // SMs given a persistent CTA (0 = all): fewer requests in flight
};
constexpr int kKnobFields = 6;

const char* const kKnobEnv[] = {"LFBP_STAGES", "LFBP_STAGE_KB", "LFBP_CONSUMER_WARPS", "LFBP_SUBWARP",
                                "LFBP_CTAS_PER_SM", "LFBP_BAND", "LFBP_STAGE_MAX_KB", "LFBP_KFLAGS",
                                "LFBP_GRID", "LFBP_TILE_Y"};

bool env_knobs_set() {
  for (const char* n : kKnobEnv) {
    const char* v = getenv(n);
    if (v && *v) return true;
  }
  return false;
}

constexpr int64_t kAutotuneMinBytes = int64_t(256) << 20;  // bytes moved (r+w): large-problem candidates
constexpr int64_t kSmallTuneMinBytes = int64_t(8) << 20;   // ... small-problem candidates from here

// Size class of a launch for the tuner: 1 large, 0 small, -1 not tuned.
int tune_class(int64_t moved_bytes) {
  return moved_bytes >= kAutotuneMinBytes ? 1 : moved_bytes >= kSmallTuneMinBytes ? 0 : -1;
}

// Untuned knobs.  Below the large-problem size a launch is latency-bound:
// fewer, busier consumer warps per CTA and more CTAs (C1: 14.5 vs 17 us).
Knobs default_knobs(int64_t moved_bytes) {
  Knobs kn;
  if (moved_bytes < kAutotuneMinBytes)
    kn.cwarps = 8;
  else
    kn.flags = HP_FLAG_DYNAMIC;  // level CTAs: the tuned plans of C2-C5 all take tickets
  return kn;
}

// Candidates tried by the autotuner (measured best plans of C1..C5 and
// neighbours; every one is bit-exact, they differ only in speed).
const Knobs kCandidates[] = {
    // Dynamic unit tickets (HP_FLAG_DYNAMIC) hold the persistent CTAs level:
    // every tuned C2-C5 plan since takes them (profiles/r02_dynamic_ab.jsonl,
    // r02_sweep_c2_c3_row.jsonl, r02_c5_tickets_sweep.jsonl).  Narrow bands and
    // 8-lane rows lead (C2 J = 4, C3 J = 1 with 3 CTAs per SM, C5 along y'
    // diagonals); the task consumer draws less power and wins on the most
    // power-limited boxes.
    {4, 48, 12, 8, HP_FLAG_DYNAMIC}, {4, 64, 12, 8, HP_FLAG_DYNAMIC}, {2, 32, 8, 8, HP_FLAG_DYNAMIC},
    {3, 32, 8, 8, HP_FLAG_DYNAMIC}, {3, 64, 12, 16, HP_FLAG_DYNAMIC}, {4, 32, 8, 8, HP_FLAG_DYNAMIC},
    {4, 48, 8, 16, HP_FLAG_DYNAMIC}, {4, 48, 12, 8, HP_FLAG_DIAGONAL | HP_FLAG_DYNAMIC},
    {3, 64, 8, 32, HP_FLAG_DIAGONAL | HP_FLAG_DYNAMIC}, {2, 96, 12, 0, HP_FLAG_TASKS | HP_FLAG_DYNAMIC},
    // static round-robin plans, the round-1 bests (C2 {3,48,8,8}, C3 J = 3
    // {2,96,12,32}, C4 and C5 {3,64,8,32}), and C5's best before tickets:
    // diagonal order, ~12 GB launches (HP_FLAG_ZCHUNK), 145 of 148 SMs
    // (profiles/r02_zchunk.jsonl, r02_grid_sweep_fine.jsonl)
    {3, 48, 8, 8}, {4, 48, 12, 16}, {2, 96, 8, 8}, {3, 64, 8, 32}, {2, 96, 12, 32},
    {4, 16, 8, 0}, {4, 16, 4, 4},
    {3, 64, 8, 32, HP_FLAG_DIAGONAL | HP_FLAG_ZCHUNK, 145},
};
// Small problems (8-256 MB moved) are latency-bound: smaller stages (narrower
// t-bands, several CTAs per SM) and short-row sub-warps; measured on the
// paper's small Table 1 geometries and C1 (profiles/r01_small_shapes.jsonl).
const Knobs kSmallCandidates[] = {
    {4, 48, 8, 0}, {4, 16, 8, 0}, {4, 16, 4, 4}, {4, 8, 8, 4},
    {4, 24, 8, 0}, {4, 32, 8, 0}, {4, 12, 4, 4}, {4, 16, 8, 8},
    {4, 48, 8, 0, HP_FLAG_DYNAMIC}, {4, 16, 8, 0, HP_FLAG_DYNAMIC}, {4, 24, 8, 0, HP_FLAG_DYNAMIC},
    {4, 16, 4, 4, HP_FLAG_DYNAMIC},
};
constexpr int kNumCandidates = int(sizeof(kCandidates) / sizeof(kCandidates[0]));
constexpr int kNumSmallCandidates = int(sizeof(kSmallCandidates) / sizeof(kSmallCandidates[0]));
static_assert(kNumSmallCandidates <= kNumCandidates, "arrays in autotune() are sized by the large set");

// Average shared-memory wavefronts per LDS of the task consumer
// (consume_unit_tasks) on the first unit of plane 0 with row pitch `rp`:
// the 32 lanes of a warp take consecutive (row, phase class) tasks.  Used
// to pick the pitch; a model, not a measurement.
double task_bank_cost(const int64_t d[5], int E, int J, int C, int32_t rp) {
  const int64_t n_s = d[0], n_t = d[1], n_x = d[2], n_y = d[3];
  const int VE = 16 / E;
  const int64_t c_s = (n_s - 1) / 2, c_t = (n_t - 1) / 2;
  const int64_t nx_off = (n_x - (c_s % n_x)) % n_x, ny_off = (n_y - (c_t % n_y)) % n_y;
  const int64_t xs16 = (n_s * n_t * E) & 15;
  const int64_t ntask = std::min<int64_t>(int64_t(J) * n_x * n_x, 32 * 16);
  const int64_t i_end = std::min<int64_t>(C, 2 * c_s + 1);
  double waves = 0;
  int n = 0;
  for (int64_t t0 = 0; t0 < ntask; t0 += 32) {
    for (int q = 0; q < VE; ++q) {
      int64_t words[32 * 2];
      int nw = 0;
      for (int64_t task = t0; task < std::min<int64_t>(t0 + 32, ntask); ++task) {
        const int64_t r = task / n_x, c = task % n_x, tl = r / n_x, xp = r % n_x;
        if (tl >= n_t) continue;
        const int64_t j = 2 * c_t - tl, yp = (tl + ny_off) % n_y;
        const int64_t o_in = n_s * j + n_s * n_t * (xp + n_x * yp);
        const int64_t gs = -(o_in & (VE - 1));
        const int64_t i = gs + VE * c + q;
        if (i < 0 || i >= i_end) continue;
        const int64_t x = (xp + i + nx_off) % n_x;
        const int64_t k = tl * n_s + 2 * c_s - i;
        const int64_t a = 80 + x * rp + ((x * xs16) & 15) + k * E;
        for (int h = 0; h < E / 4; ++h) words[nw++] = a / 4 + h;
      }
      std::sort(words, words + nw);
      const int nu = int(std::unique(words, words + nw) - words);
      int per_bank[32] = {0};
      int worst = 0;
      for (int u = 0; u < nu; ++u) worst = std::max(worst, ++per_bank[words[u] & 31]);
      waves += worst;
      ++n;
    }
  }
  return n ? waves / n : 0.0;
}

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
  p.flags = env_int("LFBP_KFLAGS", kn.flags);
  const bool tasks = (p.flags & HP_FLAG_TASKS) != 0;
  int64_t pitch = round_up(run_max + 32, 16);
  if (tasks) {
    // task consumer: any multiple of 16; pick the one with the fewest
    // shared-memory wavefronts for a warp's 32 tasks (task_bank_cost)
    const int extra = env_int("LFBP_PITCH_EXTRA16", -1);
    if (extra >= 0) {
      pitch += 16 * extra;
    } else {
      int64_t best = pitch;
      double best_cost = 1e30;
      for (int e = 0; e < 8; ++e) {
        const double c = task_bank_cost(d, E, p.J, p.C, static_cast<int32_t>(pitch + 16 * e));
        if (c < best_cost - 1e-9) {
          best_cost = c;
          best = pitch + 16 * e;
        }
      }
      pitch = best;
    }
    p.row_pitch = static_cast<int32_t>(pitch);
  } else {
    if (((pitch / 16) & 1) == 0) pitch += 16;
    pitch += env_int("LFBP_PITCH_EXTRA16", 0) * 16;
    p.row_pitch = static_cast<int32_t>(pitch + p.xs16);
  }
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
  // producer warps: one per 32 runs of a unit (the runs of one warp issue
  // serially), within the kernel's 17-warp launch bound
  int prod = env_int("LFBP_PRODUCERS", int((d[2] + 31) / 32));
  prod = std::max(1, std::min(prod, 17 - cwarps));
  p.producers = prod;
  const int threads = 32 * (prod + cwarps);  // producers + consumers
  p.threads = threads;

  const int64_t units = z_count * p.n_chunks * int64_t(p.n_bands) * d[3];
  if (units >= (1ll << 31)) return fail(LFBP_ERR_UNSUPPORTED, "too many work units (%lld)", (long long)units);
  p.n_units = units;
  int per_sm = 0;
  if (dp.real) {
    const void* fn = (E == 4) ? (tasks ? reinterpret_cast<const void*>(hp::hprime_kernel<4, true>)
                                       : reinterpret_cast<const void*>(hp::hprime_kernel<4, false>))
                              : (tasks ? reinterpret_cast<const void*>(hp::hprime_kernel<8, true>)
                                       : reinterpret_cast<const void*>(hp::hprime_kernel<8, false>));
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, p.smem_bytes);
    if (e != cudaSuccess) return fail(LFBP_ERR_CUDA, "occupancy query: %s", cudaGetErrorString(e));
  } else {
    per_sm = std::min<int>(dp.max_threads_sm / threads, int((233472) / (p.smem_bytes + 1024)));
  }
  const int cap = env_int("LFBP_CTAS_PER_SM", 0);
  if (cap > 0) per_sm = std::min(per_sm, cap);
  if (per_sm < 1) return fail(LFBP_ERR_UNSUPPORTED, "kernel does not fit on an SM");
  p.ctas_per_sm = per_sm;
  p.grid = static_cast<int32_t>(std::min<int64_t>(units, int64_t(per_sm) * dp.sm_count));
  const int grid_cap = env_int("LFBP_GRID", kn.grid_sm);  // fewer persistent CTAs
  if (grid_cap > 0) p.grid = std::min<int32_t>(p.grid, int32_t(int64_t(grid_cap) * per_sm));
  // lanes per output row: enough 16-byte groups per lane to amortise the row setup
  const int64_t groups = (std::min<int64_t>(p.C, d[0]) * E + 15) / 16 + 1;
  int W = env_int("LFBP_SUBWARP", kn.subwarp);
  if (W != 2 && W != 4 && W != 8 && W != 16 && W != 32) W = groups <= 16 ? 4 : groups <= 32 ? 8 : groups <= 64 ? 16 : 32;
  p.sub_width = W;
  p.gx_inc = static_cast<int32_t>((W * (16 / E)) % d[2]);
  p.nx_div = hp_fastdiv_make(static_cast<uint32_t>(d[2]));
  p.ny_div = hp_fastdiv_make(static_cast<uint32_t>(d[3]));
  p.nb_div = hp_fastdiv_make(static_cast<uint32_t>(p.n_bands));
  p.nc_div = hp_fastdiv_make(static_cast<uint32_t>(p.n_chunks));
  // y blocks of 4 when a unit has more than 32 source runs: concurrent units
  // then span 4 y x ~37 bands instead of all y x ~3 bands, so both the runs
  // they read and the rows they write sit in longer contiguous stretches
  // ((181,181,95,55): 0.74 -> 0.82 of copy; (307,307,51,51): 0.84 -> 0.86).
  // With n_x <= 32 (all BASELINE configs) plain y-fastest order measured best
  // (profiles/r01_order_probe.jsonl).
  int ty = env_int("LFBP_TILE_Y", (p.flags & HP_FLAG_DIAGONAL) ? 1 : d[2] > 32 ? 4 : int(d[3]));
  ty = std::max<int>(1, std::min<int>(ty, int(d[3])));
  p.tile_y = ty;
  p.n_yblocks = static_cast<int32_t>((d[3] + ty - 1) / ty);
  p.zc_div = hp_fastdiv_make(static_cast<uint32_t>(d[3] * p.n_bands));
  p.yblk_div = hp_fastdiv_make(static_cast<uint32_t>(int64_t(ty) * p.n_bands));
  p.ty_div = hp_fastdiv_make(static_cast<uint32_t>(ty));
  p.tyl_div = hp_fastdiv_make(static_cast<uint32_t>(d[3] - int64_t(ty) * (p.n_yblocks - 1)));
  return LFBP_OK;
}


int counter_slot(unsigned long long** out) {
  int dev = 0;
  HP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ctr_mu);
  auto it = g_ctr_pool.find(dev);
  if (it == g_ctr_pool.end()) {
    unsigned long long* p = nullptr;
    HP_CUDA(cudaMalloc(&p, kCounterSlots * 128));
    HP_CUDA(cudaMemset(p, 0, kCounterSlots * 128));
    it = g_ctr_pool.emplace(dev, p).first;
  }
  // one 128-byte line per slot
  *out = it->second + 16 * (g_ctr_next.fetch_add(1, std::memory_order_relaxed) % kCounterSlots);
  return LFBP_OK;
}

int launch_one(const HpPlan& p0, const void* src, void* dst, cudaStream_t st) {
  if (p0.n_units == 0) return LFBP_OK;
  HpPlan p = p0;
  if (p.flags & HP_FLAG_DYNAMIC) {
    int rc = counter_slot(&p.counter);
    if (rc) return rc;
  }
  const uint8_t* s8 = static_cast<const uint8_t*>(src);
  uint8_t* d8 = static_cast<uint8_t*>(dst);
  const bool tasks = (p.flags & HP_FLAG_TASKS) != 0;
  if (p.elem == 4) {
    if (tasks)
      hp::hprime_kernel<4, true><<<p.grid, p.threads, p.smem_bytes, st>>>(p, s8, d8);
    else
      hp::hprime_kernel<4, false><<<p.grid, p.threads, p.smem_bytes, st>>>(p, s8, d8);
  } else {
    if (tasks)
      hp::hprime_kernel<8, true><<<p.grid, p.threads, p.smem_bytes, st>>>(p, s8, d8);
    else
      hp::hprime_kernel<8, false><<<p.grid, p.threads, p.smem_bytes, st>>>(p, s8, d8);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  HP_CUDA(cudaGetLastError());
  return LFBP_OK;
}

// HP_FLAG_ZCHUNK: one launch per slab of about kZChunkBytes moved (r+w).  The
// persistent CTAs take units round-robin without synchronising, so in a long
// launch they drift apart and the units in flight spread over more rows and
// pages; on C5 a 22 ms launch falls from 6.35 to 5.6-5.8 TB/s that way
// (profiles/r02_zchunk.jsonl).  Each launch starts them level again.
constexpr int64_t kZChunkBytes = int64_t(12) << 30;

int launch(const HpPlan& p, const void* src, void* dst, cudaStream_t st) {
  if (!(p.flags & HP_FLAG_ZCHUNK)) return launch_one(p, src, dst, st);
  const int64_t plane_rw = 2 * p.n_s * p.n_t * p.n_x * p.n_y * p.elem;
  const int64_t want = int64_t(env_int("LFBP_ZCHUNK_MB", int(kZChunkBytes >> 20))) << 20;
  const int64_t k = std::max<int64_t>(1, (want + plane_rw / 2) / plane_rw);
  if (p.z_count <= k) return launch_one(p, src, dst, st);
  const int64_t per_plane = p.n_units / p.z_count;
  for (int64_t z = 0; z < p.z_count; z += k) {
    HpPlan c = p;
    c.z_begin = p.z_begin + z;
    c.z_count = std::min<int64_t>(k, p.z_count - z);
    c.n_units = per_plane * c.z_count;
    c.grid = static_cast<int32_t>(std::min<int64_t>(p.grid, c.n_units));
    int rc = launch_one(c, src, dst, st);
    if (rc) return rc;
  }
  return LFBP_OK;
}

// ---- autotuner: per (plane shape, element size, device), first large call ----
struct TuneKey {
  int64_t n_s, n_t, n_x, n_y;
  int E, dev;
  int cls;  // tune_class of the launch size: small and large launches tune separately
  bool operator<(const TuneKey& o) const {
    if (n_s != o.n_s) return n_s < o.n_s;
    if (n_t != o.n_t) return n_t < o.n_t;
    if (n_x != o.n_x) return n_x < o.n_x;
    if (n_y != o.n_y) return n_y < o.n_y;
    if (E != o.E) return E < o.E;
    if (cls != o.cls) return cls < o.cls;
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
  // every event this function creates is destroyed on every return path
  struct Events {
    std::vector<cudaEvent_t> v;
    cudaError_t make(cudaEvent_t* e) {
      cudaError_t r = cudaEventCreate(e);
      if (r == cudaSuccess) v.push_back(*e);
      return r;
    }
    ~Events() {
      for (cudaEvent_t e : v) cudaEventDestroy(e);
    }
  } events;
  cudaEvent_t e0, e1;
  HP_CUDA(events.make(&e0));
  HP_CUDA(events.make(&e1));
  // candidates interleaved over rounds (decorrelates clock / power drift);
  // each measurement is `reps` back-to-back launches (>= ~8 ms, so a plan is
  // judged at its steady-state rate, not on one launch after an idle gap);
  // score = median over rounds of the per-launch time
  constexpr int kCand = kNumCandidates;
  constexpr int kRounds = 4;
  const Knobs* cand = key.cls == 1 ? kCandidates : kSmallCandidates;
  const int n_cand = key.cls == 1 ? kNumCandidates : kNumSmallCandidates;
  HpPlan plans[kCand];
  bool ok[kCand] = {};
  float t[kCand][kRounds];
  cudaEvent_t ev[kCand][2];
  for (int c = 0; c < n_cand; ++c) {
    HP_CUDA(events.make(&ev[c][0]));
    HP_CUDA(events.make(&ev[c][1]));
  }
  float warm_ms = 0.f;
  for (int c = 0; c < n_cand; ++c) {
    ok[c] = make_plan(plans[c], dims, E, z_begin, z_count, total, key.dev, cand[c]) == LFBP_OK;
    if (ok[c]) {
      HP_CUDA(cudaEventRecord(e0, st));
      int rc = launch(plans[c], src, dst, st);  // warm
      if (rc) return rc;
      HP_CUDA(cudaEventRecord(e1, st));
      HP_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      HP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      warm_ms = std::max(warm_ms, ms);
    }
  }
  const int reps = std::max(1, std::min(64, int(8.0f / std::max(warm_ms, 1e-3f))));
  for (int r = 0; r < kRounds; ++r) {
    for (int c = 0; c < n_cand; ++c) {
      if (!ok[c]) continue;
      HP_CUDA(cudaEventRecord(ev[c][0], st));
      for (int k = 0; k < reps; ++k) {
        int rc = launch(plans[c], src, dst, st);
        if (rc) return rc;
      }
      HP_CUDA(cudaEventRecord(ev[c][1], st));
    }
    HP_CUDA(cudaStreamSynchronize(st));
    for (int c = 0; c < n_cand; ++c) {
      if (!ok[c]) continue;
      HP_CUDA(cudaEventElapsedTime(&t[c][r], ev[c][0], ev[c][1]));
      t[c][r] /= float(reps);
    }
  }
  // round 0 is a warm-up (the first window after switching plans can read
  // several % off either way); score = median of the other rounds
  float best_ms = 1e30f;
  bool found = false;
  const bool log = env_int("LFBP_TUNE_LOG", 0) != 0;
  for (int c = 0; c < n_cand; ++c) {
    if (!ok[c]) continue;
    float v[kRounds - 1];
    for (int r = 1; r < kRounds; ++r) v[r - 1] = t[c][r];
    std::sort(v, v + kRounds - 1);
    const float med = v[(kRounds - 1) / 2];
    if (log)
      fprintf(stderr, "[lfbp tune] (%lld,%lld,%lld,%lld) E=%d class=%d knobs {%d,%d,%d,%d,%d,%d}: %.4f ms\n",
              (long long)key.n_s, (long long)key.n_t, (long long)key.n_x, (long long)key.n_y, key.E, key.cls,
              cand[c].stages, cand[c].stage_kb, cand[c].cwarps, cand[c].subwarp, cand[c].flags, cand[c].grid_sm,
              med);
    if (med < best_ms) {
      best_ms = med;
      best = cand[c];
      found = true;
    }
  }
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

#include "host_pipeline.inc"

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
    const int64_t moved = 2 * plane_elems(dims) * (z_end - z_begin) * E;
    const TuneKey key{dims[0], dims[1], dims[2], dims[3], E, dev, tune_class(moved)};
    kn = default_knobs(moved);
    if (key.cls >= 0 && !tuned_knobs(key, kn) && env_int("LFBP_AUTOTUNE", 1)) {
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

int lfbp_tune(const int64_t dims[5], int dtype, int device, int64_t z_count) {
  int rc = check_common(dims, dtype, 0);
  if (rc) return rc;
  const int E = elem_size(dtype);
  if (z_count <= 0 || z_count > dims[4]) z_count = dims[4];
  const int64_t pb = plane_elems(dims) * E;
  // the two launch sizes a caller meets: z_count planes on the device API,
  // and one chunk of the host pipeline (lfbp_hprime_host / _multi / LF5)
  const int64_t jobs[2] = {z_count, host_chunk_planes(pb, dims[4])};
  int cur = 0;
  cudaGetDevice(&cur);
  HP_CUDA(cudaSetDevice(device));
  struct Restore {
    int dev;
    ~Restore() { cudaSetDevice(dev); }
  } restore{cur};
  for (int64_t planes : jobs) {
    const int cls = tune_class(2 * planes * pb);
    Knobs kn;
    const TuneKey key{dims[0], dims[1], dims[2], dims[3], E, device, cls};
    if (cls < 0 || tuned_knobs(key, kn)) continue;
    // scratch of at most ~4 GB per array (the size class, not the plane
    // count, selects the candidates; a few planes time them faithfully)
    int64_t pt = std::min<int64_t>(planes, std::max<int64_t>(1, (int64_t(4) << 30) / pb));
    while (pt < planes && tune_class(2 * pt * pb) != cls) ++pt;
    const int64_t bytes = pt * pb;
    struct Scratch {
      void* a = nullptr;
      void* b = nullptr;
      cudaStream_t s = nullptr;
      ~Scratch() {
        if (s) cudaStreamSynchronize(s), cudaStreamDestroy(s);
        if (a) cudaFree(a);
        if (b) cudaFree(b);
      }
    } sc;
    HP_CUDA(cudaMalloc(&sc.a, size_t(bytes) + 16));
    HP_CUDA(cudaMalloc(&sc.b, size_t(bytes) + 16));
    HP_CUDA(cudaMemset(sc.a, 0, size_t(bytes)));
    HP_CUDA(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    const int64_t td[5] = {dims[0], dims[1], dims[2], dims[3], pt};
    rc = autotune(key, sc.a, sc.b, td, E, 0, pt, bytes, sc.s, kn);
    if (rc) return rc;
  }
  return LFBP_OK;
}

int lfbp_plan_candidates(int size_class, int32_t* knobs, int max_n) {
  if (size_class != 0 && size_class != 1) return -fail(LFBP_ERR_ARGUMENT, "size class must be 0 or 1");
  const Knobs* cand = size_class == 1 ? kCandidates : kSmallCandidates;
  const int n = size_class == 1 ? kNumCandidates : kNumSmallCandidates;
  for (int c = 0; c < n && c < max_n && knobs; ++c) {
    int32_t* k = knobs + kKnobFields * c;
    k[0] = cand[c].stages;
    k[1] = cand[c].stage_kb;
    k[2] = cand[c].cwarps;
    k[3] = cand[c].subwarp;
    k[4] = cand[c].flags;
    k[5] = cand[c].grid_sm;
  }
  return n;
}

int lfbp_host_copy(void* dst, const void* src, int64_t bytes, int threads) {
  if (bytes < 0 || (bytes && (!dst || !src))) return fail(LFBP_ERR_ARGUMENT, "bad host_copy arguments");
  if (threads <= 0) {
    copy_pool().copy(dst, src, size_t(bytes));
  } else {
    HostPool pool(threads);
    pool.copy(dst, src, size_t(bytes));
  }
  return LFBP_OK;
}

int lfbp_synth_planes_device(void* dst, int dtype, const int64_t dims[5], int64_t n_planes, const uint64_t* pcg_state,
                             const double* tab_s, const double* tab_t, const double* disc_r2, void* stream) {
  if (!dims || !dst || !pcg_state || !tab_s || !tab_t) return fail(LFBP_ERR_ARGUMENT, "null argument");
  if (!hp_dims_valid(dims[0], dims[1], dims[2], dims[3], n_planes > 0 ? n_planes : 1))
    return fail(LFBP_ERR_INVALID_DIMS, "invalid dims");
  const int E = elem_size(dtype);
  if (!E) return fail(LFBP_ERR_ARGUMENT, "dtype code %d is not 1 (f32) or 2 (f64)", dtype);
  if (n_planes <= 0) return LFBP_OK;
  if (n_planes > 65535) return fail(LFBP_ERR_UNSUPPORTED, "at most 65535 planes per call");
  const int64_t P = plane_elems(dims);
  const int64_t per_block = int64_t(256 / 32) * 32 * hp::kSynthPer;
  const int64_t bx = (P + per_block - 1) / per_block;
  if (bx >= (int64_t(1) << 31)) return fail(LFBP_ERR_UNSUPPORTED, "plane too large");
  const dim3 grid{unsigned(bx), unsigned(n_planes), 1u};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const hp::SynthPlane* pl = reinterpret_cast<const hp::SynthPlane*>(pcg_state);
  if (E == 4)
    hp::synth_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(dst), dims[0], dims[1], dims[2], dims[3], pl,
                                                  tab_s, tab_t, disc_r2);
  else
    hp::synth_kernel<double><<<grid, 256, 0, st>>>(static_cast<double*>(dst), dims[0], dims[1], dims[2], dims[3], pl,
                                                   tab_s, tab_t, disc_r2);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  HP_CUDA(cudaGetLastError());
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
  const int64_t moved = 2 * plane_elems(dims) * dims[4] * E;
  Knobs kn = default_knobs(moved);
  const bool tuned =
      !env_knobs_set() && tuned_knobs(TuneKey{dims[0], dims[1], dims[2], dims[3], E, dev, tune_class(moved)}, kn);
  HpPlan p;
  rc = make_plan(p, dims, E, 0, dims[4], plane_elems(dims) * dims[4] * E, dev, kn);
  if (rc) return rc;
  const DevProps dp = device_props(dev);
  int w = snprintf(buf, size_t(buf_len),
                   "{\"elem\": %d, \"J\": %d, \"n_bands\": %d, \"C\": %d, \"n_chunks\": %d, \"row_pitch\": %d, "
                   "\"stage_bytes\": %d, \"stages\": %d, \"threads\": %d, \"smem_bytes\": %d, \"ctas_per_sm\": %d, "
                   "\"grid\": %d, \"n_units\": %lld, \"sub_width\": %d, \"sm_count\": %d, \"device_props\": \"%s\", "
                   "\"producers\": %d, \"tile_y\": %d, \"flags\": %d, \"autotuned\": %s, "
                   "\"knobs\": [%d, %d, %d, %d, %d, %d]}",
                   p.elem, p.J, p.n_bands, p.C, p.n_chunks, p.row_pitch, p.stage_bytes, p.stages, p.threads,
                   p.smem_bytes, p.ctas_per_sm, p.grid, (long long)p.n_units, p.sub_width, dp.sm_count,
                   dp.real ? "queried" : "b200-defaults", p.producers, p.tile_y, p.flags, tuned ? "true" : "false",
                   env_int("LFBP_STAGES", kn.stages), env_int("LFBP_STAGE_KB", kn.stage_kb),
                   env_int("LFBP_CONSUMER_WARPS", kn.cwarps), env_int("LFBP_SUBWARP", kn.subwarp),
                   env_int("LFBP_KFLAGS", kn.flags), env_int("LFBP_GRID", kn.grid_sm));
  if (w < 0 || w >= buf_len) return fail(LFBP_ERR_ARGUMENT, "buffer too small");
  return LFBP_OK;
}

#include "verify_capi.inc"

#include "projector_capi.inc"

// ---- pinned host blocks with a size-matched free cache ----
// Blocks of at least LFBP_PIN_MMAP_MB (default 1024) are anonymous mappings
// with transparent huge pages, first touched by the staging thread pool in
// parallel and then registered (cudaHostRegister); smaller ones come from
// cudaHostAlloc.  Registering pre-faulted huge pages avoids the driver's
// single-threaded fault-and-pin walk over 4 KB pages.
namespace {
struct PinBlock {
  int64_t cap;
  bool mapped;  // mmap + cudaHostRegister (else cudaHostAlloc)
};
std::mutex g_pin_mu;
std::map<void*, PinBlock> g_pin_live;           // block -> capacity, kind
std::multimap<int64_t, std::pair<void*, bool>> g_pin_cache;  // capacity -> free block
int64_t g_pin_cached = 0;

void pin_release(void* p, bool mapped, int64_t cap) {
  if (mapped) {
    cudaHostUnregister(p);
    munmap(p, size_t(cap));
  } else {
    cudaFreeHost(p);
  }
  cudaGetLastError();
}
}  // namespace

int lfbp_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(LFBP_ERR_ARGUMENT, "bad host_alloc arguments");
  *out = nullptr;
  int64_t want = std::max<int64_t>(bytes, 1);
  const bool map = want >= (int64_t(env_int("LFBP_PIN_MMAP_MB", 1024)) << 20);
  if (map) want = round_up(want, int64_t(2) << 20);
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    // smallest cached block that fits and wastes at most a quarter of it
    auto it = g_pin_cache.lower_bound(want);
    if (it != g_pin_cache.end() && it->first - want <= it->first / 4) {
      *out = it->second.first;
      g_pin_live[it->second.first] = PinBlock{it->first, it->second.second};
      g_pin_cached -= it->first;
      g_pin_cache.erase(it);
      return LFBP_OK;
    }
  }
  void* p = nullptr;
  if (map) {
    p = mmap(nullptr, size_t(want), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return fail(LFBP_ERR_CUDA, "mmap(%lld): %s", (long long)want, strerror(errno));
    madvise(p, size_t(want), MADV_HUGEPAGE);
    uint8_t* b = static_cast<uint8_t*>(p);
    copy_pool().for_range(size_t(want), size_t(2) << 20, [&](size_t a, size_t e) { memset(b + a, 0, e - a); });
    cudaError_t e = cudaHostRegister(p, size_t(want), cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      cudaGetLastError();
      munmap(p, size_t(want));
      return fail(LFBP_ERR_CUDA, "cudaHostRegister(%lld): %s", (long long)want, cudaGetErrorString(e));
    }
  } else {
    cudaError_t e = cudaHostAlloc(&p, size_t(want), cudaHostAllocPortable);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(LFBP_ERR_CUDA, "cudaHostAlloc(%lld): %s", (long long)want, cudaGetErrorString(e));
    }
  }
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_live[p] = PinBlock{want, map};
  *out = p;
  return LFBP_OK;
}

int lfbp_host_free(void* p) {
  if (!p) return LFBP_OK;
  PinBlock blk;
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_live.find(p);
    if (it == g_pin_live.end()) return fail(LFBP_ERR_ARGUMENT, "pointer was not allocated by lfbp_host_alloc");
    blk = it->second;
    g_pin_live.erase(it);
    const int64_t limit = int64_t(env_int("LFBP_PIN_CACHE_MB", 8192)) << 20;
    if (g_pin_cached + blk.cap <= limit) {
      g_pin_cache.emplace(blk.cap, std::make_pair(p, blk.mapped));
      g_pin_cached += blk.cap;
      return LFBP_OK;
    }
  }
  pin_release(p, blk.mapped, blk.cap);
  return LFBP_OK;
}

int lfbp_host_cache_release(void) {
  std::multimap<int64_t, std::pair<void*, bool>> blocks;
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    blocks.swap(g_pin_cache);
    g_pin_cached = 0;
  }
  for (auto& kv : blocks) pin_release(kv.second.first, kv.second.second, kv.first);
  return LFBP_OK;
}

int64_t lfbp_launch_count(void) { return g_launches.load(); }

const char* lfbp_last_error(void) { return g_err.c_str(); }

const char* lfbp_version(void) { return "lfbp-b200 0.1.0 (sm_100a)"; }

}  // extern "C"

#include "lf5_stream.inc"
