// Shared host/device description of one H -> H' launch.
//
// Index map (0-based, the closed form of the reference's per-axis phase
// tables, lfbp/transform.py:73-130; derivation in SURVEY.md Appendix A):
//
//   H'[i, j, x', y', z] = H[2c_s - i, 2c_t - j, (x' + i - c_s) mod n_x,
//                           (y' + j - c_t) mod n_y, z]
//   c_s = floor((n_s - 1) / 2), c_t = floor((n_t - 1) / 2);
//   rows i = n_s - 1 (even n_s) and j = n_t - 1 (even n_t) are zero
//   (np.zeros init + the dropped mirror row, transform.py:99-103, 126).
//
// The kernel is source-driven: a work unit is one (z, y, t-band, i-chunk).
// Its source is n_x contiguous runs H[s_lo:s_hi, t0:t0+J, x, y, z] (s is the
// fastest axis, t next, so J whole rows form ONE run per x), staged into
// shared memory with 1-D bulk TMA.  Each staged run feeds J*n_x output rows
// H'[i_lo:i_hi, j, x', y', z] with j = 2c_t - t and
// y' = (y + t - c_t) mod n_y, written with 16-byte stores.
//
// Shared-memory layout of one stage: a 64-byte unit header, then element k
// of the run of source phase x at byte  R0 + x * row_pitch + k * elem,
// R0 = 64 + 16 + (run byte offset mod 16).  row_pitch is congruent to (n_s * n_t * elem) mod 16, so every
// run's 16-byte-aligned superset lands on a 16-byte-aligned smem address (a
// legal bulk-copy destination) while the element address stays LINEAR in x:
// the consumer steps x -> x+1, s -> s-1 with one add.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HP_HD __host__ __device__ __forceinline__
#else
#define HP_HD inline
#endif

// Division by a runtime constant for 0 <= n < 2^31 (round-up multiplier,
// Granlund-Montgomery): q = (umulhi(n, mul) + n) >> shr.
struct HpFastDiv {
  uint32_t d, mul, shr;
};

HP_HD HpFastDiv hp_fastdiv_make(uint32_t d) {
  HpFastDiv f;
  f.d = d;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.shr = l;
  f.mul = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
  return f;
}

HP_HD uint32_t hp_umulhi(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

HP_HD uint32_t hp_div(const HpFastDiv& f, uint32_t n) {
  return (hp_umulhi(n, f.mul) + n) >> f.shr;
}

HP_HD uint32_t hp_mod(const HpFastDiv& f, uint32_t n) {
  return n - hp_div(f, n) * f.d;
}

#define HP_FLAG_LOAD_EVICT_FIRST 1  // L2 evict_first hint on the bulk loads of H
#define HP_FLAG_BAND_FASTEST 4      // unit order: t-band fastest instead of y
#define HP_FLAG_DIAGONAL 8          // unit order: t-band fastest along a y' = y + t - c_t diagonal
#define HP_FLAG_ROTATE 16           // unit u issues its runs / claims its rows starting at u mod n
#define HP_FLAG_TASKS 32            // (row, phase-class) task consumer and 16-byte row pitch (see
                                    // consume_unit_tasks in hprime_kernel.cuh)
#define HP_FLAG_ZCHUNK 64           // host side: one launch per ~12 GB z-slab (launch() in lfbp_capi.cu)
#define HP_FLAG_DYNAMIC 128         // units handed out in order by a per-launch global counter

struct HpPlan {
  // geometry of the (chunk) arrays the kernel sees
  int64_t n_s, n_t, n_x, n_y;
  int64_t z_begin, z_count;   // planes [z_begin, z_begin + z_count) are processed
  int64_t total_bytes;        // size of the source allocation (tail clamp for bulk copies)
  int32_t elem;               // 4 (f32) or 8 (f64); payload moved as integers
  int32_t c_s, c_t;           // floor((n - 1) / 2)
  int32_t v_s, v_t;           // valid mirrored rows: 2c + 1
  int32_t nx_off;             // (-c_s) mod n_x
  int32_t ny_off;             // (-c_t) mod n_y
  int32_t J;                  // t rows per unit (band)
  int32_t n_bands;            // ceil(n_t / J)
  int32_t C;                  // output i per unit (chunk); == n_s when unchunked
  int32_t n_chunks;           // ceil(n_s / C)
  int32_t row_pitch;          // smem bytes between staged runs (== xs16 mod 16; a multiple
                              // of 16 with HP_FLAG_TASKS)
  int32_t stage_bytes;        // n_x * row_pitch + 32 rounded to 128
  int32_t stages;             // smem ring depth
  int32_t threads;            // CTA size: 1 producer warp + consumer warps
  int32_t smem_bytes;         // dynamic smem per CTA
  int32_t grid;               // persistent CTAs
  int32_t ctas_per_sm;
  int32_t xs16;               // (n_s * n_t * elem) mod 16: run misalignment step per x
  int32_t flags;              // HP_FLAG_*
  int32_t sub_width;          // lanes per output row (2, 4, 8, 16 or 32)
  int32_t gx_inc;             // (sub_width * 16/elem) mod n_x: phase advance of one stride
  int32_t producers;          // producer warps (warps 0..producers-1); they split a unit's n_x runs
  int64_t n_units;            // z_count * n_chunks * n_bands * n_y  (< 2^31)
  HpFastDiv nx_div;           // mod n_x on the element path
  HpFastDiv ny_div;           // unit decode / y' wrap
  HpFastDiv nb_div;           // unit decode: bands
  HpFastDiv nc_div;           // unit decode: chunks
  // unit order inside one (z, chunk): y in blocks of tile_y, y fastest within
  // a block, then band; the last block holds the remaining y (tile_y = n_y:
  // plain y-fastest order)
  int32_t tile_y, n_yblocks;
  HpFastDiv zc_div;           // n_y * n_bands: units per (z, chunk)
  HpFastDiv yblk_div;         // tile_y * n_bands: units per full y block
  HpFastDiv ty_div, tyl_div;  // tile_y, and the last block's y count
  unsigned long long* counter;  // HP_FLAG_DYNAMIC: zeroed unit ticket counter (set per launch)
};

// Valid Dims5 (reference arrays.py:53-67): all >= 1, n_x and n_y odd,
// n_s >= n_x, n_t >= n_y.
HP_HD int hp_dims_valid(int64_t n_s, int64_t n_t, int64_t n_x, int64_t n_y, int64_t n_z) {
  if (n_s < 1 || n_t < 1 || n_x < 1 || n_y < 1 || n_z < 1) return 0;
  if ((n_x % 2) == 0 || (n_y % 2) == 0) return 0;
  if (n_s < n_x || n_t < n_y) return 0;
  return 1;
}
