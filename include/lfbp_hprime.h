/*
 * lfbp_hprime.h -- C ABI of the B200-native H -> H' rearrangement.
 *
 * Drop-in boundary for the reference's hot path, the pure-Python `lfbp`
 * package (arXiv 2003.09133).  Arrays are the reference's layout: 5-D
 * (n_s, n_t, n_x, n_y, n_z), Fortran order (s fastest, z slowest; reference
 * arrays.py:21-23, fileio.py:13), element type float32 or float64 moved
 * bit-exactly.  Every entry point takes plain pointers and sizes; no torch
 * or CUDA types appear in the signatures (streams are passed as void*,
 * a cudaStream_t / CUstream, NULL = legacy default stream).
 *
 * Which reference interface each entry point replaces:
 *   lfbp_hprime_device / lfbp_hprime_host
 *       -> lfbp.compute_backprojection(psf)            transform.py:113-135
 *          (inverse = 1) lfbp.compute_psf_from_backprojection(bp)
 *                                                    transform.py:138-155
 *   lfbp_hprime_multi
 *       -> the same, z-sharded over several GPUs; the reference permits
 *          parallelism over z-planes but runs one thread
 *   lfbp_check_dims        -> Dims5 validation        arrays.py:53-67
 *   lfbp_dropped_source_count -> dropped_source_count transform.py:106-110
 *   lfbp_compare_device    -> the bitwise np.array_equal verification of
 *                             bench.py:88 / cli.py:145-150, on the device
 *   lfbp_plane_sums_device -> sum_forward_plane / sum_backward_plane
 *                             arrays.py:211-239 (acceptance criterion 3)
 *   lfbp_lf5_*             -> read_lf5 / save / load_psf (fileio.py:46-113)
 *                             and the `lfbp transform` CLI (cli.py:115-126)
 *   lfbp_forward_project_device / lfbp_backproject_device /
 *   lfbp_safe_divide_device, lfbp_safe_divide_peak_device, lfbp_max_device,
 *   lfbp_rl_update_device   -> forward_project / backproject(_adjoint) /
 *                             _safe_divide, projector.py:55-145 (the H'
 *                             consumer; rl_run composes them)
 * Error codes mirror the reference's exceptions (errors.py:12-13, 32-33).
 */
#ifndef LFBP_HPRIME_H
#define LFBP_HPRIME_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define LFBP_OK 0
#define LFBP_ERR_INVALID_DIMS 1     /* lfbp.InvalidDims   (errors.py:12-13) */
#define LFBP_ERR_EVEN_PIXEL_DIMS 2  /* lfbp.EvenPixelDims (errors.py:32-33) */
#define LFBP_ERR_CUDA 3             /* CUDA runtime failure; see lfbp_last_error() */
#define LFBP_ERR_ARGUMENT 4         /* null / misaligned pointer, bad dtype or range */
#define LFBP_ERR_UNSUPPORTED 5      /* shape beyond the kernel's limits */
#define LFBP_ERR_FORMAT 6           /* lfbp.FormatError   (errors.py:20-21): malformed LF5 file */
#define LFBP_ERR_IO 7               /* lfbp.IoError       (errors.py:24-25): read/write failed */
#define LFBP_ERR_DIMS 8             /* lfbp.DimsError     (errors.py:16-17): file dims violate the contract */

/* element type codes: the LF5 header codes (fileio.py:35) */
#define LFBP_F32 1
#define LFBP_F64 2

/* flags for lfbp_hprime_host / lfbp_hprime_multi */
#define LFBP_HOST_REGISTER 1   /* pin pageable host buffers for the call (cudaHostRegister) */
#define LFBP_HOST_STAGE 2      /* copy pageable host buffers through pinned staging chunks
                                  (multi-threaded memcpy overlapped with the DMA); wins over
                                  LFBP_HOST_REGISTER when both are set */

/* Validate (n_s, n_t, n_x, n_y, n_z) like Dims5 (arrays.py:53-67).
 * Returns LFBP_OK or LFBP_ERR_INVALID_DIMS. No GPU needed. */
int lfbp_check_dims(const int64_t dims[5]);

/* Source elements without a target for even n_s / n_t (transform.py:106-110).
 * Returns -1 for invalid dims. No GPU needed. */
int64_t lfbp_dropped_source_count(const int64_t dims[5]);

/* H' = rearrange(H) (inverse = 0) or H = rearrange^-1(H') (inverse = 1, odd
 * n_s and n_t only; otherwise LFBP_ERR_EVEN_PIXEL_DIMS) for depth planes
 * [z_begin, z_end) of device arrays `src` and `dst` that both hold the WHOLE
 * (n_s, n_t, n_x, n_y, n_z) array, 16-byte aligned, non-overlapping.
 * Asynchronous on `stream`; the caller synchronises -- except the FIRST call
 * for a plane shape / element size / device / size class (launches moving
 * >= 8 MB) with no tuned plan: that call runs the autotuner on `src`/`dst`
 * first (about 40 candidate plans x 4 timed rounds with host
 * synchronisations on `stream`; about 3.5 s on C5) and so returns only after
 * they finish.  Call lfbp_tune() beforehand to keep every call asynchronous;
 * LFBP_AUTOTUNE=0 disables the tuner (untuned default plan).  Plans with
 * unit tickets (flag 128) take a counter slot from a per-device ring of 1024
 * per launch; a captured CUDA graph reuses its slot on every replay, so one
 * graph must not be replayed concurrently with itself. */
int lfbp_hprime_device(const void* src, void* dst, const int64_t dims[5], int dtype, int inverse,
                       int64_t z_begin, int64_t z_end, void* stream);

/* Host-to-host H' on one GPU: the z-planes are streamed through the device in
 * chunks (H2D, kernel and D2H overlapped on three streams).  `src` and `dst`
 * are host arrays of the whole shape; pinned memory gives full PCIe speed;
 * pageable memory is staged through pinned chunks (LFBP_HOST_STAGE) or
 * pinned for the call (LFBP_HOST_REGISTER), else the driver stages it.
 * Synchronous: returns when dst is complete. */
int lfbp_hprime_host(const void* src, void* dst, const int64_t dims[5], int dtype, int inverse,
                     int device, int flags);

/* Tune the kernel plan for `dims` / `dtype` on `device` ahead of time, on
 * library-owned scratch buffers (at most ~4 GB each): for launches of
 * `z_count` planes (<= 0: all n_z) and for one chunk of the host pipeline.
 * Synchronous.  Afterwards lfbp_hprime_device never synchronises, and
 * lfbp_hprime_host / _multi / the LF5 path use the tuned chunk plan (they
 * never tune by themselves).  Plans are cached per process. */
int lfbp_tune(const int64_t dims[5], int dtype, int device, int64_t z_count);

/* The autotuner's candidate plans for size class 1 (launches moving
 * >= 256 MB) or 0 (8-256 MB): writes up to `max_n` records of 6 int32
 * (smem stages, stage KB, consumer warps, lanes per row -- 0 = by row
 * length --, flags -- 8 = unit order along y' diagonals, 16 = rotated run /
 * row order, 32 = (row, phase-class) task consumer, 64 = one launch per
 * ~12 GB z-slab, 128 = units handed out by a per-launch ticket counter --,
 * SMs used -- 0 = all) into `knobs` (may be NULL) and returns the number of
 * candidates.  No GPU. */
int lfbp_plan_candidates(int size_class, int32_t* knobs, int max_n);

/* memcpy of `bytes` split over `threads` host threads (<= 0: the library's
 * staging pool, 3/4 of the host threads): the copy engine of the pageable
 * staging path.  No GPU. */
int lfbp_host_copy(void* dst, const void* src, int64_t bytes, int threads);

/* Host-to-host H' with the z-planes split into contiguous slabs, one per
 * listed device, all devices running concurrently; no inter-GPU traffic.
 * Each slab lands at its own byte offset z0 * plane_bytes of dst. */
int lfbp_hprime_multi(const void* src, void* dst, const int64_t dims[5], int dtype, int inverse,
                      int n_devices, const int* devices, int flags);

/* Contiguous balanced split of n_z planes over n_shards: shard k gets
 * [*z_begin, *z_end). No GPU needed. */
int lfbp_shard_planes(int64_t n_z, int n_shards, int shard, int64_t* z_begin, int64_t* z_end);

/* Bitwise comparison of two device buffers of `nbytes` (K2).  Writes the
 * number of differing bytes and the first differing byte offset (-1 when
 * equal).  Synchronous. */
int lfbp_compare_device(const void* a, const void* b, int64_t nbytes, int64_t* n_diff,
                        int64_t* first_diff, void* stream);

/* Sorted-order float64 sums of every (s, t) pattern slice of depth planes
 * [z_begin, z_end) of a device array (K3): out[(z - z_begin)*n_s*n_t + t*n_s + s]
 * equals, bit for bit, the reference's sum_forward_plane / sum_backward_plane
 * (arrays.py:211-239: np.sort then numpy's pairwise float64 sum).  `out` is a
 * device buffer of n_s*n_t*(z_end - z_begin) doubles.  Asynchronous on
 * `stream`.  n_x*n_y must be <= 8192. */
int lfbp_plane_sums_device(const void* src, double* out, const int64_t dims[5], int dtype, int64_t z_begin,
                           int64_t z_end, void* stream);

/* ---- LF5 container streaming (fileio.py:3-92; 32-byte header + F-order payload) ---- */

/* Parse and validate an LF5 header like read_lf5 (fileio.py:63-92): magic,
 * version 1, element code, zero reserved bytes, exact file length.  No GPU. */
int lfbp_lf5_read_header(const char* path, int64_t dims[5], int* dtype);

/* Create / truncate `path` as an LF5 file of that shape and type (header
 * written, payload sized).  No GPU. */
int lfbp_lf5_create(const char* path, const int64_t dims[5], int dtype);

/* File-to-file H' (inverse = 0) or H (inverse = 1): the `lfbp transform`
 * CLI (cli.py:115-126) without holding the array in host memory -- plane
 * chunks are pread into pinned buffers, transformed on `device` and pwritten
 * at their offsets.  Header dims are checked like load_psf (DimsError), the
 * values like PsfArray (InvalidDims for negative / NaN; no output is left). */
int lfbp_lf5_transform_file(const char* in_path, const char* out_path, int inverse, int device, int flags);

/* Planes [z_begin, z_end) of an LF5 file straight into / out of a device
 * buffer that holds exactly those planes (z-sharded loads / stores). */
int lfbp_lf5_load_device(const char* path, void* dst, int64_t z_begin, int64_t z_end, void* stream);
int lfbp_lf5_store_device(const char* path, const void* src, int64_t z_begin, int64_t z_end, void* stream);

/* ---- the H' consumer (projector.py:55-145), float64 accumulation ----
 * Volumes (nvx, nvy, n_z) and images (nvx, nvy) are F-ordered float64 device
 * arrays; the pattern arrays H / H' are float32 or float64 (dtype code). */

/* image = forward projection of the volume through H (projector.py:55-81). */
int lfbp_forward_project_device(const void* H, int dtype, const int64_t dims[5], const double* volume, int64_t nvx,
                                int64_t nvy, double* image, void* stream);

/* The same through H' when it is given and n_s, n_t are odd: each pixel's
 * own phase fixes the pattern (coalesced gather, same sums); H may be NULL
 * then.  Falls back to H for even sizes. */
int lfbp_forward_project2_device(const void* H, const void* Hp, int dtype, const int64_t dims[5], const double* volume,
                                 int64_t nvx, int64_t nvy, double* image, void* stream);

/* volume = backprojection of the image: through H' stamps (use_hprime = 1,
 * `backproject`, projector.py:103-126) or the literal adjoint through H
 * (use_hprime = 0, `backproject_adjoint`, projector.py:84-100). */
int lfbp_backproject_device(const void* P, int dtype, const int64_t dims[5], int use_hprime, const double* image,
                            int64_t npx, int64_t npy, double* volume, void* stream);

/* out = num / den where den >= eps * max(den) (and den > 0 if that is 0),
 * else 0 (`_safe_divide`, projector.py:135-145); `scratch` is one device
 * double. */
int lfbp_safe_divide_device(const double* num, const double* den, double* out, int64_t n, double eps,
                            double* scratch, void* stream);

/* *peak = max(0, max(x[0..n))) on the device (the `den.max()` of
 * `_safe_divide`, projector.py:138, for one rank's z-slab; ranks combine
 * their peaks with an all-reduce MAX before dividing). */
int lfbp_max_device(const double* x, int64_t n, double* peak, void* stream);

/* `_safe_divide` (projector.py:135-145) against a caller-supplied device
 * peak: out = num / den where den >= eps * (*peak) (and den > 0 if that is
 * 0), else 0; all zeros when *peak <= 0. */
int lfbp_safe_divide_peak_device(const double* num, const double* den, double* out, int64_t n, double eps,
                                 const double* peak, void* stream);

/* The Richardson-Lucy update `g = g * _safe_divide(back, norm, eps)`
 * (projector.py:192) in place, fused: g[i] *= (ok ? back[i] / norm[i] : 0)
 * with ok as in lfbp_safe_divide_peak_device. */
int lfbp_rl_update_device(double* g, const double* back, const double* norm, int64_t n, double eps,
                          const double* peak, void* stream);

/* Seeded synthetic H planes on the device (bench / test input generation,
 * not the hot path; K6): `n_planes` planes of shape (n_s, n_t, n_x, n_y)
 * into `dst` (F order, planes contiguous), bit-identical to the numpy
 * generator paper_2003_09133_b200.synth.baseline_plane.  Per plane p:
 * pcg_state[4p..4p+3] = the numpy PCG64 state (lo, hi) and increment
 * (lo, hi) before the plane's first draw; tab_s[p*n_s*n_x + s + n_s*x] and
 * tab_t[p*n_t*n_y + t + n_t*y] the per-axis factors; value
 * (u * tab_s) * tab_t, or with disc_r2 != NULL: u if tab_s + tab_t <=
 * disc_r2[p], else 0.  All pointers are device pointers.  Asynchronous. */
int lfbp_synth_planes_device(void* dst, int dtype, const int64_t dims[5], int64_t n_planes, const uint64_t* pcg_state,
                             const double* tab_s, const double* tab_t, const double* disc_r2, void* stream);

/* The launch plan the kernel would use, as a JSON object in `buf` (for
 * tests, tuning and DESIGN.md).  Uses the current device's properties, or
 * B200 defaults (148 SMs, 227 KB smem/CTA) when no GPU is present. */
int lfbp_plan_json(const int64_t dims[5], int dtype, char* buf, int64_t buf_len);

/* Page-locked host blocks for result arrays (the drop-ins' fresh H' / H,
 * reference transform.py:126 / 153 allocate them with np.zeros / np.empty):
 * D2H lands in them at full PCIe speed with no staging copy.  Freed blocks
 * stay cached for reuse (pinning is the expensive part, ~0.5 s per GB) up
 * to LFBP_PIN_CACHE_MB (default 8192) bytes; lfbp_host_cache_release
 * returns the cached blocks to the system. */
int lfbp_host_alloc(int64_t bytes, void** out);
int lfbp_host_free(void* p);
int lfbp_host_cache_release(void);

/* Kernel launches issued by this library since load (all entry points). */
int64_t lfbp_launch_count(void);

/* Thread-local message of the last failing call ("" if none). */
const char* lfbp_last_error(void);

/* Library version string. */
const char* lfbp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LFBP_HPRIME_H */
