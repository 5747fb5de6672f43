// The H' consumer on the GPU: forward and back
// projection of the reference's light-field model (lfbp/projector.py:55-132),
// float64 accumulation as in the reference.
//
// A voxel at (x, y, z) contributes its pattern H[:, :, x mod n_x, y mod n_y, z]
// centred on the pixel under it (pattern element a lands on image row
// S = x + a - C_s, C = pattern_centre - 1, projector.py:26-47); contributions
// past the image border are dropped.  The reference scatters ("stamps") one
// pattern per voxel / per pixel; here every output element GATHERS its own
// window, one thread per output element, so no atomics are needed:
//
//   forward   out[S,T]    = sum_z sum_{a,b} g[S-a+C_s, T-b+C_t, z] *
//                                        H[a, b, (S-a+C_s) mod n_x, (T-b+C_t) mod n_y, z]
//   adjoint   out[x,y,z]  = sum_{S,T} f[S,T] * H[S-x+C_s, T-y+C_t, x mod n_x, y mod n_y, z]
//   H'-stamp  out[X,Y,z]  = sum_{s,t} f[s,t] * H'[X-s+C_s, Y-t+C_t, s mod n_x, t mod n_y, z]
//
// (projector.py:55-81, 84-100, 103-126).  Sums run in a different order than
// the reference's, so parity is to relative 1e-12 -- the tolerance the
// reference's own tests use between its two backprojection forms
// (test_projector.py:67-82).  All arrays are F-ordered; volumes / images are
// float64.
#pragma once
#include <cuda.h>  // CUtensorMap
#include <cuda_runtime.h>
#include <stdint.h>

namespace hp {

struct ProjGeom {
  int32_t n_s, n_t, n_x, n_y, n_z;
  int32_t c_s, c_t;      // pattern_centre - 1 (0-based zero-offset element)
  int32_t nvx, nvy;      // lateral grid (image == volume lateral size)
};

template <typename T>
__global__ void forward_project_kernel(const T* __restrict__ H, const double* __restrict__ g,
                                       double* __restrict__ out, const ProjGeom q) {
  const int32_t S = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t Tt = blockIdx.y * blockDim.y + threadIdx.y;
  if (S >= q.nvx || Tt >= q.nvy) return;
  const int64_t pat = int64_t(q.n_s) * q.n_t;
  const int64_t plane = pat * q.n_x * q.n_y;
  const int64_t vplane = int64_t(q.nvx) * q.nvy;
  // pattern rows that keep the voxel inside the grid: 0 <= S - a + C < nvx
  const int32_t a_lo = max(0, S + q.c_s - (q.nvx - 1)), a_hi = min(q.n_s - 1, S + q.c_s);
  const int32_t b_lo = max(0, Tt + q.c_t - (q.nvy - 1)), b_hi = min(q.n_t - 1, Tt + q.c_t);
  double acc = 0.0;
  for (int32_t z = 0; z < q.n_z; ++z) {
    const T* Hz = H + z * plane;
    const double* gz = g + z * vplane;
    for (int32_t b = b_lo; b <= b_hi; ++b) {
      const int32_t y = Tt - b + q.c_t;
      const int64_t yoff = int64_t(y % q.n_y) * q.n_x * pat + int64_t(b) * q.n_s;
      const double* grow = gz + int64_t(y) * q.nvx;
      for (int32_t a = a_lo; a <= a_hi; ++a) {
        const int32_t x = S - a + q.c_s;
        const double w = grow[x];
        if (w != 0.0) acc = fma(w, static_cast<double>(Hz[yoff + int64_t(x % q.n_x) * pat + a]), acc);
      }
    }
  }
  out[S + int64_t(Tt) * q.nvx] = acc;
}

// forward projection through H' (odd n_s, n_t): the pixel's own phase fixes
// the pattern -- out[S,T] = sum_z sum_{i,j} g[S+i-c_s, T+j-c_t, z] *
// H'[i, j, S mod n_x, T mod n_y, z] -- so a lane walks one contiguous pattern
// row while the warp reads the volume row coalesced (same sums as the H form:
// H'[i, ., S mod n_x] = H[2c-i, ., (S+i-c) mod n_x]).
template <typename T>
__global__ void forward_project_hp_kernel(const T* __restrict__ Hp, const double* __restrict__ g,
                                          double* __restrict__ out, const ProjGeom q) {
  const int32_t S = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t Tt = blockIdx.y * blockDim.y + threadIdx.y;
  if (S >= q.nvx || Tt >= q.nvy) return;
  const int64_t pat = int64_t(q.n_s) * q.n_t;
  const int64_t plane = pat * q.n_x * q.n_y;
  const int64_t vplane = int64_t(q.nvx) * q.nvy;
  // taps that keep the voxel inside the grid: 0 <= S + i - c < nvx
  const int32_t i_lo = max(0, q.c_s - S), i_hi = min(q.n_s - 1, q.nvx - 1 - S + q.c_s);
  const int32_t j_lo = max(0, q.c_t - Tt), j_hi = min(q.n_t - 1, q.nvy - 1 - Tt + q.c_t);
  const int64_t phase = (int64_t(S % q.n_x) + int64_t(Tt % q.n_y) * q.n_x) * pat;
  double acc = 0.0;
  for (int32_t z = 0; z < q.n_z; ++z) {
    const T* K = Hp + z * plane + phase;
    const double* gz = g + z * vplane + (S - q.c_s);
    for (int32_t j = j_lo; j <= j_hi; ++j) {
      const T* krow = K + int64_t(j) * q.n_s;
      const double* grow = gz + int64_t(Tt + j - q.c_t) * q.nvx;
      for (int32_t i = i_lo; i <= i_hi; ++i) acc = fma(grow[i], static_cast<double>(krow[i]), acc);
    }
  }
  out[S + int64_t(Tt) * q.nvx] = acc;
}

// adjoint (use_hprime = 0, pattern array H, voxel phase) or the H'-stamp
// backprojection (use_hprime = 1, pattern array H', pixel phase)
template <typename T>
__global__ void backproject_kernel(const T* __restrict__ P, const double* __restrict__ f, double* __restrict__ out,
                                   const ProjGeom q, int use_hprime) {
  const int32_t X = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t Y = blockIdx.y * blockDim.y + threadIdx.y;
  const int32_t z = blockIdx.z;
  if (X >= q.nvx || Y >= q.nvy) return;
  const int64_t pat = int64_t(q.n_s) * q.n_t;
  const T* Pz = P + z * pat * q.n_x * q.n_y;
  double acc = 0.0;
  if (use_hprime) {
    // pixels s with 0 <= X - s + C_s < n_s
    const int32_t s_lo = max(0, X + q.c_s - (q.n_s - 1)), s_hi = min(q.nvx - 1, X + q.c_s);
    const int32_t t_lo = max(0, Y + q.c_t - (q.n_t - 1)), t_hi = min(q.nvy - 1, Y + q.c_t);
    for (int32_t t = t_lo; t <= t_hi; ++t) {
      const int32_t b = Y - t + q.c_t;
      const int64_t toff = int64_t(t % q.n_y) * q.n_x * pat + int64_t(b) * q.n_s;
      const double* frow = f + int64_t(t) * q.nvx;
      for (int32_t s = s_lo; s <= s_hi; ++s) {
        const double w = frow[s];
        if (w != 0.0) acc = fma(w, static_cast<double>(Pz[toff + int64_t(s % q.n_x) * pat + (X - s + q.c_s)]), acc);
      }
    }
  } else {
    // pixels S with 0 <= S - X + C_s < n_s; the voxel's phase fixes the pattern
    const int32_t S_lo = max(0, X - q.c_s), S_hi = min(q.nvx - 1, X - q.c_s + q.n_s - 1);
    const int32_t T_lo = max(0, Y - q.c_t), T_hi = min(q.nvy - 1, Y - q.c_t + q.n_t - 1);
    const T* Pxy = Pz + (int64_t(X % q.n_x) + int64_t(Y % q.n_y) * q.n_x) * pat;
    for (int32_t Tt = T_lo; Tt <= T_hi; ++Tt) {
      const T* prow = Pxy + int64_t(Tt - Y + q.c_t) * q.n_s;
      const double* frow = f + int64_t(Tt) * q.nvx;
      for (int32_t S = S_lo; S <= S_hi; ++S) acc = fma(frow[S], static_cast<double>(prow[S - X + q.c_s]), acc);
    }
  }
  out[X + int64_t(Y) * q.nvx + int64_t(z) * q.nvx * q.nvy] = acc;
}

// ---- polyphase form (odd and even sizes alike) ---------------------------
// Both directions are "fixed output phase" correlations:
//   out[P] = sum_{a,b} in[P + (a, b) - (C_s, C_t)] * K_phase(P)[a, b]
// (forward: in = g[:, :, z] summed over z, K = H' when n_s, n_t are odd;
// backward: in = f, K = H, one output plane per z).  Splitting the input into
// its n_x * n_y phase sub-images (zero-padded by a halo, PolyGeom) makes every
// tap read, for the 32 lanes of one output phase at consecutive coarse k,
// 32 consecutive doubles of one sub-image (coalesced), while the pattern
// value is one broadcast; each thread keeps 4 outputs along the coarse y axis
// and slides a 4-row register window over the taps b = r' + n_y * n.
struct PolyGeom {
  int32_t kc, lc;   // coarse extent of the output grid: ceil(nvx / n_x), ceil(nvy / n_y)
  int32_t hx, hy;   // halo (coarse cells) on each side
  int32_t kp, lp;   // padded sub-image extent: kc + 2 hx, lc + 2 hy
};

// in (nvx, nvy, planes) F-order -> sub[plane][ry][rx][ll][kk] (kk fastest)
__global__ void polyphase_pad_kernel(const double* __restrict__ in, double* __restrict__ sub, const ProjGeom q,
                                     const PolyGeom pg, int32_t planes) {
  const int64_t per = int64_t(pg.kp) * pg.lp;
  const int64_t total = per * q.n_x * q.n_y * planes;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t kk = int32_t(i % pg.kp);
    int64_t r = i / pg.kp;
    const int32_t ll = int32_t(r % pg.lp);
    r /= pg.lp;
    const int32_t rx = int32_t(r % q.n_x);
    r /= q.n_x;
    const int32_t ry = int32_t(r % q.n_y);
    const int64_t z = r / q.n_y;
    const int32_t x = rx + q.n_x * (kk - pg.hx), y = ry + q.n_y * (ll - pg.hy);
    sub[i] = (x >= 0 && x < q.nvx && y >= 0 && y < q.nvy) ? in[x + int64_t(y) * q.nvx + z * int64_t(q.nvx) * q.nvy]
                                                           : 0.0;
  }
}

__device__ __forceinline__ int32_t floordiv(int32_t a, int32_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// grid: x = (px, k) pairs / blockDim.x, y = coarse l tiles of RL rows,
//       z = py + n_y * zout; out[:, :, zout] is the backprojected plane
// (backward, input f shared by all z) or the partial image of depth plane
// zout (forward, input g[:, :, zout]; summed afterwards)
template <typename T, int RL>
__global__ void __launch_bounds__(128) poly_corr_kernel(const double* __restrict__ sub, const T* __restrict__ K,
                                                        double* __restrict__ out, const ProjGeom q, const PolyGeom pg,
                                                        int32_t forward) {
  const int32_t n_ph = q.n_x * q.n_y;
  // threads run over (px, k) with k fastest: a warp covers consecutive coarse
  // cells of at most a few x-phases, so no lanes idle when kc < 32
  const int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t px = e / pg.kc, k = e - px * pg.kc;
  const int32_t py = blockIdx.z % q.n_y;
  const int32_t zout = blockIdx.z / q.n_y;  // forward: the depth plane this block sums (partial image per z)
  const int32_t ph = px + q.n_x * py;
  const int32_t l0 = blockIdx.y * RL;
  if (px >= q.n_x || l0 >= pg.lc) return;
  const int64_t pat = int64_t(q.n_s) * q.n_t;
  const int64_t sub_plane = int64_t(pg.kp) * pg.lp;
  double acc[RL];
#pragma unroll
  for (int j = 0; j < RL; ++j) acc[j] = 0.0;
  const T* Kz = K + (int64_t(zout) * n_ph + ph) * pat;
  const double* subz = sub + (forward ? int64_t(zout) * n_ph * sub_plane : 0);
  const int64_t kstep = int64_t(q.n_y) * q.n_s;
  for (int32_t r2 = 0; r2 < q.n_y && r2 < q.n_t; ++r2) {
    const int32_t rho_y = py - q.c_t + r2;
    const int32_t ryy = ((rho_y % q.n_y) + q.n_y) % q.n_y;
    const int32_t lyy = floordiv(rho_y, q.n_y) + pg.hy;
    const int32_t n_taps = (q.n_t - r2 + q.n_y - 1) / q.n_y;   // b = r2 + n_y * n < n_t
    // tap a reads sub-image rx = (px - c_s + a) mod n_x at coarse offset
    // floordiv(px - c_s + a, n_x).  Taps are visited by residue class a0 of
    // a mod n_x: within a class the sub-image is fixed and the coarse offset
    // steps by one, so a block re-reads one small sub-image tile (L1 hits)
    // instead of cycling through all n_x of them
    const int32_t rho0 = px - q.c_s;
    const double* row0 = subz + int64_t(ryy) * q.n_x * sub_plane + k + int64_t(l0 + lyy) * pg.kp;
    const T* krow = Kz + int64_t(r2) * q.n_s;
    for (int32_t a0 = 0; a0 < q.n_x && a0 < q.n_s; ++a0) {
    const int32_t rxx = (((rho0 + a0) % q.n_x) + q.n_x) % q.n_x;
    const double* colx = row0 + int64_t(rxx) * sub_plane + floordiv(rho0 + a0, q.n_x) + pg.hx;
    for (int32_t a = a0; a < q.n_s; a += q.n_x, ++colx) {
      const double* col = colx;
      const T* kcol = krow + a;
      // register window over RL consecutive coarse rows, slid one row per
      // tap: blocks of RL taps use it as a circular buffer with static slot
      // indices (no moves), the remaining taps shift it
      double w[RL];
#pragma unroll
      for (int j = 0; j < RL - 1; ++j) w[j] = col[int64_t(j) * pg.kp];
      int32_t n = 0;
      for (; n + RL <= n_taps; n += RL) {
#pragma unroll
        for (int t = 0; t < RL; ++t) {
          w[(RL - 1 + t) % RL] = col[int64_t(n + t + RL - 1) * pg.kp];
          const double v = static_cast<double>(kcol[int64_t(n + t) * kstep]);
#pragma unroll
          for (int j = 0; j < RL; ++j) acc[j] = fma(w[(j + t) % RL], v, acc[j]);
        }
      }
      for (; n < n_taps; ++n) {
        w[RL - 1] = col[int64_t(n + RL - 1) * pg.kp];
        const double v = static_cast<double>(kcol[int64_t(n) * kstep]);
#pragma unroll
        for (int j = 0; j < RL; ++j) acc[j] = fma(w[j], v, acc[j]);
#pragma unroll
        for (int j = 0; j < RL - 1; ++j) w[j] = w[j + 1];
      }
    }
    }
  }
  const int32_t X = px + q.n_x * k;
#pragma unroll
  for (int j = 0; j < RL; ++j) {
    const int32_t Y = py + q.n_y * (l0 + j);
    if (X < q.nvx && Y < q.nvy && l0 + j < pg.lc) out[X + int64_t(Y) * q.nvx + int64_t(zout) * q.nvx * q.nvy] = acc[j];
  }
}

// ---- shared-memory tiled polyphase correlation -----------------------------
// Same sums as poly_corr_kernel, restructured around the fact that the taps of
// one residue class (a = a0 + n_x a', b = r2 + n_y n) read ONE input
// sub-image at consecutive coarse offsets.  A block owns one output phase
// (px, py), one plane and a TK x (TLT*RL) coarse tile.  Per class pair
// (r2, a0) it stages the sub-image window it needs (TK + M - 1 columns,
// TLT*RL + N - 1 rows, zero outside the padded sub-image) and the M x N
// class taps (converted to double once) in shared memory, then every thread
// runs the register-window loop of poly_corr_kernel on shared memory: per tap
// one LDS of the new window row, one broadcast LDS of the tap, RL DFMAs.
struct PolyTile {
  int32_t tk, tlt;     // block = tk x tlt threads (coarse x, groups of RL coarse rows)
  int32_t tw, th, p;   // staged window: tw columns, th rows, row pitch p (doubles)
  int32_t mmax, nmax;  // taps per class: ceil(n_s / n_x), ceil(n_t / n_y)
  int32_t conv;        // 0: correlation, K phase = output phase (H' forward, adjoint);
                       // 1: convolution, K phase = input phase (H forward, H'-stamp backprojection)
};

// resident blocks per SM the register budget is sized for: the RL
// accumulators and the RL-row window dominate the register count
constexpr int poly_tile_min_blocks(int rl) { return rl == 7 ? 7 : rl <= 8 ? 8 : rl == 12 ? 5 : rl <= 13 ? 6 : 4; }

template <typename T, int RL>
__global__ void __launch_bounds__(128, poly_tile_min_blocks(RL)) poly_tile_kernel(const double* __restrict__ sub, const T* __restrict__ K,
                                                        double* __restrict__ out, const ProjGeom q, const PolyGeom pg,
                                                        const PolyTile tg, int32_t forward) {
  extern __shared__ double psm[];
  double* tile = psm;                      // th x p
  double* ks = psm + tg.th * tg.p;         // mmax x nmax
  const int32_t nthr = tg.tk * tg.tlt;
  const int32_t tid = threadIdx.x;
  const int32_t tl = tid / tg.tk, tk = tid - tl * tg.tk;
  const int32_t n_ph = q.n_x * q.n_y;
  const int32_t ph = blockIdx.z % n_ph;
  const int32_t zout = blockIdx.z / n_ph;
  const int32_t px = ph % q.n_x, py = ph / q.n_x;
  const int32_t k0 = blockIdx.x * tg.tk;
  const int32_t L0 = blockIdx.y * tg.tlt * RL;
  const int64_t pat = int64_t(q.n_s) * q.n_t;
  const int64_t sub_plane = int64_t(pg.kp) * pg.lp;
  const T* Kz = K + (int64_t(zout) * n_ph + ph) * pat;
  const double* subz = sub + (forward ? int64_t(zout) * n_ph * sub_plane : 0);
  const int32_t tiles = tg.tw * tg.th;
  // fill walk: element tid, tid + nthr, ... of the tw x th window, as (row, col)
  const int32_t dr = nthr / tg.tw, dc = nthr - dr * tg.tw;
  const int32_t r_init = tid / tg.tw, c_init = tid - r_init * tg.tw;
  double acc[RL];
#pragma unroll
  for (int j = 0; j < RL; ++j) acc[j] = 0.0;
  const int32_t rho0 = px - q.c_s;
  for (int32_t r2 = 0; r2 < q.n_y && r2 < q.n_t; ++r2) {
    const int32_t N = (q.n_t - r2 + q.n_y - 1) / q.n_y;
    // correlation: tap b = r2 + n_y n reads input row l + floordiv(py - c_t + r2, n_y) + n;
    // convolution: it reads l + floordiv(py + c_t - r2, n_y) - n, staged with the taps
    // reversed (nn = N - 1 - n) so the compute loop below is the same
    const int32_t rho_y = tg.conv ? py + q.c_t - r2 : py - q.c_t + r2;
    const int32_t ryy = ((rho_y % q.n_y) + q.n_y) % q.n_y;
    const int32_t row_base = floordiv(rho_y, q.n_y) + pg.hy + L0 - (tg.conv ? N - 1 : 0);
    for (int32_t a0 = 0; a0 < q.n_x && a0 < q.n_s; ++a0) {
      const int32_t M = (q.n_s - a0 + q.n_x - 1) / q.n_x;
      const int32_t rho_x = tg.conv ? px + q.c_s - a0 : rho0 + a0;
      const int32_t rxx = ((rho_x % q.n_x) + q.n_x) % q.n_x;
      const int32_t col_base = floordiv(rho_x, q.n_x) + pg.hx + k0 - (tg.conv ? M - 1 : 0);
      const double* sb = subz + (int64_t(ryy) * q.n_x + rxx) * sub_plane;
      // convolution: the pattern of the class is the input phase's, H[., ., rxx, ryy, z]
      const T* Kc = tg.conv ? K + (int64_t(zout) * n_ph + rxx + int64_t(q.n_x) * ryy) * pat : Kz;
      __syncthreads();  // the previous class's compute is done with tile / ks
      {
        int32_t r = r_init, c = c_init;
        for (int32_t e = tid; e < tiles; e += nthr) {
          const int32_t gr = row_base + r, gc = col_base + c;
          double v = 0.0;
          if (gr >= 0 && gr < pg.lp && gc >= 0 && gc < pg.kp) v = sb[gc + int64_t(gr) * pg.kp];
          tile[r * tg.p + c] = v;
          c += dc;
          r += dr;
          if (c >= tg.tw) {
            c -= tg.tw;
            ++r;
          }
        }
      }
      for (int32_t e = tid; e < tg.mmax * tg.nmax; e += nthr) {
        const int32_t ap = e / tg.nmax, n = e - ap * tg.nmax;
        double v = 0.0;
        if (ap < M && n < N) {
          const int32_t ta = tg.conv ? M - 1 - ap : ap, tb = tg.conv ? N - 1 - n : n;
          v = static_cast<double>(Kc[(a0 + q.n_x * ta) + int64_t(q.n_s) * (r2 + q.n_y * tb)]);
        }
        ks[e] = v;
      }
      __syncthreads();
      for (int32_t ap = 0; ap < M; ++ap) {
        const double* col = tile + (tl * RL) * tg.p + tk + ap;
        const double* kv = ks + ap * tg.nmax;
        double w[RL];
#pragma unroll
        for (int j = 0; j < RL - 1; ++j) w[j] = col[j * tg.p];
        const double* rowp = col + (RL - 1) * tg.p;   // next window row to load
        int32_t n = 0;
        for (; n + RL <= N; n += RL) {
#pragma unroll
          for (int t = 0; t < RL; ++t) {
            w[(RL - 1 + t) % RL] = *rowp;
            rowp += tg.p;
            const double v = kv[n + t];
#pragma unroll
            for (int j = 0; j < RL; ++j) acc[j] = fma(w[(j + t) % RL], v, acc[j]);
          }
        }
        for (; n < N; ++n) {
          w[RL - 1] = *rowp;
          rowp += tg.p;
          const double v = kv[n];
#pragma unroll
          for (int j = 0; j < RL; ++j) acc[j] = fma(w[j], v, acc[j]);
#pragma unroll
          for (int j = 0; j < RL - 1; ++j) w[j] = w[j + 1];
        }
      }
    }
  }
  const int32_t k = k0 + tk;
  const int32_t l = L0 + tl * RL;
  const int32_t X = px + q.n_x * k;
#pragma unroll
  for (int j = 0; j < RL; ++j) {
    const int32_t Y = py + q.n_y * (l + j);
    if (k < pg.kc && l + j < pg.lc && X < q.nvx && Y < q.nvy)
      out[X + int64_t(Y) * q.nvx + int64_t(zout) * q.nvx * q.nvy] = acc[j];
  }
}

// ---- TMA double-buffered variant of poly_tile_kernel -----------------------
// Same sums and the same per-class compute loop.  The class's sub-image
// window is loaded by ONE thread as a 3-D tiled TMA box (kk, ll, sub-image)
// into one of two shared buffers while the block computes the previous class
// from the other, so the window fill no longer stalls the FP64 loop.  Cells
// outside the padded sub-image are zero-filled by the TMA unit.  The box's
// first column must be 16-byte aligned (an odd double offset faults with
// "illegal instruction"), so the window starts one column early when its
// origin is odd and the compute reads from column `shift`.  Shared layout:
// 2 mbarriers (128 B), two tile buffers of th x p doubles at 128-byte aligned
// offsets (p = box width, even), then the mmax x nmax taps.
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

struct PolyCls {
  int32_t r2, a0, ryy, rxx, row_base, col_base, M, N;
};

__device__ __forceinline__ PolyCls poly_class(int32_t c, const ProjGeom& q, const PolyGeom& pg, const PolyTile& tg,
                                              int32_t px, int32_t py, int32_t na0, int32_t L0, int32_t k0) {
  PolyCls g;
  g.r2 = c / na0;
  g.a0 = c - g.r2 * na0;
  g.N = (q.n_t - g.r2 + q.n_y - 1) / q.n_y;
  g.M = (q.n_s - g.a0 + q.n_x - 1) / q.n_x;
  const int32_t rho_y = tg.conv ? py + q.c_t - g.r2 : py - q.c_t + g.r2;
  g.ryy = ((rho_y % q.n_y) + q.n_y) % q.n_y;
  g.row_base = floordiv(rho_y, q.n_y) + pg.hy + L0 - (tg.conv ? g.N - 1 : 0);
  const int32_t rho_x = tg.conv ? px + q.c_s - g.a0 : px - q.c_s + g.a0;
  g.rxx = ((rho_x % q.n_x) + q.n_x) % q.n_x;
  g.col_base = floordiv(rho_x, q.n_x) + pg.hx + k0 - (tg.conv ? g.M - 1 : 0);
  return g;
}

template <typename T, int RL>
__global__ void __launch_bounds__(128, poly_tile_min_blocks(RL))
    poly_tma_kernel(const __grid_constant__ CUtensorMap tmap, const T* __restrict__ K, double* __restrict__ out,
                    const ProjGeom q, const PolyGeom pg, const PolyTile tg, int32_t forward) {
  extern __shared__ __align__(128) uint8_t psm_raw[];
  const int32_t tile_elems = tg.th * tg.p;
  const int32_t tile_stride = ((tile_elems * 8 + 127) / 128) * 128;   // bytes, 128-aligned buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(psm_raw);
  double* tiles = reinterpret_cast<double*>(psm_raw + 128);
  double* ks = reinterpret_cast<double*>(psm_raw + 128 + 2 * tile_stride);
  const int32_t nthr = tg.tk * tg.tlt;
  const int32_t tid = threadIdx.x;
  const int32_t tl = tid / tg.tk, tk = tid - tl * tg.tk;
  const int32_t n_ph = q.n_x * q.n_y;
  const int32_t ph = blockIdx.z % n_ph;
  const int32_t zout = blockIdx.z / n_ph;
  const int32_t px = ph % q.n_x, py = ph / q.n_x;
  const int32_t k0 = blockIdx.x * tg.tk;
  const int32_t L0 = blockIdx.y * tg.tlt * RL;
  const int64_t pat = int64_t(q.n_s) * q.n_t;
  const T* Kz = K + (int64_t(zout) * n_ph + ph) * pat;
  const int32_t sub0 = forward ? zout * n_ph : 0;   // first sub-image of this block's input plane
  const int32_t na0 = min(q.n_x, q.n_s);
  const int32_t ncls = min(q.n_y, q.n_t) * na0;
  const uint32_t tile_bytes = uint32_t(tile_elems) * 8u;
  const uint32_t tiles_s = smem_u32(tiles);
  if (tid == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0 && ncls > 0) {
    const PolyCls g = poly_class(0, q, pg, tg, px, py, na0, L0, k0);
    mbar_arrive_expect_tx(smem_u32(&bars[0]), tile_bytes);
    tma_load_3d(tiles_s, &tmap, g.col_base & ~1, g.row_base, sub0 + g.ryy * q.n_x + g.rxx, smem_u32(&bars[0]));
  }
  double acc[RL];
#pragma unroll
  for (int j = 0; j < RL; ++j) acc[j] = 0.0;
  for (int32_t c = 0; c < ncls; ++c) {
    const int32_t buf = c & 1;
    // the other buffer was last read by class c - 1, done before the
    // trailing barrier of the previous iteration
    if (tid == 0 && c + 1 < ncls) {
      const PolyCls g = poly_class(c + 1, q, pg, tg, px, py, na0, L0, k0);
      const uint32_t bar = smem_u32(&bars[buf ^ 1]);
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(bar, tile_bytes);
      tma_load_3d(tiles_s + uint32_t(buf ^ 1) * uint32_t(tile_stride), &tmap, g.col_base & ~1, g.row_base,
                  sub0 + g.ryy * q.n_x + g.rxx, bar);
    }
    const PolyCls g = poly_class(c, q, pg, tg, px, py, na0, L0, k0);
    const int32_t r2 = g.r2, a0 = g.a0, M = g.M, N = g.N;
    const int32_t shift = g.col_base & 1;
    const T* Kc = tg.conv ? K + (int64_t(zout) * n_ph + g.rxx + int64_t(q.n_x) * g.ryy) * pat : Kz;
    for (int32_t e = tid; e < tg.mmax * tg.nmax; e += nthr) {
      const int32_t ap = e / tg.nmax, n = e - ap * tg.nmax;
      double v = 0.0;
      if (ap < M && n < N) {
        const int32_t ta = tg.conv ? M - 1 - ap : ap, tb = tg.conv ? N - 1 - n : n;
        v = static_cast<double>(Kc[(a0 + q.n_x * ta) + int64_t(q.n_s) * (r2 + q.n_y * tb)]);
      }
      ks[e] = v;
    }
    __syncthreads();  // taps visible
    mbar_wait(smem_u32(&bars[buf]), uint32_t((c >> 1) & 1));
    const double* tile = tiles + int64_t(buf) * (tile_stride / 8) + shift;
    for (int32_t ap = 0; ap < M; ++ap) {
      const double* col = tile + (tl * RL) * tg.p + tk + ap;
      const double* kv = ks + ap * tg.nmax;
      double w[RL];
#pragma unroll
      for (int j = 0; j < RL - 1; ++j) w[j] = col[j * tg.p];
      const double* rowp = col + (RL - 1) * tg.p;
      int32_t n = 0;
      for (; n + RL <= N; n += RL) {
#pragma unroll
        for (int t = 0; t < RL; ++t) {
          w[(RL - 1 + t) % RL] = *rowp;
          rowp += tg.p;
          const double v = kv[n + t];
#pragma unroll
          for (int j = 0; j < RL; ++j) acc[j] = fma(w[(j + t) % RL], v, acc[j]);
        }
      }
      for (; n < N; ++n) {
        w[RL - 1] = *rowp;
        rowp += tg.p;
        const double v = kv[n];
#pragma unroll
        for (int j = 0; j < RL; ++j) acc[j] = fma(w[j], v, acc[j]);
#pragma unroll
        for (int j = 0; j < RL - 1; ++j) w[j] = w[j + 1];
      }
    }
    __syncthreads();  // tile[buf] and ks free for reuse
  }
  const int32_t k = k0 + tk;
  const int32_t l = L0 + tl * RL;
  const int32_t X = px + q.n_x * k;
#pragma unroll
  for (int j = 0; j < RL; ++j) {
    const int32_t Y = py + q.n_y * (l + j);
    if (k < pg.kc && l + j < pg.lc && X < q.nvx && Y < q.nvy)
      out[X + int64_t(Y) * q.nvx + int64_t(zout) * q.nvx * q.nvy] = acc[j];
  }
}

// forward: image = sum over z of the per-plane partial images (fixed order)
__global__ void sum_planes_kernel(const double* __restrict__ part, double* __restrict__ out, int64_t n, int32_t planes) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double a = 0.0;
    for (int32_t z = 0; z < planes; ++z) a += part[i + z * n];
    out[i] = a;
  }
}

// _safe_divide (projector.py:135-145): num / den where den >= eps * max(den)
// (and den > 0 when eps * max == 0), else 0; `peak` is max(den) on the device
__global__ void safe_divide_kernel(const double* __restrict__ num, const double* __restrict__ den,
                                   double* __restrict__ out, int64_t n, double eps, const double* __restrict__ peak) {
  const double pk = *peak;
  const double thr = eps * pk;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double r = 0.0;
    if (pk > 0.0) {
      const double d = den[i];
      bool ok = d >= thr;
      if (thr == 0.0) ok = ok && d > 0.0;
      if (ok) r = num[i] / d;
    }
    out[i] = r;
  }
}

// g *= _safe_divide(back, norm, eps)[i] (projector.py:192), fused
__global__ void rl_update_kernel(double* __restrict__ g, const double* __restrict__ back,
                                 const double* __restrict__ norm, int64_t n, double eps,
                                 const double* __restrict__ peak) {
  const double pk = *peak;
  const double thr = eps * pk;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double r = 0.0;
    if (pk > 0.0) {
      const double d = norm[i];
      bool ok = d >= thr;
      if (thr == 0.0) ok = ok && d > 0.0;
      if (ok) r = back[i] / d;
    }
    g[i] = g[i] * r;
  }
}

__device__ __forceinline__ void atomic_max_double(double* a, double v) {
  // nonnegative doubles order like their bit patterns; NaN / negatives never win
  if (!(v > 0.0)) return;
  atomicMax(reinterpret_cast<unsigned long long*>(a), static_cast<unsigned long long>(__double_as_longlong(v)));
}

__global__ void max_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ peak) {
  double m = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    m = fmax(m, x[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_double(peak, m);
}

}  // namespace hp
