// Solver state shared by the sweep kernels (tiled v1 fallback, streaming v2).
#pragma once

#include "pdz_internal.cuh"

namespace pdz {

constexpr int kMaxFusedRadius = 48;
constexpr int kMaxTaps = 2 * kMaxFusedRadius + 1;
constexpr int kChunk = 16;  // sweeps per captured graph chunk

// Device-resident state of one fixed_point_solve over P planes.
struct StateView {
  int32_t* stop_iter;   // [P] 0 = running, else the iteration it stopped at
  int32_t* converged;   // [P]
  int32_t* failed;      // [P] iteration that went non-finite, 0 = never
  int32_t* iters;       // [P] iterations whose norm is recorded
  double* prev_norm;    // [P]
  double* norms;        // [max_iters][P]
  double* sums;         // [max_iters][P] raw sums of r^2 (nullable; row-slab blocks all-reduce them)
  int32_t* running;     // [1] planes still running after the latest finalize
  int32_t* iter_base;   // [1] first iteration of the current graph chunk
  int32_t* chunk_ctr;   // [1]
};

// Per-iteration partial sums of r^2: [2 (iteration parity)][P][nbmax] plus a
// non-finite flag per entry.  How many entries plane p has (and which) is
// kernel specific: `tiles` (v1: every tile of the plane) or a CTA range (v2).
struct Partials {
  double* sum;
  int32_t* flag;
  int32_t nbmax;
  int32_t ring;   // iteration slots: iteration it uses slot it % ring
  // v1: count = tiles (fixed); v2: count = hi(p) - lo(p) + 1 with CTA ranges
  int32_t tiles;
  int64_t S;      // v2: total strip-rows (images x strips x H)
  int64_t U;      // v2: strip-rows per image (strips x H)
  int32_t G;      // v2: grid size
  int32_t C;      // v2: planes per image (the C channels share the CTA ranges)
  // per-strip partition (kps > 0): strip s of an image gets kps CTAs, plus
  // `bonus` for the two border strips (their mirrored pad stores make a row
  // dearer); within a strip the rows are split evenly.  kps == 0: the S
  // strip-rows are split into G even ranges (several strips per CTA).
  int32_t kps, bonus, nstr, H;
};

// Index of the CTA whose balanced range [floor(iS/G), floor((i+1)S/G)) holds
// linear strip-row L (largest i with floor(i S / G) <= L).
__host__ __device__ __forceinline__ int64_t cta_of(int64_t L, int64_t S, int64_t G) {
  return ((L + 1) * G - 1) / S;
}
__host__ __device__ __forceinline__ int64_t cta_start(int64_t i, int64_t S, int64_t G) {
  return (i * S) / G;
}

// CTAs of one image in the per-strip partition.
__host__ __device__ __forceinline__ int64_t part_per_image(const Partials& pt) {
  return int64_t(pt.nstr) * pt.kps + 2 * pt.bonus;
}
// Index of the CTA whose range holds linear strip-row L.
__host__ __device__ __forceinline__ int64_t part_cta_of(const Partials& pt, int64_t L) {
  if (pt.kps == 0) return cta_of(L, pt.S, pt.G);
  const int64_t u = L / pt.H, y = L - u * pt.H;
  const int64_t b = u / pt.nstr, s = u - b * pt.nstr;
  const int64_t ks = pt.kps + ((s == 0 || s == pt.nstr - 1) ? pt.bonus : 0);
  const int64_t base = b * part_per_image(pt) + s * pt.kps + (s > 0 ? pt.bonus : 0);
  return base + ((y + 1) * ks - 1) / pt.H;
}
// First strip-row of CTA i (i == G: S).
__host__ __device__ __forceinline__ int64_t part_start(const Partials& pt, int64_t i) {
  if (pt.kps == 0) return cta_start(i, pt.S, pt.G);
  if (i >= pt.G) return pt.S;
  const int64_t per = part_per_image(pt);
  const int64_t b = i / per;
  int64_t r = i - b * per, s, t, ks;
  if (r < pt.kps + pt.bonus) {
    s = 0, t = r, ks = pt.kps + pt.bonus;
  } else {
    r -= pt.kps + pt.bonus;
    s = 1 + r / pt.kps;
    if (s >= pt.nstr - 1) {
      s = pt.nstr - 1, t = r - int64_t(pt.nstr - 2) * pt.kps, ks = pt.kps + pt.bonus;
    } else {
      t = r - (s - 1) * pt.kps, ks = pt.kps;
    }
  }
  return (b * pt.nstr + s) * pt.H + (t * pt.H) / ks;
}

__device__ __forceinline__ int partial_count(const Partials& pt, int p) {
  if (pt.tiles > 0) return pt.tiles;
  const int64_t img = p / pt.C;
  const int64_t lo = part_cta_of(pt, img * pt.U);
  const int64_t hi = part_cta_of(pt, (img + 1) * pt.U - 1);
  return int(hi - lo + 1);
}

// Apply the stop rule of fixed_point_solve (solver.py:347-358) to plane p
// given iteration `it`'s reduced sum of r^2; returns 1 if p keeps running.
__device__ __forceinline__ int finalize_plane(const StateView& st, int P, int p, int it,
                                              int max_iters, double rel_tol, double s, int nf) {
  if (nf) {
    st.failed[p] = it;
    st.stop_iter[p] = it;
    return 0;
  }
  const double norm = sqrt(s);
  st.norms[size_t(it - 1) * P + p] = norm;
  if (st.sums) st.sums[size_t(it - 1) * P + p] = s;
  st.iters[p] = it;
  const double prev = st.prev_norm[p];
  int run = 0;
  if (it >= 2 && fabs(norm - prev) / fmax(prev, 1e-30) <= rel_tol) {
    st.converged[p] = 1;
    st.stop_iter[p] = it;
  } else if (it >= max_iters) {
    st.stop_iter[p] = it;
  } else {
    run = 1;
  }
  st.prev_norm[p] = norm;
  return run;
}

// Reduce iteration `it` for every still-running plane and apply the stop
// rule.  Executed by ONE warp, always in a fixed order so the norms are
// bitwise reproducible: planes with many partials are reduced warp-wide
// (lane-strided loads in flight together, fixed xor tree); planes with few
// partials (batches) lane-per-plane.
__device__ __forceinline__ void finalize_iteration_warp(const StateView& st, const Partials& pt,
                                                        int P, int it, int max_iters,
                                                        double rel_tol) {
  const int lane = threadIdx.x & 31;
  int running = 0;
  if (pt.nbmax > 8) {
    for (int p = 0; p < P; ++p) {
      if (st.stop_iter[p] != 0) continue;
      const size_t base = (size_t(it % pt.ring) * P + p) * pt.nbmax;
      const int n = partial_count(pt, p);
      double s = 0.0;
      int nf = 0;
      for (int b = lane; b < n; b += 32) {
        s += pt.sum[base + b];
        nf |= pt.flag[base + b];
      }
      s = warp_sum(s);
      nf = __any_sync(0xffffffffu, nf);
      if (lane == 0) running += finalize_plane(st, P, p, it, max_iters, rel_tol, s, nf);
    }
    if (lane == 0) st.running[0] = running;
    return;
  }
  for (int p = lane; p < P; p += 32) {
    if (st.stop_iter[p] != 0) continue;
    const size_t base = (size_t(it % pt.ring) * P + p) * pt.nbmax;
    const int n = partial_count(pt, p);
    double s = 0.0;
    int nf = 0;
    for (int b = 0; b < n; ++b) {
      s += pt.sum[base + b];
      nf |= pt.flag[base + b];
    }
    running += finalize_plane(st, P, p, it, max_iters, rel_tol, s, nf);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) running += __shfl_xor_sync(0xffffffffu, running, o);
  if (lane == 0) st.running[0] = running;
}

}  // namespace pdz
