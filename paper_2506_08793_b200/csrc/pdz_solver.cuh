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
};

// Index of the CTA whose balanced range [floor(iS/G), floor((i+1)S/G)) holds
// linear strip-row L (largest i with floor(i S / G) <= L).
__host__ __device__ __forceinline__ int64_t cta_of(int64_t L, int64_t S, int64_t G) {
  return ((L + 1) * G - 1) / S;
}
__host__ __device__ __forceinline__ int64_t cta_start(int64_t i, int64_t S, int64_t G) {
  return (i * S) / G;
}

__device__ __forceinline__ int partial_count(const Partials& pt, int p) {
  if (pt.tiles > 0) return pt.tiles;
  const int64_t img = p / pt.C;
  const int64_t lo = cta_of(img * pt.U, pt.S, pt.G);
  const int64_t hi = cta_of((img + 1) * pt.U - 1, pt.S, pt.G);
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
