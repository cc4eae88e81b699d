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
  int64_t S;      // v2: total strip-rows
  int64_t U;      // v2: strip-rows per plane
  int32_t G;      // v2: grid size
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
  const int64_t lo = cta_of(int64_t(p) * pt.U, pt.S, pt.G);
  const int64_t hi = cta_of(int64_t(p + 1) * pt.U - 1, pt.S, pt.G);
  return int(hi - lo + 1);
}

// Reduce iteration `it` for every still-running plane and apply the stop
// rule of fixed_point_solve (solver.py:347-358).  Executed by ONE warp:
// lane-per-plane, each lane sums its plane's partials sequentially in a
// fixed order, so the norms are bitwise reproducible.
__device__ __forceinline__ void finalize_iteration_warp(const StateView& st, const Partials& pt,
                                                        int P, int it, int max_iters,
                                                        double rel_tol) {
  const int lane = threadIdx.x & 31;
  int running = 0;
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
    if (nf) {
      st.failed[p] = it;
      st.stop_iter[p] = it;
      continue;
    }
    const double norm = sqrt(s);
    st.norms[size_t(it - 1) * P + p] = norm;
    st.iters[p] = it;
    const double prev = st.prev_norm[p];
    if (it >= 2 && fabs(norm - prev) / fmax(prev, 1e-30) <= rel_tol) {
      st.converged[p] = 1;
      st.stop_iter[p] = it;
    } else if (it >= max_iters) {
      st.stop_iter[p] = it;
    } else {
      ++running;
    }
    st.prev_norm[p] = norm;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) running += __shfl_xor_sync(0xffffffffu, running, o);
  if (lane == 0) st.running[0] = running;
}

}  // namespace pdz
