// Streaming, persistent relaxed fixed-point solve -- the production hot kernel.
//
// Same mathematics as the tiled sweep (pdz_sweep.cu; solver.py:280-302), laid
// out for B200:
//  * ONE cooperative launch runs the whole solve, one CTA per SM (15 compute
//    warps + 1 service warp).  The S = images x strips x H "strip-rows"
//    (strip = 64 output columns of one image) are split into G exactly
//    balanced ranges [floor(iS/G), floor((i+1)S/G)), aligned to strips; CTA i
//    owns range i for EVERY channel of those images, so every SM gets the
//    same pixels (+-1 row): no wave quantisation, no per-sweep launch and no
//    grid-wide barrier.
//  * a CTA walks one flat stream of blocks ordered (iteration n, channel c,
//    block of <= 120 rows; config 2 has one block per pass).  Pass (n, c)
//    reads channel c of iterate n-1, so it only
//    waits until the CTAs whose rows its stencil reads (its strip and the
//    neighbouring strips, +-R rows) have published pass (n-1, c) -- done
//    C - 1 passes earlier, so in steady state nobody waits.  A per-CTA
//    progress counter (passes completed) carries that ordering (release /
//    acquire); the same wait protects the ping-pong buffer being overwritten.
//  * the iterate buffers are PADDED, [P][H + 2R][W + 2 kPadC], so every
//    block's staged box is a plain box of the padded tensor; a block that
//    touches an image border reflects its staged pads in shared memory from
//    the interior values of the same tile (np.pad "symmetric",
//    solver.py:235) -- nothing mirrored is stored globally.  Each block's
//    input rows (64 + 2 ceil4(R) columns) arrive by ONE TMA tile load
//    (cp.async.bulk.tensor, UTMALDG)
//    into a double buffer, signalled by an mbarrier and always queued one
//    block ahead -- across pass boundaries too.
//  * horizontal Gaussian from shared memory (8 outputs per item), vertical
//    pass with packed FFMA2 over column pairs, MUFU sqrt/rcp face fluxes,
//    residual, update and r^2 fused in registers.
//  * warps 0-14 compute; warp 15 (service) does every gpu-scope
//    synchronisation: it releases the CTA's pass counter to global memory
//    and grants the compute warps the passes whose inputs are published, so
//    compute warps never execute a gpu-scope fence.
//  * one extra CTA finalises sweep n once every CTA published it: it reduces
//    the r^2 partials in a fixed order (bitwise reproducible), applies the
//    stop rule (solver.py:347-358) and releases `fin = n`.  Partials live in
//    a ring of kRing iteration slots: pass (n, c) waits for fin >= n - kRing,
//    and with the stop rule for fin >= n - 2 so planes stopped at <= n-2 are
//    skipped (their answer stays in buf[stop & 1]).
// Requirements: width % 4 == 0 (TMA strides), H >= 2R and W >= 2 ceil4(R)
// (one reflection fold), a compiled radius, and all G + 1 CTAs co-resident
// (cooperative launch; G + 1 <= SMs); otherwise the tiled kernel is used.
// Every spin has a 10 s timeout that sets an abort flag instead of hanging.
#pragma once
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "pdz_solver.cuh"

namespace pdz {

constexpr int kSTW = 64;                    // strip width (output columns)
// Block geometry V (a template parameter of the kernel, picked per solve from
// the partition, pdz_sweep.cu):
//  V = 0: 19 compute warps x 6 output rows (114-row blocks; 5 rows / 95 for
//         R = 24, whose wider staging would not fit shared memory otherwise),
//         20 warps x 96 registers (5 warps per SM sub-partition fill its
//         16K-register file).  Best when a CTA's rows of a strip fit one block
//         (config 2: ~114 rows per CTA).
//  V = 1: 15 compute warps x 8 rows (120-row blocks) at 128 registers (4 warps
//         per sub-partition), for CTAs that walk several blocks per pass
//         (configs 3 and 4): fewer blocks per strip and more registers per
//         thread for the vertical pass.
__host__ __device__ constexpr int geo_scw(int V) { return V ? 15 : 19; }
// R = 24: 5 rows per warp (95-row blocks, 215 KB of shared memory); 4 rows
// (76-row blocks) cost 9 % more per sweep on config 5 (1.63x horizontal-pass
// rows per output row instead of 1.51x, 1024 H items on 608 threads).
#ifndef PDZ_RPW24
#define PDZ_RPW24 5
#endif
__host__ __device__ constexpr int geo_rpw(int R, int V) { return V ? 8 : (R <= 12 ? 6 : PDZ_RPW24); }
__host__ __device__ constexpr int geo_srb(int R, int V) { return geo_scw(V) * geo_rpw(R, V); }
__host__ __device__ constexpr int geo_threads(int V) { return (geo_scw(V) + 1) * 32; }  // + service warp
__host__ __device__ constexpr int geo_nreg(int V) { return V ? 128 : 96; }
// A block's input rows arrive in two TMA boxes, rows [0, split) and
// [split, ROWS), with their own mbarriers: the first wave of horizontal-pass
// items (one per compute thread, 8-row groups) only touches rows < split, so
// it starts as soon as the first box lands.
__host__ __device__ constexpr int geo_split(int V) { return (geo_scw(V) * 32 / 64) * 8 + 8; }
constexpr int kSCWMax = 19;                 // mailbox slots
constexpr int kRing = 4;
constexpr int kNBuf = 3;                    // iterate buffers (iteration n in buf[n % 3])
// Column pad of the padded iterates: 32 floats (128 B) each side, so padded
// rows and every strip's first image column are 128-byte aligned (only the
// ceil4(R) columns next to the image are ever written or read).
constexpr int kPadC = 32;
constexpr long long kSpinTimeoutNs = 10000000000ll;

// Shared-memory row pitches are an ODD number of float4s, so the 8 lanes of a
// quarter-warp that read / write 16 bytes each in 8 different rows of the same
// column group hit 8 distinct bank quads (conflict-free LDS.128 / STS.128).
template <int R, int V>
struct SGeo {
  static constexpr int SCW = geo_scw(V);       // compute warps
  static constexpr int CT = SCW * 32;          // compute threads
  static constexpr int NT = geo_threads(V);    // threads per CTA
  static constexpr int SPLIT = geo_split(V);   // rows of the first TMA box
  static constexpr int RPW = geo_rpw(R, V);    // output rows per compute warp
  static constexpr int SRB = geo_srb(R, V);    // output rows per block
  static constexpr int RP = (R + 3) & ~3;      // column halo rounded to float4
  static constexpr int PWD = kSTW + 2 * RP;    // staged floats per row used (even # float4)
  static constexpr int PITCH = PWD + 4;        // staged row pitch = TMA box width
  static constexpr int HP = kSTW + 4;          // H row pitch
  static constexpr int ROWS = SRB + 2 * R;     // staged input rows / H rows = TMA box height
  static constexpr int IN_FLOATS = (ROWS * PITCH + 31) & ~31;  // 128-byte aligned buffers
  static constexpr int H_FLOATS = (ROWS * HP + 31) & ~31;
  static constexpr int PL_FLOATS = SRB * kSTW;  // Phi or lambda tile of the block
  static constexpr size_t SMEM = size_t(2 * IN_FLOATS + H_FLOATS + 2 * PL_FLOATS) * 4 + 128;
  static constexpr bool FITS = SMEM <= 227 * 1024;
};

struct StreamArgs {
  // TMA maps of the two padded iterate buffers [P][H + 2R][W + 2 kPadC], box
  // {PITCH, SRB + 2R, 1}.
  CUtensorMap tm[kNBuf];
  CUtensorMap tm2[kNBuf];  // the same buffers, box {PITCH, ROWS - SPLIT, 1} (second part)
  CUtensorMap tm_phi;   // Phi [P][H][W], box {64, SRB, 1}
  CUtensorMap tm_lam;   // lambda [P / C][H][W], box {64, SRB, 1}
  float* buf[kNBuf];   // iterate n in buf[n % kNBuf] (padded planes)
  const float* phi;
  const float* lam;
  Partials pt;          // ring of kRing slots
  StateView st;         // st.stop_iter == nullptr: single step (no finalisation)
  int32_t* done;        // [G] passes published by each CTA
  int32_t* fin;         // [1] last iteration finalised
  int32_t* flags;       // [0] iteration by which every plane stopped, [1] abort
  int32_t H, W, P, C, nstrips;
  int32_t iter_last, max_iters;  // sweeps 1..iter_last
  int32_t srb;          // output rows per block (geo_srb(R, V))
  int32_t stop_rule;    // rel_tol active: pass (n, c) needs fin >= n - 2
  int32_t chan_inner;   // block order (iteration, block, channel) instead of (iteration, channel, block)
  int32_t cnt_lo, cnt_hi;  // rows whose r^2 / non-finite flags are counted (0, H: all)
  float eps, tau;
  double rel_tol;
  long long* prof;      // -DPDZ_PROFILE builds + PDZ_PROF=1: [2G+1][16] wait times
  float w[kMaxTaps];
  float2 w2[kMaxTaps];  // (w, w) pairs: the FFMA2 operand
  float2 wp[kMaxTaps + 1];  // (w[k], w[k-1]), w[-1] = w[K] = 0: horizontal-pass output pairs
};

// Profiling instrumentation (tools/prof_stream.py): compiled only with
// -DPDZ_PROFILE (build with PDZ_PROFILE=1), absent from the product build.
#ifdef PDZ_PROFILE
// timeline (ns, globaltimer): kind 0 progress >= k published, 1 pass k's IN
// issued, 2 pass k's IN wanted (generated, buffer free), 3 / 4 compute warps
// start / end waiting for pass k's IN
#ifdef PDZ_TIMELINE
#define PDZ_TL(a, kind, cta, k)                                                              \
  do {                                                                                       \
    if ((a).prof && (k) > 0 && (k) < 2048 && (cta) < 256)                                     \
      (a).prof[131072 + ((size_t(kind) * 256 + (cta)) * 2048 + (k))] = global_ns();           \
  } while (0)
#else
#define PDZ_TL(a, kind, cta, k) \
  do {                          \
  } while (0)
#endif
#define PDZ_P(...) __VA_ARGS__
#define PDZ_PT(slot, stmt)            \
  {                                   \
    const long long t_ = global_ns(); \
    stmt;                             \
    pf[slot] += global_ns() - t_;     \
  }
#else
#define PDZ_P(...)
#define PDZ_PT(slot, stmt) stmt
#endif

// ------------------------------------------------------------ primitives --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// Bulk global -> shared copy (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 3-D tile load (TMA): box at (x, y, z) -> dst, completion counted on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// Order this thread's generic-proxy view (after an acquire) before its later
// async-proxy (TMA) reads of global memory.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Polling load: relaxed (no L1 invalidation per poll); one acquire fence
// follows once the condition holds.
__device__ __forceinline__ int ld_relaxed(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta_shared(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <int CT>
__device__ __forceinline__ void compute_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// d = a * b + c on packed float pairs (FFMA2).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

template <bool EDGE>
__device__ __forceinline__ float sflux(float jump, float along, float eps) {
  if (!EDGE) return jump;
  // explicit roundings: no fma contraction with the caller's adds, so every
  // kernel instantiation (block geometry, border variant) rounds alike
  const float s = fmaf(jump, jump, __fmul_rn(along, along));
  return __fmul_rn(jump, rcp_approx(__fadd_rn(sqrt_approx(s), eps)));
}

// Packed float pairs (FADD2 / FMUL2): per-lane IEEE round-to-nearest, so a
// packed op is bitwise the two scalar ops.
__device__ __forceinline__ unsigned long long f2bits(float2 a) {
  return *reinterpret_cast<unsigned long long*>(&a);
}
__device__ __forceinline__ float2 bits2f(unsigned long long d) {
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2bits(a)), "l"(f2bits(b)));
  return bits2f(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2bits(a)), "l"(f2bits(b)));
  return bits2f(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2bits(a)), "l"(f2bits(b)));
  return bits2f(d);
}
// sflux on a pair of faces (same per-lane arithmetic as sflux).
template <bool EDGE>
__device__ __forceinline__ float2 sflux2(float2 jump, float2 along, float2 eps2) {
  if (!EDGE) return jump;
  const float2 s = ffma2(jump, jump, mul2(along, along));
  const float2 q = add2(make_float2(sqrt_approx(s.x), sqrt_approx(s.y)), eps2);
  return mul2(jump, make_float2(rcp_approx(q.x), rcp_approx(q.y)));
}

// 1 / (|(jump, along)| + eps) per lane (1 when !EDGE): the coefficient of a
// face whose flux enters the divergence as an explicit fused multiply-add
// (ptxas otherwise contracts the packed product with the add or sub that
// follows in SOME unrolled rows only, and a pixel's rounding would depend on
// its row's position in the warp's row group, i.e. on the launch plan).
template <bool EDGE>
__device__ __forceinline__ float2 sflux2_coef(float2 jump, float2 along, float2 eps2) {
  if (!EDGE) return make_float2(1.f, 1.f);
  const float2 s = ffma2(jump, jump, mul2(along, along));
  const float2 q = add2(make_float2(sqrt_approx(s.x), sqrt_approx(s.y)), eps2);
  return make_float2(rcp_approx(q.x), rcp_approx(q.y));
}

// ----------------------------------------------------------- iteration --
struct SBlock {
  int p, x0, yb, n;  // plane, strip origin, first row, rows
  int iter, c;       // pass (iter, c)
  int img;           // image of the plane (p / C)
};

// One pass over the CTA's range [L0, L1) of strip-rows: (image b, strip s,
// row y) advance incrementally.  Planes frozen at <= iter-2 are skipped.
struct RangeIter {
  int L, L0, L1, b, s, y;
  int b0, s0, y0;
  bool check_stop;  // some plane has stopped: look up frozen planes (uniform per pass)
  template <class A>
  __device__ __forceinline__ void init(int l0, int l1, const A& a) {
    L = L0 = l0;
    L1 = l1;
    check_stop = false;
    const int u = l0 / a.H;
    y0 = l0 - u * a.H;
    b0 = u / a.nstrips;
    s0 = u - b0 * a.nstrips;
    reset();
  }
  __device__ __forceinline__ void reset() {
    L = L0;
    b = b0;
    s = s0;
    y = y0;
  }
  template <class A>
  __device__ __forceinline__ void wrap(const A& a) {
    y = 0;
    if (++s == a.nstrips) {
      s = 0;
      ++b;
    }
  }
  template <bool STOP, class A>
  __device__ __forceinline__ bool next(const A& a, int iter, int c, SBlock& blk) {
    while (L < L1) {
      const int seg_end = min(L1, L - y + a.H);
      const int p = b * a.C + c;
      if (STOP && check_stop) {
        const int st = a.st.stop_iter[p];
        if (st != 0 && st <= iter - kNBuf) {  // its answer buf[st % 3] is kept
          L = seg_end;
          wrap(a);
          continue;
        }
      }
      blk.p = p;
      blk.img = b;
      blk.x0 = s * kSTW;
      blk.yb = y;
      blk.n = min(a.srb, seg_end - L);
      L += blk.n;
      y += blk.n;
      if (y == a.H) wrap(a);
      return true;
    }
    return false;
  }
  // Channel-inner order: the next block POSITION of the range and the mask of
  // its image's channels still running (segments whose planes are all frozen
  // are skipped).  blk.p = the image's first plane.
  template <bool STOP, class A>
  __device__ __forceinline__ bool next_pos(const A& a, int iter, SBlock& blk, int& mask) {
    while (L < L1) {
      const int seg_end = min(L1, L - y + a.H);
      mask = (1 << a.C) - 1;
      if (STOP && check_stop) {
        for (int c = 0; c < a.C; ++c) {
          const int st = a.st.stop_iter[b * a.C + c];
          if (st != 0 && st <= iter - kNBuf) mask &= ~(1 << c);
        }
        if (mask == 0) {
          L = seg_end;
          wrap(a);
          continue;
        }
      }
      blk.p = b * a.C;
      blk.img = b;
      blk.x0 = s * kSTW;
      blk.yb = y;
      blk.n = min(a.srb, seg_end - L);
      L += blk.n;
      y += blk.n;
      if (y == a.H) wrap(a);
      return true;
    }
    return false;
  }
};

// The few kernel arguments the service warp's iterator reads on every block,
// copied into registers once: read as kernel parameters they are constant-bank
// loads, and the compute warps' tap streams keep evicting those lines, so a
// handful of them per block cost the service warp ~1k cycles.
__device__ __forceinline__ int reg_copy(int v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}
template <class T>
__device__ __forceinline__ T* reg_copy(T* p) {
  asm volatile("mov.b64 %0, %0;" : "+l"(p));
  return p;
}
struct SvcView {
  int H, C, srb, nstrips, iter_last, ci;
  struct {
    int32_t* stop_iter;
  } st;
  int32_t* flags;
  __device__ __forceinline__ explicit SvcView(const StreamArgs& a) {
    ci = reg_copy(a.chan_inner);
    H = reg_copy(a.H);
    C = reg_copy(a.C);
    srb = reg_copy(a.srb);
    nstrips = reg_copy(a.nstrips);
    iter_last = reg_copy(a.iter_last);
    st.stop_iter = reg_copy(a.st.stop_iter);
    flags = reg_copy(a.flags);
  }
};

// Progress counter value once pass (n, c) is complete.
__device__ __forceinline__ int pass_index(int iter, int c, int C) { return (iter - 1) * C + c + 1; }

// Progress value that the CTAs a block reads from must have published, and
// that is published once the block's own unit is complete.  Channel-outer
// order: the unit is the pass (n, c) and it needs the neighbours' pass
// (n-1, c).  Channel-inner order: the channels of a sweep complete together,
// so the unit is the sweep: every block of sweep n carries (n-1) C + 1 and
// needs (n-1) C, the neighbours' whole previous sweep.
__device__ __forceinline__ int prog_index(int iter, int c, int C, int ci) {
  return ci ? (iter - 1) * C + 1 : pass_index(iter, c, C);
}
__device__ __forceinline__ int prog_need(int kprog, int C, int ci) { return ci ? kprog - 1 : kprog - C; }

// Flat stream of (iteration, channel, block) run by the service warp.
// Passes with no blocks (every plane of the range frozen) are skipped.  With
// the stop rule a pass of iteration n first needs the stop decisions of
// n - 3 (fin >= n - 3: its answer buffer is then final); next() returns
// kWaitFin until they are known.
enum { kIterEnd = 0, kIterBlock = 1, kIterWaitFin = 2 };
// Channel-inner order (a.ci; CTAs that walk several blocks per pass): the
// stream is (iteration, block position, channel), so the three channel
// blocks of a position run back to back and share one lambda tile (lambda is
// a third of the Phi / lambda / u traffic of a block and was re-read for every
// channel: measured DRAM traffic 1.4x algorithmic on configs 3 and 4).
struct SvcIter {
  RangeIter r;
  int iter, c;
  bool fresh;  // the next block starts a new pass (channel-inner: a new sweep)
  bool ended;
  SBlock pos;  // channel-inner: the current block position
  int mask;    // and its channels still to emit
  template <bool STOP, class A>
  __device__ __forceinline__ int next(const A& a, SBlock& blk, int fin_seen,
                                      bool anystop) {
    while (!ended && iter <= a.iter_last) {
      if (STOP && fresh && a.st.stop_iter && iter > kNBuf) {
        if (fin_seen < iter - kNBuf) return kIterWaitFin;
        // Only once some plane has stopped are the stop records consulted.
        r.check_stop = anystop;
        if (anystop) {
          const int all = ld_relaxed(a.flags);
          if (all != 0 && all <= iter - kNBuf) {
            ended = true;
            break;
          }
        }
      }
      if (a.ci) {
        if (mask == 0) {
          if (!r.template next_pos<STOP>(a, iter, pos, mask)) {
            ++iter;
            r.reset();
            fresh = true;
            continue;
          }
          c = 0;
        }
        while (!(mask & (1 << c))) ++c;
        mask &= ~(1 << c);
        blk = pos;
        blk.p = pos.p + c;
        blk.iter = iter;
        blk.c = c;
        fresh = false;
        return kIterBlock;
      }
      if (r.template next<STOP>(a, iter, c, blk)) {
        blk.iter = iter;
        blk.c = c;
        fresh = false;
        return kIterBlock;
      }
      if (++c == a.C) {
        c = 0;
        ++iter;
      }
      r.reset();
      fresh = true;
    }
    ended = true;
    return kIterEnd;
  }
  // Progress index of the last pass before the iterator position.
  template <class A>
  __device__ __forceinline__ int completed(const A& a) const {
    if (ended) return pass_index(a.iter_last, a.C - 1, a.C);
    return a.ci ? (iter - 1) * a.C : pass_index(iter, c, a.C) - 1;
  }
};

// ----------------------------------------------------------- row loads --
// ONE TMA tile load brings a block's input rows: staged row i holds image row
// yb - R + i (padded row yb + i); rows beyond the block's n + 2R are
// over-fetch, never read.  Pad rows / columns of the box are reflected by
// the readers (the pads of the iterates carry no data).
template <int R, int V>
__device__ __forceinline__ void issue_block(const StreamArgs& a, const SBlock& q, float* in,
                                            uint64_t* bar) {
  using Gm = SGeo<R, V>;
  constexpr int kSplit = Gm::SPLIT;
  const int buf = (q.iter - 1) % kNBuf;  // the buffer iteration `iter` reads
  static_assert(Gm::ROWS > kSplit, "two-part row load");
  mbar_expect_tx(bar, uint32_t(kSplit) * Gm::PITCH * 4u);
  tma_load_3d(in, &a.tm[buf], q.x0 + kPadC - Gm::RP, q.yb, q.p, bar);
  mbar_expect_tx(bar + 5, uint32_t(Gm::ROWS - kSplit) * Gm::PITCH * 4u);
  tma_load_3d(in + kSplit * Gm::PITCH, &a.tm2[buf], q.x0 + kPadC - Gm::RP, q.yb + kSplit, q.p,
              bar + 5);
}

// --------------------------------------------------------- service warp --
// CTAs whose output rows a CTA's stencil reads: up to 3 intervals of CTA
// indices (the strips left / right and its own strip, rows +-R); a range that
// spans several strips uses one covering interval.
struct DepSet {
  int lo[3], hi[3], n;  // three intervals (hi < lo: empty)
};
__device__ __forceinline__ DepSet dep_set(const StreamArgs& a, int L0, int L1, int R) {
  DepSet d;
  const int S = int(a.pt.S), H = a.H;
  const int u0 = L0 / H, u1 = (L1 - 1) / H;
  if (u0 != u1) {
    d.n = 3;
    d.lo[0] = int(part_cta_of(a.pt, max(0, L0 - H - R)));
    d.hi[0] = int(part_cta_of(a.pt, min(S - 1, L1 - 1 + H + R)));
    d.lo[1] = d.lo[2] = 1;
    d.hi[1] = d.hi[2] = 0;
    return d;
  }
  const int b = u0 / a.nstrips, s = u0 - b * a.nstrips;
  const int y0 = max(0, L0 - u0 * H - R), y1 = min(H, L1 - u0 * H + R);
  d.n = 3;
#pragma unroll
  for (int i = 0; i < 3; ++i) {  // strips s-1, s, s+1 (empty interval if absent)
    const int s2 = s + i - 1;
    const int base = (b * a.nstrips + s2) * H;
    const bool ok = s2 >= 0 && s2 < a.nstrips;
    d.lo[i] = ok ? int(part_cta_of(a.pt, base + y0)) : 1;
    d.hi[i] = ok ? int(part_cta_of(a.pt, base + y1 - 1)) : 0;
  }
  return d;
}

__device__ __forceinline__ void st_relaxed(int32_t* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Non-blocking mbarrier phase test (acquire at CTA scope when complete).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Shared-memory mailbox between the service warp and the compute warps.
struct Mailbox {
  SBlock desc[2];        // block of IN buffer ib (n == 0: end of the stream)
  SBlock q[4];           // service warp: generated blocks, ring by block number
  double red[2][kSCWMax];  // per-warp r^2 of block b in red[b & 1]
  int nf[2][kSCWMax];      // per-warp non-finite flag
  PDZ_P(long long t_issue[2];)  // profiling: clock64 of IN(ib)'s TMA issue
};

// The service warp (the last warp) runs the CTA's whole schedule, so the compute
// warps only wait for data, compute and report:
//  * it walks the block stream (SvcIter) and posts each block's descriptor
//    with the TMA load of its input rows into IN(b & 1), once the pass is
//    granted: the CTAs whose rows the stencil reads have published pass
//    (n-1, c), partial slot n % kRing is free (fin >= n - kRing), and the
//    buffer's previous block b-2 is done;
//  * when the compute warps report block b done (mbarrier bars[3 + (b & 1)],
//    one arrival per warp), it sums their r^2 in a fixed order into the
//    (CTA, plane, iteration) partial slot and publishes the CTA's progress
//    (passes completed) to done[cta];
//  * with the stop rule it mirrors `fin` for the iterator.
// Every gpu-scope fence of the CTA is executed here, one per round for all
// purposes (release of the progress, acquire of neighbours / fin).
template <int R, int V, bool STOP>
__device__ void service_loop(const StreamArgs& a, Mailbox* mb, float* in0, float* in1,
                             uint64_t* bars, const DepSet& dep, int L0, int L1) {
  const int lane = threadIdx.x & 31;
  const int C = reg_copy(a.C);
  const bool fin_on = a.st.stop_iter != nullptr;
  int32_t* const done_ctr = reg_copy(a.done);
  int32_t* const fin_ctr = reg_copy(a.fin);
  SvcIter it;
  const SvcView sv(a);
  it.r.init(L0, L1, sv);
  it.iter = 1;  // pass numbering (done[], grants) starts at sweep 1
  it.c = 0;
  it.fresh = true;
  it.ended = false;
  it.mask = 0;
  const int ci = sv.ci;
  // flattened dependency list: lane l checks CTAs #l and #l + 32 of the
  // (disjoint) intervals; more than 64: the generic per-interval loop
  int ndep = 0, dep0 = -1, dep1 = -1;
  for (int i = 0; i < 3; ++i) {
    const int n = dep.hi[i] >= dep.lo[i] ? dep.hi[i] - dep.lo[i] + 1 : 0;
    if (lane >= ndep && lane < ndep + n) dep0 = dep.lo[i] + lane - ndep;
    if (lane + 32 >= ndep && lane + 32 < ndep + n) dep1 = dep.lo[i] + lane + 32 - ndep;
    ndep += n;
  }
  SBlock* const q = mb->q;  // generated blocks (at most 3 not done), ring by block number
  int gen = 0, iss = 0, dn = 0;  // blocks generated / issued / done
  int published = 0, fin_seen = 0, granted_k = 0, fin_probe = 0;
  bool anystop = false, aborted = false;
  // open partial: (plane, iteration) of the blocks summed so far
  int acc_p = -1, acc_it = 0, acc_img = 0, slot_img = -1, slot_k = 0;
  double acc = 0.0;
  int acc_nf = 0;
  static_assert((kRing & (kRing - 1)) == 0, "ring slots by mask");
  auto flush = [&]() {
    if (acc_p < 0) return;
    if (lane == 0) {
      if (acc_img != slot_img) {  // the CTA's index within the image's range
        slot_img = acc_img;
        slot_k = int(blockIdx.x - part_cta_of(a.pt, int64_t(acc_img) * a.pt.U));
      }
      const size_t slot = (size_t(acc_it & (kRing - 1)) * a.P + acc_p) * a.pt.nbmax + slot_k;
      a.pt.sum[slot] = acc;
      a.pt.flag[slot] = acc_nf;
    }
    acc_p = -1;
  };
  // channel-inner order: the blocks of an image's channels alternate, so the
  // open partials are per channel, keyed by (image, iteration)
  double cacc0 = 0.0, cacc1 = 0.0, cacc2 = 0.0, cacc3 = 0.0;
  int cmask = 0, cnf = 0, c_img = -1, c_it = 0;
  auto flush_ci = [&]() {
    if (cmask == 0) return;
    if (lane == 0) {
      if (c_img != slot_img) {
        slot_img = c_img;
        slot_k = int(blockIdx.x - part_cta_of(a.pt, int64_t(c_img) * a.pt.U));
      }
      const double v[4] = {cacc0, cacc1, cacc2, cacc3};
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (cmask >> c & 1) {
          const size_t slot =
              (size_t(c_it & (kRing - 1)) * a.P + c_img * C + c) * a.pt.nbmax + slot_k;
          a.pt.sum[slot] = v[c];
          a.pt.flag[slot] = cnf >> c & 1;
        }
    }
    cmask = 0;
    cnf = 0;
  };
  long long t0 = global_ns();
  int idle = 0;
  // [0] rounds [1] dependency-scan cycles [2] publications [3] sleeps
  // [4] done events [5] cycles from a block's IN issue to its done being seen
  PDZ_P(long long sp[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long t_iss[4] = {0, 0, 0, 0}; int want_k = 0;)
  PDZ_P(long long tr = clock64(); long long rp[8] = {0, 0, 0, 0, 0, 0, 0, 0};)
  // rp: cycles in [0] done tests [1] generation [2] scan [3] grant + TMA
  // [4] sleeping [5] rest [6] r^2 reduction of done blocks [7] the release store
  while (true) {
    bool progressed = false;
    PDZ_P(sp[0] += 1;)
    PDZ_P(auto lap = [&](int i) { const long long t = clock64(); rp[i] += t - tr; tr = t; };)
    // 1. blocks the compute warps finished (in order)
    while (true) {
      const bool fin_blk = dn < iss && mbar_test(&bars[3 + (dn & 1)], uint32_t((dn >> 1) & 1));
      PDZ_P(lap(0);)
      if (!fin_blk) break;
      const SBlock& b = q[dn & 3];
      // lane w holds warp w's value; a fixed butterfly sums them (lane 0's
      // result is the one stored: deterministic)
      const double s = warp_sum(lane < geo_scw(V) ? mb->red[dn & 1][lane] : 0.0);
      const int f = __any_sync(0xffffffffu, lane < geo_scw(V) && mb->nf[dn & 1][lane] != 0);
      if (ci) {
        if (cmask != 0 && (c_img != b.img || c_it != b.iter)) flush_ci();
        c_img = b.img;
        c_it = b.iter;
        const bool had = cmask >> b.c & 1;
        if (b.c == 0) cacc0 = had ? cacc0 + s : s;
        if (b.c == 1) cacc1 = had ? cacc1 + s : s;
        if (b.c == 2) cacc2 = had ? cacc2 + s : s;
        if (b.c == 3) cacc3 = had ? cacc3 + s : s;
        cmask |= 1 << b.c;
        cnf |= (f ? 1 : 0) << b.c;
      } else {
        if (acc_p != b.p || acc_it != b.iter) {
          flush();
          acc_p = b.p;
          acc_it = b.iter;
          acc_img = b.img;
          acc = 0.0;
          acc_nf = 0;
        }
        acc += s;
        acc_nf |= f;
      }
      PDZ_P(sp[4] += 1; sp[5] += clock64() - t_iss[dn & 3];)
      ++dn;
      progressed = true;
      PDZ_P(lap(6);)
    }
    // 2. generate the schedule ahead (at most 3 blocks not yet done)
    bool wait_fin = false;
    while (!aborted && gen < dn + 3) {
      SBlock nb;
      const int k = it.template next<STOP>(sv, nb, fin_seen, anystop);
      if (k != kIterBlock) {
        wait_fin = k == kIterWaitFin;
        // stop rule: the decisions of iteration n - 3 are needed; fin_probe
        // was loaded at the end of the previous round (its latency hidden)
        if (wait_fin && fin_probe > fin_seen) {  // (loaded with acquire: the stop records)
          fin_seen = fin_probe;
          if (!anystop && a.st.running[0] < a.P) anystop = true;  // written before fin
          progressed = true;
          continue;  // retry the pass start
        }
        break;
      }
      if (lane == 0) q[gen & 3] = nb;
      __syncwarp();
      ++gen;
    }
    // the open partial is complete once no block of its (plane, iteration)
    // is pending: the oldest pending block has another key, or everything
    // generated is done and the iterator moved on (it is then at a pass start)
    if (acc_p >= 0 && (dn < gen ? (q[dn & 3].p != acc_p || q[dn & 3].iter != acc_it)
                                : (it.fresh || it.ended)))
      flush();
    if (cmask != 0 && (dn < gen ? (q[dn & 3].img != c_img || q[dn & 3].iter != c_it)
                                : (it.fresh || it.ended)))
      flush_ci();
    PDZ_P(lap(1);)
    // 3. scan for the next TMA load (block iss): acquire loads of the
    // neighbours' progress, one per lane (the flattened dependency list; an
    // acquire load is a strong load + L1 invalidation, no fence)
    const bool want = !aborted && iss < gen && iss < dn + 2;
    int kpass = 0, need = 0, need_fin = 0;
    int v0 = 0x7fffffff, v1 = 0x7fffffff, vf = 0x7fffffff;
    bool scan = false;
    if (want) {
      const SBlock& b = q[iss & 3];
      kpass = prog_index(b.iter, b.c, C, ci);
      PDZ_P(if (lane == 0 && want_k != kpass) { want_k = kpass; PDZ_TL(a, 2, blockIdx.x, kpass); })
      if (kpass > granted_k) {
        scan = true;
        need = prog_need(kpass, C, ci);  // pass (n-1, c) / the whole sweep n-1
        if (b.iter >= 2) {
          if (ndep <= 64) {
            if (dep0 >= 0) v0 = ld_acquire_gpu(done_ctr + dep0);
            if (dep1 >= 0) v1 = ld_acquire_gpu(done_ctr + dep1);
          } else {
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 3; ++i)
              for (int j = dep.lo[i] + lane; j <= dep.hi[i]; j += 32)
                ok &= ld_acquire_gpu(done_ctr + j) >= need;
            v0 = ok ? 0x7fffffff : -1;
          }
        }
        need_fin = b.iter - kRing;
        if (fin_on && !STOP && need_fin > 0) vf = ld_acquire_gpu(fin_ctr);
      }
    }
    // stop rule: probe fin for the next round while the iterator waits for it
    // (in flight together with the scan loads)
    int fprobe = 0;
    if (wait_fin) fprobe = ld_acquire_gpu(fin_ctr);  // every lane: they all read the records
    PDZ_P(lap(2);)
    // 4. grant: every dependency met -> the TMA (before the publication, whose
    // release fence would otherwise delay it)
    if (want) {
      bool grant = !scan;
      if (scan) {
        PDZ_P(const long long ts = clock64();)
        const bool ok = v0 >= need && v1 >= need && (need_fin <= 0 || vf >= need_fin);
        grant = __all_sync(0xffffffffu, ok);
        __syncwarp();  // every lane's acquire -> lane 0's TMA
        PDZ_P(sp[1] += clock64() - ts;)
      }
      if (grant) {
        const SBlock& b = q[iss & 3];
        granted_k = max(granted_k, kpass);
        if (lane == 0) {
          mb->desc[iss & 1] = b;
          fence_proxy_async_global();  // acquired data -> TMA (async proxy) reads
          issue_block<R, V>(a, b, (iss & 1) ? in1 : in0, &bars[iss & 1]);
          PDZ_P(mb->t_issue[iss & 1] = clock64(); PDZ_TL(a, 1, blockIdx.x, kpass);)
        }
        PDZ_P(t_iss[iss & 3] = clock64();)
        ++iss;
        progressed = true;
      }
    }
    PDZ_P(lap(3);)
    // 5. progress: every pass before the oldest pending block is complete;
    // one release store (the block outputs the done barrier made visible to
    // this warp, and the partials above)
    const int upto =
        dn < gen ? prog_index(q[dn & 3].iter, q[dn & 3].c, C, ci) - 1 : it.completed(sv);
    if (upto > published) {
      PDZ_P(lap(5);)
      if (lane == 0) st_release(done_ctr + blockIdx.x, upto);
      __syncwarp();
      PDZ_P(lap(7);)
      PDZ_P(if (lane == 0) for (int kk = published + 1; kk <= upto; ++kk)
                PDZ_TL(a, 0, blockIdx.x, kk);)
      PDZ_P(sp[2] += 1;)
      published = upto;
      progressed = true;
    }
    if (wait_fin) fin_probe = __shfl_sync(0xffffffffu, fprobe, 0);
    PDZ_P(lap(5);)
    // 6. end of the stream: everything done and published (or, after an
    // abort, every issued block done: the compute warps then leave cleanly)
    if ((it.ended && dn == gen && iss == gen && published >= it.completed(sv)) ||
        (aborted && dn == iss)) {
      if (lane == 0) {
        mb->desc[iss & 1].n = 0;
        mbar_arrive(&bars[iss & 1]);  // completes the phase with no bytes
      }
      PDZ_P(if (a.prof && lane == 0) {
        for (int i = 0; i < 8; ++i) a.prof[(2 * a.pt.G + 2 + blockIdx.x) * 16 + i] = sp[i];
        for (int i = 0; i < 8; ++i) a.prof[(2 * a.pt.G + 2 + blockIdx.x) * 16 + 8 + i] = rp[i];
      })
      return;
    }
    if (progressed) {
      idle = 0;
      PDZ_P(lap(5);)
      continue;
    }
    // nothing moved: the abort flag and the clock cost a global round trip
    // each, so they are looked at every 64th idle round only
    if ((++idle & 63) == 1) {
      if (idle == 1) t0 = global_ns();
    }
    if (!aborted && (idle & 63) == 0 &&
        (ld_relaxed(a.flags + 1) || global_ns() - t0 > kSpinTimeoutNs)) {
      // a dependency never arrived (or another CTA gave up): flag the abort,
      // stop generating, let the issued blocks drain and end the stream --
      // the launch completes, the host raises, the context stays usable
      if (lane == 0) atomicExch(a.flags + 1, 1);
      aborted = true;
      gen = iss;
      continue;
    }
    PDZ_P(sp[3] += 1; lap(5);)
    __nanosleep(wait_fin || want ? 32 : 64);
    PDZ_P(lap(4);)
  }
}

// ------------------------------------------------------------ finaliser --
// The extra CTA (index G) finalises sweeps in order: once every compute CTA
// has published sweep n, it reduces sweep n's r^2 partials in a fixed order
// (bitwise reproducible), applies the stop rule (solver.py:347-358) and
// releases fin = n; it ends when every plane has stopped.
template <int kSThreads>
__device__ void finalizer_cta(const StreamArgs& a) {
  if (!a.st.stop_iter) return;
  __shared__ int s_run;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kSThreads / 32;
  const int G = a.pt.G, C = a.C, P = a.P;
  const Partials& pt = a.pt;
  for (int n = 1; n <= a.iter_last; ++n) {
    const int need = pass_index(n, C - 1, C);
    const long long t0 = global_ns();
    while (true) {
      bool ok = true;
      for (int i = tid; i < G; i += kSThreads) ok &= ld_relaxed(a.done + i) >= need;
      if (__syncthreads_and(ok)) break;
      const bool bad = ld_relaxed(a.flags + 1) != 0 || global_ns() - t0 > kSpinTimeoutNs;
      if (__syncthreads_or(bad)) {
        if (tid == 0) atomicExch(a.flags + 1, 1);
        return;
      }
      __nanosleep(100);
    }
    fence_acq_rel_gpu();
    if (tid == 0) s_run = 0;
    __syncthreads();
    int running = 0;
    if (pt.nbmax <= 32) {  // many planes, few partials each: thread per plane
      for (int p = tid; p < P; p += kSThreads) {
        if (a.st.stop_iter[p] != 0) continue;
        const size_t base = (size_t(n % pt.ring) * P + p) * pt.nbmax;
        const int cnt = partial_count(pt, p);
        double s = 0.0;
        int nf = 0;
#pragma unroll 8
        for (int b = 0; b < cnt; ++b) {
          s += pt.sum[base + b];
          nf |= pt.flag[base + b];
        }
        running += finalize_plane(a.st, P, p, n, a.max_iters, a.rel_tol, s, nf);
      }
    } else {  // few planes, many partials: warp per plane, lane-strided
      for (int p = warp; p < P; p += NW) {
        if (a.st.stop_iter[p] != 0) continue;
        const size_t base = (size_t(n % pt.ring) * P + p) * pt.nbmax;
        const int cnt = partial_count(pt, p);
        double s = 0.0;
        int nf = 0;
#pragma unroll 8
        for (int b = lane; b < cnt; b += 32) {
          s += pt.sum[base + b];
          nf |= pt.flag[base + b];
        }
        s = warp_sum(s);
        nf = __any_sync(0xffffffffu, nf);
        if (lane == 0) running += finalize_plane(a.st, P, p, n, a.max_iters, a.rel_tol, s, nf);
      }
    }
    if (running) atomicAdd(&s_run, running);
    __syncthreads();
    const int run = s_run;
    if (tid == 0) {
      a.st.running[0] = run;
      if (run == 0) a.flags[0] = n;
      fence_acq_rel_gpu();
      st_relaxed(a.fin, n);
    }
    if (run == 0) return;
    __syncthreads();  // s_run is reset next round
  }
}

// ------------------------------------------------------------- kernel --
template <int R, int V, bool EDGE, bool STOP>  // STOP: the relative-change stop rule is armed
__global__ void __maxnreg__(geo_nreg(V))  // the whole register file: one CTA per SM
    stream_kernel(const __grid_constant__ StreamArgs a) {
  using Gm = SGeo<R, V>;
  constexpr int kSCW = Gm::SCW, kComputeThreads = Gm::CT, kSplit = Gm::SPLIT;
  extern __shared__ __align__(128) float smem[];
  float* const in0 = smem;
  float* const in1 = smem + Gm::IN_FLOATS;
  float* const hbuf = smem + 2 * Gm::IN_FLOATS;
  float* const sphi = hbuf + Gm::H_FLOATS;
  float* const slam = sphi + Gm::PL_FLOATS;
  // bars[0..1]: IN double buffer; bars[2]: the block's Phi / lambda tiles;
  // bars[3 + (b & 1)]: block b done (one arrival per compute warp; two
  // barriers, as the compute warps may finish b and b + 1 before the service
  // warp looks, which one barrier's phase parity could not tell apart)
  uint64_t* const bars = reinterpret_cast<uint64_t*>(slam + Gm::PL_FLOATS);
  __shared__ Mailbox mb;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    mbar_init(&bars[3], kSCW);
    mbar_init(&bars[4], kSCW);
    mbar_init(&bars[5], 1);  // IN(0) rows >= kSplit
    mbar_init(&bars[6], 1);  // IN(1) rows >= kSplit
    mbar_fence_init();
  }
  __syncthreads();

  const int H = a.H, W = a.W;
  constexpr int RP = Gm::RP;
  const int WP = W + 2 * kPadC;                          // padded iterate row
  const size_t plane_pad = size_t(H + 2 * R) * WP;       // padded iterate plane
  if (blockIdx.x == a.pt.G) {  // the extra CTA: finaliser
    finalizer_cta<Gm::NT>(a);
    return;
  }
  if (warp == kSCW) {
    const int L0 = int(part_start(a.pt, blockIdx.x));
    const int L1 = int(part_start(a.pt, blockIdx.x + 1));
    service_loop<R, V, STOP>(a, &mb, in0, in1, bars, dep_set(a, L0, L1, R), L0, L1);
    return;
  }

  // thread roles for the vertical pass / update: column pair, kRPW-row group
  const int c = 2 * lane;      // strip-local output column of the pair
  constexpr int kRPW = Gm::RPW;
  const int j0 = warp * kRPW;  // block-local first row
  uint32_t ph_in = 0, ph_pl = 0;  // bit ib: phase of IN(ib)
  int ib = 0;
  int lam_img = -1, lam_yb = -1, lam_x0 = -1;  // rows of the lambda tile held
  // H rows carried from block to block down a strip (large radii only): the H
  // buffer is a ring of ROWS rows, local row i of the block lives in physical
  // row (i + hbase) % ROWS.  A block that continues the previous one (same
  // plane and strip, yb = the previous yb + n) finds its first 2R rows there
  // already -- they are the previous block's rows [n, n + 2R) -- and blurs
  // only its n new rows: (n + 2R) / n = 1.5x less horizontal-pass work at
  // K = 49.  (At R <= 12 the ring's address arithmetic costs more than the
  // saved rows: measured slower on configs 3 and 4.)
  constexpr bool kCarry = R > 12;
  int hbase = 0, prev_p = -1, prev_x0 = 0, prev_end = 0, prev_yb = 0;
  // profile rows (PDZ_PROFILE builds): lane 0 of warps 0 and kSCW-1, clock64
  // [0] total [1] IN wait [2] H pass [3] H barrier [4] Phi/lambda wait
  // [5] V pass [6] report + end barrier [7] blocks
  PDZ_P(long long pf[16] = {0}; const long long tk0 = clock64(); long long tq = tk0;)
  // [8] waits that found the load not yet issued [9] sum of (issue - wait start)
  // for those [10] waits on an issued load [11] sum of (ready - issue) for those

  // Per block b: wait IN(b) (posted by the service warp with its descriptor);
  // blur its n + 2R rows into H; barrier; wait Phi / lambda; vertical pass +
  // divergence + update; report the warp's r^2 and arrive on "done"; barrier
  // (H is reused by the next block).
  while (true) {
    const uint32_t par = (ph_in >> ib) & 1u;
    PDZ_P(const long long tw0 = global_ns();)
    mbar_wait(&bars[ib], par);
    ph_in ^= 1u << ib;
    bool got2 = false;  // second part of the rows (bars[5 + ib], same parity)
    const SBlock cur = mb.desc[ib];
    PDZ_P(if (tid == 0 && cur.n) {
      const int kk = pass_index(cur.iter, cur.c, a.C);
      if (a.prof && kk < 2048 && blockIdx.x < 256) {
        a.prof[131072 + ((size_t(3) * 256 + blockIdx.x) * 2048 + kk)] = tw0;
        PDZ_TL(a, 4, blockIdx.x, kk);
      }
    })
    PDZ_P({
      const long long t = clock64();
      const long long ti = mb.t_issue[ib];
      if (t - tq > 300) {  // actually waited
        if (ti > tq) { pf[8] += 1; pf[9] += ti - tq; } else { pf[10] += 1; pf[11] += t - ti; }
      }
      pf[1] += t - tq; tq = t; pf[7] += 1;
    })
    if (cur.n == 0) break;
    // the block's Phi / lambda tiles (iteration invariant; the buffer is free
    // since the previous block's closing barrier), hidden by the H pass
    if (tid == kComputeThreads - 32) {
      // the C channels of an image share lambda: kept while the block covers
      // the same rows of the same image
      const int img = cur.img;
      const bool lam = img != lam_img || cur.yb != lam_yb || cur.x0 != lam_x0;
      mbar_expect_tx(&bars[2], (lam ? 2u : 1u) * Gm::PL_FLOATS * 4u);
      tma_load_3d(sphi, &a.tm_phi, cur.x0, cur.yb, cur.p, &bars[2]);
      if (lam) {
        tma_load_3d(slam, &a.tm_lam, cur.x0, cur.yb, img, &bars[2]);
        lam_img = img;
        lam_yb = cur.yb;
        lam_x0 = cur.x0;
      }
    }
    float* const in_cur = ib ? in1 : in0;
    float* const h_cur = hbuf;
    const int gx = cur.x0 + c;
    const bool col_ok = gx < W;
    float* __restrict__ uout_all = a.buf[cur.iter % kNBuf];
    double acc_r2 = 0.0;
    float acc_nf = 0.0f;

    const int hn = cur.n + 2 * R;
    int hfirst = 0;  // first H row to blur
    if (kCarry) {
      if (cur.p == prev_p && cur.x0 == prev_x0 && cur.yb == prev_end) {
        hbase += cur.yb - prev_yb;
        if (hbase >= Gm::ROWS) hbase -= Gm::ROWS;
        hfirst = 2 * R;
      } else {
        hbase = 0;
      }
      prev_p = cur.p;
      prev_x0 = cur.x0;
      prev_yb = cur.yb;
      prev_end = cur.yb + cur.n;
    }
    // ---- image borders (np.pad "symmetric", solver.py:235: -1-i <- i,
    // H+i <- H-1-i): nothing mirrored is stored globally and the pads of the
    // global iterates never carry data.  The horizontal pass reads a pad
    // row's mirror source row and patches pad columns in registers; the
    // vertical pass patches its border loads.  When W % 64 != 0 the strips
    // whose staged columns reach past W (the last one or two) reflect their
    // right pad columns in shared memory first.
    const int ylo = cur.yb - R;  // image row of staged row 0
    const bool lbord = cur.x0 == 0;
    const int wl = W - cur.x0;   // image columns of the strip
    const bool rbord = wl == kSTW;
    if (wl != kSTW && wl < kSTW + Gm::RP) {  // CTA-uniform
      const int xr = Gm::RP + wl;  // staged column of image column W
      constexpr int SL = Gm::RP <= 16 ? 16 : 32;  // pad-column slots per row
      static_assert(Gm::RP <= SL, "pad columns per row slot");
      const int k = tid % SL;
      // every staged row is patched, so the second TMA box must have landed
      // first (else it overwrites the reflected columns with the NaN pads)
      mbar_wait(&bars[5 + ib], par);
      got2 = true;
      if (k < Gm::RP && xr + k < Gm::PWD)
        for (int sr = tid / SL; sr < hn; sr += kComputeThreads / SL)
          in_cur[sr * Gm::PITCH + xr + k] = in_cur[sr * Gm::PITCH + xr - 1 - k];
      compute_bar<kComputeThreads>();
    }
    // ---- H rows: horizontal blur of the n + 2R staged rows
    // 8 adjacent outputs per item: 8 independent FMA chains, (8 + 2R)
    // staged values per 8 outputs.
    // Item -> (row i, column group g): 8 consecutive items = 8 consecutive rows
    // of one group (a conflict-free quarter-warp, see SGeo).
    const int hitems = ((hn - hfirst + 7) & ~7) * (kSTW / 8);
    constexpr int OFF = Gm::RP - R;
    constexpr int NQ = (OFF + 2 * R + 8 + 3) / 4;
    // staged values of one item -> registers (false: no such item)
    auto hfetch = [&](int item, float (&v)[4 * NQ], int& i, int& g) -> bool {
      if (item >= hitems) return false;
      i = hfirst + (item >> 6) * 8 + (item & 7);
      g = (item >> 3) & 7;
      if (i >= hn) return false;
      const int y = ylo + i;  // a pad row reads its mirror source row
      const int si = (y < 0 ? -1 - y : (y >= H ? 2 * H - 1 - y : y)) - ylo;
      if (!got2 && si >= kSplit) {
        mbar_wait(&bars[5 + ib], par);
        got2 = true;
      }
      const float* row = in_cur + si * Gm::PITCH + 8 * g;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 t = reinterpret_cast<const float4*>(row)[q];
        v[4 * q] = t.x;
        v[4 * q + 1] = t.y;
        v[4 * q + 2] = t.z;
        v[4 * q + 3] = t.w;
      }
      return true;
    };
    auto hcompute = [&](float (&v)[4 * NQ], int i, int g) {
      // pad columns in registers, compile-time indices per group: left
      // (staged column 8g + t < RP) <- 2 RP - 1 - 8g - t, in the groups that
      // reach it (8g + OFF < RP, i.e. g < R / 8); right (full last strip,
      // staged column 8g + t >= RP + 64) <- 2 RP + 127 - 8g - t.
      if (lbord && 8 * g + OFF < Gm::RP) {
        auto lpatch = [&](auto gtag) {
          constexpr int GG = decltype(gtag)::value;
#pragma unroll
          for (int t = OFF; t < OFF + 2 * R + 8; ++t) {
            const int tp = 2 * Gm::RP - 1 - 16 * GG - t;
            if (8 * GG + t < Gm::RP && tp >= 0 && tp < 4 * NQ) v[t] = v[tp];
          }
        };
        static_assert(R < 24 || Gm::RP <= 24, "left patch covers groups 0..2");
        if (g == 0)
          lpatch(std::integral_constant<int, 0>{});
        else if (g == 1)
          lpatch(std::integral_constant<int, 1>{});
        else
          lpatch(std::integral_constant<int, 2>{});
      }
      if (rbord && g >= 5) {
        auto patch = [&](auto gtag) {
          constexpr int GG = decltype(gtag)::value;
#pragma unroll
          for (int t = OFF; t < OFF + 2 * R + 8; ++t) {
            const int tp = 2 * Gm::RP + 127 - 16 * GG - t;
            if (8 * GG + t >= Gm::RP + kSTW && tp >= 0 && tp < 4 * NQ) v[t] = v[tp];
          }
        };
        if (g == 7)
          patch(std::integral_constant<int, 7>{});
        else if (g == 6)
          patch(std::integral_constant<int, 6>{});
        else
          patch(std::integral_constant<int, 5>{});
      }
      // packed FFMA2 over output pairs (2m, 2m+1): staged value j, broadcast
      // to both lanes (FFMA2 .F32 operand, no register-pair shuffles), meets
      // taps (w[j-2m], w[j-2m-1]).  Per lane the terms arrive in tap order,
      // plus one exact +0*v at the unused end, so each output is bitwise the
      // scalar fma chain.
      float2 o[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) o[m] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 2 * R + 8; ++j) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int t = j - 2 * m;
#ifdef PDZ_KO_COMPUTE  // timing-only build (profiles/r2_knockouts.txt): no arithmetic
          if (t == R) o[m] = make_float2(v[OFF + j], v[OFF + j + 1]);
#else
          if (t >= 0 && t <= 2 * R + 1)
            o[m] = ffma2(make_float2(v[OFF + j], v[OFF + j]), a.wp[t], o[m]);
#endif
        }
      }
      int hr = i;  // physical H row
      if (kCarry) {
        hr += hbase;
        if (hr >= Gm::ROWS) hr -= Gm::ROWS;
      }
      float4* dst = reinterpret_cast<float4*>(h_cur + hr * Gm::HP + 8 * g);
      dst[0] = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
      dst[1] = make_float4(o[2].x, o[2].y, o[3].x, o[3].y);
    };
    for (int item = tid; item < hitems; item += kComputeThreads) {
      float v[4 * NQ];
      int i, g;
      if (hfetch(item, v, i, g)) hcompute(v, i, g);
    }
    if (!got2) mbar_wait(&bars[5 + ib], par);  // the vertical pass reads every row
    PDZ_P({ const long long t = clock64(); pf[2] += t - tq; tq = t; })
    compute_bar<kComputeThreads>();
    PDZ_P({ const long long t = clock64(); pf[3] += t - tq; tq = t; })
    mbar_wait(&bars[2], ph_pl);
    ph_pl ^= 1;
    PDZ_P({ const long long t = clock64(); pf[4] += t - tq; tq = t; })

    // ---- vertical pass (FFMA2 over the column pair), divergence, update
    if (j0 < cur.n) {
      float2 G2[kRPW];
#pragma unroll
      for (int j = 0; j < kRPW; ++j) G2[j] = make_float2(0.f, 0.f);
      const float* hrow = h_cur + c;  // kCarry: walks the ring
      if (kCarry) {
        int hr = j0 + hbase;
        if (hr >= Gm::ROWS) hr -= Gm::ROWS;
        hrow += hr * Gm::HP;
      }
      const float* const hend = h_cur + Gm::ROWS * Gm::HP;
#pragma unroll
      for (int k = 0; k < kRPW + 2 * R; ++k) {
        float2 hv;
        if (kCarry) {
          hv = *reinterpret_cast<const float2*>(hrow);
          hrow += Gm::HP;
          if (hrow >= hend) hrow -= Gm::ROWS * Gm::HP;
        } else {
          hv = *reinterpret_cast<const float2*>(h_cur + (j0 + k) * Gm::HP + c);
        }
#pragma unroll
        for (int j = 0; j < kRPW; ++j) {
          const int t = k - j;
#ifdef PDZ_KO_COMPUTE
          if (t == R) G2[j] = hv;
#else
          if (t >= 0 && t <= 2 * R) G2[j] = ffma2(a.w2[t], hv, G2[j]);
#endif
        }
      }

      // rolling window of u rows (A = y-1, B = y, C = y+1) at columns c-1 .. c+2
      // (staged column RP + c is 8-byte aligned)
      const float* urow = in_cur + (R + j0 - 1) * Gm::PITCH + Gm::RP + c;
      // np.gradient factors (1 at the one-sided ends, else 1/2) times the 1/2
      // of the face average, applied once to the summed raw differences:
      // both are powers of two, so this is bitwise the factored form
      const float2 hx2 = make_float2((gx == 0) ? 0.5f : 0.25f,            // column c
                                     (gx + 1 == W - 1) ? 0.5f : 0.25f);  // column c+1
      const float2 eps2 = make_float2(a.eps, a.eps);
      float2 r2p = make_float2(0.f, 0.f), nfp = make_float2(0.f, 0.f);
      const float2 zero2 = make_float2(0.f, 0.f), tau2 = make_float2(a.tau, a.tau);
      float* __restrict__ uout = uout_all + cur.p * plane_pad + size_t(R) * WP + kPadC;
      const int y0 = cur.yb + j0;  // image row of j = 0
      const int jz0 = -y0, jz1 = H - 1 - y0;  // rows 0 / H-1: one-sided differences
      // warps holding row 0 or H-1 run the loop with the per-row factor test
      // and the row-pad patches; warps of a border strip patch the pad
      // columns of their loads (u[-1] = u[0], u[W] = u[W-1])
      const bool edge_row = (jz0 >= 0 && jz0 < kRPW) || (jz1 >= 0 && jz1 < kRPW);
      const bool edge_col = lbord || wl <= kSTW;
      const bool pcl = gx == 0, pcr = gx + 1 == W - 1;
      const int nrows = col_ok ? min(kRPW, cur.n - j0) : 0;
      // counted rows [jc0, jc1) of the warp's (row-slab blocks count only the
      // rank's own rows, pdz_fixed_point_sweeps_from)
      const int jc0 = a.cnt_lo - y0, jc1 = min(nrows, a.cnt_hi - y0);
      float* orow = uout + ptrdiff_t(y0) * WP + gx;
      const float* pl_row = sphi + j0 * kSTW + c;  // Phi / lambda tiles: row pitch 64
      const float* lm_row = slam + j0 * kSTW + c;
      auto rows = [&](auto erow_tag, auto ecol_tag) {
        constexpr bool EROW = decltype(erow_tag)::value;
        constexpr bool ECOL = decltype(ecol_tag)::value;
        // Column pairs in packed float2: c = (u[c], u[c+1]), e = (u[c-1], u[c+2]).
        auto load = [&](float2& e, float2& cc) {
          e = make_float2(urow[-1], urow[2]);
          cc = *reinterpret_cast<const float2*>(urow);
          if (ECOL) {
            if (pcl) e.x = cc.x;
            if (pcr) e.y = cc.y;
          }
        };
        float2 eA, cA, eB, cB;
        load(eA, cA);
        urow += Gm::PITCH;
        load(eB, cB);
        if (EROW && jz0 == 0) {  // row -1 = row 0
          eA = eB;
          cA = cB;
        }
        float2 xA = make_float2(cA.y - eA.x, eA.y - cA.x);  // raw centred x-differences
        float2 xB = make_float2(cB.y - eB.x, eB.y - cB.x);
        // south face of the row above the first output row: jump and coefficient
        float2 ju = sub2(cB, cA);
        float2 ru = sflux2_coef<EDGE>(ju, mul2(hx2, add2(xA, xB)), eps2);
#pragma unroll
        for (int j = 0; j < kRPW; ++j) {
          urow += Gm::PITCH;
          float2 eC, cC;
          load(eC, cC);
          if (EROW && j == jz1) {  // row H = row H-1
            eC = eB;
            cC = cB;
          }
          const float2 xC = make_float2(cC.y - eC.x, eC.y - cC.x);
          const float hy = (EROW && (j == jz0 || j == jz1)) ? 0.5f : 0.25f;
          const float2 hy2 = make_float2(hy, hy);
          // raw centred vertical differences: d = columns (c, c+1), de = (c-1, c+2)
          const float2 d = sub2(cC, cA);
          const float2 de = sub2(eC, eA);
          const float u0 = cB.x, u1 = cB.y;
          // east faces c-1|c and c+1|c+2 as one pair: the second with its jump
          // negated, (u0 - l, u1 - r) = cB - eB; sflux is odd in the jump, so
          // the pair is (fw, -fe) exactly
          const float2 fwe = sflux2<EDGE>(sub2(cB, eB), mul2(hy2, add2(de, d)), eps2);
          const float fm = sflux<EDGE>(__fsub_rn(u1, u0), __fmul_rn(hy, __fadd_rn(d.x, d.y)), a.eps);  // face c|c+1
          const float2 jd = sub2(cC, cB);
          const float2 rd = sflux2_coef<EDGE>(jd, mul2(hx2, add2(xB, xC)), eps2);
          // div0 = ((fm - fw) + s0) - n0, div1 = ((fe - fm) + s1) - n1, with
          // fe - fm = -(fm + (-fe)) exactly; the south and north fluxes
          // s = jd * rd, n = ju * ru enter as fused multiply-adds
#ifdef PDZ_KO_COMPUTE
          const float2 div = cC;
#else
          const float2 we = make_float2(__fsub_rn(fm, fwe.x), -__fadd_rn(fm, fwe.y));
          const float2 div = ffma2(make_float2(-ju.x, -ju.y), ru, ffma2(jd, rd, we));
#endif
          const float2 cB_old = cB;
          ju = jd;
          ru = rd;
          eA = eB;
          cA = cB;
          xA = xB;
          eB = eC;
          cB = cC;
          xB = xC;
          const float2 phv = *reinterpret_cast<const float2*>(pl_row + j * kSTW);
          const float2 lmv = *reinterpret_cast<const float2*>(lm_row + j * kSTW);
          const float2 rr = add2(ffma2(make_float2(-lmv.x, -lmv.y), G2[j], div), phv);
          const float2 nn = ffma2(tau2, rr, cB_old);
          const float r0 = rr.x, r1 = rr.y, n0 = nn.x, n1 = nn.y;
          if (j < nrows) *reinterpret_cast<float2*>(orow) = make_float2(n0, n1);
          if (j >= jc0 && j < jc1) {
            r2p = ffma2(rr, rr, r2p);
            nfp = ffma2(nn, zero2, nfp);  // NaN iff non-finite update
          }
          orow += WP;
        }
      };
      if (edge_row) {  // warp-uniform (the warp's rows) / CTA-uniform (the strip)
        if (edge_col)
          rows(std::true_type{}, std::true_type{});
        else
          rows(std::true_type{}, std::false_type{});
      } else if (edge_col) {
        rows(std::false_type{}, std::true_type{});
      } else {
        rows(std::false_type{}, std::false_type{});
      }
      acc_r2 += double(r2p.x + r2p.y);
      acc_nf += nfp.x + nfp.y;
    }

    PDZ_P({ const long long t = clock64(); pf[5] += t - tq; tq = t; })
    // ---- report the block: the warp's r^2 and non-finite flag, then done
    {
      const double s = warp_sum(acc_r2);
      const int nfw = __any_sync(0xffffffffu, !(acc_nf == 0.0f));
      if (lane == 0) {
        mb.red[ib][warp] = s;  // block parity == IN buffer index
        mb.nf[ib][warp] = nfw;
        mbar_arrive(&bars[3 + ib]);
      }
    }
    // every read of IN / H / Phi / lambda of the block precedes this barrier
    // (H is rewritten by the next block's horizontal pass)
    compute_bar<kComputeThreads>();
    PDZ_P({ const long long t = clock64(); pf[6] += t - tq; tq = t; })
    ib ^= 1;
  }
  PDZ_P(if (a.prof && lane == 0 && (warp == 0 || warp == kSCW - 1)) {
    pf[0] = clock64() - tk0;
    for (int i = 0; i < 16; ++i) a.prof[(blockIdx.x * 2 + (warp != 0)) * 16 + i] = pf[i];
  })
}

// ------------------------------------------------------------------- host --
using StreamFn = void (*)(const StreamArgs);

template <int R, int V, bool EDGE, bool STOP>
static StreamFn stream_prepared(size_t* smem) {
  static_assert(SGeo<R, V>::FITS, "staging buffers exceed shared memory");
  static_assert(SGeo<R, V>::ROWS > SGeo<R, V>::SPLIT, "two-part row load");
  static std::atomic<uint64_t> done{0};
  *smem = SGeo<R, V>::SMEM;
  if (first_use_on_device(&done))
    cudaFuncSetAttribute(stream_kernel<R, V, EDGE, STOP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(SGeo<R, V>::SMEM));
  return stream_kernel<R, V, EDGE, STOP>;
}

template <int V, bool EDGE, bool STOP>
static StreamFn stream_pick_radius(int R, size_t* smem) {
  switch (R) {  // radii whose staging fits in shared memory (SGeo<R, V>::FITS)
#ifdef PDZ_ONLY_R  // experiment builds (tools/): one radius, a minute to compile
    case PDZ_ONLY_R:
      if (PDZ_ONLY_R > 12 && V != 0) return nullptr;  // like the full table: V = 1 up to R = 12
      return stream_prepared<PDZ_ONLY_R, (PDZ_ONLY_R > 12) ? 0 : V, EDGE, STOP>(smem);
#else
    case 1: return stream_prepared<1, V, EDGE, STOP>(smem);
    case 2: return stream_prepared<2, V, EDGE, STOP>(smem);
    case 3: return stream_prepared<3, V, EDGE, STOP>(smem);
    case 4: return stream_prepared<4, V, EDGE, STOP>(smem);
    case 6: return stream_prepared<6, V, EDGE, STOP>(smem);
    case 9: return stream_prepared<9, V, EDGE, STOP>(smem);
    case 12: return stream_prepared<12, V, EDGE, STOP>(smem);
    case 16: return V == 0 ? stream_prepared<16, 0, EDGE, STOP>(smem) : nullptr;
    case 20: return V == 0 ? stream_prepared<20, 0, EDGE, STOP>(smem) : nullptr;
    case 24: return V == 0 ? stream_prepared<24, 0, EDGE, STOP>(smem) : nullptr;
#endif
    default: return nullptr;
  }
}
// Smallest compiled radius >= R (0: none).  Keep in step with
// stream_pick_radius.
static int stream_compiled_radius(int R) {
#ifdef PDZ_ONLY_R
  return R <= PDZ_ONLY_R ? PDZ_ONLY_R : 0;
#else
  static const int kCompiled[] = {1, 2, 3, 4, 6, 9, 12, 16, 20, 24};
  for (int r : kCompiled)
    if (r >= R) return r;
  return 0;
#endif
}

template <bool EDGE>
static StreamFn stream_pick(int R, int V, bool stop, size_t* smem) {
  if (V == 0)
    return stop ? stream_pick_radius<0, EDGE, true>(R, smem)
                : stream_pick_radius<0, EDGE, false>(R, smem);
  return stop ? stream_pick_radius<1, EDGE, true>(R, smem)
              : stream_pick_radius<1, EDGE, false>(R, smem);
}

}  // namespace pdz
