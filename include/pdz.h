/*
 * pdz.h -- C ABI of the B200 (sm_100a) dehazing library  libpdz.so
 *
 * Drop-in boundary for the hot path of pdehaze 0.1.0 (arXiv 2506.08793).
 * The reference has no FFI: its boundary is the Python API of
 * pdehaze.solver / pdehaze.scattering (re-exported by pdehaze/__init__.py:10-36).
 * Each entry point below replaces one of those functions; the Python package
 * paper_2506_08793_b200 binds them with ctypes and keeps
 * the reference names, signatures and exceptions.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers unless the parameter name ends in
 *     `_host`.  Buffers are caller-owned; the library keeps no pointer after a
 *     call returns and allocates no device memory: scratch comes from a caller
 *     workspace whose size the matching *_workspace_bytes() reports.
 *   - Images are interleaved [H][W][C] (the reference's (H, W, C) C-order
 *     layout, image.py:3-6), float64 or float32 (`image_is_f64`).
 *   - Solver fields are planar float32: plane p of P = batch*C planes at
 *     offset p*H*W, rows of W samples.  The transmission-driven weight
 *     lambda has one plane per image (shared by its C channels).
 *   - Every call is stream-ordered on `stream` (a cudaStream_t) and returns a
 *     status code; pdz_last_error() holds a thread-local message.
 *       PDZ_OK         success
 *       PDZ_EINVAL     bad shape / range / configuration  -> ValueError
 *       PDZ_ENONFINITE solver produced non-finite values  -> FloatingPointError
 *       PDZ_ECUDA      CUDA runtime failure               -> RuntimeError
 *       PDZ_EWORKSPACE workspace too small                -> ValueError
 */
#ifndef PDZ_H_
#define PDZ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDZ_OK 0
#define PDZ_EINVAL 1
#define PDZ_ENONFINITE 2
#define PDZ_ECUDA 3
#define PDZ_EWORKSPACE 4

/* lambda_mode values (solver.py:262, :414-417) */
#define PDZ_LAMBDA_AS_PRINTED 0 /* lambda0 * exp(-beta * (1 - t))      */
#define PDZ_LAMBDA_PROSE 1      /* lambda0 * exp(-beta * t)            */
#define PDZ_LAMBDA_ZERO 2       /* ablation "no-nonlocal": lambda == 0 */
#define PDZ_LAMBDA_CONST 3      /* ablation "no-adaptive": == lambda0  */

/* Geometry + numerics of one relaxed fixed-point solve over P planes.
 * Mirrors the solver fields of SolverConfig (solver.py:78-89). */
typedef struct pdz_solve_params {
  int32_t height;          /* H >= 2 (divergence_term, solver.py:200-201)   */
  int32_t width;           /* W >= 2                                        */
  int32_t planes;          /* P = batch * channels                          */
  int32_t channels;        /* C: planes p share lambda plane p / C          */
  int32_t kernel_size;     /* odd >= 1, Gaussian support (solver.py:80)     */
  int32_t edge_preserving; /* 0: D == 1 (ablation "no-edge", solver.py:420) */
  int32_t max_iters;       /* >= 1                                          */
  int32_t reserved;
  double sigma;            /* Gaussian width (solver.py:79)                 */
  double epsilon;          /* diffusion stabiliser (solver.py:78)           */
  double tau;              /* relaxation step, 0 allowed for one step       */
  double rel_tol;          /* relative residual-change stop (solver.py:88)  */
} pdz_solve_params;

/* ---- library ----------------------------------------------------------- */
int32_t pdz_version(void);
const char* pdz_last_error(void);

/* Normalised 1-D Gaussian factor g/sum(g), g = exp(-d^2/2 sigma^2): the 2-D
 * kernel of gaussian_kernel (solver.py:213-222) is outer(w, w).  Host call. */
int32_t pdz_gaussian_taps(double sigma, int32_t kernel_size, double* taps_host);

/* ---- DCP front end (scattering.py:48-139) ------------------------------ */
/* Scratch needed by pdz_dark_channel / pdz_multiscale_dark_channel. */
size_t pdz_dark_channel_workspace_bytes(int32_t height, int32_t width);

/* dark_channel (scattering.py:48-65): min over channels of I_c / A_c (float64
 * divide, :60), border-truncated (2r+1)^2 window minimum (van Herk/Gil-Werman,
 * :61-64), capped at 1 (:65).  `airlight` is a device float64[C]. */
int32_t pdz_dark_channel(const void* image, int32_t image_is_f64, int32_t height,
                         int32_t width, int32_t channels, const double* airlight,
                         int32_t radius, double* dark, void* workspace,
                         size_t workspace_bytes, void* stream);

/* multiscale_dark_channel (scattering.py:68-85): w0*d0 + w1*d1 + ... in
 * radius order, float64 multiply-then-add (no FMA contraction). */
int32_t pdz_multiscale_dark_channel(const void* image, int32_t image_is_f64, int32_t height,
                                    int32_t width, int32_t channels, const double* airlight,
                                    const int32_t* radii_host, const double* weights_host,
                                    int32_t n_radii, double* dark, void* workspace,
                                    size_t workspace_bytes, void* stream);

/* Number of pixels estimate_atmospheric_light averages: ceil(fraction*H*W)
 * in float64 (scattering.py:102). */
int64_t pdz_airlight_count(int32_t height, int32_t width, double fraction);
size_t pdz_airlight_workspace_bytes(int32_t height, int32_t width, double fraction);

/* estimate_atmospheric_light (scattering.py:88-107): radix-select the count
 * largest dark values, order them by (value desc, flat index asc) exactly like
 * the stable argsort at :105, average I over them with a sequential float64
 * sum in that order (:106-107), clip to [0.05, 1].  Writes airlight (device
 * float64[C]) and, if non-NULL, the ordered flat indices (device int64[count]). */
int32_t pdz_atmospheric_light(const void* image, int32_t image_is_f64, int32_t height,
                              int32_t width, int32_t channels, const double* dark,
                              double fraction, double* airlight, int64_t* picked,
                              void* workspace, size_t workspace_bytes, void* stream);

/* estimate_transmission (scattering.py:110-121): t = 1 - omega * dark. */
int32_t pdz_transmission(const double* dark, int32_t height, int32_t width, double omega,
                         double* transmission, void* stream);

/* The whole front end of dehaze (solver.py:393-419 without the guided
 * refinement) for a BATCH of equal-shaped images stored back to back
 * ([batch][H][W][C]), every stage ONE launch sequence for the batch (the
 * kernels take the image from the grid): (multiscale) dark channel at A = 1,
 * the airlight selection, the dark channel normalised by each image's A, the
 * transmission, and -- when the outputs are non-NULL -- Phi (planar float32
 * [batch * C][H][W]), lambda (float32 [batch][H][W]) and the float64 Phi
 * ([batch][H][W][C]).  radii / weights: the n_radii scales of
 * multiscale_dark_channel (host arrays; one radius with weight 1 = the plain
 * dark channel).  airlight: device float64 [batch][C]; transmission: device
 * float64 [batch][H][W].  Each image's results are bitwise those of the
 * single-image entry points.  Replaces the per-image loop of a caller that
 * maps dehaze over a batch (BASELINE config 3). */
size_t pdz_front_end_batch_workspace_bytes(int32_t batch, int32_t height, int32_t width,
                                           int32_t n_radii, double fraction);
int32_t pdz_front_end_batch(const void* images, int32_t image_is_f64, int32_t batch,
                            int32_t height, int32_t width, int32_t channels,
                            const int32_t* radii_host, const double* weights_host,
                            int32_t n_radii, double fraction, double omega, double t_floor,
                            int32_t lambda_mode, double lambda0, double beta, double* airlight,
                            double* transmission, float* phi, float* lambda_map, double* phi64,
                            void* workspace, size_t workspace_bytes, void* stream);

/* Solver inputs for one image: Phi_c = (I_c - A_c (1 - t)) / max(t, t0)
 * (solver.py:324, scattering.py:138-139) as planar float32 [C][H][W], and
 * lambda(t) (solver.py:244-263 or the ablation overrides :414-417) as float32
 * [H][W].  Also returns the float64 Phi if phi64 != NULL (for "no-pde"). */
int32_t pdz_solver_fields(const void* image, int32_t image_is_f64, int32_t height,
                          int32_t width, int32_t channels, const double* transmission,
                          const double* airlight, double t_floor, int32_t lambda_mode,
                          double lambda0, double beta, float* phi, float* lambda_map,
                          double* phi64, void* stream);

/* adaptive_lambda (solver.py:244-263) in float64 over n samples of t;
 * mode is PDZ_LAMBDA_AS_PRINTED or PDZ_LAMBDA_PROSE. */
int32_t pdz_adaptive_lambda(const double* transmission, int64_t n, int32_t mode,
                            double lambda0, double beta, double* out, void* stream);

/* ---- guided-filter refinement (refine.py:21-80), SURVEY 8(f) next #1 ---- */
size_t pdz_guided_workspace_bytes(int32_t height, int32_t width);
/* box_mean (refine.py:21-40): border-truncated (2r+1)^2 mean from an integral
 * image built with the reference's sequential cumsum order (bit-exact). */
int32_t pdz_box_mean(const double* field, int32_t height, int32_t width, int32_t radius,
                     double* out, void* workspace, size_t workspace_bytes, void* stream);
/* guided_filter (refine.py:43-62). */
int32_t pdz_guided_filter(const double* guide, const double* target, int32_t height,
                          int32_t width, int32_t radius, double reg, double* out,
                          void* workspace, size_t workspace_bytes, void* stream);
/* refine_transmission (refine.py:65-80): luminance guide, clip to [0, 1]. */
int32_t pdz_refine_transmission(const void* image, int32_t image_is_f64, int32_t height,
                                int32_t width, int32_t channels, const double* t_raw,
                                int32_t radius, double reg, double* t_out, void* workspace,
                                size_t workspace_bytes, void* stream);

/* ---- PDE operators (solver.py:152-302) --------------------------------- */
/* diffusion_coefficient (solver.py:152-164): 1 / (g + eps) over n samples. */
int32_t pdz_diffusion_coefficient(const double* grad_magnitude, int64_t n, double epsilon,
                                  double* out, void* stream);

/* tau_stability_bound (solver.py:266-277) per plane at u: 2/(8 max D + max(max
 * lambda, 0)), D edge-preserving.  bound: device float64[P]. */
size_t pdz_tau_bound_workspace_bytes(const pdz_solve_params* params);
int32_t pdz_tau_bound(const pdz_solve_params* params, const float* u, const float* lambda_map,
                      double* bound, void* workspace, size_t workspace_bytes, void* stream);
/* Same bound from a float64 interleaved [H][W][C] iterate (the float64 Phi of
 * pdz_solver_fields) and the float32 lambda plane; planes == channels. */
int32_t pdz_tau_bound_hwc(const pdz_solve_params* params, const double* u_hwc,
                          const float* lambda_map, double* bound, void* workspace,
                          size_t workspace_bytes, void* stream);
int32_t pdz_tau_bound_f64(const pdz_solve_params* params, const double* u,
                          const double* lambda_map, double* bound, void* workspace,
                          size_t workspace_bytes, void* stream);

/* Operator probes for the API functions divergence_term (solver.py:190-210)
 * and gaussian_convolve (:225-241) on P planes (float32 in/out). */
int32_t pdz_divergence(const pdz_solve_params* params, const float* u, float* div,
                       void* stream);
int32_t pdz_divergence_f64(const pdz_solve_params* params, const double* u, double* div,
                           void* stream);
size_t pdz_gaussian_workspace_bytes(const pdz_solve_params* params, int32_t is_f64);
int32_t pdz_gaussian(const pdz_solve_params* params, const float* u, float* out,
                     void* workspace, size_t workspace_bytes, void* stream);
int32_t pdz_gaussian_f64(const pdz_solve_params* params, const double* u, double* out,
                         void* workspace, size_t workspace_bytes, void* stream);

/* ---- relaxed fixed-point sweep (the hot kernel) ------------------------- */
size_t pdz_step_workspace_bytes(const pdz_solve_params* params);

/* One sweep of a ROW SLAB of a larger image (multi-GPU row-slab mode, SURVEY
 * 8(e); paper_2506_08793_b200/parallel.py).  `params->height` rows of u /
 * Phi / lambda are given; array row y is global row y + row_offset of a
 * global_height-row image.  The caller fills the halo rows (neighbour rows,
 * or the symmetric reflection at the global top / bottom); only rows
 * [row_lo, row_hi) are written to u_out and counted.  Per plane,
 * sumsq[p] = sum of r^2 over those rows (the caller all-reduces and takes the
 * square root, solver.py:301), nonfinite[p] as in pdz_fixed_point_step.
 * Workspace: pdz_step_workspace_bytes(params). */
int32_t pdz_fixed_point_step_rows(const pdz_solve_params* params, const float* u, float* u_out,
                                  const float* phi, const float* lambda_map, int32_t row_offset,
                                  int32_t global_height, int32_t row_lo, int32_t row_hi,
                                  double* sumsq, int32_t* nonfinite, void* workspace,
                                  size_t workspace_bytes, void* stream);
/* fixed_point_step (solver.py:280-302) on all P planes at once: one fused
 * sweep u_out = u + tau * r, r = div(D grad u) - lambda G(u) + Phi, with
 * ||r||_2 per plane (device float64[P]) and a per-plane non-finite flag
 * (device int32[P]). */
int32_t pdz_fixed_point_step(const pdz_solve_params* params, const float* u, float* u_out,
                             const float* phi, const float* lambda_map, double* norms,
                             int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                             void* stream);

size_t pdz_solve_workspace_bytes(const pdz_solve_params* params);

/* fixed_point_solve (solver.py:305-359) for all P planes: u0 = Phi, sweeps
 * until each plane's relative residual change <= rel_tol (never at iteration
 * 1) or max_iters.  Planes stop independently, like the reference's
 * per-channel loop.  u_out (device float32 [P][H][W]) receives each plane's
 * final iterate (after its stopping update, unclamped).  Host outputs:
 * norms_host [max_iters][P] (row it-1 = iteration it), iterations_host[P],
 * converged_host[P], failed_host[P] (0, or the iteration whose values went
 * non-finite).  Returns PDZ_ENONFINITE if any plane failed.  Synchronises
 * `stream` before returning. */
int32_t pdz_fixed_point_solve(const pdz_solve_params* params, const float* phi,
                              const float* lambda_map, float* u_out, double* norms_host,
                              int32_t* iterations_host, int32_t* converged_host,
                              int32_t* failed_host, void* workspace, size_t workspace_bytes,
                              void* stream);

/* pdz_fixed_point_solve without the host synchronisation: queues the solve
 * on `stream` and, behind it, copies its outcome into the caller's DEVICE
 * buffer `state` of pdz_solve_state_bytes(params) bytes: double
 * norms[max_iters][P], then int32 iterations[P], converged[P], failed[P],
 * abort[1] (1: a persistent-kernel dependency wait timed out).  The caller
 * queues more work (clamp, result copy) and reads `state` once; dehaze()
 * does.  Returns after queueing. */
size_t pdz_solve_state_bytes(const pdz_solve_params* params);
int32_t pdz_fixed_point_solve_async(const pdz_solve_params* params, const float* phi,
                                    const float* lambda_map, float* u_out, void* state,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* Asynchronous fixed-iteration variant for benchmarking: exactly
 * params->max_iters sweeps (rel_tol ignored) captured in a CUDA graph,
 * norms left on the device in the workspace.  Returns immediately. */
int32_t pdz_fixed_point_sweeps_async(const pdz_solve_params* params, const float* phi,
                                     const float* lambda_map, void* workspace,
                                     size_t workspace_bytes, void* stream);
/* A block of a row-slab solve (multi-GPU row-slab mode with k sweeps per
 * halo exchange; paper_2506_08793_b200/parallel.py): exactly
 * params->max_iters sweeps (rel_tol ignored) of the float32 field u_init
 * (device [P][H][W], H = params->height: the rank's rows plus up to k*R
 * neighbour rows above and below) instead of u0 = Phi, rows 0 and H-1
 * treated as image borders (np.gradient ends, symmetric reflection).  Rows
 * further than n*R from a non-border edge are exact after n sweeps, which is
 * why the caller exchanges k*R rows every k sweeps.  Device outputs: u_out
 * [P][H][W] the final iterate; sumsq[(n-1)*P + p] = sum of r^2 of sweep n
 * over rows [count_lo, count_hi) (the caller all-reduces, takes the square
 * root and applies the stop rule, solver.py:301,347-358); failed[p] = the
 * first sweep whose counted values went non-finite, 0 if none.
 * Asynchronous.  Workspace: pdz_solve_workspace_bytes(params).
 * Replaces the per-sweep loop of fixed_point_solve (solver.py:343-358) for a
 * slab. */
int32_t pdz_fixed_point_sweeps_from(const pdz_solve_params* params, const float* u_init,
                                    const float* phi, const float* lambda_map, int32_t count_lo,
                                    int32_t count_hi, float* u_out, double* sumsq,
                                    int32_t* failed, void* workspace, size_t workspace_bytes,
                                    void* stream);
/* The same block with the iterates RESIDENT in the workspace between calls
 * (the production engine of row-slab mode): nothing is copied into or out of
 * the padded iterate layout per block.  pdz_slab_layout reports where the
 * nbuf iterate buffers live inside a workspace of
 * pdz_solve_workspace_bytes(params): info_host[0..8) <- {nbuf, byte offset
 * of buffer 0, 1, 2 (-1: absent), pad rows, pad columns, padded rows per
 * plane, padded row pitch in floats}; buffer b holds float32
 * [P][H + 2 pad_rows][W + 2 pad_cols] with the field at [pad_rows, pad_cols).
 * The offsets do not depend on params->max_iters, so one workspace sized for
 * the largest block serves every block.  pdz_fixed_point_sweeps_resident
 * runs params->max_iters sweeps starting from buffer `base`: when u_init is
 * non-NULL (the first block) that buffer is first filled from u_init
 * (device [P][H][W]) and every buffer's pads are poisoned; otherwise the
 * buffer's field is taken as it is -- the caller has written the k*R halo
 * rows it received straight into it (the rest is the previous block's
 * result).  The final iterate is left in buffer (base + max_iters) % nbuf.
 * sumsq / failed as in pdz_fixed_point_sweeps_from.  Asynchronous. */
#define PDZ_SLAB_LAYOUT_LEN 8
int32_t pdz_slab_layout(const pdz_solve_params* params, int64_t* info_host, int32_t n);
int32_t pdz_fixed_point_sweeps_resident(const pdz_solve_params* params, const float* u_init,
                                        const float* phi, const float* lambda_map,
                                        int32_t count_lo, int32_t count_hi, int32_t base,
                                        double* sumsq, int32_t* failed, void* workspace,
                                        size_t workspace_bytes, void* stream);
/* Number of kernels pdz_fixed_point_sweeps_async launches for `params`
 * (benchmark bookkeeping). */
int64_t pdz_solve_kernel_launches(const pdz_solve_params* params);
/* Which sweep kernel `params` runs on: 2 = persistent (width % 4 == 0,
 * H >= 2R, W >= 2 ceil4(R), a compiled radius, every CTA co-resident),
 * 1 = tiled fallback, -1 = invalid params. */
int32_t pdz_sweep_kernel_kind(const pdz_solve_params* params);
/* The launch plan `params` gets (host call, no device work), for tests and
 * benchmarks: info_host[0..n) <- {kind (2 persistent / 1 tiled), CTAs (G,
 * or tiles for the tiled kernel), CTAs per strip (kps; 0 = even split of
 * strip-rows, ranges may span strips and images), border bonus, block
 * geometry V, radius R, partial slots per plane, strips per image, output
 * rows per block, threads per CTA, stop rule armed, channel-inner block
 * order (1: (iteration, block, channel), the channel blocks of a position
 * share one lambda tile; 0: (iteration, channel, block))}. */
#define PDZ_PLAN_INFO_LEN 12
int32_t pdz_solve_plan_info(const pdz_solve_params* params, int32_t* info_host, int32_t n);
/* Name of the sweep kernel template `params` launches (e.g.
 * "pdz::stream_kernel<9, 0, 1, 1>"), NUL-terminated into buf_host[n]. */
int32_t pdz_solve_kernel_name(const pdz_solve_params* params, char* buf_host, int32_t n);
/* Device pointer to the plane-p final iterate (dense [H][W]) inside a solve
 * workspace after pdz_fixed_point_sweeps_async (`iterations` is ignored: the
 * solve already copied every plane's final iterate into the dense area). */
const float* pdz_solve_result_plane(const pdz_solve_params* params, const void* workspace,
                                    int32_t plane, int32_t iterations);
/* Measurement hook: enable != 0 makes later solves record a CUDA event pair
 * around the sweep kernel launch(es) on the solve's stream;
 * pdz_last_sweep_kernel_ms() returns the elapsed device time of the last such
 * solve (synchronising on its end event), or -1 if none was recorded. */
void pdz_time_sweep_kernels(int32_t enable);
float pdz_last_sweep_kernel_ms(void);

/* clamp01 + interleave (solver.py:434, image.py:56-61): planar float32 P=C
 * planes -> [H][W][C] float32 or float64 in [0, 1]. */
int32_t pdz_clamp_interleave(const float* planes, int32_t height, int32_t width,
                             int32_t channels, void* out, int32_t out_is_f64, void* stream);

/* ---- image I/O and evaluation ------------------------ */
/* save_image quantisation (image.py:128-145): out[i] = floor(clamp(v, 0, 1) *
 * 255 + 0.5) in float64 for n samples; *flag = 1 if any sample is non-finite
 * (clamp01 rejects those, image.py:56-61).  flag is a device int32. */
int32_t pdz_quantize_u8(const double* image, int64_t n, uint8_t* out, int32_t* flag,
                        void* stream);
/* synthesize_haze (scattering.py:142-158): out = J * t + A * (1 - t) in
 * float64, J interleaved (pixels, channels), t (pixels), A (channels). */
int32_t pdz_synthesize_haze(const double* clean, const double* transmission,
                            const double* airlight, int64_t pixels, int32_t channels,
                            double* out, void* stream);
/* metrics.compare (metrics.py:20-37): sums[0] = sum (x - y)^2, sums[1] =
 * sum |x - y| over n samples (fixed-order fp64 reduction); *flag bit 1 / 2:
 * first / second image has a value outside [0, 1] or non-finite. */
size_t pdz_compare_workspace_bytes(void);
int32_t pdz_compare(const double* x, const double* y, int64_t n, double* sums, int32_t* flag,
                    void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PDZ_H_ */
