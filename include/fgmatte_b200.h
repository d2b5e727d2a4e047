/*
 * fgmatte_b200 -- C ABI of the B200 (sm_100a) multi-level foreground /
 * background estimator (arXiv 2006.14970).
 *
 * Every entry point replaces one reference interface (paths relative to
 * /root/reference/proj):
 *
 *   fgm_params               <- fgmatte::MlParams            include/fgmatte/multilevel.hpp:12-20
 *   fgm_params_validate      <- MlParams::validate           src/multilevel.cpp:10-15
 *   fgm_level_schedule       <- fgmatte::level_schedule      src/multilevel.cpp:17-44
 *   fgm_ml_solve_f32         <- fgmatte::ml_foreground_background  src/multilevel.cpp:141-166
 *   fgm_ml_solve_host_f32/64 <- the same, host buffers (the reference's own
 *                               call shape: planar Image in, planar Image out,
 *                               include/fgmatte/image.hpp:12-26)
 *   fgm_ml_solve_levels_f32  <- the same, plus every level's F/B (debug hook
 *                               for per-level parity; the reference keeps them
 *                               internal, multilevel.cpp:157-164)
 *   fgm_batch_solve_f32      <- N independent ml_foreground_background calls
 *                               (the reference is reentrant)
 *   fgm_resize_f32           <- fgmatte::resize              src/image.cpp:114-133
 *   fgm_ml_solve_hwc         <- _fgmatte.ml_foreground_background with its
 *                               HWC conversion loops     python/bindings.cpp:20-53,146-157
 *   fgm_metrics_f32          <- fgmatte::evaluate_metrics    src/metrics.cpp:75-145
 *
 *   fgm_compose_f32          <- fgmatte::compose             src/image.cpp:39-57
 *                               (python/bindings.cpp:89-95)
 *   fgm_sweep_passes_f32     <- `iterations` x sweep         src/multilevel.cpp:81-121, 162-163
 *
 * Conventions: planar fp32 (plane(c)[y*w + x], as image.hpp:22-26), image = 3
 * planes, alpha = 1 plane, fg/bg = 3 planes each.  "Device" entry points take
 * device pointers and enqueue on `stream` (a cudaStream_t, NULL = legacy
 * default stream) without synchronising; "host" entry points take host
 * pointers and return when the result is in host memory.
 *
 * Status codes: FGM_OK (0); FGM_INVALID_ARGUMENT (1) where the reference
 * throws std::invalid_argument (same message text, fgm_last_error());
 * FGM_RUNTIME_ERROR (2) for CUDA / runtime failures.  There is no CPU
 * fallback: without a usable sm_100 device every solve returns 2.
 * fgm_last_error() is thread-local.  The solve entry points are reentrant
 * (concurrent calls on distinct buffers and streams are safe, from any host
 * thread and for any current device); the fgm_set_* / fgm_debug_* / profiling
 * switches below are process-wide settings (atomic) meant for tests and tools.
 */
#ifndef FGMATTE_B200_H
#define FGMATTE_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define FGM_OK 0
#define FGM_INVALID_ARGUMENT 1
#define FGM_RUNTIME_ERROR 2

/* MlParams (multilevel.hpp:12-20), named as in BASELINE.json's north_star. */
typedef struct fgm_params {
    double regularization;  /* eps_r  (> 0)               multilevel.hpp:14 */
    double gradient_weight; /* omega  (>= 0)              multilevel.hpp:13 */
    int n_small_iterations; /* iters_low  (>= 1)          multilevel.hpp:16 */
    int n_big_iterations;   /* iters_high (>= 1)          multilevel.hpp:17 */
    int small_size;         /* low_res_threshold (>= 1)   multilevel.hpp:15 */
} fgm_params;

/* Reference defaults (multilevel.hpp:13-17): eps_r 5e-3, omega 0.1, 10, 2, 32. */
void fgm_params_default(fgm_params* p);

int fgm_params_validate(const fgm_params* p);

/* Writes up to `cap` levels (coarse -> full); returns the level count, or
 * -FGM_INVALID_ARGUMENT. */
int fgm_level_schedule(int w, int h, const fgm_params* p, int* out_w, int* out_h, int* out_iters, int cap);

/* Device pointers, asynchronous on `stream`. */
int fgm_ml_solve_f32(const float* image, const float* alpha, int w, int h, const fgm_params* p, float* fg, float* bg,
                     void* stream);

/* Host pointers (pageable or pinned); synchronous. */
int fgm_ml_solve_host_f32(const float* image, const float* alpha, int w, int h, const fgm_params* p, float* fg,
                          float* bg);
/* fp64 host planes, as the reference's Image/AlphaMatte hold them; converted to
 * fp32 on the device (K5), results converted back.  Used by the C++ drop-in. */
int fgm_ml_solve_host_f64(const double* image, const double* alpha, int w, int h, const fgm_params* p, double* fg,
                          double* bg);

/* Device pointers.  level_fg[l] / level_bg[l] (3 planes of level l's size, or
 * NULL) receive each level's F/B after its sweeps. */
int fgm_ml_solve_levels_f32(const float* image, const float* alpha, int w, int h, const fgm_params* p, float* fg,
                            float* bg, float* const* level_fg, float* const* level_bg, int n_levels, void* stream);

/* A batch of independent images, device pointers, one stream, batched
 * level-by-level launches. */
int fgm_batch_solve_f32(int n_images, const float* const* images, const float* const* alphas, const int* widths,
                        const int* heights, const fgm_params* p, float* const* fgs, float* const* bgs, void* stream);

/* The same batch from HOST buffers (pinned for full PCIe speed): the images
 * are split into sub-batches whose host->device copies, solve and
 * device->host copies overlap on separate streams (two sub-batches of device
 * workspace in flight).  Synchronous.
 * The reference has no batch entry point; this is the end-to-end path the
 * benchmark's e2e figure is measured through. */
int fgm_batch_solve_host_f32(int n_images, const float* const* images, const float* const* alphas, const int* widths,
                             const int* heights, const fgm_params* p, float* const* fgs, float* const* bgs);

/* Bilinear, centre-aligned, edge-clamped resize of `nplanes` planes with
 * clamp01, identity copy at equal size (image.cpp:71-133).  Device pointers. */
int fgm_resize_f32(const float* src, int sw, int sh, int nplanes, float* dst, int dw, int dh, void* stream);

/* The Python binding's boundary on the device (bindings.cpp:20-53, 146-157):
 * interleaved (h, w, 3) image and (h, w) alpha of float (f64 = 0) or double
 * (f64 = 1), clamped to [0, 1] on the way in as the binding does, solved, and
 * written back interleaved in the same type.  Device pointers, enqueued on
 * `stream` (zero-copy for torch / DLPack callers). */
int fgm_ml_solve_hwc(const void* image_hwc, const void* alpha, int w, int h, int f64, const fgm_params* p,
                     void* fg_hwc, void* bg_hwc, void* stream);

/* Quality metrics of an estimate against ground truth over the translucent
 * region 0 < alpha < 1 (metrics.cpp:75-145): out[0] = SAD, out[1] = MSE (the
 * reference's alpha-weighted sum), out[2] = GRAD (Gaussian-derivative filter,
 * sigma, radius = kernel_radius or ceil(4 sigma)), out[3] = translucent pixel
 * count.  fp64 accumulation, deterministic.  Device pointers in, host `out`;
 * synchronises `stream`.  Errors as GradParams::validate (metrics.cpp:13-16). */
int fgm_metrics_f32(const float* est, const float* gt, const float* alpha, int w, int h, int nch, double sigma,
                    int kernel_radius, double* out, void* stream);

/* Composite: out_c = clamp01(alpha * fg_c + (1 - alpha) * bg_c) for `nch`
 * planes (image.cpp:39-57); the epilogue that puts an estimated foreground on
 * a new background.  Device pointers; out may alias fg or bg. */
int fgm_compose_f32(const float* fg, const float* bg, const float* alpha, int w, int h, int nch, float* out,
                    void* stream);

/* `iterations` exact Gauss-Seidel scanline sweeps of one level, given the
 * level's image/alpha and initial F/B (device pointers; fg_out/bg_out may not
 * alias the inputs).  The GPU counterpart of multilevel.cpp:162-163. */
int fgm_sweep_passes_f32(const float* image, const float* alpha, const float* fg_in, const float* bg_in, int w,
                         int h, int iterations, double regularization, double gradient_weight, float* fg_out,
                         float* bg_out, void* stream);
/* The same with the sweep kernel chosen explicitly (parity tests of both):
 * 0 automatic (as fgm_sweep_passes_f32: one image is a latency-bound launch),
 * 1 the latency kernel (one warp-specialised CTA per 32-row band), 2 the throughput
 * kernel (64-row bands, two rows per lane) that solves batches. */
int fgm_sweep_passes_kernel_f32(const float* image, const float* alpha, const float* fg_in, const float* bg_in,
                                int w, int h, int iterations, double regularization, double gradient_weight,
                                float* fg_out, float* bg_out, int kernel, void* stream);

/* Tuning/debug (process-wide, atomic): 1 computes the I/alpha pyramid of all
 * sub-top levels in one pass over the full-res input (pyramid_kernel), 0
 * (default) with one resample launch per level (image.cpp:114-133 each).  Both
 * are bitwise identical. */
void fgm_set_pyramid_mode(int fused);

/* Failure detection.  A big-level sweep band waits for the band above
 * through a boundary stream; every such wait is bounded (default 2000 ms,
 * fgm_set_spin_timeout_ms).  A wait that times out aborts its launch (every
 * other waiter of the launch gives up at once), increments a per-device fault
 * counter, and makes the synchronous (host-buffer) entry points return
 * FGM_RUNTIME_ERROR.  fgm_device_faults() synchronises the current device and
 * returns the counter (reset != 0 clears it), or -FGM_RUNTIME_ERROR.
 * fgm_debug_fault(1) makes band 0 of every sweep skip publishing its boundary
 * stream (a deliberate hand-over fault for tests); 0 turns it off.  These three
 * settings are process-wide and atomic. */
void fgm_set_spin_timeout_ms(int ms);
int fgm_device_faults(int reset);
void fgm_debug_fault(int code);

/* Debug: 1 surrounds every workspace region of a solve with a guard band and
 * checks it (synchronously) when the solve's work is done; an overrun fails
 * the call with FGM_RUNTIME_ERROR.  0 (default) off. */
void fgm_set_debug_guards(int on);

/* Profiling: when enabled, every kernel launch of the solver is bracketed by
 * CUDA events on its stream; fgm_kernel_stats() synchronises on the recorded
 * events and reports, for kernel class `which` (0 = big-level sweep K3,
 * 1 = I/alpha pyramid K1, 2 = coarse levels K4, 3 = F/B upsample K2), the
 * launch count, the summed device milliseconds and the algorithmic HBM bytes
 * of those launches
 * ("Roofline").  fgm_profile_reset() clears the counters. */
void fgm_profile_enable(int on);
void fgm_profile_reset(void);
int fgm_kernel_stats(int which, long long* launches, double* ms, double* alg_bytes);
/* Diagnostic: the launches of the last drained profile window, in enqueue
 * order: kernel class, start and end (ms from the first launch's start).
 * Writes at most `max` entries; returns the number of launches. */
int fgm_profile_timeline(int max, int* which, double* t0, double* t1);

/* Workspace comes from the library's own stream-ordered memory pool on each
 * device, kept mapped between calls (the process's default pool is not
 * touched).  fgm_release_memory() synchronises the current device and returns
 * that pool's unused memory to the system. */
int fgm_release_memory(void);

const char* fgm_last_error(void);
int fgm_device_count(void);
const char* fgm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FGMATTE_B200_H */
