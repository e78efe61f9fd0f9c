/*
 * convtact_b200.h -- C ABI of the B200-native convtact hot path.
 *
 * Every entry point is extern "C", takes plain pointers and sizes, runs
 * stream-ordered on the CUDA stream passed as `stream` (a cudaStream_t, or
 * NULL for the legacy default stream), and returns a status code:
 *   CT_OK (0)       success
 *   CT_EINVAL (1)   invalid arguments; the reference raises ValueError here
 *   CT_ECUDA (2)    a CUDA runtime error (launch/config); see ct_last_error()
 *   CT_EUNSUPPORTED (3) a shape/dtype this build does not handle
 * The library never allocates device memory: callers own every input,
 * output and workspace buffer (sizes via the *_workspace_bytes queries), and
 * it never calls back into the caller.  All data pointers are DEVICE
 * pointers unless the name says `host`.
 *
 * Reference interface each entry replaces (paths under /root/reference/pkg/src/convtact):
 *   ct_xcorr_nd / ct_direct   conv._direct + _loops.xcorr_{valid,zpad}_{1,2,3}d +
 *                             xcorr_valid_nd  (conv.py:105-158, _loops.py:27-208)
 *   ct_ttc_derivatives        ttc.derivatives_3d        (ttc.py:82-91)
 *   ct_radial_gradient        ttc.radial_gradient       (ttc.py:94-99)
 *   ct_normal_system          ttc.build_normal_system   (ttc.py:102-120)
 *   ct_ttc_moments            derivatives_3d + radial_gradient + build_normal_system
 *                             fused, over every consecutive pair (ttc.py:82-120, 282-305)
 *   ct_ttc_solve              ttc._ldlt_solve + solve_ttc + _estimate_at FOE scaling
 *                             (ttc.py:123-184, 215-225)
 *   ct_pyramid_down           ttc.downsample            (ttc.py:187-204)
 *   ct_ttc_multiscale_select  estimate_multiscale greedy level walk (ttc.py:248-279)
 *   ct_run_sequence           ttc.run_sequence / estimate_fixed / estimate_multiscale
 *                             (ttc.py:228-305) for a stack of frames
 *   ct_zoom_frames            synth.zoom_frame / _axis_taps (synth.py:88-126), used to
 *                             generate synthetic inputs on the device
 *   ct_gradient               kernels.gradient (kernels.py:63-72), fused SAME/REPLICATE
 *                             pair correlation + hypot/atan2
 *   ct_decode_samples         tensor.image_read_pgm raster decode (tensor.py:104-136) on the
 *                             device, for PGM frame ingestion
 */
#ifndef CONVTACT_B200_H
#define CONVTACT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { CT_OK = 0, CT_EINVAL = 1, CT_ECUDA = 2, CT_EUNSUPPORTED = 3 };
enum { CT_F64 = 0, CT_F32 = 1 };                     /* element type            */
enum { CT_FULL = 0, CT_SAME = 1, CT_VALID = 2 };     /* conv.ConvShape          */
enum { CT_ZERO = 0, CT_REPLICATE = 1 };              /* conv.BoundaryPolicy     */
enum { CT_MAXDIM = 8 };                              /* ranks handled on device */
enum { CT_NSUMS = 11 };  /* m00 m01 m02 m11 m12 m22, rhs0 rhs1 rhs2 (negated), et2, count */
enum { CT_NEST = 10 };   /* a b c x0 y0 ttc residual misfit level degenerate           */

/* Message of the last failing call on this host thread ("" if none). */
const char* ct_last_error(void);
/* Library version string. */
const char* ct_version(void);

/* Generic zero/replicate-extended correlation of `batch` signals with one
 * kernel: out[b][o] = sum_j k[j] * s_ext[b][o - pad_left + j], taps in
 * row-major order.  s_ext is s extended by zeros (CT_ZERO) or by clamping to
 * the nearest edge sample (CT_REPLICATE).  `k` is the kernel in device
 * memory; `k_host` may be NULL or a host copy of the same taps, which lets the
 * register-tiled kernels take the taps through the parameter bank without a
 * device->host copy (and without synchronising the stream).  Ranks 1-3 run on
 * register-tiled kernels for every kernel width (compile-time widths 1-9, 11,
 * 15, 31; any other width on the runtime-width strip kernel); ranks >= 4 on
 * the one-thread-per-output kernel.  float64 results are bit-identical to the
 * reference loops. */
int ct_xcorr_nd(int dtype, int ndim, const void* s, const int64_t* s_shape, int64_t batch,
                const void* k, const void* k_host, const int64_t* k_shape,
                const int64_t* pad_left, const int64_t* out_shape, int boundary, void* out,
                void* stream);

/* conv_direct (flip=1) / xcorr_direct (flip=0) with the reference's shape and
 * boundary semantics (FULL m+n-1, SAME m anchored at ceil((n-1)/2), VALID
 * m-n+1).  `k` is the kernel as the caller passed it; flip reflects it. */
int ct_direct(int dtype, int ndim, const void* s, const int64_t* s_shape, int64_t batch,
              const void* k, const void* k_host, const int64_t* k_shape, int shape,
              int boundary, int flip, void* out, void* stream);

/* Ex, Ey, Et on the (h-1) x (w-1) half-pixel grid of one frame pair. */
int ct_ttc_derivatives(int dtype, const void* first, const void* second, int64_t h, int64_t w,
                       void* ex, void* ey, void* et, void* stream);

/* G = xc*Ex + yc*Ey with centred coordinates on a gh x gw grid. */
int ct_radial_gradient(int dtype, const void* ex, const void* ey, int64_t gh, int64_t gw,
                       void* g, void* stream);

/* The 11 normal-system sums over the window [border:-border, border:-border]. */
size_t ct_normal_system_workspace_bytes(int64_t gh, int64_t gw);
int ct_normal_system(int dtype, const void* ex, const void* ey, const void* g, const void* et,
                     int64_t gh, int64_t gw, int64_t border, double* sums, void* workspace,
                     size_t workspace_bytes, void* stream);

/* Fused K5: for each of `n_videos` stacks of `n_frames` frames (h x w, row
 * major, contiguous), the 11 sums of every consecutive pair, written to
 * sums[v][i][11].  Frames are read once; no derivative field touches HBM. */
size_t ct_ttc_moments_workspace_bytes(int dtype, int64_t n_videos, int64_t n_frames, int64_t h,
                                      int64_t w);
int ct_ttc_moments(int dtype, const void* frames, int64_t n_videos, int64_t n_frames, int64_t h,
                   int64_t w, double* sums, void* workspace, size_t workspace_bytes, void* stream);

/* K7: solve `count` normal systems (rows of 11 sums) into estimate rows of 10
 * doubles; `level` scales the FOE by 2^level and is written to the level field. */
int ct_ttc_solve(const double* sums, int64_t count, double c_min, int level, double* est,
                 void* stream);

/* K6: ttc.downsample of `n_images` images (h x w) into (h/2) x (w/2). */
int ct_pyramid_down(int dtype, const void* in, int64_t n_images, int64_t h, int64_t w, void* out,
                    void* stream);

/* Greedy level walk of estimate_multiscale over precomputed per-level
 * estimates est_levels[count][n_levels][10] -> best[count][10]. */
int ct_ttc_multiscale_select(const double* est_levels, int64_t count, int n_levels, double* best,
                             void* stream);

/* Multiscale normal-system sums (SURVEY.md 8(b) ct_ttc_pyramid_moments): for
 * pyramid levels l = 0..levels-1 (level l = l-fold ttc.downsample of the
 * frames, ttc.py:187-204) the 11 sums of every consecutive pair, as
 * ttc_moments writes them, laid out [levels][n_videos][n_frames-1][11].  These
 * are the systems estimate_multiscale solves per level (ttc.py:248-279).
 * Errors: fewer than two frames, levels outside [1, 30], or a level smaller
 * than 4 pixels (the reference's _level_extents guard, ttc.py:235-241). */
size_t ct_ttc_pyramid_moments_workspace_bytes(int dtype, int64_t n_videos, int64_t n_frames, int64_t h,
                                              int64_t w, int levels);
int ct_ttc_pyramid_moments(int dtype, const void* frames, int64_t n_videos, int64_t n_frames, int64_t h,
                           int64_t w, int levels, double* sums, void* workspace, size_t workspace_bytes,
                           void* stream);

/* run_sequence for `n_videos` independent stacks [n_videos][n_frames][h][w]:
 * max_level < 0 -> estimate_fixed(level), else estimate_multiscale(max_level).
 * Writes est[n_videos][n_frames-1][10]; a `None` multiscale result has level -1. */
size_t ct_run_sequence_workspace_bytes(int dtype, int64_t n_videos, int64_t n_frames, int64_t h,
                                       int64_t w, int level, int max_level);
int ct_run_sequence(int dtype, const void* frames, int64_t n_videos, int64_t n_frames, int64_t h,
                    int64_t w, int level, int max_level, double c_min, double* est,
                    void* workspace, size_t workspace_bytes, void* stream);

/* run_sequence from HOST frames (f64 or f32 host buffer), streaming them to
 * the device in chunks that overlap the copy with compute; est_host receives
 * [n_videos][n_frames-1][10].  Device workspace via the query below.
 * Page-locked frames are copied directly; pageable frames (a plain numpy
 * array) are staged through a page-locked ring of two 8 MB slots owned by the
 * library (one per calling host thread, reused across calls), filled by a
 * small pool of host copy threads while the previous chunk crosses PCIe. */
size_t ct_run_sequence_host_workspace_bytes(int dtype, int64_t n_videos, int64_t n_frames,
                                            int64_t h, int64_t w, int level, int max_level);
int ct_run_sequence_host(int dtype, const void* frames_host, int64_t n_videos, int64_t n_frames,
                         int64_t h, int64_t w, int level, int max_level, double c_min,
                         double* est_host, void* workspace, size_t workspace_bytes, void* stream);

/* Synthetic generator: frames[t] = zoom_frame(texture, foe_px, mags[t]) for
 * t < n, written as f64 (dtype CT_F64) or rounded to f32 (CT_F32).  The
 * texture is f64 [h][w] on the device; mags is a host array. */
int ct_zoom_frames(int dtype, const double* texture, int64_t h, int64_t w, double foe_x,
                   double foe_y, const double* mags_host, int64_t n, void* frames, void* workspace,
                   size_t workspace_bytes, void* stream);
size_t ct_zoom_frames_workspace_bytes(int64_t h, int64_t w);

/* Gradient fields of `n_images` h x w images with a named kernel pair (host
 * taps kx, ky, kh x kw <= 64): ex, ey = SAME/REPLICATE correlations, mag =
 * hypot(ex, ey), dir = atan2(ey, ex); outputs are h x w per image. */
int ct_gradient(int dtype, const void* img, int64_t n_images, int64_t h, int64_t w, const double* kx_host,
                const double* ky_host, int64_t kh, int64_t kw, void* ex, void* ey, void* mag, void* dir,
                void* stream);

/* out[i] = float64(sample_i) / maxval for n raw PGM samples on the device:
 * bytes_per_sample 1 (maxval 255) or 2 (big-endian, maxval 65535). */
int ct_decode_samples(int bytes_per_sample, const void* raw, int64_t n, double maxval, double* out,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CONVTACT_B200_H */
