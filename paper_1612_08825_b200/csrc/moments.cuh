// Internal interface of the fused moments kernel (moments.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ct {

// Workspace bytes for `n_videos` stacks of `n_frames` h x w frames.
size_t moments_workspace(int dtype, int64_t n_videos, int n_frames, int h, int w);

// sums[v][pair][11] for every consecutive pair (see ct_ttc_moments).  With
// `dec` non-null the kernel also writes the 2x2 block means of every frame
// ([n_videos][n_frames][h/2][w/2]), the first half of the next pyramid level.
int moments_launch(int dtype, const void* frames, int64_t n_videos, int n_frames, int h, int w, int border,
                   double* sums, void* ws, size_t ws_size, cudaStream_t st, void* dec = nullptr);

// Band partials ([n_videos][n_pairs][units][10], rhs negated) of several
// pyramid levels of the same videos, one kernel launch when possible (no
// finalize).  Level l's frames are lv[l].frames (h x w), its partials go to
// lv[l].partials (moments_workspace bytes), and with lv[l].dec non-null its
// 2x2 block means are written as well.
struct MomentLevel {
  const void* frames;
  int h, w;
  double* partials;
  void* dec;
  int chunk = 0;  // pairs per CTA (0: the automatic plan; >0 e.g. one chunk per video so no frame is read twice)
};
constexpr int kMomentLevelsPerLaunch = 8;  // n_levels <= this
int moments_levels_launch(int dtype, const MomentLevel* lv, int n_levels, int64_t n_videos, int n_frames, int border,
                          cudaStream_t st);

// Band partials per pair (the `units` of a moments launch for these extents).
int moments_units(int dtype, int64_t n_videos, int n_frames, int h, int w);

// sums[i] = fixed-order sum over `units` 10-value partials, plus count.
int partials_finalize(const double* partials, int64_t n_sys, int units, double count, double* sums,
                      cudaStream_t st);

}  // namespace ct
