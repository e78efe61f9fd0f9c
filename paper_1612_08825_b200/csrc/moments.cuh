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

// sums[i] = fixed-order sum over `units` 10-value partials, plus count.
int partials_finalize(const double* partials, int64_t n_sys, int units, double count, double* sums,
                      cudaStream_t st);

}  // namespace ct
