// run_sequence from host memory: frames are streamed to the device in chunks
// (a one-frame temporal halo between chunks) on a copy stream while the
// previous chunk is computed on the caller's stream, so the host->device
// transfer overlaps the kernels.  This is the end-to-end path the public
// Python API takes for numpy inputs (ttc.run_sequence, ttc.py:282-305).
#include <algorithm>

#include "common.cuh"

namespace ct {
namespace {

constexpr size_t kChunkBudget = 512ull << 20;  // device bytes per frame chunk buffer

int64_t chunk_frames(int dtype, int64_t n_frames, int64_t h, int64_t w) {
  const size_t fb = (size_t)h * w * (dtype == CT_F64 ? 8 : 4);
  int64_t k = (int64_t)std::max<size_t>(2, kChunkBudget / std::max<size_t>(fb, 1));
  return std::min<int64_t>(k, n_frames);
}

inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct HostLayout {
  int64_t K;
  size_t frame_bytes, buf_bytes, est_bytes, seq_ws;
  size_t total;
};

HostLayout layout(int dtype, int64_t n_frames, int64_t h, int64_t w, int level, int max_level) {
  HostLayout L{};
  L.K = chunk_frames(dtype, n_frames, h, w);
  L.frame_bytes = (size_t)h * w * (dtype == CT_F64 ? 8 : 4);
  L.buf_bytes = al(L.frame_bytes * L.K);
  L.est_bytes = al((size_t)(L.K - 1) * CT_NEST * sizeof(double));
  L.seq_ws = al(ct_run_sequence_workspace_bytes(dtype, 1, L.K, h, w, level, max_level));
  L.total = 2 * L.buf_bytes + 2 * L.est_bytes + L.seq_ws;
  return L;
}

}  // namespace
}  // namespace ct

using namespace ct;

extern "C" size_t ct_run_sequence_host_workspace_bytes(int dtype, int64_t n_videos, int64_t n_frames, int64_t h,
                                                       int64_t w, int level, int max_level) {
  (void)n_videos;
  if (n_frames < 2 || h < 1 || w < 1) return 0;
  return layout(dtype, n_frames, h, w, level, max_level).total;
}

extern "C" int ct_run_sequence_host(int dtype, const void* frames_host, int64_t n_videos, int64_t n_frames, int64_t h,
                                    int64_t w, int level, int max_level, double c_min, double* est_host,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  clear_error();
  CT_REQUIRE(dtype == CT_F64 || dtype == CT_F32, "dtype must be CT_F64 or CT_F32");
  CT_REQUIRE(n_frames >= 2, "need at least two frames");
  CT_REQUIRE(n_videos >= 0, "bad n_videos");
  const HostLayout L = layout(dtype, n_frames, h, w, level, max_level);
  CT_REQUIRE(workspace && workspace_bytes >= L.total, "workspace too small (%zu < %zu)", workspace_bytes, L.total);
  if (n_videos == 0) return CT_OK;
  cudaStream_t st = as_stream(stream);
  char* ws = reinterpret_cast<char*>(workspace);
  char* buf[2] = {ws, ws + L.buf_bytes};
  double* est_dev[2] = {reinterpret_cast<double*>(ws + 2 * L.buf_bytes),
                        reinterpret_cast<double*>(ws + 2 * L.buf_bytes + L.est_bytes)};
  void* seq_ws = ws + 2 * L.buf_bytes + 2 * L.est_bytes;

  cudaStream_t cs;
  CT_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaEvent_t copied[2], computed[2], start;
  for (int i = 0; i < 2; ++i) {
    CT_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    CT_CUDA(cudaEventCreateWithFlags(&computed[i], cudaEventDisableTiming));
  }
  CT_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  CT_CUDA(cudaEventRecord(start, st));
  CT_CUDA(cudaStreamWaitEvent(cs, start, 0));  // copies are ordered after prior work on `stream`

  // work items: (video, first frame, frames in chunk)
  struct Item {
    int64_t v, f0, len;
  };
  const int64_t step = L.K - 1;
  const int64_t per_video = (n_frames - 1 + step - 1) / step;
  const int64_t n_items = n_videos * per_video;
  auto item = [&](int64_t i) {
    Item it;
    it.v = i / per_video;
    it.f0 = (i % per_video) * step;
    it.len = std::min<int64_t>(L.K, n_frames - it.f0);
    return it;
  };
  const char* hbase = reinterpret_cast<const char*>(frames_host);
  auto h2d = [&](int64_t i) -> int {
    const Item it = item(i);
    const char* src = hbase + ((size_t)it.v * n_frames + it.f0) * L.frame_bytes;
    CT_CUDA(cudaMemcpyAsync(buf[i & 1], src, (size_t)it.len * L.frame_bytes, cudaMemcpyHostToDevice, cs));
    CT_CUDA(cudaEventRecord(copied[i & 1], cs));
    return CT_OK;
  };
  int rc = h2d(0);
  for (int64_t i = 0; i < n_items && rc == CT_OK; ++i) {
    const Item it = item(i);
    if (i + 1 < n_items) {
      if (i >= 1) CT_CUDA(cudaStreamWaitEvent(cs, computed[(i + 1) & 1], 0));  // buffer of item i-1 free
      rc = h2d(i + 1);
      if (rc) break;
    }
    CT_CUDA(cudaStreamWaitEvent(st, copied[i & 1], 0));
    rc = ct_run_sequence(dtype, buf[i & 1], 1, it.len, h, w, level, max_level, c_min, est_dev[i & 1], seq_ws,
                         L.seq_ws, stream);
    if (rc) break;
    double* dst = est_host + ((size_t)it.v * (n_frames - 1) + it.f0) * CT_NEST;
    CT_CUDA(cudaMemcpyAsync(dst, est_dev[i & 1], (size_t)(it.len - 1) * CT_NEST * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
    CT_CUDA(cudaEventRecord(computed[i & 1], st));
  }
  // join the copy stream back into the caller's stream, then release helpers
  cudaEvent_t done;
  CT_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  CT_CUDA(cudaEventRecord(done, cs));
  CT_CUDA(cudaStreamWaitEvent(st, done, 0));
  cudaEventDestroy(done);
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(computed[i]);
  }
  cudaEventDestroy(start);
  cudaStreamDestroy(cs);  // resources are released once its pending work completes
  return rc;
}
