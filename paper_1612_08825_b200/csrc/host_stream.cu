// run_sequence from host memory: frames are streamed to the device in chunks
// (a one-frame temporal halo between chunks) on a copy stream while the
// previous chunk is computed on the caller's stream, so the host->device
// transfer overlaps the kernels.  This is the end-to-end path the public
// Python API takes for numpy inputs (ttc.run_sequence, ttc.py:282-305).
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

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

// Pageable host frames (a numpy array from the reference-style call) cannot be
// copied asynchronously: the driver stages them through its own small pinned
// buffer at a fraction of the link rate.  Instead they are staged through a
// reused pinned ring of two slots (per host thread), the host-side copy split
// over worker threads and overlapped with the previous chunk's H2D and
// compute; chunks are smaller (8 MB) so the host copy of
// chunk k+1 runs while chunk k crosses PCIe.
size_t pageable_chunk() {  // CT_PAGEABLE_CHUNK_MB: probing only
  static const size_t mb = getenv("CT_PAGEABLE_CHUNK_MB") ? (size_t)atoi(getenv("CT_PAGEABLE_CHUNK_MB")) : 8;
  return std::max<size_t>(1, mb) << 20;
}

struct PinnedRing {
  void* slot[2] = {nullptr, nullptr};
  size_t bytes = 0;
  ~PinnedRing() {
    for (void* p : slot)
      if (p) cudaFreeHost(p);
  }
};

int pinned_ring(size_t bytes, void* (&out)[2]) {
  static thread_local PinnedRing ring;
  if (ring.bytes < bytes) {
    for (void*& p : ring.slot) {
      if (p) cudaFreeHost(p);
      p = nullptr;
    }
    ring.bytes = 0;
    for (void*& p : ring.slot) CT_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocPortable));
    ring.bytes = bytes;
  }
  out[0] = ring.slot[0];
  out[1] = ring.slot[1];
  return CT_OK;
}

// A small persistent pool of copy threads (created on first use; a thread
// spawn per chunk costs more than the copy of a few MB).  Host memcpy into
// pinned memory measured on the box: 13 GB/s on one thread, 30-45 GB/s on 8-16;
// the drop-in run_sequence(numpy video) call went from 2.6 to 2.0-2.1 ms per
// 64 x 256^2 f64 video with 8 copy threads and 8 MB chunks (16 threads: slower).
class CopyPool {
 public:
  static CopyPool& get() {
    // never destroyed: the detached workers block on its condition variable
    // until process exit, so running its destructor at exit would be unsafe.
    // A forked child has none of the parent's worker threads: it builds its own
    // pool (the parent's copy is leaked in the child).
    static std::mutex make_mu;
    static CopyPool* pool = nullptr;
    static pid_t owner = 0;
    std::lock_guard<std::mutex> lk(make_mu);
    if (pool == nullptr || owner != getpid()) {
      pool = new CopyPool();
      owner = getpid();
    }
    return *pool;
  }
  int threads() const { return (int)workers_.size() + 1; }
  void copy(void* dst, const void* src, size_t bytes) {
    const int n = threads();
    const size_t per = (bytes / n + 4095) & ~size_t(4095);
    if (n == 1 || bytes < (4u << 20)) {
      memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);  // one job at a time (callers on several host threads)
    {
      std::unique_lock<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      per_ = per;
      pending_ = (int)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    memcpy(dst, src, std::min(bytes, per));  // slice 0 on the calling thread
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  CopyPool() {
    const char* e = getenv("CT_COPY_THREADS");
    const int hw = (int)std::thread::hardware_concurrency();
    const int n = e ? std::max(1, atoi(e)) : std::max(1, std::min(8, hw / 2));
    for (int t = 1; t < n; ++t) workers_.emplace_back([this, t] { run(t); });
    for (auto& w : workers_) w.detach();  // live for the process; never joined at exit
  }
  void run(int t) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      char* d = dst_;
      const char* s = src_;
      const size_t a = std::min(bytes_, (size_t)t * per_), b = std::min(bytes_, a + per_);
      lk.unlock();
      if (a < b) memcpy(d + a, s + a, b - a);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, per_ = 0;
};

void parallel_copy(void* dst, const void* src, size_t bytes) { CopyPool::get().copy(dst, src, bytes); }

bool is_pageable(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return attr.type == cudaMemoryTypeUnregistered;
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
  // pageable input: smaller chunks through the pinned ring (device buffers of
  // the full layout are larger than these, so the same workspace serves)
  const bool pageable = is_pageable(frames_host);
  const int64_t K = pageable ? std::min<int64_t>(L.K, std::max<int64_t>(2, (int64_t)(pageable_chunk() / L.frame_bytes)))
                             : L.K;
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t staged[2] = {nullptr, nullptr};
  if (pageable) {
    int rc0 = pinned_ring((size_t)K * L.frame_bytes, stage);
    if (rc0) return rc0;
    for (int i = 0; i < 2; ++i) CT_CUDA(cudaEventCreateWithFlags(&staged[i], cudaEventDisableTiming));
  }
  const int64_t step = K - 1;
  const int64_t per_video = (n_frames - 1 + step - 1) / step;
  const int64_t n_items = n_videos * per_video;
  auto item = [&](int64_t i) {
    Item it;
    it.v = i / per_video;
    it.f0 = (i % per_video) * step;
    it.len = std::min<int64_t>(K, n_frames - it.f0);
    return it;
  };
  const char* hbase = reinterpret_cast<const char*>(frames_host);
  auto h2d = [&](int64_t i) -> int {
    const Item it = item(i);
    const char* src = hbase + ((size_t)it.v * n_frames + it.f0) * L.frame_bytes;
    const size_t bytes = (size_t)it.len * L.frame_bytes;
    if (pageable) {  // host copy into the pinned slot the H2D of item i - 2 has finished reading
      if (i >= 2) CT_CUDA(cudaEventSynchronize(staged[i & 1]));
      parallel_copy(stage[i & 1], src, bytes);
      src = static_cast<const char*>(stage[i & 1]);
    }
    CT_CUDA(cudaMemcpyAsync(buf[i & 1], src, bytes, cudaMemcpyHostToDevice, cs));
    if (pageable) CT_CUDA(cudaEventRecord(staged[i & 1], cs));
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
    if (staged[i]) {
      cudaEventSynchronize(staged[i]);  // the ring is reused by the next call on this thread
      cudaEventDestroy(staged[i]);
    }
  }
  cudaEventDestroy(start);
  cudaStreamDestroy(cs);  // resources are released once its pending work completes
  return rc;
}
