"""Benchmark of the B200 convtact hot path (driver contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[1], the config the TTC metric is
quoted on): single-scale TTC in float64 over synthetic approaching-plane
videos of 64 frames x 256 x 256 (the reference generator's construction,
seeded, generated on the device).  One step = run_sequence(level=0) over a
batch of V such videos per GPU (frames resident in HBM, V*33.5 MB >> L2):
fused moments kernel + solve, every pair of every video.  value = estimates
(frame pairs) per second over all ranks; scaling is weak (V videos per rank,
no data-path collective -- videos are independent).

Also reported on the same line:
  roofline     the fused moments kernel (ttc_moments_kernel), algorithmic
               bytes = 8*256*256 B per estimate (each frame read once,
               SURVEY.md 8(d)), timed live with CUDA events on its stream;
  e2e          the same metric through the public host API
               (run_sequence_host on pinned numpy frames, H2D of every frame
               and D2H of every estimate inside the timed region);
  cpu_baseline the CPU oracle port (C restatement of the reference) as a
               pinned process pool over videos, all host cores and one core,
               plus the unmodified Python reference (baseline/_ref) on one
               core and on all cores; rank 0, bounded samples;
  secondary    the other BASELINE configs (conv Gpix/s, multiscale TTC).

--impl reference times the CPU reference restatement (oracle/, one pinned
worker process per host core) on the same workload and prints the same line
with impl=reference (plus the unmodified Python reference's numbers).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H = W = 256
NFRAMES = 64
BYTES_PER_EST = 8 * H * W  # each frame read once per estimate
METRIC = "TTC frames/s (estimates/s), single-scale fp64, 64x256x256 approach videos"
UNIT = "estimates/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_ncu_traffic(key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """Polls SM clocks and throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.005):
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        # CT_DIST_BACKEND=gloo exercises the multi-rank plumbing with several
        # ranks on one GPU (host-side barriers only; kernels never wait on peers)
        backend = os.environ.get("CT_DIST_BACKEND", backend)
        if torch.cuda.is_available():
            torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local % torch.cuda.device_count())
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_videos(V: int, seed0: int = 0):
    """V cfg2 videos [V, 64, 256, 256] f64 on the device; video v uses seed seed0+v
    (video 0 is BASELINE config 2 itself: seed 0, FOE centre, t0 = 100)."""
    import torch
    import paper_1612_08825_b200 as ct
    frames = torch.empty((V, NFRAMES, H, W), dtype=torch.float64, device="cuda")
    mags = [100.0 / (100.0 - t) for t in range(NFRAMES)]
    for v0 in range(0, V, 64):
        seeds = list(range(seed0 + v0, seed0 + min(V, v0 + 64)))
        tex = ct.make_textures(W, H, seeds)
        for j in range(len(seeds)):
            ct.zoom_frames(tex[j].contiguous(), (0.5 * W, 0.5 * H), mags, out=frames[v0 + j])
    return frames


# ---------------------------------------------------------------- CPU legs ---
# The CPU baselines run as a pool of single-threaded worker processes, one per
# host core (pinned), over independent cfg2 videos (a
# process pool over videos; the reference is serial by design).  A step = every
# worker processes `per_worker` videos; steps are separated by a barrier and
# timed on the host clock, so a step lasts as long as its slowest worker.
#   kind "port":   oracle.run_sequence (the C restatement of the reference,
#                  oracle/convtact_oracle.c), the tier's reference arm;
#   kind "python": the unmodified reference package (Python + numba) installed
#                  into baseline/_ref (pip --target, git-ignored, travels to the
#                  box), numba JIT warmed in every worker before timing.
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _host_cpus():
    return sorted(os.sched_getaffinity(0))


def _cpu_worker(kind, cpu, per_worker, n_steps, barrier, q):
    try:
        os.sched_setaffinity(0, {cpu})
        if kind == "python":
            sys.path.insert(0, REF_DIR)
            import convtact
            f = convtact.generate(convtact.SynthConfig(width=W, height=H, frames=NFRAMES, t0=100.0, foe=(0.5, 0.5),
                                                       seed=0)).frames
            run = lambda: convtact.run_sequence(f, level=0)  # noqa: E731
        else:
            import oracle
            f = oracle.generate(W, H, NFRAMES, 100.0, (0.5, 0.5), 0, 0.0)
            run = lambda: oracle.run_sequence(f, level=0, nthreads=1)  # noqa: E731
        ttc0 = run()[0]
        ttc0 = ttc0.ttc if kind == "python" else ttc0[5]
        assert abs(ttc0 - 97.315722253398093) <= 1e-9 * 97.3, ttc0  # SURVEY 8(c) anchor: the real computation
        q.put(("ready", cpu))
    except Exception as exc:  # reported by the parent, never hangs it
        q.put(("error", repr(exc)))
        barrier.abort()
        return
    barrier.wait()
    for _ in range(n_steps):
        for _ in range(per_worker):
            run()
        barrier.wait()


def cpu_pool(kind: str, workers: int, per_worker: int, steps: int, warmup: int = 1):
    """Run `warmup + steps` pool steps; returns per-step wall times of the timed steps."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    cpus = _host_cpus()[:workers]
    barrier = ctx.Barrier(len(cpus) + 1, timeout=900)
    q = ctx.Queue()
    env_old = {k: os.environ.get(k) for k in ("NUMBA_CACHE_DIR", "NUMBA_NUM_THREADS", "OMP_NUM_THREADS")}
    os.environ.update(NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/ct_numba_cache"),
                      NUMBA_NUM_THREADS="1", OMP_NUM_THREADS="1")
    procs = [ctx.Process(target=_cpu_worker, args=(kind, c, per_worker, warmup + steps, barrier, q), daemon=True)
             for c in cpus]
    try:
        for p in procs:
            p.start()
        for _ in procs:
            tag, info = q.get(timeout=900)
            if tag == "error":
                raise RuntimeError(f"{kind} worker failed: {info}")
        barrier.wait()  # every worker set up (inputs built, JIT warm, anchor checked)
        times = []
        t = time.perf_counter()
        for k in range(warmup + steps):
            barrier.wait()
            now = time.perf_counter()
            if k >= warmup:
                times.append(now - t)
            t = now
        for p in procs:
            p.join(timeout=60)
        return times, len(cpus)
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
        for k, v in env_old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def cpu_measure(kind: str, workers: int, per_worker: int, steps: int, warmup: int = 1):
    times, n = cpu_pool(kind, workers, per_worker, steps, warmup)
    n_est = n * per_worker * (NFRAMES - 1) * steps
    tot = sum(times)
    what = ("C restatement of the reference (oracle/convtact_oracle.c)" if kind == "port"
            else "unmodified reference package convtact (Python + numba, baseline/_ref)")
    return {"value": n_est / tot, "unit": UNIT, "cores": n, "kind": "port" if kind == "port" else "reference",
            "seconds": tot, "steps": steps, "ms_per_step": tot / steps * 1e3,
            "sample": f"{n} pinned single-threaded worker process(es) x {per_worker} cfg2 video(s) (64x256x256 f64, "
                      f"run_sequence level 0) per step, {steps} timed steps after {warmup} warm-up, {tot:.1f} s; "
                      f"{what}"}


def cpu_baselines(seconds_scale: float = 1.0):
    """Port on all cores (the headline CPU number) and on one core, plus the
    unmodified Python reference on one core and on all cores."""
    ncpu = len(_host_cpus())
    out = cpu_measure("port", ncpu, 16, max(2, int(10 * seconds_scale)))
    out["one_core"] = cpu_measure("port", 1, 16, max(2, int(6 * seconds_scale)))
    py = {}
    if os.path.isdir(os.path.join(REF_DIR, "convtact")):
        try:
            py["one_core"] = cpu_measure("python", 1, 2, max(2, int(5 * seconds_scale)))
            py["all_cores"] = cpu_measure("python", ncpu, 2, max(2, int(5 * seconds_scale)))
        except Exception as exc:
            py["error"] = repr(exc)
    else:
        py["unavailable"] = "baseline/_ref missing (pip install --no-index --no-deps --target baseline/_ref <reference>)"
    out["reference_python"] = py
    return out


def run_reference(args, world, rank):
    """The reference arm: the port (the tier's CPU reference implementation of
    the path) on every host core as a pinned process pool, K timed steps of
    `ref_videos` videos per worker after W warm-up steps; rank 0 only."""
    if rank != 0:
        return
    ncpu = len(_host_cpus())
    m = cpu_measure("port", ncpu, max(1, args.ref_videos), args.steps, args.warmup)
    py = {}
    if os.path.isdir(os.path.join(REF_DIR, "convtact")) and not args.quick:
        try:
            py["one_core"] = cpu_measure("python", 1, 2, 4)
            py["all_cores"] = cpu_measure("python", ncpu, 2, 4)
        except Exception as exc:
            py["error"] = repr(exc)
    line = {
        "impl": "reference", "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2 single-scale TTC fp64, 64x256x256 approach video",
                   "videos_per_worker_per_step": m["sample"], "parallelism": f"cpu x{ncpu} processes (rank 0 only)"},
        "cpu_baseline": {k: m[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "reference_python": py,
        "e2e": {"value": m["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


DP_PER_PX = 711.539e6 * 32 / (256 * 63 * 255 * 255)  # ncu FP64 warp instructions x 32 lanes per grid pixel (21.7)


def fma_peaks():
    """FP32 (FFMA) and FP64 (DFMA) TFLOP/s measured in this run by the FMA-chain
    probe (tools/fp_peak_lib.cu, built by __graft_entry__.build()), plus the
    theoretical peaks at the maximum SM clock NVML reports (148 SMs x 128 / 64 lanes x 2)."""
    import ctypes
    import torch
    out = {}
    so = os.path.join(ROOT, "tools", "libfp_peak.so")
    try:
        lib = ctypes.CDLL(so)
        lib.ct_probe_fma_tflops.restype = ctypes.c_double
        lib.ct_probe_fma_tflops.argtypes = [ctypes.c_int]
        out["fp32"] = float(lib.ct_probe_fma_tflops(0))
        out["fp64"] = float(lib.ct_probe_fma_tflops(1))
        out["kind"] = "measured in this run (FMA-chain probe, tools/fp_peak_lib.cu)"
    except OSError:
        out["fp32"], out["fp64"] = 72.2, 30.2
        out["kind"] = "fallback: round-2 fp_peak.cu measurement on a B200 box (probe library missing)"
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    try:
        import pynvml
        pynvml.nvmlInit()
        # the maximum SM clock (the hardware limit the kernels are rated against;
        # the instantaneous clock after a long run can sit lower)
        mhz = pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device()),
                                               pynvml.NVML_CLOCK_SM)
    except Exception:
        mhz = 1965
    out["theoretical_at_clock"] = {"sm_mhz": mhz, "fp32": sms * 128 * 2 * mhz * 1e6 / 1e12,
                                   "fp64": sms * 64 * 2 * mhz * 1e6 / 1e12}
    return out


def secondary_configs(quick: bool, peaks):
    """Other BASELINE configs, each timed with CUDA events (not the headline)."""
    import torch
    import paper_1612_08825_b200 as ct
    out = {}
    # rated against the theoretical FMA peak at the SM clock (the hardware limit); the
    # FMA-chain rate measured in this run is reported beside it (frac_vs_measured_rate)
    p32, p64 = peaks["theoretical_at_clock"]["fp32"], peaks["theoretical_at_clock"]["fp64"]
    m32, m64 = peaks["fp32"], peaks["fp64"]
    pnote = ("theoretical FMA peak at the maximum SM clock: 148 SMs x %s lanes x 2 flop x %d MHz"
             % ("{128 fp32 | 64 fp64}", peaks["theoretical_at_clock"]["sm_mhz"]))
    st = torch.cuda.current_stream()

    def timeit(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    hbm, _ = load_peaks()
    # cfg1: 2-D FULL fp64 256^2 * 5^2, batch of distinct images (>> L2)
    B = 512 if quick else 2048
    s = torch.rand((B, 256, 256), dtype=torch.float64, device="cuda")
    s[0] = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).random((256, 256)))
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((5, 5))
    o = torch.empty((B, 260, 260), dtype=torch.float64, device="cuda")
    t = timeit(lambda: ct.direct_batch(s, k, out=o), 10)
    bytes_ = B * 8 * (256 * 256 + 260 * 260)
    out["cfg1_conv2d_fp64_5x5"] = {"gpix_s": B * 260 * 260 / t / 1e9, "batch": B, "ms_per_launch": t * 1e3,
                                   "roofline": {"bound": "hbm", "achieved": bytes_ / t / 1e9, "peak": hbm,
                                                "unit": "GB/s", "frac": bytes_ / t / 1e9 / hbm}}
    s1, o1 = s[:1].contiguous(), o[:1].contiguous()
    out["cfg1_conv2d_fp64_5x5"]["single_call_ms"] = timeit(lambda: ct.direct_batch(s1, k, out=o1), 50) * 1e3
    del s, o, s1, o1
    # cfg3: 3-D FULL fp32 128^3 * 7^3
    B3 = 8
    s3 = torch.rand((B3, 128, 128, 128), dtype=torch.float32, device="cuda")
    k3 = np.random.Generator(np.random.PCG64(1)).standard_normal((7, 7, 7)).astype(np.float32)
    o3 = torch.empty((B3, 134, 134, 134), dtype=torch.float32, device="cuda")
    t = timeit(lambda: ct.direct_batch(s3, k3, out=o3), 20)
    fl = B3 * 2.0 * 128 ** 3 * 343
    out["cfg3_conv3d_fp32_7^3"] = {"gpix_s": B3 * 134 ** 3 / t / 1e9, "batch": B3, "ms_per_launch": t * 1e3,
                                   "roofline": {"bound": "fp32", "achieved": fl / t / 1e12, "peak": p32,
                                                "unit": "TFLOP/s", "frac": fl / t / 1e12 / p32, "peak_note": pnote,
                                                "frac_vs_measured_rate": fl / t / 1e12 / m32}}
    s1, o1 = s3[:1].contiguous(), o3[:1].contiguous()
    out["cfg3_conv3d_fp32_7^3"]["single_call_ms"] = timeit(lambda: ct.direct_batch(s1, k3, out=o1), 20) * 1e3
    del s3, o3, s1, o1
    # cfg4: large-kernel 2-D FULL fp32 2048^2 * 31^2
    B4 = 2
    s4 = torch.rand((B4, 2048, 2048), dtype=torch.float32, device="cuda")
    k4 = np.random.Generator(np.random.PCG64(1)).standard_normal((31, 31)).astype(np.float32)
    o4 = torch.empty((B4, 2078, 2078), dtype=torch.float32, device="cuda")
    t = timeit(lambda: ct.direct_batch(s4, k4, out=o4), 20)
    fl = B4 * 2.0 * 2048 ** 2 * 961
    out["cfg4_conv2d_fp32_31x31"] = {"gpix_s": B4 * 2078 ** 2 / t / 1e9, "batch": B4, "ms_per_launch": t * 1e3,
                                     "roofline": {"bound": "fp32", "achieved": fl / t / 1e12, "peak": p32,
                                                  "unit": "TFLOP/s", "frac": fl / t / 1e12 / p32, "peak_note": pnote,
                                                  "frac_vs_measured_rate": fl / t / 1e12 / m32}}
    s1, o1 = s4[:1].contiguous(), o4[:1].contiguous()
    out["cfg4_conv2d_fp32_31x31"]["single_call_ms"] = timeit(lambda: ct.direct_batch(s1, k4, out=o1), 10) * 1e3
    del s4, o4, s1, o1
    # widths without a tiled instantiation (the width-generic strip kernel):
    # 13x13 fp64 (the reference's direct/FFT crossover, test_output.txt:206) on
    # cfg1-sized images, and 33x33 fp32 on cfg4-sized images; FP-bound
    for name, dt, shp, kw, bt, pk, mk in (
            ("w13_conv2d_fp64_13x13", torch.float64, (256, 256), 13, 2 if quick else 512, p64, m64),
            ("w33_conv2d_fp32_33x33", torch.float32, (2048, 2048), 33, 2, p32, m32)):
        sw = torch.rand((bt,) + shp, dtype=dt, device="cuda")
        kwt = np.random.Generator(np.random.PCG64(1)).standard_normal((kw, kw))
        if dt == torch.float32:
            kwt = kwt.astype(np.float32)
        ow = torch.empty((bt, shp[0] + kw - 1, shp[1] + kw - 1), dtype=dt, device="cuda")
        t = timeit(lambda: ct.direct_batch(sw, kwt, out=ow), 20)
        fl = bt * 2.0 * shp[0] * shp[1] * kw * kw
        out[name] = {"gpix_s": ow.numel() / t / 1e9, "batch": bt, "ms_per_launch": t * 1e3,
                     "kernel": ("xcorr_tma2d_strip (runtime width, 8-tap strips, TMA-staged tiles)" if kw * kw <= 400
                                else "xcorr_strip (runtime width, 8-tap strips)"),
                     "roofline": {"bound": "fp64" if dt == torch.float64 else "fp32", "achieved": fl / t / 1e12,
                                  "peak": pk, "unit": "TFLOP/s", "frac": fl / t / 1e12 / pk, "peak_note": pnote,
                                  "frac_vs_measured_rate": fl / t / 1e12 / mk}}
        del sw, ow
    return out


def cfg5_sharded(quick: bool, world: int, rank: int):
    """BASELINE config 5, the full multiscale stream (8 videos x 1024 frames of 1080x1920 fp32,
    max_level=3), frames sharded over the ranks with a one-frame temporal halo:
    rank r owns pairs [p0, p1) of EVERY video and builds only frames p0..p1 of each on its own
    GPU; the step is parallel.run_sequence_sharded (the local multiscale pipeline over all
    eight shards in one call, then one all_gather of the 80-byte estimate rows).  Timed with
    CUDA events between barriers, max over ranks; est/s = every pair of every video / that time
    (strong scaling: the 8-video job is fixed; any N <= 1023 is valid).  quick: 1 video x 64 frames."""
    import torch
    import paper_1612_08825_b200 as ct
    from paper_1612_08825_b200 import parallel
    nv_total, nf = (1, 64) if quick else (8, 1024)
    me = parallel.shard_pairs(nf, world)[rank]
    a, b = me.frames
    fr = torch.empty((nv_total, b - a, 1080, 1920), dtype=torch.float32, device="cuda")
    for v in range(nv_total):
        ct.approach_stream(nf, 1080, 1920, seed=1000 + v, dtype=torch.float32, out=fr[v], frame_range=(a, b))
    st = torch.cuda.current_stream()
    group = None

    def step(**kw):
        if kw.get("level") == 0:  # the level-0 fused kernel alone on this rank's shards
            return ct.run_sequence_batch(fr, **kw) if me.n_pairs else None
        return parallel.run_sequence_sharded(fr, max_level=3, frames_are_local=True, n_frames=nf, group=group)

    def timed(**kw):
        rows = step(**kw)  # warm (workspace allocation)
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record(st)
        for _ in range(reps):
            rows = step(**kw)
        e1.record(st)
        e1.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / reps * 1e-3, world), rows

    t, rows = timed(max_level=3)
    if rank == 0 and not quick:  # the sharded rows are the whole job's, in order
        assert tuple(rows.shape) == (nv_total, nf - 1, 10), rows.shape
    t0, _ = timed(level=0)
    del fr
    torch.cuda.empty_cache()
    hbm, _ = load_peaks()
    n_est = nv_total * (nf - 1)
    bytes_ = n_est * 4 * 1080 * 1920
    ext = [(1080, 1920)]
    for _ in range(3):
        ext.append((ext[-1][0] // 2, ext[-1][1] // 2))
    pipe_bpf = 4 * (ext[0][0] * ext[0][1] + 4 * sum(hh * ww for hh, ww in ext[1:]))
    pipe_bytes = nv_total * nf * pipe_bpf
    return {"est_s": n_est / t, "videos": nv_total, "frames": nf, "n_gpus": world,
            "pairs_per_gpu_per_video": f"{(nf - 1) // world}-{-(-(nf - 1) // world)}", "ms_per_step": t * 1e3,
            "input_bytes": nv_total * nf * 1080 * 1920 * 4,
            "api": "paper_1612_08825_b200.parallel.run_sequence_sharded (frames_are_local, 4-D)",
            "scaling": "strong (the 8-video job split by frame ranges with a one-frame halo; one all_gather of "
                       "the estimate rows)",
            "roofline": {"bound": "hbm", "achieved": bytes_ / t / 1e9 / world, "peak": hbm, "unit": "GB/s per GPU",
                         "frac": bytes_ / t / 1e9 / world / hbm,
                         "note": "whole pipeline (level-0 moments + block means, blurs, levels 1-3, epilogue)"},
            "pipeline_traffic_roofline": {
                "bound": "hbm", "bytes_per_frame": pipe_bpf, "achieved": pipe_bytes / t / 1e9 / world, "peak": hbm,
                "unit": "GB/s per GPU", "frac": pipe_bytes / t / 1e9 / world / hbm,
                "note": "HBM bytes the 4-level pipeline moves as designed: level-0 frames read once; per level "
                        "l >= 1 the block means written and read once, the blurred level written and read once, "
                        "and the next level's block means written: 4*(h0*w0 + 4*sum_l h_l*w_l) B per frame; "
                        "band partials (< 0.5 %) not counted"},
            "level0_fused_kernel": {
                "ms_per_step": t0 * 1e3, "est_s": n_est / t0,
                "roofline": {"bound": "hbm", "achieved": bytes_ / t0 / 1e9 / world, "peak": hbm,
                             "unit": "GB/s per GPU", "frac": bytes_ / t0 / 1e9 / world / hbm,
                             "note": "ttc_moments_ws_kernel<float> + finalize + solve over the level-0 frames"}}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--videos", type=int, default=256, help="cfg2 videos per GPU per step")
    ap.add_argument("--ref-videos", type=int, default=16, help="videos per worker process per step for --impl reference")
    ap.add_argument("--e2e-videos", type=int, default=32)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import paper_1612_08825_b200 as ct

    V = args.videos
    frames = make_videos(V, seed0=rank * V)
    out = torch.empty((V, NFRAMES - 1, 10), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()

    # one step = the single-scale run_sequence pass over V videos, issued as its
    # two C-ABI stages (ct_ttc_moments = fused moments kernel + fixed-order
    # finalize, then ct_ttc_solve) -- exactly what ct_run_sequence does for
    # level 0 -- so the dominant kernel can be bracketed by CUDA events on its
    # own stream inside the timed region (the roofline's kernel time)
    from paper_1612_08825_b200 import _lib
    L = _lib.load()
    sums = torch.empty((V, NFRAMES - 1, 11), dtype=torch.float64, device="cuda")
    nb = L.ct_ttc_moments_workspace_bytes(_lib.CT_F64, V, NFRAMES, H, W)
    ws = _lib.workspace(nb, "cuda")

    def step(ev=None):
        if ev is not None:
            ev[0].record(st)
        _lib.check(L.ct_ttc_moments(_lib.CT_F64, _lib.ptr(frames), V, NFRAMES, H, W, _lib.ptr(sums), _lib.ptr(ws),
                                    nb, st.cuda_stream))
        if ev is not None:
            ev[1].record(st)
        _lib.check(L.ct_ttc_solve(_lib.ptr(sums), V * (NFRAMES - 1), 1e-9, 0, _lib.ptr(out), st.cuda_stream))

    for _ in range(args.warmup):
        step()
    ref_out = ct.run_sequence_batch(frames[:1], level=0)  # the public entry gives the same rows
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(st)
        for k in range(args.steps):
            step(kev[k])
        e1.record(st)
        e1.synchronize()
    t_k = max_over_ranks(sum(a.elapsed_time(b) for a, b in kev) / args.steps * 1e-3, world)
    barrier(world)
    torch.cuda.synchronize()
    dt = max_over_ranks(e0.elapsed_time(e1) * 1e-3, world)
    n_est = world * V * (NFRAMES - 1) * args.steps
    value = n_est / dt
    # launches per step: ttc_moments + moments_finalize + ttc_solve
    launches = 3 * args.steps

    # sanity: the timed output is the real thing (pair 0 of video 0 is cfg2 pair 0)
    if rank == 0:
        ttc0 = float(out[0, 0, 5])
        assert abs(ttc0 - 97.315722253398093) <= 1e-9 * 97.3, ttc0
        assert torch.equal(out[:1].nan_to_num(7.0), ref_out.nan_to_num(7.0))

    # roofline of the dominant kernel: its CUDA-event time inside the timed region (t_k above)
    hbm, peak_kind = load_peaks()
    peaks = fma_peaks()  # FP32 / FP64 FMA rates measured now, outside the timed region
    fp64_lane_peak = peaks["theoretical_at_clock"]["fp64"] * 1e12 / 2  # hardware DFMA lane-ops/s at the clock
    achieved = V * (NFRAMES - 1) * BYTES_PER_EST / t_k / 1e9
    tr = load_ncu_traffic("ttc_moments_ws_kernel<double>/cfg2")
    traffic = None
    if tr and tr.get("videos"):
        traffic = tr["bytes_per_launch"] * V / tr["videos"]  # scaled to this launch's video count
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": traffic, "traffic_unit": "bytes/launch (dram read+write, ncu --set full, profiles/)",
            "algorithmic_bytes_per_launch": V * (NFRAMES - 1) * BYTES_PER_EST, "kernel": "ttc_moments_ws_kernel<double> (+ finalize)", "peak_kind": peak_kind,
            "kernel_ms": t_k * 1e3, "step_ms": dt / args.steps * 1e3,
            "kernel_timing": "CUDA events around ct_ttc_moments in every timed step, on its stream, max over ranks",
            # the kernel is FP64-issue bound (profiles/r01_ttc_moments_ws_f64_cfg2.txt):
            # 711.5 M FP64 warp instructions per 256-video launch = 21.7 per thread-pixel
            # (sweep 20 + 7/16 band-halo row + the per-pair epilogue and warp reduction)
            "fp64_pipe": {"dp_instr_per_grid_px": DP_PER_PX,
                          "achieved_lane_ops_per_s": DP_PER_PX * V * (NFRAMES - 1) * 255 * 255 / t_k,
                          "peak_lane_ops_per_s": fp64_lane_peak,
                          "frac": DP_PER_PX * V * (NFRAMES - 1) * 255 * 255 / t_k / fp64_lane_peak,
                          "peak_note": "theoretical DFMA rate at the maximum SM clock (148 x 64 lanes x MHz)",
                          "frac_vs_measured_rate": DP_PER_PX * V * (NFRAMES - 1) * 255 * 255 / t_k / (peaks["fp64"] * 1e12 / 2)},
            "hbm_read_only_probe_gbs": 7500, "hbm_read_only_note": "TMA stream of the same boxes/ring/grid without compute (tools/tma_stream2.cu); above the copy peak"}

    # end to end through the public host API: pinned frames in, estimates out
    Ve = min(args.e2e_videos, V)
    host = torch.empty((Ve, NFRAMES, H, W), dtype=torch.float64).pin_memory()
    host.copy_(frames[:Ve])
    hnp = host.numpy()
    ct.run_sequence_host(hnp, level=0)
    torch.cuda.synchronize()
    barrier(world)
    e_steps = max(3, args.steps // 4)
    t0 = time.perf_counter()
    for _ in range(e_steps):
        est_h = ct.run_sequence_host(hnp, level=0)
    torch.cuda.synchronize()
    e_dt = max_over_ranks((time.perf_counter() - t0) / e_steps, world)
    if rank == 0:  # rank 0's video 0 is BASELINE config 2 itself
        assert abs(est_h[0, 0, 5] - 97.315722253398093) <= 1e-9 * 97.3
    # the e2e bound: pinned host->device copy bandwidth on this box (the frames dominate the step's bytes)
    hb = host.view(-1)[: 1 << 27]  # 1 GiB of the pinned frames
    db = torch.empty_like(hb, device="cuda")
    db.copy_(hb, non_blocking=True)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(st)
    for _ in range(3):
        db.copy_(hb, non_blocking=True)
    c1.record(st)
    c1.synchronize()
    h2d_gbs = 3 * hb.numel() * 8 / (c0.elapsed_time(c1) * 1e-3) / 1e9
    del db
    e2e_val = world * Ve * (NFRAMES - 1) / e_dt
    e2e = {"value": e2e_val, "unit": UNIT,
           "pcie_roofline": {"bound": "h2d", "h2d_gbs_measured": h2d_gbs,
                             "ceiling_est_s": world * h2d_gbs * 1e9 / (NFRAMES * H * W * 8 / (NFRAMES - 1)),
                             "frac": e2e_val / (world * h2d_gbs * 1e9 / (NFRAMES * H * W * 8 / (NFRAMES - 1))),
                             "note": "pinned 1 GiB cudaMemcpy H2D timed with CUDA events on this box; ceiling = "
                                     "that bandwidth / the frame bytes per estimate"},
           "h2d_bytes_per_step": Ve * NFRAMES * H * W * 8, "d2h_bytes_per_step": Ve * (NFRAMES - 1) * 10 * 8,
           "videos_per_step": Ve, "api": "paper_1612_08825_b200.run_sequence_host (ct_run_sequence_host)"}
    del host
    # the drop-in call a reference user makes (ttc.py:282-305): run_sequence on one
    # pageable float64 numpy video at a time, a list of TtcEstimate back
    Vd = min(8, V)
    vids = [frames[v].cpu().numpy() for v in range(Vd)]
    warm = ct.run_sequence(vids[0], level=0)
    if rank == 0:  # rank 0's video 0 is BASELINE config 2 itself
        assert abs(warm[0].ttc - 97.315722253398093) <= 1e-9 * 97.3, warm[0]
    torch.cuda.synchronize()
    barrier(world)
    d_reps = 3
    t0 = time.perf_counter()
    for _ in range(d_reps):
        for vid in vids:
            ests = ct.run_sequence(vid, level=0)
    d_dt = max_over_ranks((time.perf_counter() - t0) / d_reps, world)
    assert len(ests) == NFRAMES - 1
    e2e["drop_in_run_sequence"] = {
        "value": world * Vd * (NFRAMES - 1) / d_dt, "unit": UNIT, "videos_per_step": Vd,
        "h2d_bytes_per_step": Vd * NFRAMES * H * W * 8, "d2h_bytes_per_step": Vd * (NFRAMES - 1) * 10 * 8,
        "api": "paper_1612_08825_b200.run_sequence(numpy [64,256,256] float64, pageable) -> list[TtcEstimate], "
               "one call per video (host wall clock, max over ranks)"}
    del vids

    secondary = None
    if not args.no_secondary:
        if rank == 0:
            try:
                secondary = secondary_configs(args.quick, peaks)
            except Exception as exc:  # reported, never silently dropped
                secondary = {"error": repr(exc)}
        # config 5 runs on every rank (its videos shard over the GPUs)
        try:
            c5 = cfg5_sharded(args.quick, world, rank)
        except Exception as exc:
            c5 = {"error": repr(exc)}
        if rank == 0:
            secondary["cfg5_multiscale_fp32_1080p"] = c5
    cpu = cpu_baselines(args.cpu_seconds / 10.0) if (rank == 0 and world == 1) else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2 single-scale TTC fp64: 64-frame 256x256 approach videos (t0=100, FOE centre)",
                       "videos_per_gpu_per_step": V, "estimates_per_step": world * V * (NFRAMES - 1),
                       "input_bytes_per_gpu": V * NFRAMES * H * W * 8,
                       "l2": f"inputs larger than L2 ({V * NFRAMES * H * W * 8 / 1e9:.1f} GB per GPU vs 126 MB)",
                       "parallelism": f"dp{world} (independent videos per rank)"},
            "roofline": roof,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "fma_peaks": peaks,
            "clocks": clk.summary(),
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
