"""Multi-process (world_size 2 and 3, gloo on CPU) tests of the sharding host
logic: temporal pair shards with a one-frame halo + ordered all_gather, and
row-slab halo exchange for one large image.  The compute step is the CPU
oracle here (no GPU in this container); on GPUs parallel.py uses the CUDA
path with NCCL.  Results must equal the unsharded computation bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1612_08825_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _seq_compute(frames, level, max_level, c_min):
    return torch.from_numpy(O.run_sequence(np.asarray(frames), level=level, max_level=max_level, c_min=c_min,
                                           nthreads=1))


def _worker_seq(rank, world, port, frames, level, max_level, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = parallel.run_sequence_sharded(frames, level=level, max_level=max_level, compute=_seq_compute)
        # local-shard form: each rank holds only frames p0..p1
        me = parallel.shard_pairs(frames.shape[0], world)[rank]
        out2 = parallel.run_sequence_sharded(frames[me.frames[0]:me.frames[1]], level=level, max_level=max_level,
                                             compute=_seq_compute, frames_are_local=True, n_frames=frames.shape[0])
        q.put((rank, out.numpy(), out2.numpy()))
    finally:
        dist.destroy_process_group()


def _slab_compute(rows, k, pad_left, out_shape):
    r = np.asarray(rows, dtype=np.float64)
    full = np.zeros(out_shape)
    lib = O.lib()
    import ctypes
    out = np.empty(out_shape)
    rc = lib.or_xcorr_zpad(r.ndim, r.ctypes.data_as(ctypes.c_void_p),
                           np.array(r.shape, dtype=np.int64).ctypes.data_as(ctypes.c_void_p),
                           np.ascontiguousarray(k, dtype=np.float64).ctypes.data_as(ctypes.c_void_p),
                           np.array(k.shape, dtype=np.int64).ctypes.data_as(ctypes.c_void_p),
                           np.array(pad_left, dtype=np.int64).ctypes.data_as(ctypes.c_void_p),
                           np.array(out_shape, dtype=np.int64).ctypes.data_as(ctypes.c_void_p),
                           out.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0
    del full
    return torch.from_numpy(out)


def _worker_slab(rank, world, port, img, k, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m0 = img.shape[0]
        n0 = k.shape[0]
        pl0 = {"full": n0 - 1, "same": (n0 - 1) - (n0 - 1) // 2, "valid": 0}[mode]
        o0 = {"full": m0 + n0 - 1, "same": m0, "valid": m0 - n0 + 1}[mode]
        me = parallel.slab_plan(m0, o0, pl0, n0, world)[rank]
        local = torch.from_numpy(img[me.in0:me.in1].copy())
        out = parallel.xcorr_rows_sharded(local, m0, k, mode, compute=_slab_compute)
        q.put((rank, me.out0, out.numpy()))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


def test_shard_plan_covers_every_pair_once():
    for n in (2, 3, 9, 64, 1024):
        for world in (1, 2, 3, 8):
            plan = parallel.shard_pairs(n, world)
            pairs = [p for s in plan for p in range(s.p0, s.p1)]
            assert pairs == list(range(n - 1))
            assert max(s.n_pairs for s in plan) - min(s.n_pairs for s in plan) <= 1
            for s in plan:
                if s.n_pairs:
                    assert s.frames == (s.p0, s.p1 + 1)  # one-frame temporal halo


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kw", [dict(level=0, max_level=None), dict(level=0, max_level=3)])
def test_temporal_sharding_matches_unsharded(world, kw):
    frames = O.generate(64, 48, 11, 40.0, (0.45, 0.55), 5, 0.02)
    ref = O.run_sequence(frames, level=kw["level"], max_level=kw["max_level"])
    for rank, out, out2 in _spawn(_worker_seq, world, frames, kw["level"], kw["max_level"]):
        assert np.array_equal(out, ref, equal_nan=True), rank
        assert np.array_equal(out2, ref, equal_nan=True), rank


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["full", "same", "valid"])
def test_row_slab_halo_exchange_matches_unsharded(world, mode):
    rng = np.random.default_rng(9)
    img = rng.random((37, 23))
    k = rng.standard_normal((7, 5))
    ref = O.direct(img, k, mode, "zero", flip=False)
    got = np.zeros_like(ref)
    for rank, out0, out in _spawn(_worker_slab, world, img, k, mode):
        got[out0:out0 + out.shape[0]] = out
    assert np.array_equal(got, ref)


def _worker_seq_more_ranks(rank, world, port, frames, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = parallel.run_sequence_sharded(frames, level=0, compute=_seq_compute)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def test_more_ranks_than_pairs():
    # 3 frames = 2 pairs over 3 ranks: rank 2 computes nothing but joins the gather
    frames = O.generate(32, 32, 3, 40.0, (0.45, 0.55), 8, 0.0)
    ref = O.run_sequence(frames, level=0)
    assert parallel.shard_pairs(3, 3)[2].n_pairs == 0
    for rank, out in _spawn(_worker_seq_more_ranks, 3, frames):
        assert np.array_equal(out, ref, equal_nan=True), rank


def _seq_compute_batched(frames, level, max_level, c_min):
    f = np.asarray(frames)
    if f.ndim == 3:
        return _seq_compute(f, level, max_level, c_min)
    return torch.stack([_seq_compute(v, level, max_level, c_min) for v in f])


def _worker_seq_batched(rank, world, port, vids, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        me = parallel.shard_pairs(vids.shape[1], world)[rank]
        out = parallel.run_sequence_sharded(vids[:, me.frames[0]:me.frames[1]], max_level=2, frames_are_local=True,
                                            n_frames=vids.shape[1], compute=_seq_compute_batched)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def test_batched_videos_sharded_by_frames():
    # the bench's config-5 layout: every rank holds frames p0..p1 of EVERY video
    vids = np.stack([O.generate(48, 40, 7, 30.0 + 10 * v, (0.45, 0.55), 20 + v, 0.01) for v in range(3)])
    ref = np.stack([O.run_sequence(v, max_level=2) for v in vids])
    for rank, out in _spawn(_worker_seq_batched, 3, vids):
        assert out.shape == (3, 6, 10)
        assert np.array_equal(out, ref, equal_nan=True), rank
