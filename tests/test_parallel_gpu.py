"""The multi-GPU data plane (parallel.py) with its DEFAULT compute -- the CUDA
kernels -- on a GPU box: two ranks share cuda:0 over gloo (host-side
collectives; no kernel waits on another rank, so one GPU is a faithful stand-in
for the plumbing).  The sharded results must equal the unsharded single-GPU
run bit for bit (pairs are independent, ttc.py:299-304; the slab halo gives
each output row exactly the taps of the unsharded correlation, _loops.py:104-145)
and the oracle within the north_star tolerances."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, frames, img, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1612_08825_b200 import parallel
        res = {}
        # temporal shards: whole stack given, each rank slices p0..p1 (CUDA compute)
        res["seq"] = parallel.run_sequence_sharded(frames, level=0).cpu().numpy()
        res["ms"] = parallel.run_sequence_sharded(frames.astype(np.float32), max_level=3).cpu().numpy()
        # local-shard form on device tensors (rank r holds only frames p0..p1)
        me = parallel.shard_pairs(frames.shape[0], world)[rank]
        loc = torch.from_numpy(frames[me.frames[0]:me.frames[1]]).cuda()
        res["seq_local"] = parallel.run_sequence_sharded(loc, level=0, frames_are_local=True,
                                                         n_frames=frames.shape[0]).cpu().numpy()
        # every video sharded by frames (the bench's config-5 layout), one call for all shards
        vids = torch.from_numpy(np.stack([frames, frames[::-1].copy()])).float().cuda()
        res["batched"] = parallel.run_sequence_sharded(vids[:, me.frames[0]:me.frames[1]], max_level=2,
                                                       frames_are_local=True, n_frames=frames.shape[0]).cpu().numpy()
        # row slabs of one image, K-1 halo rows exchanged (CUDA ct_xcorr_nd per slab)
        m0, n0 = img.shape[0], k.shape[0]
        plan = parallel.slab_plan(m0, m0 + n0 - 1, n0 - 1, n0, world)
        mine = plan[rank]
        local = torch.from_numpy(img[mine.in0:mine.in1].copy()).cuda()
        out = parallel.xcorr_rows_sharded(local, m0, k, "full")
        assert out.is_cuda
        res["slab"] = (mine.out0, out.cpu().numpy())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_data_plane_cuda_compute(world):
    import paper_1612_08825_b200 as ct
    frames = O.generate(256, 160, 9, 60.0, (0.5, 0.5), 4, 0.0)
    rng = np.random.default_rng(12)
    img = rng.random((203, 150))
    k = rng.standard_normal((7, 5))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, frames, img, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = ct.run_sequence_batch(torch.from_numpy(frames).cuda()[None], level=0)[0].cpu().numpy()
    full_ms = ct.run_sequence_batch(torch.from_numpy(frames.astype(np.float32)).cuda()[None],
                                    max_level=3)[0].cpu().numpy()
    vids = torch.from_numpy(np.stack([frames, frames[::-1].copy()])).float().cuda()
    full_b = ct.run_sequence_batch(vids, max_level=2).cpu().numpy()
    ref = O.run_sequence(frames, level=0)
    ref_conv = O.direct(img, k, "full", "zero", flip=False)
    got_conv = np.zeros_like(ref_conv)
    for rank, r in res:
        assert np.array_equal(r["seq"], full, equal_nan=True), rank
        assert np.array_equal(r["seq_local"], full, equal_nan=True), rank
        assert np.array_equal(r["ms"], full_ms, equal_nan=True), rank
        assert np.array_equal(r["batched"], full_b, equal_nan=True), rank
        o0, out = r["slab"]
        got_conv[o0:o0 + out.shape[0]] = out
    fin = np.isfinite(ref[:, 5])
    assert np.max(np.abs(full[fin, 5] - ref[fin, 5]) / np.abs(ref[fin, 5])) <= 1e-9
    assert np.array_equal(got_conv, ref_conv)  # fp64 conv is bit-exact to the oracle


def test_approach_stream_frame_range_is_a_shard_of_the_stream():
    # config-5 temporal shards build only their frames; they equal the whole stream's
    import paper_1612_08825_b200.synth as S
    full, truth = S.approach_stream(40, 64, 96, seed=1004, dtype=torch.float32)
    for a, b in ((0, 40), (25, 35), (31, 32), (10, 10)):
        part, tr = S.approach_stream(40, 64, 96, seed=1004, dtype=torch.float32, frame_range=(a, b))
        assert torch.equal(part, full[a:b])
        assert np.array_equal(tr, truth[a:b], equal_nan=True)
    with pytest.raises(ValueError):
        S.approach_stream(40, 64, 96, seed=1004, frame_range=(5, 41))
