"""Multi-GPU drivers (one process per GPU, torch.distributed over NCCL).

Two sharding schemes, both from SURVEY.md 8(e):

* Temporal sharding of a frame stack (run_sequence over a long video):
  pairs are independent (ttc.py:299-304), so rank r takes a contiguous pair
  range [p0, p1) and the frames p0..p1 -- one frame of temporal halo shared
  with the next rank, duplicated at load/generation time.  There is no
  exchange during compute; the per-pair estimate rows (10 float64 each) are
  gathered to every rank with one all_gather at the end.

* Row-slab sharding of one large image for direct convolution: rank r owns
  input rows [a_r, b_r) and produces a contiguous block of output rows; the
  K-1 halo rows it needs from its neighbours arrive by point-to-point
  send/recv (one batched NCCL group), then the local slab runs through the
  same single-GPU kernel with adjusted padding.

The compute step is injectable (``compute``) so the host-side logic -- plans,
halos, gathers, ordering -- is testable on CPU with the gloo backend; on GPUs
the default compute is this package's CUDA path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class PairShard:
    rank: int
    p0: int  # first pair (== first frame)
    p1: int  # one past the last pair; frames p0..p1 inclusive

    @property
    def frames(self) -> tuple[int, int]:
        return self.p0, self.p1 + 1

    @property
    def n_pairs(self) -> int:
        return self.p1 - self.p0


def shard_pairs(n_frames: int, world: int) -> list[PairShard]:
    """Split the n_frames - 1 pairs of a stack into `world` contiguous ranges (sizes differ by <= 1)."""
    if n_frames < 2:
        raise ValueError("need at least two frames")
    n_pairs = n_frames - 1
    base, extra = divmod(n_pairs, world)
    out, p = [], 0
    for r in range(world):
        cnt = base + (1 if r < extra else 0)
        out.append(PairShard(r, p, p + cnt))
        p += cnt
    return out


def collective_device(group=None) -> torch.device:
    """Where tensors must live for this group's collectives: the current CUDA
    device under NCCL, the host under gloo (CUDA results are staged through
    host memory there; gloo is the CPU test backend)."""
    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _default_compute(frames_local, level, max_level, c_min):
    from .ttc import run_sequence_batch
    t = frames_local if isinstance(frames_local, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(frames_local))
    if t.ndim == 4:  # a batch of videos' shards [V, frames, h, w]
        return run_sequence_batch(t.cuda(), level=level, max_level=max_level, c_min=c_min)
    return run_sequence_batch(t.cuda()[None], level=level, max_level=max_level, c_min=c_min)[0]


def run_sequence_sharded(frames, level=0, max_level=None, c_min=1e-9, group=None, compute=None,
                         frames_are_local: bool = False, n_frames: int | None = None) -> torch.Tensor:
    """Estimate rows [n_frames - 1, 10] for a stack sharded over the ranks of `group`.

    ``frames`` is either the whole stack (each rank slices its shard) or, with
    frames_are_local=True, this rank's shard frames p0..p1 already (then pass
    n_frames, the global frame count).  A 4-D ``frames`` [V, n, h, w] shards
    every video the same way (one launch for all videos' shards, one
    all_gather) and returns [V, n_frames - 1, 10].  Every rank returns the
    full, ordered result (gathered with one all_gather; rows identical to the
    1-GPU run) on collective_device(group): the GPU under NCCL, the host
    under gloo.  Ranks beyond the pair count compute nothing and still join
    the gather.
    """
    compute = compute or _default_compute
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    batched = frames.ndim == 4
    n = n_frames if frames_are_local else frames.shape[1 if batched else 0]
    if n is None:
        raise ValueError("n_frames is required with frames_are_local=True")
    plan = shard_pairs(n, world)
    me = plan[rank]
    a, b = me.frames
    local = frames if frames_are_local else (frames[:, a:b] if batched else frames[a:b])
    lead = (frames.shape[0],) if batched else ()
    if me.n_pairs > 0:
        rows = compute(local, level, max_level, c_min)
        rows = torch.as_tensor(rows, dtype=torch.float64)
    else:  # more ranks than pairs: this rank only takes part in the gather
        rows = torch.empty(lead + (0, 10), dtype=torch.float64)
    if world == 1:
        return rows
    dev = collective_device(group)
    rows = rows.to(dev)
    width = max(s.n_pairs for s in plan)
    buf = torch.full(lead + (width, 10), float("nan"), dtype=torch.float64, device=dev)
    buf[..., :me.n_pairs, :] = rows
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf, group=group)
    return torch.cat([g[..., :s.n_pairs, :] for g, s in zip(gathered, plan)], dim=-2)


# ----------------------------------------------------------- row slabs ---

@dataclass(frozen=True)
class RowSlab:
    rank: int
    in0: int   # owned input rows [in0, in1)
    in1: int
    out0: int  # produced output rows [out0, out1)
    out1: int


def slab_plan(m0: int, o0: int, pl0: int, n0: int, world: int) -> list[RowSlab]:
    """Owned input rows and produced output rows per rank for a correlation
    along axis 0 with left pad pl0, kernel extent n0 and output extent o0.

    Output row y reads input rows [y - pl0, y - pl0 + n0); outputs are split
    evenly, inputs are split evenly, and halos cover the difference.
    """
    def split(n):
        base, extra = divmod(n, world)
        cuts, p = [], 0
        for r in range(world):
            c = base + (1 if r < extra else 0)
            cuts.append((p, p + c))
            p += c
        return cuts

    ins, outs = split(m0), split(o0)
    return [RowSlab(r, ins[r][0], ins[r][1], outs[r][0], outs[r][1]) for r in range(world)]


def needed_rows(slab: RowSlab, pl0: int, n0: int, m0: int) -> tuple[int, int]:
    lo = max(0, slab.out0 - pl0)
    hi = min(m0, slab.out1 - 1 - pl0 + n0)
    return lo, max(lo, hi)


def exchange_halo(local_in: torch.Tensor, plan: list[RowSlab], rank: int, pl0: int, n0: int, m0: int,
                  group=None) -> tuple[torch.Tensor, int]:
    """Assemble this rank's needed input rows from its own slab plus
    neighbours' rows (batched point-to-point).  Returns (rows, first_row)."""
    me = plan[rank]
    lo, hi = needed_rows(me, pl0, n0, m0)
    home = local_in.device
    local_in = local_in.to(collective_device(group))  # gloo: stage CUDA rows through the host
    ops, recv = [], []
    for other in plan:
        # rows `other` needs from me
        olo, ohi = needed_rows(other, pl0, n0, m0)
        a, b = max(olo, me.in0), min(ohi, me.in1)
        if other.rank != rank and a < b:
            ops.append(dist.P2POp(dist.isend, local_in[a - me.in0:b - me.in0].contiguous(), other.rank, group=group))
        # rows I need from `other`
        a, b = max(lo, other.in0), min(hi, other.in1)
        if other.rank != rank and a < b:
            t = torch.empty((b - a,) + tuple(local_in.shape[1:]), dtype=local_in.dtype, device=local_in.device)
            ops.append(dist.P2POp(dist.irecv, t, other.rank, group=group))
            recv.append((a, t))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    pieces = recv + [(max(lo, me.in0), local_in[max(lo, me.in0) - me.in0:max(min(hi, me.in1), max(lo, me.in0)) - me.in0])]
    pieces = [(a, t) for a, t in pieces if t.shape[0] > 0]
    pieces.sort(key=lambda p: p[0])
    rows = torch.cat([t for _, t in pieces]) if pieces else local_in[:0]
    return rows.to(home), lo


def xcorr_rows_sharded(local_in: torch.Tensor, m0: int, kernel, shape_mode: str = "full", group=None,
                       compute=None) -> torch.Tensor:
    """Row-slab sharded zero-extended correlation of one image (axis 0 split).

    ``local_in`` is this rank's owned input rows (per slab_plan over m0 rows).
    Returns this rank's output rows [out0, out1).  ``compute(rows, kernel,
    pad_left, out_shape)`` runs the local correlation (default: ct_xcorr_nd).
    """
    k = np.asarray(kernel)
    n0 = k.shape[0]
    if shape_mode == "full":
        pl = [n - 1 for n in k.shape]
        o0 = m0 + n0 - 1
    elif shape_mode == "same":
        pl = [(n - 1) - (n - 1) // 2 for n in k.shape]
        o0 = m0
    else:
        pl = [0] * k.ndim
        o0 = m0 - n0 + 1
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = slab_plan(m0, o0, pl[0], n0, world)
    rows, first = exchange_halo(local_in, plan, rank, pl[0], n0, m0, group)
    me = plan[rank]
    # global output row y reads global input rows y - pl0 + j; `rows` starts at
    # global row `first` >= out0 - pl0, so the local left pad is non-negative
    local_pad0 = first - (me.out0 - pl[0])
    out_shape = [me.out1 - me.out0] + [
        (s + n - 1 if shape_mode == "full" else (s if shape_mode == "same" else s - n + 1))
        for s, n in zip(local_in.shape[1:], k.shape[1:])]
    compute = compute or _xcorr_local
    return compute(rows, k, [local_pad0] + pl[1:], out_shape)


def _xcorr_local(rows, k, pad_left, out_shape):
    """Zero-extended correlation of the assembled rows on this rank's GPU (ct_xcorr_nd)."""
    import ctypes

    from . import _lib
    L = _lib.load()
    src = rows.contiguous()
    pads = list(pad_left)
    out = torch.empty(out_shape, dtype=rows.dtype, device=rows.device)
    kk = np.ascontiguousarray(k, dtype=np.float64 if rows.dtype == torch.float64 else np.float32)
    kd = torch.from_numpy(kk).to(rows.device)
    _lib.check(L.ct_xcorr_nd(_lib.dtype_code(src), kk.ndim, _lib.ptr(src), _lib.i64_array(src.shape), 1, _lib.ptr(kd),
                             kk.ctypes.data_as(ctypes.c_void_p), _lib.i64_array(kk.shape), _lib.i64_array(pads),
                             _lib.i64_array(out_shape), _lib.CT_ZERO, _lib.ptr(out), _lib.stream_ptr()))
    return out
