"""K7 — outer product + merge sharded over GPUs (one process per GPU).

Path (no reference equivalent; the paper lists distributed memory as future
work):

1. every rank builds the SAME merge plan from the replicated A and B, so the
   key-range splitters (a deterministic sample of the full product) agree
   without a collective;
2. rank r generates the raw products of B columns [r*Mb/G, (r+1)*Mb/G) -- the
   reference's thread split over j-blocks (sums.py:161-173) -- and buckets
   them by key range (``pl_outer_partition``);
3. one all-to-all over NCCL sends bucket range q to rank q (``exchange``);
4. each rank merges what it received (``pl_merge_received``).

Concatenating the ranks' shards in rank order is bit-identical to the
single-GPU result: runs of equal keys never straddle buckets and each run is
summed in raw-row order by one thread.  The bitmatrix path shards by row
blocks with no collective (``sharded_bitmatrix``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from ._device import cuda_device, ptr, stream_ptr
from .sums import (PauliSumSoA, _alloc_planes, _download, _fitted, _new_sum, _remember,
                   _zero_planes)


def block_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced block [lo, hi) of range(n) for `rank` of `world`."""
    return rank * n // world, (rank + 1) * n // world


def exchange(send: torch.Tensor, bucket_counts: torch.Tensor, item_bytes: int, group=None):
    """All-to-all of bucket-contiguous records by bucket range.

    ``send`` holds this rank's records grouped by bucket (uint8, bucket-major
    over all nb buckets); ``bucket_counts`` (nb,) int32 the records per bucket.
    Rank q receives buckets ``block_range(nb, G, q)`` from every source.
    Returns (recv uint8 tensor, counts (G, nb_local) int32 on send's device,
    b0, b1).  Works with any backend (NCCL on GPUs, gloo on CPU tensors).
    """
    world = dist.get_world_size(group) if group is not None or dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    nb = bucket_counts.numel()
    if world == 1:
        return send, bucket_counts.view(1, nb), 0, nb
    home = send.device
    # gloo moves host tensors only: device records are staged through host
    # memory (the multi-process tests on one GPU); NCCL moves device memory
    staged = home.type == "cuda" and dist.get_backend(group) == "gloo"
    wire = torch.device("cpu") if staged else home
    counts = bucket_counts.to(wire)
    gathered = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(gathered, counts, group=group)
    cm = torch.stack(gathered).to("cpu", torch.int64).numpy()  # (G, nb)
    ranges = [block_range(nb, world, q) for q in range(world)]
    b0, b1 = ranges[rank]
    send_split = [int(cm[rank, lo:hi].sum()) * item_bytes for lo, hi in ranges]
    recv_split = [int(cm[s, b0:b1].sum()) * item_bytes for s in range(world)]
    recv = torch.empty(max(sum(recv_split), 1), dtype=torch.uint8, device=wire)
    recv_view = recv[:sum(recv_split)]
    send_view = send[:sum(send_split)].to(wire)
    dist.all_to_all_single(recv_view, send_view, recv_split, send_split, group=group)
    local = torch.from_numpy(np.ascontiguousarray(cm[:, b0:b1]).astype(np.int32)).to(home)
    return recv_view.to(home), local, b0, b1


def partition(A, B, plan, j0: int, j1: int, dev):
    """Stage 1 on this device: (send bytes, bucket counts (nb,) int32)."""
    lib = _native.load()
    nb = int(plan.n_buckets)
    item = int(lib.pl_dist_item_bytes(C.byref(plan)))
    n_local = A.M * (j1 - j0)
    ws_bytes = int(lib.pl_dist_workspace_bytes(C.byref(plan), n_local, nb))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    send = torch.empty(max(n_local * item, 1), dtype=torch.uint8, device=dev)
    counts = torch.empty(nb, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _native.call("pl_outer_partition", C.byref(plan), ptr(A.x), ptr(A.z), ptr(A.k), A.ld,
                     ptr(B.x), ptr(B.z), ptr(B.k), B.ld, j0, j1, ptr(ws), ws.numel(),
                     ptr(send), ptr(counts), stream_ptr(dev))
    return send[:n_local * item], counts, item


def merge_received(A, B, plan, recv, counts, b0: int, b1: int, eps: float, dev, n: int):
    """Stage 3: merge received records into this rank's output shard."""
    lib = _native.load()
    item = int(lib.pl_dist_item_bytes(C.byref(plan)))
    n_recv = recv.numel() // item
    G = counts.shape[0]
    ws_bytes = int(lib.pl_dist_workspace_bytes(C.byref(plan), n_recv, b1 - b0))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    x, z, k, c = _alloc_planes(A.W, n_recv, dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    counts = counts.to(dev, torch.int32).contiguous()
    with torch.cuda.device(dev):
        _native.call("pl_merge_received", C.byref(plan), ptr(recv), n_recv, ptr(counts), G, b0, b1,
                     ptr(A.x), ptr(A.z), ptr(A.k), ptr(A.c), A.ld,
                     ptr(B.x), ptr(B.z), ptr(B.k), ptr(B.c), B.ld, float(eps), ptr(ws), ws.numel(),
                     ptr(x), ptr(z), ptr(k), ptr(c), x.stride(0), ptr(cnt), stream_ptr(dev))
    return _fitted(n, x, z, k, c, int(cnt.item()))


def _plan(A, B, dev):
    plan = _native.MergePlan()
    with torch.cuda.device(dev):
        _native.call("pl_outer_plan", A.W, A.M, B.M, ptr(A.x), ptr(A.z), A.ld, ptr(B.x),
                     ptr(B.z), B.ld, C.byref(plan), stream_ptr(dev))
    _remember(plan)
    return plan


def sharded_outer_multiply(a: PauliSumSoA, b: PauliSumSoA, *, group=None, eps: float = 0.0,
                           device=None) -> PauliSumSoA:
    """This rank's shard of the canonical A*B (sums.py:293-305 with combine).

    A and B are replicated on every rank.  Host inputs are uploaded and the
    shard is returned to host memory (end-to-end path)."""
    a._check_same_n(b)
    back = a.device.type != "cuda" and b.device.type != "cuda"
    dev = cuda_device(device if device is not None else (a.device if not back else None))
    A = a.to(dev).planes()
    B = b.to(dev).planes()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if A.M * B.M == 0:
        out = PauliSumSoA.empty(a.n, device=dev)
        return _download(out) if back else out
    plan = _plan(A, B, dev)
    j0, j1 = block_range(B.M, world, rank)
    send, counts, item = partition(A, B, plan, j0, j1, dev)
    recv, cm, b0, b1 = exchange(send, counts, item, group)
    if b1 > b0:
        out = merge_received(A, B, plan, recv, cm, b0, b1, eps, dev, a.n)
    else:  # fewer buckets than ranks: this rank owns no key range (still joined the exchange)
        out = PauliSumSoA.empty(a.n, device=dev)
    return _download(out, *_zero_planes(plan), True) if back else out


def emulate_sharded(a: PauliSumSoA, b: PauliSumSoA, world: int, *, eps: float = 0.0):
    """Run the K7 stages for `world` virtual ranks on ONE device (sequentially,
    exchange done by slicing) and return the per-rank shards.  Used by the
    tests to check that the sharded result equals the single-GPU one."""
    dev = a.device if a.device.type == "cuda" else cuda_device()
    A, B = a.to(dev).planes(), b.to(dev).planes()
    plan = _plan(A, B, dev)
    nb = int(plan.n_buckets)
    sends, counts = [], []
    for r in range(world):
        j0, j1 = block_range(B.M, world, r)
        s, c, item = partition(A, B, plan, j0, j1, dev)
        sends.append(s)
        counts.append(c.to("cpu", torch.int64).numpy())
    cm = np.stack(counts)
    shards = []
    for q in range(world):
        b0, b1 = block_range(nb, world, q)
        pieces = []
        for s in range(world):
            lo = int(cm[s, :b0].sum()) * item
            hi = int(cm[s, :b1].sum()) * item
            pieces.append(sends[s][lo:hi])
        recv = torch.cat(pieces) if pieces else torch.empty(0, dtype=torch.uint8, device=dev)
        local = torch.from_numpy(np.ascontiguousarray(cm[:, b0:b1]).astype(np.int32))
        if b1 > b0:
            shards.append(merge_received(A, B, plan, recv, local, b0, b1, eps, dev, a.n))
        else:
            shards.append(PauliSumSoA.empty(a.n, device=dev))
    return shards


def concat(shards) -> PauliSumSoA:
    """Rank-order concatenation of shards (the global canonical sum)."""
    n = shards[0].n
    return _new_sum(n, torch.cat([s.x for s in shards], 1), torch.cat([s.z for s in shards], 1),
                    torch.cat([s.flags for s in shards]), torch.cat([s.coeffs for s in shards]))


def sharded_bitmatrix(s: PauliSumSoA, *, group=None, out=None, method: str = "auto"):
    """Row block [r*M/G, (r+1)*M/G) of the commutation bitmatrix on this rank
    (inputs replicated, no collective)."""
    from .bitmatrix import commutation_bitmatrix

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    r0, r1 = block_range(len(s), world, rank)
    return commutation_bitmatrix(s, row0=r0, rows=r1 - r0, out=out, method=method), (r0, r1)
