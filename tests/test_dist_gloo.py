"""CPU, world_size 2 over gloo: the K7 key-range exchange (dist.exchange) moves
every bucket's records to its owner in (source, bucket) order."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_25974_b200.dist import block_range, exchange

ITEM = 16  # bytes per synthetic record


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_send(rank, nb, seed):
    r = np.random.default_rng(seed + rank)
    counts = r.integers(0, 7, nb).astype(np.int32)
    recs = []
    for b in range(nb):
        for i in range(counts[b]):
            recs.append(np.array([rank, b, i, 12345], dtype=np.int32))
    buf = np.concatenate(recs).view(np.uint8) if recs else np.zeros(0, np.uint8)
    return torch.from_numpy(buf.copy()), torch.from_numpy(counts)


def _worker(rank, world, port, nb, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        send, counts = make_send(rank, nb, seed)
        recv, cm, b0, b1 = exchange(send, counts, ITEM)
        got = recv.numpy().view(np.int32).reshape(-1, 4) if recv.numel() else np.zeros((0, 4), np.int32)
        exp = []
        for s in range(world):
            _, cs = make_send(s, nb, seed)
            for b in range(b0, b1):
                for i in range(int(cs[b])):
                    exp.append([s, b, i, 12345])
        exp = np.array(exp, dtype=np.int32).reshape(-1, 4)
        ok = np.array_equal(got, exp) and tuple(cm.shape) == (world, b1 - b0)
        ok = ok and (b0, b1) == block_range(nb, world, rank)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nb", [(2, 7), (2, 64), (3, 10)])
def test_exchange_gloo(world, nb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nb, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_block_range_partitions():
    for n in (0, 1, 7, 512, 10_000):
        for w in (1, 2, 3, 8):
            parts = [block_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
