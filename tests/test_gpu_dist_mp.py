"""GPU, real multi-process K7: world_size 2 and 3 processes over gloo, every
rank running the partition / merge kernels on the one visible GPU (the
exchange goes through host memory, so no rank's kernel ever waits on
another's).  The rank-order concatenation of the shards returned by
``dist.sharded_outer_multiply`` must equal the single-GPU merge bit for bit,
including when there are fewer buckets than ranks (ranks with an empty key
range), and the ``sharded_bitmatrix`` row blocks must tile the full matrix."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _operands(case):
    from paper_2605_25974_b200 import rng

    if case == "c2":
        return (500,) + rng.config_columns(2, 0.3)
    if case == "tiny":  # 5 x 4 products: one bucket, fewer than the ranks
        a, b = rng.config_columns(2, 0.005)
        return (500, a, tuple(v[:4] for v in b))
    if case == "hh":  # heavy cancellation, runs longer than a leaf
        h = rng.local_columns(64, 700, rng.SplitMix64(3), 12, (1, 3))
        return (64, h, h)
    raise KeyError(case)


def _worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2605_25974_b200 as pl
        from paper_2605_25974_b200 import dist as pdist

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        n, a, b = _operands(case)
        A = pl.PauliSumSoA.from_columns(n, *a, device=dev)
        B = pl.PauliSumSoA.from_columns(n, *b, device=dev)
        shard = pdist.sharded_outer_multiply(A, B)
        words, (r0, r1) = pdist.sharded_bitmatrix(A)
        q.put((rank, shard.columns(), words.cpu().numpy(), r0, r1, None))
    except Exception as exc:  # reported to the parent
        q.put((rank, None, None, 0, 0, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("c2", 2), ("c2", 3), ("tiny", 2), ("hh", 2)])
def test_sharded_processes_equal_single(cuda, case, world):
    import paper_2605_25974_b200 as pl

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=120)
    errors = {r: v[5] for r, v in res.items() if v[5]}
    assert not errors, errors

    n, a, b = _operands(case)
    A = pl.PauliSumSoA.from_columns(n, *a, device=cuda)
    B = pl.PauliSumSoA.from_columns(n, *b, device=cuda)
    sx, sz, sf, sc = pl.outer_multiply(A, B).columns()
    gx = np.concatenate([res[r][1][0] for r in range(world)])
    gz = np.concatenate([res[r][1][1] for r in range(world)])
    gf = np.concatenate([res[r][1][2] for r in range(world)])
    gc = np.concatenate([res[r][1][3] for r in range(world)])
    assert np.array_equal(gx, sx) and np.array_equal(gz, sz) and np.array_equal(gf, sf)
    assert np.array_equal(gc.view(np.uint64), sc.view(np.uint64))  # bit-identical sums

    full = pl.commutation_bitmatrix(A).cpu().numpy()
    assert res[0][3] == 0 and res[world - 1][4] == len(A)
    assert all(res[r][4] == res[r + 1][3] for r in range(world - 1))
    rows = np.concatenate([res[r][2] for r in range(world)])
    assert np.array_equal(rows, full)
