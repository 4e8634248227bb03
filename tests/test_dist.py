"""Multi-process host path on CPU (gloo, world_size 2).

The GHN path shards by queries: every rank holds the same index (replica)
and answers its own query shard; no collective touches the data path
(SURVEY §8(e)).  This test runs that sharding with the oracle standing in
for the device kernel on each rank and checks that the gathered answers
equal a single-process run -- the host logic bench.py uses for --gpus N.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard(nq, world, rank):
    per = (nq + world - 1) // world
    return slice(rank * per, min(nq, (rank + 1) * per))


def _worker(rank, world, port, out):
    import torch

    import oracle
    from paper_2004_02290_b200 import datagen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = datagen.cfg0(n=20_000, nq=1_001, seed=7)          # identical replica on every rank
    ref = oracle.COracle(w.X, w.widths)
    sl = _shard(w.Q.shape[0], world, rank)
    keys, idx, stats = ref.query(w.Q[sl], w.k, threads=1)
    lab, _ = oracle.classify(keys, idx, w.y.astype(np.int64))
    # gather variable-size shards (pad to the largest)
    per = (w.Q.shape[0] + world - 1) // world
    buf = torch.full((per,), -1, dtype=torch.int64)
    buf[: lab.shape[0]] = torch.from_numpy(lab)
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    # max-over-ranks timing reduction used by bench.py
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        allv = torch.cat(gathered)[: w.Q.shape[0]].numpy()
        np.save(out, np.concatenate([allv, [int(t.item())]]))
    dist.barrier()
    dist.destroy_process_group()


def test_query_sharding_gloo_world2(tmp_path):
    import oracle
    from paper_2004_02290_b200 import datagen

    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    w = datagen.cfg0(n=20_000, nq=1_001, seed=7)
    ref = oracle.COracle(w.X, w.widths)
    keys, idx, _ = ref.query(w.Q, w.k, threads=1)
    want, _ = oracle.classify(keys, idx, w.y.astype(np.int64))
    assert np.array_equal(got[:-1], want)
    assert got[-1] == 2          # max over ranks
