"""N > 1 path of the weak-scaling bench on CPU: world_size 2 over gloo (no GPU needed).

Ciphertexts shard over ranks with no data-path collective; these tests check the
sharding arithmetic, that the sharded inputs are exactly the single-rank job's, and the
max-over-ranks timing reduction over a real process group.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2502_00847_b200 import shard


def test_shard_partitions_exactly():
    for n in (0, 1, 7, 8, 16, 33):
        for ws in (1, 2, 3, 8):
            blocks = [shard.shard(n, ws, r) for r in range(ws)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.shard(4, 2, 2)


def test_sharded_inputs_equal_single_rank_job():
    n, cfg = 16, 5
    single = [shard.input_seed(cfg, i) for i in range(n)]
    sharded = []
    for r in range(4):
        b, e = shard.shard(n, 4, r)
        sharded += [shard.input_seed(cfg, i) for i in range(b, e)]
    assert sharded == single and len(set(single)) == n


def test_job_throughput():
    assert shard.job_throughput(2048 * 8, 2, 100.0) == pytest.approx(2048 * 8 * 2 / 0.1)
    with pytest.raises(ValueError):
        shard.job_throughput(1, 1, 0.0)


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        ms = 10.0 + 5.0 * rank  # rank-local device time
        mx = shard.max_over_ranks(ms)
        b, e = shard.shard(10, ws, rank)
        q.put((rank, mx, b, e))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert [r[1] for r in res] == [15.0, 15.0]  # every rank sees the slowest rank's time
    assert [(r[2], r[3]) for r in res] == [(0, 5), (5, 10)]
