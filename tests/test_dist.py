# SPDX-License-Identifier: Apache-2.0
"""The N>1 host path on CPU: world_size-2 gloo processes shard ciphertext batches
with no overlap and reduce device times with MAX (bench.py's multi-GPU logic)."""
import os
import socket

import pytest

from paper_1908_04172_b200.dist import shard


def test_shard_partition():
    for n in (1, 7, 64, 65):
        for w in (1, 2, 3, 8):
            got = [i for r in range(w) for i in shard(n, r, w)]
            assert got == list(range(n))
            sizes = [len(shard(n, r, w)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_04172_b200.dist import env, max_over_ranks, shard
    ws, r, lr = env()
    mine = list(shard(64, r, ws))  # config 5a: 64 independent batches
    t = max_over_ranks(10.0 + r)
    q.put((r, mine, t))
    dist.destroy_process_group()


def test_gloo_world2_batch_sharding():
    mp = pytest.importorskip("torch.multiprocessing")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] + res[1][1] == list(range(64))
    assert res[0][2] == res[1][2] == 11.0
