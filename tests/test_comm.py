# SPDX-License-Identifier: Apache-2.0
"""The C-ABI multi-GPU pieces (include/henet_b200.h: hg_shard_range, hg_comm_*,
hg_allgather_tensor, hg_broadcast_tensor).

CPU (gloo, world size 2): every rank asks the library for its block of the output neurons
and ships its rows with the same padded-block exchange hg_allgather_tensor performs
(ncclAllGather of max-width blocks, then each rank's rows moved to its block start); the
blocks must tile [0, total) exactly once, agree with dist.shard, and reassemble bit-exactly.
GPU (one device, so world size 1 over NCCL): the gather and broadcast through the library
leave the residue words unchanged, and an output-sharded c5b-shaped layer gathered by the
library equals the unsharded layer, residue for residue.
"""
import os
import socket

import numpy as np
import pytest

from paper_1908_04172_b200 import dist


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_04172_b200 import henet as H
    out = []
    for total in (4096, 4095, 13, 1, 0):
        mine = H.shard_range(total, rank, world)
        assert mine == dist.shard(total, rank, world)
        blocks = [H.shard_range(total, r, world) for r in range(world)]
        width = max(len(b) for b in blocks)
        send = torch.zeros((width, 5), dtype=torch.int64)
        send[:len(mine)] = torch.tensor([[7 * i + c for c in range(5)] for i in mine], dtype=torch.int64).reshape(-1, 5)
        parts = torch.empty((world * width, 5), dtype=torch.int64)
        tdist.all_gather_into_tensor(parts, send)
        full = torch.full((total, 5), -1, dtype=torch.int64)
        for r, b in enumerate(blocks):
            full[b.start:b.stop] = parts[r * width: r * width + len(b)]
        out.append((total, [(b.start, b.stop) for b in blocks], full.numpy()))
    q.put((rank, out))
    tdist.destroy_process_group()


def test_shard_blocks_and_padded_gather_gloo_world2():
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
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        for total, blocks, full in res[r]:
            covered = sorted(i for b in blocks for i in range(*b))
            assert covered == list(range(total))
            want = np.array([[7 * i + c for c in range(5)] for i in range(total)], dtype=np.int64).reshape(-1, 5)
            assert np.array_equal(full, want)


@pytest.mark.gpu
def test_native_gather_broadcast_world1():
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200 import workloads as W
    for p in (W.N8192, W.N16384):
        ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
        comm = H.Communicator(ctx, H.comm_unique_id(), 1, 0)
        x = W.random_ciphertexts(p, 5, seed=3, level=3)
        t = H.CipherTensor.from_words(ctx, x, 2.0 ** 40)
        g = comm.allgather(t, 5)
        assert g.info()[:4] == (5, 2, 3, 2.0 ** 40)
        assert np.array_equal(g.to_words(), x)
        comm.broadcast(t, 0)
        assert np.array_equal(t.to_words(), x)
        with pytest.raises(H.ValidationError):
            comm.allgather(t, 9)  # 9 outputs over 1 rank: the local block must hold all 9


@pytest.mark.gpu
def test_output_sharded_dense_native_gather_bit_exact():
    """c5b topology (K -> M dense, one rescale per output, N = 16384 with the 40-bit limb):
    the rank's column block evaluated and gathered by hg_allgather_tensor equals the whole
    layer evaluated at once."""
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200 import workloads as W
    from paper_1908_04172_b200.sharded import OutputShardedDense
    p = W.N16384
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    K, M = 160, 150
    w = W.wide_dense_weights(k=K, m=M)
    x = H.CipherTensor.from_words(ctx, W.random_ciphertexts(p, K, seed=5), p["scale"], shape=[K])
    whole = OutputShardedDense(ctx, w, 0, 1)
    comm = H.Communicator(ctx, H.comm_unique_id(), 1, 0)
    got = whole.gather_native(whole.local(x), comm)
    want = H.execute(ctx, whole.model, whole.plan, x)
    assert got.scale == want.scale
    assert np.array_equal(got.to_words(), want.to_words())
