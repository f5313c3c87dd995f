# SPDX-License-Identifier: Apache-2.0
"""Config 5b: a dense layer sharded by output neuron across ranks, outputs all-gathered.

CPU: the row all-gather (gloo, world 2, equal and unequal blocks) and the plan patch
against the reference's own patched plan.  GPU: every shard of a 3-way split computed
on one device and assembled in rank order equals the reference's unsharded layer."""
import os
import socket

import numpy as np
import pytest

from paper_1908_04172_b200 import dist
from paper_1908_04172_b200 import workloads as W


def _gather_worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_04172_b200.sharded import gather_rows
    out = []
    for total in (5, 6, 1):
        rows = dist.shard(total, rank, world)
        local = torch.tensor([[1000 * i + c for c in range(7)] for i in rows], dtype=torch.int64).reshape(-1, 7)
        out.append(gather_rows(local, total, world).numpy())
    q.put((rank, out))
    tdist.destroy_process_group()


def _chunk_worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_04172_b200.sharded import gather_chunk_into
    out = []
    for total in (5, 6, 13, 2):
        for chunks in (1, 2, 3):
            blocks = dist.chunk_shards(total, world, chunks)
            dst = torch.full((total, 7), -1, dtype=torch.int64)
            for c in range(chunks):
                mine = blocks[c][rank]
                local = torch.tensor([[1000 * i + k for k in range(7)] for i in mine], dtype=torch.int64).reshape(-1, 7)
                gather_chunk_into(dst, local, blocks[c])
            out.append(dst.numpy())
    q.put((rank, out))
    tdist.destroy_process_group()


def test_chunked_gather_gloo_world2():
    """Chunk c of every rank's shard lands in its global rows (the overlapped c5b gather)."""
    mp = pytest.importorskip("torch.multiprocessing")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_chunk_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    k = 0
    for total in (5, 6, 13, 2):
        for chunks in (1, 2, 3):
            want = np.array([[1000 * i + c for c in range(7)] for i in range(total)], dtype=np.int64)
            assert np.array_equal(res[0][k], want) and np.array_equal(res[1][k], want), (total, chunks)
            k += 1
    # every row is produced exactly once
    for total in (5, 6, 13, 2):
        for world in (1, 2, 3, 8):
            for chunks in (1, 2, 4):
                rows = [i for c in dist.chunk_shards(total, world, chunks) for b in c for i in b]
                assert sorted(rows) == list(range(total)), (total, world, chunks)


def test_gather_rows_gloo_world2():
    mp = pytest.importorskip("torch.multiprocessing")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, total in enumerate((5, 6, 1)):
        want = np.array([[1000 * i + c for c in range(7)] for i in range(total)], dtype=np.int64)
        assert np.array_equal(res[0][k], want) and np.array_equal(res[1][k], want), total


def test_patch_terminal_rescale_matches_reference():
    from oracle import refbind as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200.sharded import patch_terminal_rescale
    p = W.N16384
    for wl, counts in ((W.wide_dense(k=96, m=40), {"input": 96, "fc": 40, "out": 40}),
                       (W.dense_layer(), {"input": 845, "fc": 100, "out": 100})):
        pp = W.N16384 if "c5b" in wl.name else W.N8192
        ref = R.RefContext(pp["n"], pp["chain"], pp["special"], pp["scale"])
        rp = ref.plan(wl.manifest, wl.blob, patch=True)
        model = H.PlainModel.load(wl.manifest, wl.blob)
        plan = H.RescalePlan.plan_params(pp["chain"], pp["scale"], model)
        got = patch_terminal_rescale(pp["chain"], pp["scale"], wl.manifest, plan, counts)
        assert got.planned_rescale_ops == rp["planned_rescale_ops"]
        for n in rp["nodes"]:
            dec, lin, lout, sc = got.node(n["id"])
            want_sc = np.array([n["scale_out_bits"]], dtype=np.uint64).view(np.float64)[0]
            assert (lin, lout, sc) == (n["level_in"], n["level_out"], want_sc), n["id"]
    del p


@pytest.mark.gpu
def test_output_sharded_dense_bit_exact():
    from oracle import refbind as R
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200.sharded import OutputShardedDense, assemble
    p = W.N16384
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    k, m = 64, 29
    wl = W.wide_dense(k=k, m=m)
    x = W.random_ciphertexts(p, k, seed=21)
    want, want_sc, _ = ref.execute(None, wl.manifest, wl.blob, x, p["scale"], patch=True)
    wts = W.wide_dense_weights(k=k, m=m)
    xt = H.CipherTensor.from_words(ctx, x, p["scale"], shape=[k])
    world = 3
    parts = [OutputShardedDense(ctx, wts, r, world).local(xt) for r in range(world)]
    assert [pt.count for pt in parts] == [len(dist.shard(m, r, world)) for r in range(world)]
    full = assemble(parts)
    assert full.scale == want_sc
    assert np.array_equal(full.to_words(), want)
    one = OutputShardedDense(ctx, wts, 0, 1)
    assert np.array_equal(one.forward(xt).to_words(), want)  # world 1: local + gather path
    chunked = OutputShardedDense(ctx, wts, 0, 1, chunks=3)  # overlapped-gather path
    assert np.array_equal(chunked.forward(xt).to_words(), want)
