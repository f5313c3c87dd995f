# SPDX-License-Identifier: Apache-2.0
"""Output-neuron sharding of a dense layer across GPUs (BASELINE config 5b).

Every rank holds all K input ciphertexts; rank r evaluates the output neurons
`dist.shard(M, r, G)` (a column block of W, so each output residue is computed by
exactly one rank with the same arithmetic as the unsharded layer), then the output
ciphertexts are all-gathered as raw residue words.  The gather is a byte copy, so the
sharded result is bit-identical to `henet::execute` on the whole layer.

The reference has no multi-device executor; the per-rank computation is the
reference's `eval_dot` (henet/graph.hpp:935-954) on a column slice, and the plan is
`plan_rescaling` (henet/graph.hpp:504-584) with the harness's terminal-rescale patch
(c1/c5b: one rescale per output).
"""
from __future__ import annotations

import json
from typing import List, Optional, Sequence

from . import dist
from . import henet as H


def patch_terminal_rescale(chain: Sequence[int], default_scale: float, manifest: str, plan: H.RescalePlan,
                           out_counts: dict) -> H.RescalePlan:
    """The harness's plan patch for configs 1 / 5b: every Dot/Convolution the lazy planner
    leaves at Skip rescales after accumulation (level - 1, scale * s / q_{level-1}), and
    pass-through Reshape/Output nodes follow.  Same rule as oracle/ref/ref_capi.cpp
    `patch_terminal_rescale`.  out_counts: node id -> output element count."""
    s = float(default_scale)
    nodes = {}
    planned = plan.planned_rescale_ops
    for n in json.loads(manifest)["nodes"]:
        nid, op = n["id"], n["op"]
        dec, lin, lout, sc = plan.node(nid)
        ins = n.get("inputs", [])
        if op in ("Dot", "Convolution") and dec == H.SKIP:
            _, _, _, in_sc = nodes[ins[0]]
            dec, lout, sc = H.RESCALE_AFTER, lin - 1, (in_sc * s) / float(chain[lin - 1])
            planned += out_counts[nid]
        elif op in ("Reshape", "Output") and ins:
            _, _, p_out, p_sc = nodes[ins[0]]
            lin, lout, sc = p_out, p_out, p_sc
        nodes[nid] = (dec, lin, lout, sc)
    return H.RescalePlan.from_nodes(H.RESCALE_LAZY, planned, nodes)


def gather_rows(local, total: int, world: int, group=None):
    """All-gather row blocks of a 2-D tensor partitioned by `dist.shard(total, r, world)`.

    local: this rank's rows (torch tensor, CUDA for NCCL or CPU for gloo).  Returns the
    (total, cols) tensor, identical on every rank.  Equal blocks are gathered straight
    into the result; unequal ones through a padded staging buffer."""
    import torch
    import torch.distributed as tdist
    cols = local.shape[1]
    counts = [len(dist.shard(total, r, world)) for r in range(world)]
    width = max(counts)
    if world == 1:
        return local.clone()
    send = local
    if local.shape[0] != width:
        send = torch.zeros((width, cols), dtype=local.dtype, device=local.device)
        send[: local.shape[0]] = local
    parts = [torch.empty((width, cols), dtype=local.dtype, device=local.device) for _ in range(world)]
    tdist.all_gather(parts, send.contiguous(), group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def gather_chunk_into(dst, local, blocks, group=None):
    """All-gather one chunk: `blocks[r]` is the global row range rank r contributes (its
    `local` rows on this rank); every rank's rows land in place in `dst` (total, cols)."""
    import torch
    import torch.distributed as tdist
    world = len(blocks)
    if world == 1:
        dst[blocks[0].start:blocks[0].stop].copy_(local)
        return
    width = max(len(b) for b in blocks)
    cols = dst.shape[1]
    send = local
    if local.shape[0] != width:
        send = torch.zeros((width, cols), dtype=local.dtype, device=local.device)
        send[: local.shape[0]] = local
    parts = torch.empty((world * width, cols), dtype=local.dtype, device=local.device)
    tdist.all_gather_into_tensor(parts, send.contiguous(), group=group)
    for r, b in enumerate(blocks):
        dst[b.start:b.stop].copy_(parts[r * width: r * width + len(b)])


class OutputShardedDense:
    """One dense layer K -> M (W row-major K x M, f32) split by output neuron over
    `world` ranks; `forward` returns all M output ciphertexts on every rank."""

    def __init__(self, ctx: H.CkksContext, weights, rank: int, world: int, preset: str = "P14",
                 rescale: bool = True, bias: Optional[Sequence[float]] = None, chunks: int = 1):
        """chunks > 1: the rank's neurons are evaluated in `chunks` column blocks, and each
        block's all-gather (torch's stream) overlaps the next block's evaluation (the
        context stream).  Chunks of >= 128 neurons cost no extra input traffic: the
        tensor-core kernel already re-reads the inputs per 128-neuron tile."""
        import numpy as np
        self.ctx, self.rank, self.world = ctx, rank, world
        w = np.asarray(weights, dtype=np.float32)
        self.K, self.M = w.shape
        self.rows = dist.shard(self.M, rank, world)
        self.blocks = dist.chunk_shards(self.M, world, max(1, chunks))
        b = np.asarray(bias, np.float32) if bias is not None else None
        self.parts = [self._build(w, b, blk[rank], preset, rescale, f"c{c}") for c, blk in enumerate(self.blocks)]
        self.model, self.plan = self.parts[0] if len(self.parts) == 1 else (None, None)

    def _build(self, w, b, rows, preset, rescale, tag):
        from . import workloads as Wk
        blob = Wk.Blob()
        blob.add("fc_w", [self.K, len(rows)], w[:, rows.start:rows.stop])
        nodes = [Wk._node("input", "Input", attrs={"shape": [self.K]}),
                 Wk._node("fc", "Dot", ["input"], weight_ref="fc_w"),
                 Wk._node("out", "Output", ["fc"])]
        if b is not None:
            blob.add("fc_b", [len(rows)], b[rows.start:rows.stop])
            nodes[1] = Wk._node("fc", "Dot", ["input"], weight_ref="fc_w", bias_ref="fc_b")
        manifest = json.dumps({"name": f"dense-{self.K}-{self.M}-shard{self.rank}of{self.world}-{tag}",
                               "packing": "real", "preset": preset, "weights": blob.table, "nodes": nodes})
        model = H.PlainModel.load(manifest, blob.bytes())
        plan = H.RescalePlan.plan(self.ctx, model)
        if rescale:
            n = len(rows)
            plan = patch_terminal_rescale(self.ctx.chain, self.ctx.default_scale, manifest, plan,
                                          {"input": self.K, "fc": n, "out": n})
        return model, plan

    def local(self, x: H.CipherTensor) -> H.CipherTensor:
        """This rank's output ciphertexts (rows `self.rows`; single-chunk layers)."""
        assert len(self.parts) == 1, "local() is for single-chunk layers; use forward()"
        return H.execute(self.ctx, self.model, self.plan, x)

    def forward(self, x: H.CipherTensor, group=None) -> H.CipherTensor:
        if len(self.parts) == 1:
            return self.gather(self.local(x), group)
        import torch
        dev = self.ctx.device
        ext = torch.cuda.ExternalStream(self.ctx.stream(), device=dev)
        cur = torch.cuda.current_stream(dev)
        full = None
        keep = []
        for c, (model, plan) in enumerate(self.parts):
            y = H.execute(self.ctx, model, plan, x)  # enqueued on the context stream
            if full is None:
                cnt, polys, level, scale, packing = y.info()
                full = H.CipherTensor(self.ctx, self.M, polys, level, scale, packing, shape=[self.M])
            ev = torch.cuda.Event()
            ev.record(ext)
            cur.wait_event(ev)  # chunk c's gather waits for chunk c only
            gather_chunk_into(full.torch_view(dev), y.torch_view(dev), self.blocks[c], group)
            keep.append(y)  # freed after the gathers (ext waits on cur below)
        ext.wait_stream(cur)
        del keep
        return full

    def gather_native(self, y: H.CipherTensor, comm: "H.Communicator") -> H.CipherTensor:
        """All-gather through the C ABI (hg_allgather_tensor, NCCL inside the library, on the
        context stream): the same byte copy as gather(), without torch."""
        assert comm.nranks == self.world and comm.rank == self.rank
        assert list(H.shard_range(self.M, self.rank, self.world)) == list(self.rows)
        return comm.allgather(y, self.M)

    def gather(self, y: H.CipherTensor, group=None) -> H.CipherTensor:
        """All-gather the output ciphertexts.  Stream-ordered, no host synchronisation:
        the collective runs on torch's current stream after the context stream's work,
        and later context work (downloads, frees of `y`) waits for it."""
        import torch
        cnt, polys, level, scale, packing = y.info()
        dev = self.ctx.device
        full = H.CipherTensor(self.ctx, self.M, polys, level, scale, packing, shape=[self.M])
        ext = torch.cuda.ExternalStream(self.ctx.stream(), device=dev)
        cur = torch.cuda.current_stream(dev)
        cur.wait_stream(ext)
        dst, src = full.torch_view(dev), y.torch_view(dev)
        counts = [len(dist.shard(self.M, r, self.world)) for r in range(self.world)]
        if self.world > 1 and len(set(counts)) == 1:
            import torch.distributed as tdist
            tdist.all_gather_into_tensor(dst, src, group=group)  # straight into place
        else:
            dst.copy_(gather_rows(src, self.M, self.world, group))
        ext.wait_stream(cur)
        return full


def assemble(parts: List[H.CipherTensor]) -> H.CipherTensor:
    """Concatenate per-shard output tensors in rank order (single-process check of the
    sharding: the same layout the all-gather produces)."""
    import torch
    first = parts[0]
    cnt = sum(p.count for p in parts)
    _, polys, level, scale, packing = first.info()
    full = H.CipherTensor(first.ctx, cnt, polys, level, scale, packing, shape=[cnt])
    dev = first.ctx.device
    ext = torch.cuda.ExternalStream(first.ctx.stream(), device=dev)
    cur = torch.cuda.current_stream(dev)
    cur.wait_stream(ext)
    torch.cat([p.torch_view(dev) for p in parts], dim=0, out=full.torch_view(dev))
    ext.wait_stream(cur)
    return full
