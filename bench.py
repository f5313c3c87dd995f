#!/usr/bin/env python
# SPDX-License-Identifier: Apache-2.0
"""Benchmark of the B200 encrypted-inference hot path (BASELINE.json metric).

One step = one batch of 4096 encrypted 28x28 images (batch-axis packed, one
image per slot) through the full CryptoNets-shaped network of BASELINE config 2
(conv 5x5/2 -> square+relin+rescale -> dense 845->100 -> square -> dense
100->10, lazy rescaling), N=8192, 7-prime chain, scale 2^24, executed by
libhenet_b200.so's graph executor (hg_execute).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun, one process per GPU): independent 4096-image batches per
rank (config 5a: batch sharding, no collective), weak scaling; time = max over
ranks of the device time.

`value` is whole-job images/s with inputs resident in HBM (input tensor 308 MB >
126 MB L2, so every step streams it from HBM).  `e2e` is the same metric through
the C ABI with host buffers: per step the reference-format u64 input words are
uploaded from pinned host memory (hg_tensor_upload), the graph executed, and the
logits downloaded (hg_tensor_download).  Inputs are seeded uniform residues mod
q_i: fresh RLWE ciphertexts are uniform, so the work is identical to real
encryptions (parity on real encryptions is covered by tests/).

--impl reference times the reference's own CPU implementation (the unmodified
henet headers compiled into oracle/_ref/libhenet_ref.so, execute() with all host
threads) on the same network, parameters and batch.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted images/sec, CryptoNets-shaped N=8192 net; % of HBM/INT32 roofline"
IMAGES_PER_STEP = 4096


def _h2d_bytes(words, host_narrow):
    """Bytes hg_tensor_upload moves over PCIe: with host narrowing, the last
    HG_UPLOAD_DIRECT_FRAC of the ciphertexts (default 0.15, hg_upload.cpp
    upload_direct_fraction) cross raw as u64 and the rest as packed u32."""
    if not host_narrow:
        return int(words.nbytes)
    f = min(1.0, max(0.0, float(os.environ.get("HG_UPLOAD_DIRECT_FRAC", "0.15"))))
    count = words.shape[0]
    per_ct = words.nbytes // count
    direct = int(count * f)
    return int((count - direct) * per_ct // 2 + direct * per_ct)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lanes", type=int, default=2,
                    help="c2: independent batches in flight per GPU (contexts / streams the steps alternate over)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c5b", "c4", "c1", "c3"],
                    help="c2 (default, the BASELINE metric); c1: the dense 845->100 layer; c3: CryptoNets-ReLU "
                         "under complex packing with GPU refreshes; c4: the MobileNetV2 block (tiled); c5b: wide "
                         "dense 4096->4096 at N=16384, output-sharded over the ranks with an NCCL all-gather")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_config(n_gpus):
    return {
        "workload": "c2 CryptoNets-shaped net: conv5x5/2(5)->sq->fc845x100->sq->fc100x10, lazy rescale",
        "images_per_step_per_gpu": IMAGES_PER_STEP,
        "ring": "N=8192, chain [30,24x5]+30-bit special, scale 2^24",
        "input_ciphertexts": 784,
        "l2": "input tensor 308 MB > 126 MB L2 (no flush needed)",
        "parallelism": f"batch-sharded replicas x{n_gpus} (config 5a), no collective",
    }


# ---------------------------------------------------------------------------
# Clock sampling during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    def __init__(self, device):
        self.f = tempfile.NamedTemporaryFile(prefix="clocks", suffix=".csv", delete=False)
        if os.environ.get("HG_BENCH_NO_CLOCKS"):  # diagnostic runs only: no clock evidence
            self.p = None
            return
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# Algorithmic work model: IMAD-class ops (modular MAC = 1,
# NTT butterfly = 3, modmul = 3) and compulsory HBM bytes (u32 residues).
# ---------------------------------------------------------------------------
def work_model(n=8192):
    """Algorithmic work of one c2 step per kernel: (modmul, mac, bytes).

    modmul = Shoup modular products (one per NTT butterfly + one per point-wise
    product), the unit the NTT-family kernels are bound by: each is IMAD.HI + 2 IMAD,
    and IMAD.HI issues at a quarter of the FFMA rate on sm_100 (scripts/int_pipe_probe.cu).
    mac = 32x32->64-bit multiply-accumulates (IMAD.WIDE) of the MAC kernels.
    bytes = compulsory HBM traffic (inputs read once, outputs written once)."""
    import math
    logn = int(math.log2(n))
    bf = n // 2 * logn  # butterflies per transform
    W = 4               # bytes per residue
    m = {}

    def add(name, modmul=0.0, mac=0.0, byts=0.0):
        o = m.get(name, (0.0, 0.0, 0.0))
        m[name] = (o[0] + modmul, o[1] + mac, o[2] + byts)

    # conv1: 784 inputs at level 6 -> 845 outputs, 20480 valid taps
    L = 6
    add("k_mac_conv", mac=20480 * 2 * L * n, byts=(784 + 845) * 2 * L * n * W)
    # rescale after conv1: 845 cts at level 6 -> 5; after fc1: 100 cts 4 -> 3
    # (per poly: INTT of the dropped limb + NTT of l-1 corrections, then l-1 scalings)
    for C_, l in ((845, 6), (100, 4)):
        add("k_rescale", modmul=C_ * (2 * l * bf + 2 * (l - 1) * n), byts=C_ * (2 * l + 2 * (l - 1)) * n * W)
    # square+relin+rescale: act1 845 cts at level 5, act2 100 cts at level 3
    for C_, l in ((845, 5), (100, 3)):
        add("k_relin_digits", modmul=C_ * (l * bf + l * n), byts=C_ * 2 * l * n * W)
        key_bytes = 2 * l * (l + 1) * n * 8
        # l(l-1) + l forward transforms (digit j under prime t != j, and the special prime),
        # 2 inverse transforms of the special accumulators, 2 key products per digit/limb
        add("k_relin_keysw", modmul=C_ * ((l * l + 2) * bf + 2 * l * (l + 1) * n),
            byts=C_ * (l * n * W + 2 * l * n * W + 2 * n * W) + key_bytes)
        # mod-down with the rescale merged: per polynomial l-1 forward transforms (kept limbs)
        # and one inverse (the dropped limb, INTT(d + acc P^-1) - cps P^-1)
        add("k_relin_moddown", modmul=C_ * (2 * l * bf + (6 * l - 2) * n),
            byts=C_ * (2 * l * n * W + 2 * l * n * W + 2 * n * W + 2 * (l - 1) * n * W))
    # fc1 845 -> 100 at level 4, fc2 100 -> 10 at level 2
    dense_macs = 845 * 100 * 2 * 4 * n + 100 * 10 * 2 * 2 * n
    dense_bytes = (845 + 100) * 2 * 4 * n * W + (100 + 10) * 2 * 2 * n * W
    add("k_mac_dense", mac=dense_macs, byts=dense_bytes)
    add("k_mac_dense_tc", mac=dense_macs, byts=dense_bytes)
    return m


def tc_work():
    """int8 tensor-core MACs the byte-plane contraction needs (fc1 + fc2 of c2):
    planes^2 byte products per modular MAC, planes = 4 for the 30-bit limb 0, 3 else."""
    n = 8192
    per_limb = lambda K, M, L: sum((16 if i == 0 else 9) for i in range(L)) * K * M * 2 * n
    return per_limb(845, 100, 4) + per_limb(100, 10, 2)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# Reference arm
# ---------------------------------------------------------------------------
def reference_run(args, ws, rank):
    from oracle import refbind as R
    from paper_1908_04172_b200 import workloads as Wk

    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhenet_ref.so not built"}))
        return 0
    p = Wk.N8192
    wl = Wk.cryptonets()
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(7, True)
    imgs = Wk.synthetic_images(wl.input_shape, wl.batch, 1)
    words, sc = ref.encrypt_tensor(keys, imgs, 2, threads=cores)
    # each step is one full 4096-image batch (~5-15 s on the host cores); cap the
    # run so --steps K --warmup W finishes within a few minutes.
    warm = min(args.warmup, 1)
    steps = max(1, min(args.steps, 5))
    for _ in range(warm):
        ref.execute(keys, wl.manifest, wl.blob, words, sc, threads=cores)
    times = []
    for _ in range(steps):
        _, _, st = ref.execute(keys, wl.manifest, wl.blob, words, sc, threads=cores)
        times.append(st["exec_ms"])
    ms = sum(times) / len(times)
    v = IMAGES_PER_STEP / (ms / 1e3)
    unit = "images/s"
    line = {
        "metric": METRIC, "value": v, "unit": unit, "impl": "reference", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64 (RNS residues)", "data": "synthetic (seeded uniform pixels, real encryptions)",
        "config": workload_config(1) | {"parallelism": f"reference execute() on {cores} host threads"},
        "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "reference",
                         "sample": f"{steps} x full 4096-image batch through henet::execute (oracle/_ref)"},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline_sample():
    """The reference CPU path timed on this host (rank 0, N=1): one full batch."""
    from oracle import refbind as R
    from paper_1908_04172_b200 import workloads as Wk
    if not R.available():
        return None
    cores = os.cpu_count() or 1
    p = Wk.N8192
    wl = Wk.cryptonets()
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(7, True)
    imgs = Wk.synthetic_images(wl.input_shape, wl.batch, 1)
    words, sc = ref.encrypt_tensor(keys, imgs, 2, threads=cores)
    _, _, st = ref.execute(keys, wl.manifest, wl.blob, words, sc, threads=cores)
    ms = st["exec_ms"]
    return {"value": IMAGES_PER_STEP / (ms / 1e3), "unit": "images/s", "cores": cores, "kind": "reference",
            "sample": "one 4096-image batch of the same network through henet::execute (oracle/_ref), "
                      f"{ms / 1e3:.1f} s"}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def bind_gpu_numa(local):
    """Restrict this process to the CPUs of the GPU's NUMA node (sysfs), so pinned host
    buffers are first-touched next to the GPU's PCIe root: host<->device copies then do not
    cross the socket interconnect.  Returns the node, or None when unknown."""
    import torch
    try:
        pr = torch.cuda.get_device_properties(local)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/numa_node") as f:
            node = int(f.read().strip())
        if node < 0:
            return None
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return node
    except (OSError, ValueError, AttributeError):
        pass
    return None


def b200_run(args, ws, rank, local):
    import torch
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200 import workloads as Wk

    torch.cuda.set_device(local)
    numa = bind_gpu_numa(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p = Wk.N8192
    wl = Wk.cryptonets()
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"], device=local)
    L = len(p["chain"])
    rng = np.random.default_rng(100 + rank)
    key_words = np.empty((L, 2, L + 1, p["n"]), dtype=np.uint64)
    for t, q in enumerate(p["chain"] + [p["special"]]):
        key_words[:, :, t, :] = rng.integers(0, q, size=(L, 2, p["n"]), dtype=np.uint64)
    rk = H.RelinKey(ctx, key_words)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    plan = H.RescalePlan.plan(ctx, model)
    words = Wk.random_ciphertexts(p, wl.input_count, seed=7 + rank)
    inp = H.CipherTensor.from_words(ctx, words, p["scale"], shape=wl.input_shape)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=local)

    def step():
        return H.execute(ctx, model, plan, inp, rk)

    # Lanes: config 5a's batches are independent, so a GPU may keep more than one in flight.
    # Lane 0 is the context above; every further lane is another context (own stream, own copy
    # of the resident inputs and key) and the timed steps alternate over the lanes, so one
    # batch's latency-bound kernels (convolution, Dot) share the SMs with another's transforms.
    n_lanes = max(1, args.lanes)
    lanes = [(ctx, rk, plan, inp, stream)]
    for _ in range(1, n_lanes):
        c2_ = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"], device=local)
        lanes.append((c2_, H.RelinKey(c2_, key_words), H.RescalePlan.plan(c2_, model),
                      H.CipherTensor.from_words(c2_, words, p["scale"], shape=wl.input_shape),
                      torch.cuda.ExternalStream(c2_.stream(), device=local)))

    def lane_step(i):
        c_, rk_, plan_, inp_, _ = lanes[i % len(lanes)]
        return H.execute(c_, model, plan_, inp_, rk_)

    def timed_steps(nl, k):
        """k steps alternating over the first nl lanes; device time between an event on lane
        0's stream (all streams idle) and one recorded there after every lane's work."""
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        l0 = sum(l[0].launch_count() for l in lanes)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for l in lanes[1:nl]:
            l[4].wait_event(e0)
        outs = []
        marks = []  # per-step completion events (each on its lane's stream)
        calls = []  # host time of every execute call
        for i in range(k):
            c_, rk_, plan_, inp_, st_ = lanes[i % nl]
            tc = time.perf_counter()
            outs.append(H.execute(c_, model, plan_, inp_, rk_))
            calls.append((time.perf_counter() - tc) * 1e3)
            if len(outs) > 2 * nl:
                outs.pop(0)
            m = torch.cuda.Event(enable_timing=True)
            m.record(st_)
            marks.append(m)
        for l in lanes[1:nl]:
            ev = torch.cuda.Event()
            ev.record(l[4])
            stream.wait_event(ev)
        e1.record(stream)
        e1.synchronize()
        nlaunch = sum(l[0].launch_count() for l in lanes) - l0
        dev = e0.elapsed_time(e1)
        # completion-to-completion intervals: their median is the steady step time, a large
        # maximum a stall (a host hiccup that let the launch queue run dry)
        done = sorted(e0.elapsed_time(m) for m in marks)
        gaps = [b - a for a, b in zip([0.0] + done[:-1], done)]
        timed_steps.intervals = {"median_ms": statistics.median(gaps), "max_ms": max(gaps),
                                 "ms": [round(g, 3) for g in gaps] if len(gaps) <= 64 else None,
                                 "host_call_ms": [round(c, 3) for c in calls] if len(calls) <= 64 else None}
        host = (time.perf_counter() - t0) * 1e3
        torch.cuda.synchronize()
        t = torch.tensor([dev], dtype=torch.float64, device=f"cuda:{local}")
        if ws > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item()), host, nlaunch, outs[-1]

    clocks = Clocks(local)  # started before warm-up so nvidia-smi start-up is not inside the timed region
    for i in range(max(args.warmup, 3) * n_lanes):
        out = lane_step(i)
    torch.cuda.synchronize()
    time.sleep(0.5)
    for i in range(2 * n_lanes):
        out = lane_step(i)
    torch.cuda.synchronize()
    max_ms, host_ms, launches, out = timed_steps(n_lanes, args.steps)
    step_intervals = timed_steps.intervals
    clk = clocks.stop()
    ms_per_step = max_ms / args.steps
    value = IMAGES_PER_STEP * ws / (ms_per_step / 1e3)
    one_lane = None
    if n_lanes > 1:
        # the same K steps with one batch in flight (lane 0 only), reported beside the value
        ms1, _, _, out1 = timed_steps(1, args.steps)
        one_lane = {"ms_per_step": ms1 / args.steps, "value": IMAGES_PER_STEP * ws / (ms1 / args.steps / 1e3)}
        assert np.array_equal(out1.to_words(), out.to_words()), "lanes disagree"
    out_words = out.to_words()
    assert out_words.shape == (10, 2, 2, p["n"])

    # ---- e2e through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        # End to end through the C ABI with host buffers.  Every step uploads its own 617 MB of
        # reference-format u64 words from pinned memory (hg_tensor_upload: residue validation +
        # narrowing to u32 by host threads, chunk by chunk, each chunk's H2D overlapping the
        # packing of the next -- 308 MB over PCIe; HG_UPLOAD_HOST_NARROW=0 copies the u64 words
        # and narrows on the GPU), executes, and downloads its logits (hg_tensor_download).  As a
        # serving loop would, step i+1's upload runs on a second stream from a helper thread
        # while step i executes (ctypes calls release the GIL); the sequential loop is reported
        # beside it.
        import concurrent.futures
        import ctypes
        host_in = torch.empty(words.size, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        host_in[:] = words.reshape(-1)
        host_in = host_in.reshape(words.shape)
        out_host = torch.empty(10 * 2 * 2 * p["n"], dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        bufs = [H.CipherTensor(ctx, wl.input_count, 2, L, p["scale"], shape=wl.input_shape) for _ in range(2)]
        from paper_1908_04172_b200._lib import check, lib
        copy_stream = torch.cuda.Stream(device=local)
        used = [torch.cuda.Event(), torch.cuda.Event()]

        up_ms, step_ms = [], []

        def upload(k, strm=None):
            t0 = time.perf_counter()
            if strm is not None:
                copy_stream.wait_event(used[k])  # the step that last read buffer k is done with it
            check(lib.hg_tensor_upload(bufs[k].handle, H._ptr(host_in),
                                       ctypes.c_void_p(strm.cuda_stream) if strm is not None else None))
            up_ms.append((time.perf_counter() - t0) * 1e3)

        def run_step(k):
            t0 = time.perf_counter()
            o = H.execute(ctx, model, plan, bufs[k], rk)
            used[k].record(stream)
            check(lib.hg_tensor_download(o.handle, H._ptr(out_host), None))
            step_ms.append((time.perf_counter() - t0) * 1e3)

        def sequential(n):
            for _ in range(n):
                upload(0)
                run_step(0)

        def pipelined(n, pool):
            fut = pool.submit(upload, 0, copy_stream)
            for i in range(n):
                fut.result()
                if i + 1 < n:
                    fut = pool.submit(upload, (i + 1) % 2, copy_stream)
                run_step(i % 2)

        def timed(fn, n):
            if ws > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            fn(n)
            f1.record(stream)
            f1.synchronize()
            ms = max(f0.elapsed_time(f1), (time.perf_counter() - t0) * 1e3) / n
            te = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
            if ws > 1:
                torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
            return float(te.item())

        host_narrow = os.environ.get("HG_UPLOAD_HOST_NARROW", "1") != "0"
        n_e2e = max(10, args.steps)
        # three trials of each loop, medians reported (the helper thread makes single trials
        # sensitive to host scheduling)
        with concurrent.futures.ThreadPoolExecutor(1) as pool:
            # warm-up: both buffers and both streams, and on a fresh box the host side itself
            # (packer threads, pinned pages, CPU clocks): the first 10-20 loop steps of a
            # process ran 10-30% slower than the rest (profiles/r3_experiments.md)
            pipelined(max(args.warmup, 3) + 17, pool)
            up_ms.clear()
            step_ms.clear()
            pipe_trials = [timed(lambda n: pipelined(n, pool), n_e2e) for _ in range(3)]
            pipe_up, pipe_step = statistics.median(up_ms), statistics.median(step_ms)
        up_ms.clear()
        step_ms.clear()
        seq_trials = [timed(sequential, n_e2e) for _ in range(3)]
        seq_up, seq_step = statistics.median(up_ms), statistics.median(step_ms)
        e_ms, seq_ms = statistics.median(pipe_trials), statistics.median(seq_trials)
        # the bytes the library's last upload actually put on the bus (3-byte words for the
        # 24-bit primes when the host packs them, + the raw share); the model as a fallback
        import ctypes
        lib_h2d = ctypes.c_uint64(0)
        H.lib.hg_last_upload_h2d_bytes(ctypes.byref(lib_h2d))
        h2d_bytes = int(lib_h2d.value) if (host_narrow and lib_h2d.value) else _h2d_bytes(words, host_narrow)
        e2e = {"value": IMAGES_PER_STEP * ws / (e_ms / 1e3), "unit": "images/s",
               "h2d_bytes_per_step": h2d_bytes,
               "d2h_bytes_per_step": int(out_host.nbytes),
               "host_input_bytes_per_step": int(words.nbytes),
               "ms_per_step": e_ms, "steps": n_e2e, "trials_ms_per_step": pipe_trials,
               "sequential": {"value": IMAGES_PER_STEP * ws / (seq_ms / 1e3), "ms_per_step": seq_ms,
                              "trials_ms_per_step": seq_trials},
               "host_numa_node": numa,
               "host_ms_median": {"pipelined": {"upload": pipe_up, "execute_download": pipe_step},
                                  "sequential": {"upload": seq_up, "execute_download": seq_step}},
               "path": "hg_tensor_upload(u64 host words, " +
                       ("validated and packed to u32 by host threads, chunked H2D" if host_narrow else
                        "u64 H2D, GPU narrowing") +
                       ", second stream, next step) + hg_execute + hg_tensor_download, double-buffered"}

    # ---- per-kernel roofline pass (CUDA events around every launch) ----
    H.prof_enable(True)
    n_prof = 3
    for _ in range(n_prof):
        step()
    ctx.synchronize()
    H.prof_enable(False)
    prof = H.prof_report()
    hbm_gbs, hbm_src = load_peaks()
    shoup_peak = H.bench_int_peak(local, 3)  # Shoup modular products / s
    wide_peak = H.bench_int_peak(local, 1)   # IMAD.WIDE MACs / s
    imad_peak = H.bench_int_peak(local, 0)
    model_w = work_model(p["n"])
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    i8_peak = H.bench_int_peak(local, 4)  # measured int8 tcgen05 MMA MAC/s (raw, static operands)
    kernels = {}
    total_ms = sum(v["ms"] for v in prof.values()) / n_prof
    for name, v in prof.items():
        ms = v["ms"] / n_prof
        mm, mac, byts = model_w.get(name, (0.0, 0.0, 0.0))
        t_int = (mm / shoup_peak + mac / wide_peak) * 1e3
        t_hbm = byts / (hbm_gbs * 1e9) * 1e3
        k = {"ms_per_step": ms, "launches_per_step": v["launches"] / n_prof,
             "share": ms / total_ms if total_ms else 0,
             "modmul_t_per_s": mm / (ms * 1e-3) / 1e12 if ms else 0,
             "mac_t_per_s": mac / (ms * 1e-3) / 1e12 if ms else 0,
             "hbm_gbs": byts / (ms * 1e-3) / 1e9 if ms else 0,
             "int32_floor_ms": t_int, "hbm_floor_ms": t_hbm,
             "roofline_frac": max(t_int, t_hbm) / ms if ms else 0,
             "bound": "int32" if t_int >= t_hbm else "hbm"}
        if name == "k_mac_dense_tc":
            # the contraction runs on the tensor cores: its roofline is int8 MMA throughput
            t_tc = tc_work() / i8_peak * 1e3
            k.update({"bound": "tensor", "tensor_int8_macs_per_s": tc_work() / (ms * 1e-3),
                      "tensor_floor_ms": t_tc, "roofline_frac": max(t_tc, t_hbm) / ms if ms else 0,
                      "tensor_peak_note": "measured raw tcgen05.mma.kind::i8 rate (hg_bench_int_peak kind 4)"})
        kernels[name] = k
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    dk = kernels[dom]
    mm, mac, byts = model_w.get(dom, (0.0, 0.0, 0.0))
    if dk["bound"] == "int32" and mm >= mac:
        roof = {"bound": "int32", "kernel": dom, "achieved": dk["modmul_t_per_s"], "peak": shoup_peak / 1e12,
                "unit": "T modmul/s (Shoup: IMAD.HI + 2 IMAD)", "frac": dk["modmul_t_per_s"] / (shoup_peak / 1e12),
                "peak_source": "measured register-only Shoup-product probe (hg_bench_int_peak kind 3) on this GPU",
                "imad_peak": imad_peak / 1e12, "imad_wide_peak": wide_peak / 1e12,
                "hbm_gbs_achieved": dk["hbm_gbs"], "hbm_peak": hbm_gbs, "traffic": None}
    elif dk["bound"] == "int32":
        roof = {"bound": "int32", "kernel": dom, "achieved": dk["mac_t_per_s"], "peak": wide_peak / 1e12,
                "unit": "T MAC/s (IMAD.WIDE)", "frac": dk["mac_t_per_s"] / (wide_peak / 1e12),
                "peak_source": "measured register-only IMAD.WIDE probe (hg_bench_int_peak kind 1) on this GPU",
                "hbm_gbs_achieved": dk["hbm_gbs"], "hbm_peak": hbm_gbs, "traffic": None}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": dk["hbm_gbs"], "peak": hbm_gbs, "unit": "GB/s",
                "frac": dk["hbm_gbs"] / hbm_gbs, "peak_source": hbm_src, "traffic": None}
    roof["algorithmic_per_step"] = {"modmul": mm, "mac": mac, "hbm_bytes": byts}
    # measured DRAM traffic of the dominant kernel's first launch (act1 for the key switch),
    # from the committed `ncu --set full` capture summarised in profiles/ncu_traffic.json
    try:
        nt = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        hits = {k: v for k, v in nt["kernels"].items() if k.split("<")[0].split("(")[0] == dom}
        if hits:
            roof["traffic"] = sum(v["dram_bytes_read"] + v["dram_bytes_write"] for v in hits.values())
            roof["traffic_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one launch of " +
                                    ", ".join(sorted(hits)) + "; " + nt["source"])
    except (OSError, ValueError, KeyError):
        pass
    whole_t = sum(max(k["int32_floor_ms"] if k["bound"] != "tensor" else k["tensor_floor_ms"], k["hbm_floor_ms"])
                  for k in kernels.values())
    roof["whole_step"] = {"floor_ms": whole_t, "measured_ms": ms_per_step,
                          "frac": whole_t / ms_per_step if ms_per_step else 0}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample()
        except Exception as e:  # reported, not fatal
            cpu = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32 (RNS residues mod 24/30-bit primes)",
            "data": "synthetic (seeded uniform residues = fresh-ciphertext distribution; random relin key)",
            "config": workload_config(ws), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps, "clocks": clk,
            "host_wall_ms_per_step": host_ms / args.steps,
            "kernels": kernels,
        }
        line["config"] = line["config"] | {
            "batches_in_flight": n_lanes,
            "lanes": f"the {args.steps} timed steps alternate over {n_lanes} contexts (one stream each) on the GPU; "
                     "every step is one full 4096-image batch"}
        line["step_completion_intervals"] = step_intervals
        if one_lane:
            line["one_batch_in_flight"] = one_lane
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# Config 5b: wide dense layer, output-neuron sharded
# ---------------------------------------------------------------------------
C5B_K = C5B_M = 4096
C5B_IMAGES = 8192  # images per ciphertext at N=16384 (one pass of the layer)
C5B_METRIC = "encrypted images/sec, c5b wide dense 4096->4096 N=16384, output-sharded + all-gather"


def c5b_config(ws):
    return {"workload": f"c5b wide dense {C5B_K}->{C5B_M}, one rescale per output (patched plan, as c1)",
            "ring": "N=16384, chain [40,30x7]+40-bit special, scale 2^30 (u64 residue storage)",
            "images_per_step": C5B_IMAGES, "input_ciphertexts": C5B_K,
            "l2": "input tensor 8.6 GB > 126 MB L2 (no flush needed)",
            "parallelism": f"output-neuron sharded x{ws}, all inputs on every rank, NCCL all-gather of outputs"}


def c5b_work(n=16384, L=8):
    """(mac, bytes) of the layer: K*M*2*L*N MACs (limb 0 40-bit: 128-bit MACs); u64 words."""
    return C5B_K * C5B_M * 2 * L * n, (C5B_K * 2 * L + C5B_M * 2 * (L - 1)) * n * 8


def c5b_reference_sample(cores):
    """Reference execute() on a K_s x M_s slice of the layer (same parameters, per-tap cost
    is uniform), extrapolated to K x M (subset of outputs, labelled)."""
    from oracle import refbind as R
    from paper_1908_04172_b200 import workloads as Wk
    p = Wk.N16384
    ks, ms = 128, max(cores, 4)
    wl = Wk.wide_dense(k=ks, m=ms)
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    x = Wk.random_ciphertexts(p, ks, seed=31)
    _, _, st = ref.execute(None, wl.manifest, wl.blob, x, p["scale"], patch=True, threads=cores)
    ms_full = st["exec_ms"] * (C5B_K * C5B_M) / (ks * ms)
    return C5B_IMAGES / (ms_full / 1e3), f"K={ks} x M={ms} slice of the layer through henet::execute " \
        f"(oracle/_ref, {st['exec_ms'] / 1e3:.1f} s), extrapolated x{C5B_K * C5B_M // (ks * ms)} to 4096x4096"


def c5b_run(args, ws, rank, local):
    import torch
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200 import workloads as Wk
    from paper_1908_04172_b200.sharded import OutputShardedDense

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p = Wk.N16384
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"], device=local)
    L = len(p["chain"])
    # ranks > 1: 4 column chunks per rank, each chunk's NCCL all-gather overlapping the next
    # chunk's evaluation (each chunk is >= 128 neurons: no extra input traffic)
    layer = OutputShardedDense(ctx, Wk.wide_dense_weights(k=C5B_K, m=C5B_M), rank, ws, chunks=4 if ws > 1 else 1)
    # inputs generated on the device (seeded uniform residues per limb; 8.6 GB)
    x = H.CipherTensor(ctx, C5B_K, 2, L, p["scale"], shape=[C5B_K])
    ctx.synchronize()
    xv = x.torch_view(local).view(C5B_K, 2, L, p["n"])
    g = torch.Generator(device=f"cuda:{local}")
    g.manual_seed(41)  # identical inputs on every rank
    for i, q in enumerate(p["chain"]):
        xv[:, :, i, :] = torch.randint(0, q, (C5B_K, 2, p["n"]), device=f"cuda:{local}", dtype=torch.int64,
                                       generator=g)
    torch.cuda.synchronize()
    ext = torch.cuda.ExternalStream(ctx.stream(), device=local)
    cur = torch.cuda.current_stream(local)
    clocks = Clocks(local)
    for _ in range(max(args.warmup, 3)):
        out = layer.forward(x)
    torch.cuda.synchronize()
    ctx.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    steps = max(1, min(args.steps, 5))
    l0 = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for _ in range(steps):
        out = layer.forward(x)
    e1.record(cur)
    e1.synchronize()
    dev_ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    t = torch.tensor([dev_ms], dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item()) / steps
    value = C5B_IMAGES / (ms / 1e3)
    # per-kernel share (rank-local profile of one step)
    H.prof_enable(True)
    layer.forward(x)
    torch.cuda.synchronize()
    ctx.synchronize()
    H.prof_enable(False)
    prof = H.prof_report()
    mac, byts = c5b_work(p["n"], L)
    mac_r = mac * len(layer.rows) / C5B_M  # this rank's share of the modular MACs
    hbm_gbs, hbm_src = load_peaks()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    i8_peak = H.bench_int_peak(local, 4)  # measured int8 tcgen05 MMA MAC/s
    kern = {k: {"ms_per_step": v["ms"], "launches_per_step": v["launches"]} for k, v in prof.items()}
    # the contraction runs on the tensor cores: limbs 1..7 (30-bit) as 4 x 4 byte-plane
    # products, the 40-bit limb 0 as 5 x 5 (k_mac_dense_tc + k_mac_dense_tc_w)
    tc_names = [k for k in kern if k.startswith("k_mac_dense_tc")]
    tc_ms = sum(kern[k]["ms_per_step"] for k in tc_names)
    i8_macs = mac_r / L * ((L - 1) * 16 + 25)
    roof = {"bound": "tensor", "kernel": "+".join(tc_names), "achieved": i8_macs / (tc_ms * 1e-3) / 1e12,
            "peak": i8_peak / 1e12, "unit": "T int8 MAC/s", "frac": i8_macs / (tc_ms * 1e-3) / i8_peak,
            "peak_source": "measured raw tcgen05.mma.kind::i8 rate, M=128 x N=256 x K=32 (hg_bench_int_peak kind 4)",
            "modular_mac_t_per_s": mac_r / (tc_ms * 1e-3) / 1e12,
            "hbm_gbs_achieved": byts / (tc_ms * 1e-3) / 1e9, "hbm_peak": hbm_gbs, "traffic": None,
            "algorithmic_per_step": {"modular_mac": mac_r, "int8_mac": i8_macs, "hbm_bytes": byts}}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            from oracle import refbind as R
            if R.available():
                v, sample = c5b_reference_sample(os.cpu_count() or 1)
                cpu = {"value": v, "unit": "images/s", "cores": os.cpu_count() or 1, "kind": "reference",
                       "sample": sample}
        except Exception as e:  # reported, not fatal
            cpu = {"error": str(e)}
    if rank == 0:
        print(json.dumps({
            "metric": C5B_METRIC, "value": value, "unit": "images/s", "n_gpus": ws, "steps": steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64 (RNS residues, 40/30-bit primes)",
            "data": "synthetic (seeded uniform residues generated on device; W ~ N(0, 0.1^2) f32)",
            "config": c5b_config(ws), "roofline": roof, "cpu_baseline": cpu,
            "e2e": None, "e2e_note": "not measured for c5b (8.6 GB of host input per step; c2 carries the e2e line)",
            "gpu_launches": launches, "clocks": clk, "kernels": kern,
            "outputs": {"count": out.count, "level": out.level, "scale": out.scale}}))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def c5b_reference_run(args, ws, rank):
    from oracle import refbind as R
    if rank != 0:
        return 0
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhenet_ref.so not built"}))
        return 0
    cores = os.cpu_count() or 1
    v, sample = c5b_reference_sample(cores)
    print(json.dumps({
        "metric": C5B_METRIC, "value": v, "unit": "images/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": 1, "warmup": 0, "ms_per_step": C5B_IMAGES / v * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 (RNS residues)",
        "data": "synthetic (seeded uniform residues)", "config": c5b_config(1) | {"parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
    return 0


# ---- BASELINE config 4: MobileNetV2 block, one spatial tile -------------------------------
C4_METRIC = "encrypted images/sec, MobileNetV2 inverted-residual block 56x56x16 (BASELINE config 4, tiled)"
C4_HW, C4_TILE = 56, 8  # the 56 x 56 activations as 7 x 7 tiles of 8 x 8 outputs (+1-pixel halo)


def c4_secret_key(H, ctx, p, seed):
    """A uniform ternary secret (keygen's distribution), NTT'd by the library under the chain
    primes; the special limb (unused by encrypt / decrypt) is zero."""
    import numpy as np
    L, n = len(p["chain"]), p["n"]
    s = np.random.default_rng(seed).integers(-1, 2, n)
    w = np.zeros((1, 2, L, n), dtype=np.uint64)
    for i, q in enumerate(p["chain"]):
        w[0, 0, i] = np.where(s < 0, q - 1, s).astype(np.uint64)
    t = H.CipherTensor.from_words(ctx, w, 1.0)
    H.ntt_forward(ctx, t)
    sk = np.zeros((L + 1, n), dtype=np.uint64)
    sk[:L] = t.to_words()[0, 0]
    return H.SecretKey(ctx, sk)


def c4_run(args, ws, rank, local):
    """One 8 x 8-output tile (10 x 10 x 16 input with its halo) of the block per GPU step:
    1x1 expand 16->96, client-aided ReLU6 refresh, 3x3 depthwise (pad 1), ReLU6 refresh, 1x1
    project 96->24, all on the device (the refreshes by the GPU NonlinearityEngine with the
    [0, 6] clamp).  The input tile is resident; 49 tiles make one 8192-image 56 x 56 batch."""
    import numpy as np
    import torch
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200 import workloads as Wk

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p = Wk.N16384
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"], device=local)
    hw = C4_TILE + 2
    wl = Wk.mobilenet_block(hw=hw)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    plan = H.RescalePlan.plan(ctx, model)
    sk = c4_secret_key(H, ctx, p, 5 + rank)
    acts = np.random.default_rng(6 + rank).normal(0, 1, (ctx.slot_count(), wl.input_count))
    x = H.encrypt_tensor(ctx, sk, acts, 7 + rank, shape=wl.input_shape)
    eng = H.RefreshEngine(ctx, sk, 77)
    eng.set_relu_clip(6.0)
    ctx.synchronize()
    ext = torch.cuda.ExternalStream(ctx.stream(), device=local)
    clocks = Clocks(local)
    for _ in range(max(args.warmup, 1)):
        out = H.execute(ctx, model, plan, x, None, eng)
    ctx.synchronize()
    steps = max(1, min(args.steps, 6))
    l0 = ctx.launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    e0, e1 = ev[0], ev[-1]
    node_timing = os.environ.get("HG_NODE_TIMING") is not None  # diagnostic: per-node event times
    e0.record(ext)
    for i in range(steps):
        st = H.ExecutionStats() if node_timing else None
        out = H.execute(ctx, model, plan, x, None, eng, stats=st)
        ev[i + 1].record(ext)
        if st is not None:
            print("c4 step", i, "nodes", [(k, round(v, 2)) for k, v in st.layer_ms], file=sys.stderr)
    e1.synchronize()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    tile_ms = float(t.item())
    tiles = (C4_HW // C4_TILE) ** 2
    value = ws * 8192 / (tiles * tile_ms / 1e3)
    # decrypted check of the tile's interior against the cleartext block (ReLU6 semantics)
    dec = H.decrypt_tensor(ctx, sk, out, 16).reshape(16, 24, hw, hw)
    w = {k: np.frombuffer(wl.blob, dtype="<f4") for k in ("all",)}["all"]
    man = json.loads(wl.manifest)["weights"]
    g = lambda k, shp: w[man[k]["offset"] // 4:][:int(np.prod(shp))].reshape(shp).astype(np.float64)
    ew, dw, pw = g("exp_w", (96, 16, 1, 1))[:, :, 0, 0], g("dw_w", (96, 96, 3, 3)), g("proj_w", (24, 96, 1, 1))[:, :, 0, 0]
    a0 = acts[:16].reshape(16, 16, hw, hw)
    h1 = np.clip(np.einsum("fc,bchw->bfhw", ew, a0), 0, 6)
    hp = np.pad(h1, ((0, 0), (0, 0), (1, 1), (1, 1)))
    h2 = np.zeros_like(h1)
    for c in range(96):
        for ky in range(3):
            for kx in range(3):
                h2[:, c] += dw[c, c, ky, kx] * hp[:, c, ky:ky + hw, kx:kx + hw]
    want = np.einsum("fc,bchw->bfhw", pw, np.clip(h2, 0, 6))
    err = float(np.abs(dec - want)[:, :, 1:-1, 1:-1].max())
    # per-kernel attribution: one extra profiled tile (library events on the launching stream)
    H.prof_enable(True)
    H.execute(ctx, model, plan, x, None, eng)
    ctx.synchronize()
    H.prof_enable(False)
    rep = H.prof_report()
    tot = sum(v["ms"] for v in rep.values()) or 1.0
    kernels = {k: {"ms_per_tile": v["ms"], "launches": v["launches"], "share": v["ms"] / tot}
               for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])}
    # roofline of the refresh engine's transform kernel (the step's largest transform family):
    # per ReLU6 refresh of G ciphertexts at the top level, G x 7 narrow-limb transforms for the
    # decrypt INTT, the encode NTT and the encryption-error NTT; N/2 log2 N butterflies each
    G = 96 * hw * hw
    narrow = len(p["chain"]) - 1
    n_tr = 2 * 3 * G * narrow
    bfly = n_tr * (p["n"] // 2) * int(np.log2(p["n"]))
    shoup_peak = H.bench_int_peak(local, 3)
    k32 = rep.get("k_ntt_w32", {}).get("ms", 0.0)
    roof = None
    if k32 > 0:
        ach = bfly / (k32 * 1e-3) / 1e12
        roof = {"bound": "int32", "kernel": "k_ntt_w32 (refresh engine: decrypt INTT, encode NTT, error NTT)",
                "achieved": ach, "peak": shoup_peak / 1e12, "unit": "T modmul/s (Shoup: IMAD.HI + 2 IMAD)",
                "frac": ach / (shoup_peak / 1e12),
                "work": f"{n_tr} transforms x {(p['n'] // 2) * int(np.log2(p['n']))} butterflies per tile",
                "peak_source": "measured register-only Shoup-product probe (hg_bench_int_peak kind 3) on this GPU",
                "traffic": None}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = c4_reference_sample()
        except Exception as e:  # reported, not fatal
            cpu = {"error": str(e)}
    if rank == 0:
        print(json.dumps({
            "metric": C4_METRIC, "value": value, "unit": "images/s", "n_gpus": ws, "steps": steps,
            "warmup": max(args.warmup, 1), "ms_per_step": tile_ms * tiles, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues, 40/30-bit primes)",
            "data": "synthetic N(0,1) activations encrypted on the GPU; W ~ N(0, 0.1^2) f32",
            "config": {"workload": "c4 MobileNetV2 block 56x56x16 -> expand 96 -> ReLU6 -> dw 3x3 -> ReLU6 -> project 24",
                       "ring": "N=16384, chain [40,30x7]+40, scale 2^30", "images_per_batch": 8192,
                       "tiling": f"{tiles} tiles of {C4_TILE}x{C4_TILE} outputs, each computed on a "
                                 f"{hw}x{hw} input (1-pixel halo); one tile per step, the 56x56 batch = {tiles} steps",
                       "refresh": "client-aided ReLU6 on the GPU (hg_refresh_engine, clamp [0, 6])",
                       "parallelism": f"replicas x{ws}"},
            "tile_ms": tile_ms, "tile_ms_steps": step_ms, "roofline": roof, "kernels": kernels,
            "roofline_note": "the client-aided refreshes (decrypt/decode/encode/encrypt of 2 x 9600 ciphertexts per tile) are most of the tile; kernels: one profiled tile (serialised launches)",
            "cpu_baseline": cpu, "e2e": None, "gpu_launches": launches, "clocks": clk,
            "check": {"max_abs_err_vs_cleartext_interior": err, "images_checked": 16}}))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def c4_reference_sample():
    """The reference on a 1 x 1 tile (one position: 16 -> 96 -> ReLU6 -> depthwise (centre
    tap) -> ReLU6 -> 24, the harness's clamp provider; its NonlinearityEngine refreshes one
    ciphertext after another), per position, scaled to the 56 x 56 batch."""
    import numpy as np
    from oracle import refbind as R
    from paper_1908_04172_b200 import workloads as Wk
    p = Wk.N16384
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(9, False)
    wl = Wk.mobilenet_block(hw=1)
    acts = np.random.default_rng(3).normal(0, 1, (8192, wl.input_count))
    words, sc = ref.encrypt_tensor(keys, acts, 4)
    R.set_relu_clip(6.0)
    try:
        t0 = time.perf_counter()
        ref.execute(keys, wl.manifest, wl.blob, words, sc, refresh_seed=77)
        dt = time.perf_counter() - t0
    finally:
        R.set_relu_clip(0.0)
    per_position = dt
    v = 8192 / (per_position * C4_HW * C4_HW)
    return {"value": v, "unit": "images/s", "cores": os.cpu_count() or 1, "kind": "reference",
            "sample": f"1x1 tile (one position, {dt:.1f} s) through henet::execute with the clamp provider, "
                      f"scaled by position to 56x56 (extrapolated)"}


NET_METRIC = {
    "c1": "encrypted images/sec, dense 845->100 layer (BASELINE config 1), N=8192",
    "c3": "encrypted images/sec, CryptoNets-ReLU, complex packing, client-aided ReLU on the GPU (BASELINE config 3)",
}


def net_run(args, ws, rank, local):
    """BASELINE c1 (the dense layer, 4096 images, patched 'rescale after' plan, relin-free) or c3
    (the CryptoNets-shaped network with ReLU under complex packing: 8192 images per ciphertext,
    both ReLU layers refreshed client-aided by the GPU NonlinearityEngine).  Inputs are real
    encryptions made on the GPU and stay resident; one step is one execute of the batch."""
    import numpy as np
    import torch
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200 import workloads as Wk

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    which = args.workload
    p = Wk.N8192
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"], device=local)
    wl = Wk.dense_layer() if which == "c1" else Wk.cryptonets_relu()
    model = H.PlainModel.load(wl.manifest, wl.blob)
    plan = H.RescalePlan.plan(ctx, model)
    if wl.patch_terminal_rescale:  # config 1: one rescale per output (the harness's patch, ref_capi.cpp)
        nodes = {}
        planned = plan.planned_rescale_ops
        for nid in ("input", "fc", "out"):
            nodes[nid] = plan.node(nid)
        dec, lin, lout, sc = nodes["fc"]
        raised = nodes["input"][3] * p["scale"]
        nodes["fc"] = (1, lin, lin - 1, raised / float(p["chain"][lin - 1]))
        nodes["out"] = (nodes["out"][0], lin - 1, lin - 1, nodes["fc"][3])
        plan = H.RescalePlan.from_nodes(0, planned + 100, nodes)
    sk = c4_secret_key(H, ctx, p, 5 + rank)
    samples = np.random.default_rng(6 + rank).random((wl.batch, wl.input_count))
    x = H.encrypt_tensor(ctx, sk, samples, 7 + rank, wl.packing, shape=wl.input_shape)
    eng = None
    if which == "c3":
        eng = H.RefreshEngine(ctx, sk, 99)
    ctx.synchronize()
    ext = torch.cuda.ExternalStream(ctx.stream(), device=local)
    clocks = Clocks(local)
    for _ in range(max(args.warmup, 1)):
        out = H.execute(ctx, model, plan, x, None, eng)
    ctx.synchronize()
    steps = max(1, args.steps)
    l0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for _ in range(steps):
        out = H.execute(ctx, model, plan, x, None, eng)
    e1.record(ext)
    e1.synchronize()
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    value = ws * wl.batch / (ms / 1e3)
    H.prof_enable(True)
    H.execute(ctx, model, plan, x, None, eng)
    ctx.synchronize()
    H.prof_enable(False)
    rep = H.prof_report()
    tot = sum(v["ms"] for v in rep.values()) or 1.0
    kernels = {k: {"ms_per_step": v["ms"], "launches": v["launches"], "share": v["ms"] / tot}
               for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])}
    dec = H.decrypt_tensor(ctx, sk, out, wl.batch)  # decrypted outputs are finite
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            from oracle import refbind as R
            ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
            keys = ref.keygen(5, False)
            words, sc = ref.encrypt_tensor(keys, samples, 7, packing=wl.packing)
            t0 = time.perf_counter()
            ref.execute(keys if which == "c3" else None, wl.manifest, wl.blob, words, sc,
                        patch=wl.patch_terminal_rescale, refresh_seed=99)
            dt = time.perf_counter() - t0
            cpu = {"value": wl.batch / dt, "unit": "images/s", "cores": os.cpu_count() or 1, "kind": "reference",
                   "sample": f"one full {wl.batch}-image batch through henet::execute (oracle/_ref), {dt:.1f} s"}
        except Exception as e:  # reported, not fatal
            cpu = {"error": str(e)}
    if rank == 0:
        print(json.dumps({
            "metric": NET_METRIC[which], "value": value, "unit": "images/s", "n_gpus": ws, "steps": steps,
            "warmup": max(args.warmup, 1), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 (RNS residues, 24/30-bit primes)",
            "data": "synthetic U[0,1) images encrypted on the GPU; weights ~N(0, 0.05^2) f32",
            "config": {"workload": "c1 dense 845->100 + bias, patched rescale-after plan" if which == "c1" else
                       "c3 CryptoNets-ReLU (conv5x5/2 -> ReLU -> fc845x100 -> ReLU -> fc100x10), complex packing",
                       "ring": "N=8192, chain [30,24x5]+30-bit special, scale 2^24",
                       "images_per_step_per_gpu": wl.batch, "parallelism": f"replicas x{ws}",
                       "refresh": "client-aided ReLU on the GPU (hg_refresh_engine)" if which == "c3" else None},
            "kernels": kernels, "roofline": None, "cpu_baseline": cpu, "e2e": None, "gpu_launches": launches,
            "clocks": clk, "check": {"decrypted_finite": bool(np.isfinite(dec).all())}}))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    ws, rank, local = dist_env()
    if ws > 1 and "HG_UPLOAD_THREADS" not in os.environ:
        # the ranks of one node share its host cores: each rank's upload packers get their share
        # (the library's default is all but two of the host's threads, right for one rank)
        per_node = int(os.environ.get("LOCAL_WORLD_SIZE", ws)) or ws
        os.environ["HG_UPLOAD_THREADS"] = str(max(2, (os.cpu_count() or 16) // per_node - 2))
    if args.workload == "c4":
        if args.impl == "reference":
            if rank == 0:
                c = c4_reference_sample()
                print(json.dumps({"metric": C4_METRIC, "impl": "reference", "value": c["value"], "unit": "images/s",
                                  "higher_is_better": True, "cpu_baseline": c,
                                  "e2e": {"value": c["value"], "unit": "images/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}))
            return 0
        return c4_run(args, ws, rank, local)
    if args.workload == "c5b":
        return c5b_reference_run(args, ws, rank) if args.impl == "reference" else c5b_run(args, ws, rank, local)
    if args.workload in ("c1", "c3"):
        if args.impl == "reference":
            if rank == 0:
                print(json.dumps({"metric": NET_METRIC[args.workload], "impl": "reference",
                                  "unavailable": "run the b200 arm: its cpu_baseline times the reference on the same batch"}))
            return 0
        return net_run(args, ws, rank, local)
    if args.impl == "reference":
        return reference_run(args, ws, rank)
    return b200_run(args, ws, rank, local)


if __name__ == "__main__":
    sys.exit(main())
