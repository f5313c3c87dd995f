# SPDX-License-Identifier: Apache-2.0
"""Times hg_tensor_upload of the c2 input (784 ciphertexts, 617 MB of reference u64 words)
from pinned host memory: ms per upload and effective host-word GB/s."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1908_04172_b200 import henet as H, workloads as Wk
from paper_1908_04172_b200._lib import check, lib

p = Wk.N8192
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
words = Wk.random_ciphertexts(p, 784, seed=7)
host = torch.empty(words.size, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
host[:] = words.reshape(-1)
t = H.CipherTensor(ctx, 784, 2, 6, p["scale"])
for _ in range(3):
    check(lib.hg_tensor_upload(t.handle, H._ptr(host), None))
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    check(lib.hg_tensor_upload(t.handle, H._ptr(host), None))
    ts.append(time.perf_counter() - t0)
ms = 1e3 * float(np.median(ts))
assert np.array_equal(t.to_words().reshape(-1), words.reshape(-1))
print(f"threads={os.environ.get('HG_UPLOAD_THREADS', 'default')} host_narrow={os.environ.get('HG_UPLOAD_HOST_NARROW', '1')} "
      f"upload {ms:.2f} ms  {words.nbytes / ms / 1e6:.1f} GB/s of u64 words (nproc {os.cpu_count()})")
