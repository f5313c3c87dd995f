# SPDX-License-Identifier: Apache-2.0
"""The C ABI boundary (include/henet_b200.h): the in-tree library loads, exports
every declared symbol, and fails loudly (no CPU fallback) without a B200."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "henet_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1908_04172_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True, check=True)
    exported = {line.split()[-1] for line in out.stdout.splitlines() if line.strip()}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert len(declared_symbols()) >= 50


def test_python_binding_covers_header():
    from paper_1908_04172_b200 import _lib
    missing = [s for s in declared_symbols() if s not in _lib.PROTOTYPES]
    assert not missing, missing


def test_abi_version():
    from paper_1908_04172_b200._lib import lib
    assert lib.hg_abi_version() == 1


def test_library_is_sm100a_only():
    from paper_1908_04172_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_no_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1908_04172_b200 import henet as H
    from paper_1908_04172_b200 import workloads as W
    p = W.N8192
    with pytest.raises(H.HeError if hasattr(H, "HeError") else Exception):
        H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])


def test_product_does_not_touch_oracle():
    """The product package never imports or links anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_1908_04172_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".hpp", ".cuh", ".h")) or f == "Makefile":
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "henet_oracle" not in txt and "libhenet_ref" not in txt, f
    from paper_1908_04172_b200 import _lib
    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True)
    assert "oracle" not in out.stdout and "henet_ref" not in out.stdout
