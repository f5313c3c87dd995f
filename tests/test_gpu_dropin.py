# SPDX-License-Identifier: Apache-2.0
"""The C++ drop-in (include/henet_b200.hpp) against the unmodified reference:
oracle/ref/dropin_test.cpp runs henet::execute and henet::gpu::execute on the
reference's own model generators (make_cryptonets, make_cryptonets_relu under
complex packing with LocalProvider refresh, the shaped toy) and op-level calls,
and requires bit-identical ciphertexts, scales, statistics and exceptions."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref not built (needs /root/reference at build time)")
def test_dropin_matches_reference_bit_exactly():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN OK" in r.stdout
