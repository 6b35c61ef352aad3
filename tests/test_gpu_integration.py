"""The drop-in boundary from callers that are not this package:
integration/c_abi_demo.c (plain C + CUDA runtime) and
integration/lanehash_cuda_backend.py (the reference-side ctypes backend of
INTEGRATION.md, no torch), checked against the reference's vectors."""
import importlib.util
import os
import struct
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_abi_demo_reproduces_reference_vectors():
    exe = os.path.join(ROOT, "integration", "c_abi_demo")
    if not os.path.exists(exe):
        import __graft_entry__

        __graft_entry__.build_c_demo()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def _stub():
    spec = importlib.util.spec_from_file_location(
        "lanehash_cuda_backend", os.path.join(ROOT, "integration", "lanehash_cuda_backend.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_reference_side_backend_stub(oracle, golden):
    from paper_1612_06257_b200.highway import Key256

    be = _stub().CudaBackend()
    ramp_key = Key256.from_bytes(bytes(range(32)))
    for n, hexd in golden["frozen_64"].items():
        assert be.hash64(ramp_key, bytes(i & 0xFF for i in range(int(n)))) == int(hexd, 16)
    for n, hexd in golden["frozen_256_hex"].items():
        d = be.hash256(ramp_key, bytes(i & 0xFF for i in range(int(n))))
        assert struct.pack("<4Q", *d).hex() == hexd
    rng = np.random.default_rng(2)
    for _ in range(200):  # T/test_acceptance.py:75-98 protocol, reduced
        key = Key256.from_bytes(rng.integers(0, 256, 32, dtype=np.uint8).tobytes())
        msg = rng.integers(0, 256, int(rng.integers(0, 1025)), dtype=np.uint8).tobytes()
        assert be.hash64(key, msg) == oracle.highway(key.lanes, msg)[0]
    msgs = rng.integers(0, 256, (16, 37), dtype=np.uint8)
    got = be.hash64_batch(ramp_key, msgs)
    assert np.array_equal(got, oracle.batch_fixed(oracle.ALG_HIGHWAY, ramp_key.lanes, msgs, 64, 4))
    with pytest.raises(ValueError):
        be._run(ramp_key, msgs, 96, 4)
