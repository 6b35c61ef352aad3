"""No kernel reads outside the caller's batch.

compute-sanitizer is not available on the GPU pool, so the bounds check is
done with guard pages instead: tests/_guard_child.py places each batch so
that it ends exactly at (or starts exactly at) an unmapped virtual page,
runs every kernel on it and compares the digests with the CPU oracle.  A
read of one byte past the end (or before the start) is an illegal-address
fault in the child, which poisons its CUDA context; the child runs in its
own process so a fault fails this test instead of the whole session.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("mode", ["end", "start"])
def test_kernels_stay_inside_the_batch(mode):
    r = subprocess.run([sys.executable, os.path.join(HERE, "_guard_child.py"), mode],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MISMATCH" not in r.stdout
    assert r.stdout.count(" ok") >= 20, r.stdout


def test_guard_page_catches_an_overrun():
    """Positive control: hashing one row past the mapped end faults."""
    r = subprocess.run([sys.executable, os.path.join(HERE, "_guard_child.py"), "control"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode != 0 and "no fault" not in r.stdout, r.stdout + r.stderr[-2000:]
