"""Both stage-(d) kernels (DYNRAD_K6: db = double-buffered single tile, the
default below 64 MiB of K + V per head; rp = block-row pairs sharing K/V,
the default above) pass the same bf16 parity tests.
The variant is fixed per process, so it runs the attention test module in a
subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("variant", ["db", "rp"])
def test_variant_passes_attention_parity(cuda, variant):
    env = dict(os.environ, DYNRAD_K6=variant)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_attention_gpu.py"),
                        "-k", "bf16 or wan_shape or empty_row or host_pipeline"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
