"""Library build-time/run-time variants stay bit-exact: the GPU parity checks of
test_gpu_parity.py re-run in a subprocess under each environment switch the
library reads once per process (FHE_LANES: key-switch lanes; FHE_KS_FUSED=1: ModUp
fused into the key inner product with TMEM accumulators; FHE_FUSED_MODDOWN:
the q primes' inner product inside the ModDown rescale; FHE_KS_BATCH: sub-batch
size; FHE_KS_VARIANT: inner-product thread mapping and key placement)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# sub-batches of 2 physical ciphertexts, so the small parity cases span several
# sub-batches and every lane
VARIANTS = [
    {"FHE_LANES": "3", "FHE_KS_BATCH": "2"},
    {"FHE_LANES": "1", "FHE_KS_BATCH": "2"},
    # ModUp fused into the key inner product, accumulators in TMEM (ks_fused.cuh)
    {"FHE_KS_FUSED": "1", "FHE_KS_BATCH": "2"},
    {"FHE_KS_FUSED": "1"},
    {"FHE_FUSED_MODDOWN": "1", "FHE_KS_BATCH": "2"},
    {"FHE_KS_BATCH": "3", "FHE_KS_VARIANT": "1"},
    # inner product: register keys (the earlier default), shared-memory keys without / with the
    # prefetch of the next ciphertext's digits at 8 ciphertexts per thread (default: 9 = 16 per thread)
    {"FHE_KS_BATCH": "11", "FHE_KS_VARIANT": "2"},
    {"FHE_KS_BATCH": "11", "FHE_KS_VARIANT": "6"},
    {"FHE_KS_BATCH": "19", "FHE_KS_VARIANT": "7"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_bit_exact(env):
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_parity.py"),
           "-k", "ops_bit_exact or rotate_many or rotate_multi or rotate_hoisted or cluster"]
    r = subprocess.run(cmd, cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
