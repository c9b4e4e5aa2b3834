"""The producer conv's pinned variants (cgbn_conv.cu): 128- / 256-pixel tiles, split-K
ranges, cta_group::2 CTA pairs, 64- / 128-row weight boxes for Cout <= 64. The per-layer plan picks among them, so one process sees
only the planned ones; each variant here runs the producer parity tests
(tests/test_gpu_producer.py: z against an fp64 reference, the fused partial against the
oracle's statistics of z as stored, the fused BN forward / backward against the oracle)
in a subprocess with the plan pinned through the experiment knobs (read once per process).
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = [
    {"CGBN_CONV_TBN": "128"},
    {"CGBN_CONV_TBN": "256"},
    {"CGBN_CONV_TBN": "128", "CGBN_CONV_SPLITS": "2"},
    {"CGBN_CONV_TBN": "128", "CGBN_CONV_SPLITS": "3"},
    {"CGBN_CONV_PAIR": "1"},
    {"CGBN_CONV_PAIR": "1", "CGBN_CONV_TBN": "256"},
    {"CGBN_CONV_WROWS": "128"},  # 128-row weight boxes also for Cout <= 64
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: "-".join(f"{k[10:]}{v}" for k, v in e.items()))
def test_producer_parity_with_pinned_plan(env):
    full = dict(os.environ)
    full.update(env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_producer.py")],
                       cwd=ROOT, env=full, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
