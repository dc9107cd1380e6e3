"""The library's device memory pool gives scratch back (an idle library
must not pin the tens of GB a large factorisation uses)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import torch, paper_1812_06007_b200 as u
from paper_1812_06007_b200 import _lib
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
free0 = torch.cuda.mem_get_info()[0]
f = u.power_urv(a, q=1, seed=3, redundant_qr=False)
torch.cuda.synchronize()
free1 = torch.cuda.mem_get_info()[0]
_lib.release_memory()
free2 = torch.cuda.mem_get_info()[0]
out = torch.empty(3 * n * n, dtype=torch.float64, device="cuda")  # outputs u, r, v are still alive
print("HELD", (free0 - free1) / 2**20, (free0 - free2) / 2**20)
"""


def _held(env):
    p = subprocess.run([sys.executable, "-c", CODE], cwd=ROOT, capture_output=True, text=True,
                       env=dict(os.environ, **env), timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("HELD")][0]
    after_call, after_release = map(float, line.split()[1:])
    return after_call, after_release


def test_pool_released_after_call_without_cache():
    # keep 0: the scratch (Z = 512 MiB, QR buffers) goes back at the call's final sync;
    # only the three outputs (3 x 512 MiB) stay allocated
    outputs_mib = 3 * 8192 * 8192 * 8 / 2**20
    after_call, after_release = _held({"URV_POOL_KEEP_MB": "0"})
    assert after_call <= outputs_mib + 256, after_call
    assert after_release <= outputs_mib + 256, after_release


def test_release_memory_trims_cached_scratch():
    outputs_mib = 3 * 8192 * 8192 * 8 / 2**20
    after_call, after_release = _held({"URV_POOL_KEEP_MB": "8192"})
    assert after_call >= outputs_mib + 256, after_call  # scratch cached for the next call
    assert after_release <= outputs_mib + 256, after_release
