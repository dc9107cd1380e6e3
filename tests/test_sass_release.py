"""The GEMM's ring-slot release must wait for the warp's shared-memory reads (CPU: SASS only)."""

import os
import shutil
import subprocess

import pytest

from sass_release import pending_loads_at_releases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1812_06007_b200", "liburv_b200.so")


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not available")
def test_no_lds_pending_at_consumer_release():
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    gemm = [r for r in pending_loads_at_releases(sass) if "dgemm_tma_dmma" in r[0]]
    assert gemm, "no GEMM kernels found in the SASS"
    racy = [(f[-60:], a, p) for f, a, p in gemm if p]
    assert not racy, f"LDS still in flight at a ring release: {racy[:3]}"
    # the fragment loads must be true shared-memory loads (a generic LD to smem is slower)
    assert "LDS.64" in sass
