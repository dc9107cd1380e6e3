"""GPU: the sharded path's product backend (CudaOps: liburv_b200.so kernels on CUDA
tensors, NCCL collectives) on a single-rank NCCL group, against power_urv."""

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    yield None
    dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(300, 64), (128, 128)])
def test_sharded_cuda_backend_matches_power_urv(nccl_group, shape):
    import paper_1812_06007_b200 as urvb
    from paper_1812_06007_b200.distributed import CudaOps, power_urv_sharded

    m, n = shape
    a = urvb.gaussian_matrix(m, n, urvb.RngSeed(5))
    a[:, n // 2:] *= 1e-7
    ops = CudaOps(0)
    u, r, v, prov = power_urv_sharded(ops.from_numpy(a), [m], q=2, seed=9, ops=ops)
    f = urvb.power_urv(a, q=2, seed=9)
    np.testing.assert_allclose(r.cpu().numpy(), f.r, atol=1e-13)
    np.testing.assert_allclose(v.cpu().numpy(), f.v, atol=1e-13)
    np.testing.assert_allclose(u.cpu().numpy(), f.u, atol=1e-13)
    assert prov.warnings == f.provenance.warnings


def test_matrix_stats_entry_point():
    import torch

    from paper_1812_06007_b200 import _lib

    x = np.arange(12.0).reshape(4, 3)
    x[1, 1] = np.inf
    out = np.zeros(3)
    _lib.check(_lib.lib().urv_matrix_stats_f64(np.asfortranarray(x).ctypes.data, 4, 3, 4, 0, out.ctypes.data, None))
    assert out[1] == 1 and out[2] == 11
    t = torch.from_numpy(np.asfortranarray(np.ones((5, 2)))).cuda()
    _lib.check(_lib.lib().urv_matrix_stats_f64(t.data_ptr(), 5, 2, 5, 1, out.ctypes.data, None))
    assert out.tolist() == [10.0, 0.0, 10.0]
