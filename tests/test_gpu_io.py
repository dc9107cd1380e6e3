"""GPU: URVK1 payloads streamed between files and HBM (urv_read_f64_file /
urv_write_f64_file) -- byte-exact against the reference's host format."""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1812_06007_b200 as urvb

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("shape", [(1, 1), (7, 5), (1001, 333), (3, 4000)])
def test_device_load_matches_host(tmp_path, shape):
    a = urvb.gaussian_matrix(*shape, urvb.RngSeed(11))
    path = tmp_path / "a.urv"
    urvb.save_matrix_binary(path, a)
    t = urvb.load_matrix_binary_device(path)
    assert t.is_cuda and tuple(t.shape) == shape and t.stride(0) == 1 and t.stride(1) % 2 == 0
    assert np.array_equal(t.cpu().numpy(), a)


@pytest.mark.parametrize("layout", ["F", "C", "slice"])
def test_device_save_matches_host_format(tmp_path, layout):
    import torch

    a = urvb.gaussian_matrix(301, 77, urvb.RngSeed(12))
    t = torch.from_numpy(np.asfortranarray(a)).cuda()
    if layout == "C":
        t = t.contiguous()
    elif layout == "slice":
        big = torch.zeros(310, 90, dtype=torch.float64, device="cuda").t().contiguous().t()
        big[:301, :77] = t
        t = big[:301, :77]
    path, ref = tmp_path / "d.urv", tmp_path / "h.urv"
    urvb.save_matrix_binary_device(path, t)
    urvb.save_matrix_binary(ref, a)
    assert path.read_bytes() == ref.read_bytes()


def test_chunked_pipeline_round_trip(tmp_path):
    # 1 MiB chunks: many column blocks through the three pinned staging buffers,
    # with a ragged last block (run in a child so the chunk size is read fresh)
    code = ("import numpy as np, paper_1812_06007_b200 as u; a = u.gaussian_matrix(3001, 777, u.RngSeed(5));"
            "u.save_matrix_binary(%r, a); t = u.load_matrix_binary_device(%r);"
            "assert np.array_equal(t.cpu().numpy(), a); u.save_matrix_binary_device(%r, t);"
            "assert open(%r, 'rb').read() == open(%r, 'rb').read()")
    p1, p2 = str(tmp_path / "a.urv"), str(tmp_path / "b.urv")
    subprocess.run([sys.executable, "-c", code % (p1, p1, p2, p1, p2)], check=True, cwd=ROOT,
                   env=dict(os.environ, URV_IO_CHUNK_MB="1"))


def test_truncated_payload_rejected_before_any_copy(tmp_path):
    path = tmp_path / "short.urv"
    path.write_bytes(b"URVK1" + np.array([100, 10], dtype="<u8").tobytes() + bytes(8 * 999))
    with pytest.raises(ValueError, match="expected 1000 entries, got 999"):
        urvb.load_matrix_binary_device(path)


def test_power_urv_from_streamed_file(tmp_path):
    a = urvb.gaussian_matrix(500, 300, urvb.RngSeed(13))
    path = tmp_path / "a.urv"
    urvb.save_matrix_binary(path, a)
    f_dev = urvb.power_urv(urvb.load_matrix_binary_device(path), q=1, seed=2)
    f_host = urvb.power_urv(a, q=1, seed=2)
    assert np.array_equal(f_dev.r.cpu().numpy(), f_host.r)
