"""The library baselines used by tools/kv_microbench.py copy the bytes they
are asked to (one cudaMemcpyAsync per page)."""

import numpy as np
import pytest
import torch

from paper_2605_05467_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method", [0])
def test_baseline_copy_pages(method):
    src = torch.randint(0, 255, (1 << 20,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros_like(src)
    offs = np.random.default_rng(method).permutation(256)[:40].astype(np.uint64) * 4096
    s = np.ascontiguousarray(src.data_ptr() + offs, dtype=np.uint64)
    d = np.ascontiguousarray(dst.data_ptr() + offs[::-1].copy(), dtype=np.uint64)
    b = np.full(len(offs), 4096, np.uint64)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    _native.call("tpr_baseline_copy_pages", s.ctypes.data, d.ctypes.data, b.ctypes.data, len(s),
                 method, side.cuda_stream)
    torch.cuda.synchronize()
    hs, hd = src.cpu().numpy(), dst.cpu().numpy()
    for so, do in zip(offs, offs[::-1]):
        assert np.array_equal(hd[do:do + 4096], hs[so:so + 4096])
    with pytest.raises(_native.NativeError):
        _native.call("tpr_baseline_copy_pages", s.ctypes.data, d.ctypes.data, b.ctypes.data, 1, 7,
                     torch.cuda.current_stream().cuda_stream)
