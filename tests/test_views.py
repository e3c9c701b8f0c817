"""DeviceView host logic (numpy ufunc / torch function protocols), exercised on
CPU tensors -- the same code drives the CUDA bucket views."""
import numpy as np
import torch

from paper_2209_00103_b200.views import DeviceView


def test_ufunc_out_in_place_and_casting():
    t = torch.arange(10, dtype=torch.int32)
    v = DeviceView(t)
    r = np.add(v, 1, out=v)
    assert r is v and torch.equal(t, torch.arange(10, dtype=torch.int32) + 1)
    np.multiply(v, np.int32(3), out=v, casting="unsafe")
    assert torch.equal(t, (torch.arange(10, dtype=torch.int32) + 1) * 3)
    np.subtract(v, np.asarray(2, np.int32), out=v)
    assert t.dtype == torch.int32 and int(t[0]) == 1


def test_ufunc_without_out_and_reductions_via_array():
    t = torch.arange(6, dtype=torch.float32)
    v = DeviceView(t)
    w = np.negative(v)
    assert isinstance(w, DeviceView) and torch.equal(w.tensor, -t)
    assert np.asarray(v).sum() == 15.0                  # __array__: host copy
    assert len(v) == 6 and v.shape == t.shape            # attribute delegation


def test_torch_functions_and_methods():
    t = torch.zeros(4, dtype=torch.int64)
    v = DeviceView(t)
    v.add_(5)                                            # tensor method
    assert torch.equal(torch.cat([v, v]), torch.full((8,), 5))   # __torch_function__ unwrap
    v[1] = np.int64(9)
    assert int(t[1]) == 9 and int(v[1]) == 9


def test_wrapping_int8_like_numpy():
    t = torch.tensor([127, -128], dtype=torch.int8)
    np.add(DeviceView(t), 1, out=DeviceView(t), casting="unsafe")
    want = (np.array([127, -128], np.int8) + np.int8(1)).astype(np.int8)
    assert t.numpy().tolist() == want.tolist()
