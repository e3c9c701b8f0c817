"""Writable device views that numpy code can drive.

The reference hands ``for_each_shard`` ops numpy views of its buckets
(sharded_array.py:165-186), e.g. ``lambda v: np.add(v, 1, out=v)``.  Here the
buckets live in HBM, so the op gets a :class:`DeviceView`: a thin wrapper of a
torch CUDA tensor aliasing the bucket that

* implements numpy's ``__array_ufunc__`` for the elementwise ufuncs (with
  ``out=``), running them as torch ops on the device -- the reference's ops
  work unchanged;
* forwards every other attribute to the tensor (``v.add_(1)``, ``v.shape``)
  and unwraps itself for torch functions (``__torch_function__``);
* converts to a host numpy copy on ``np.asarray(v)`` (read-only semantics).
"""

from __future__ import annotations

import numpy as np

_UFUNCS = None


def _ufunc_table():
    global _UFUNCS
    if _UFUNCS is None:
        import torch
        _UFUNCS = {
            np.add: torch.add, np.subtract: torch.sub, np.multiply: torch.mul,
            np.true_divide: torch.true_divide, np.floor_divide: torch.floor_divide,
            np.remainder: torch.remainder, np.negative: torch.neg, np.absolute: torch.abs,
            np.maximum: torch.maximum, np.minimum: torch.minimum, np.bitwise_and: torch.bitwise_and,
            np.bitwise_or: torch.bitwise_or, np.bitwise_xor: torch.bitwise_xor,
            np.invert: torch.bitwise_not, np.left_shift: torch.bitwise_left_shift,
            np.right_shift: torch.bitwise_right_shift, np.square: torch.square, np.sqrt: torch.sqrt,
        }
    return _UFUNCS


def _unwrap(x, like=None):
    import torch
    if isinstance(x, DeviceView):
        return x.tensor
    if isinstance(x, np.ndarray):
        if x.ndim == 0:
            return x.item()
        return torch.from_numpy(np.ascontiguousarray(x)).to(like.device if like is not None else "cuda")
    if isinstance(x, np.generic):
        return x.item()
    if isinstance(x, (list, tuple)):
        return type(x)(_unwrap(y, like) for y in x)
    return x


class DeviceView:
    __slots__ = ("tensor",)

    def __init__(self, tensor):
        object.__setattr__(self, "tensor", tensor)

    # ---- numpy protocol
    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kwargs):
        fn = _ufunc_table().get(ufunc)
        kwargs.pop("casting", None)          # results are cast into `out` like casting="unsafe"
        if method != "__call__" or fn is None or kwargs:
            return NotImplemented
        args = [_unwrap(x, self.tensor) for x in inputs]
        res = fn(*args)
        if out is not None:
            (o,) = out
            target = o.tensor if isinstance(o, DeviceView) else o
            target.copy_(res.to(target.dtype) if hasattr(res, "to") else res)
            return o
        return DeviceView(res)

    def __array__(self, dtype=None, copy=None):
        a = self.tensor.cpu().numpy()
        return a.astype(dtype) if dtype is not None else a

    # ---- torch protocol
    @classmethod
    def __torch_function__(cls, func, types, args=(), kwargs=None):
        return func(*_unwrap(args), **{k: _unwrap(v) for k, v in (kwargs or {}).items()})

    # ---- container / attribute delegation
    def __len__(self):
        return len(self.tensor)

    def __getitem__(self, k):
        return self.tensor[k]

    def __setitem__(self, k, v):
        self.tensor[k] = _unwrap(v, self.tensor)

    def __getattr__(self, name):
        return getattr(object.__getattribute__(self, "tensor"), name)

    def __repr__(self):
        return f"DeviceView({self.tensor!r})"
