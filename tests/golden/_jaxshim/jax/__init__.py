"""Minimal stand-in for the `jax` API surface the reference package touches.

The reference (srsim, /root/reference/pkg) differentiates its reduced
squared-distance formulas and the prismatic/hinge energies with jax, which is
not installed in this image. This shim maps the handful of calls it uses onto
torch.func (float64, CPU) so the *unmodified* reference code can be imported
and run to generate golden fixtures. Test infrastructure only: never imported
by the product package.
"""
import numpy as _np
import torch as _torch
import torch.func as _tf

from . import numpy  # noqa: F401  (jax.numpy)


class _Config:
    def update(self, *args, **kwargs):
        return None


config = _Config()


def _to_t(a):
    if isinstance(a, _np.ndarray):
        return _torch.as_tensor(a, dtype=_torch.float64)
    if isinstance(a, float):
        return _torch.tensor(a, dtype=_torch.float64)
    return a


def _to_np(out):
    if isinstance(out, tuple):
        return tuple(_to_np(o) for o in out)
    if isinstance(out, _torch.Tensor):
        return out.detach().numpy()
    return out


def jit(fn):
    def wrapped(*args):
        return _to_np(fn(*[_to_t(a) for a in args]))
    return wrapped


def vmap(fn):
    return _tf.vmap(fn)


def grad(fn):
    return _tf.grad(fn)


def hessian(fn):
    return _tf.hessian(fn)


def value_and_grad(fn):
    g = _tf.grad_and_value(fn)

    def wrapped(*args):
        gr, val = g(*args)
        return val, gr
    return wrapped
