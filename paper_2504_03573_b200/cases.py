"""Manufactured solutions of the reference (sipg.py:85-121: `ManufacturedCase`, `sinusoidal_case`,
`gaussian_pulse_case`), written once for both numpy arrays and CUDA torch tensors.

The reference's own cases call numpy ufuncs, so `rhs_assemble` / `l2_error` evaluate them on the
host at host points (the reference's behaviour).  These versions are pointwise in any array
namespace: given CUDA tensors they run on the device, and `rhs_assemble` / `l2_error` then keep
the whole computation — physical points, forcing, boundary data, products, reductions — on the GPU
(rhs.py / rhs3d.py detect this with a one-point probe).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["ManufacturedCase", "sinusoidal_case", "gaussian_pulse_case", "device_callable"]


def _ns(x):
    mod = type(x).__module__
    if mod.startswith("torch"):
        import torch
        return torch
    return np


@dataclass
class ManufacturedCase:
    name: str
    dim: int
    lambda_: float
    exact: object
    forcing: object


def sinusoidal_case(k: float, dim: int, lambda_: float = 1.0) -> ManufacturedCase:
    """u = prod sin(k x_i), f = -(lambda + d k^2) u (reference sipg.py:88-100)."""

    def exact(x):
        xp = _ns(x)
        u = xp.sin(k * x[0])
        for i in range(1, dim):
            u = u * xp.sin(k * x[i])
        return u

    def forcing(x):
        return -(lambda_ + dim * k * k) * exact(x)

    return ManufacturedCase(f"sin(k={k:g})", dim, lambda_, exact, forcing)


def gaussian_pulse_case(a: float, dim: int, lambda_: float = 1.0) -> ManufacturedCase:
    """u = exp(-r^2/a^2), f = lap(u) - lambda u (reference sipg.py:103-116)."""

    def exact(x):
        xp = _ns(x)
        r2 = sum(x[i] ** 2 for i in range(dim))
        return xp.exp(-r2 / (a * a))

    def forcing(x):
        xp = _ns(x)
        r2 = sum(x[i] ** 2 for i in range(dim))
        return (4.0 * r2 / a ** 4 - 2.0 * dim / (a * a) - lambda_) * xp.exp(-r2 / (a * a))

    return ManufacturedCase(f"gauss(a={a:g})", dim, lambda_, exact, forcing)


def device_callable(fn, dim: int) -> bool:
    """Does `fn` map a CUDA float64 tensor of points (dim, 1, 1) to a CUDA tensor?"""
    import torch
    try:
        r = fn(torch.full((dim, 1, 1), 0.25, dtype=torch.float64, device="cuda"))
    except Exception:
        return False
    return isinstance(r, torch.Tensor) and r.is_cuda
