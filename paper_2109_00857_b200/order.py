"""Order reduction of a raw velocity ensemble on the GPU (SURVEY.md 8(f)
row 4): drop-in for synthesis.reduce_order (synthesis.py:267-313), the step
upstream of the planner that turns per-realization snapshots into the DO
form (mean + modes + coefficients) the build consumes.

Per time step (all steps batched on the device): subtract the ensemble
mean, take the top ``n_modes`` right-singular vectors of the centred
(realization x stacked-component) matrix as modes -- sign fixed so each
mode's largest-magnitude entry is positive -- and project the centred
realizations onto them.  The SVD is cuSOLVER's (torch.linalg.svd, f64),
so results agree with the reference's LAPACK SVD to rounding (tolerances
in tests/test_gpu_order.py), not bit for bit.
"""

from __future__ import annotations

import numpy as np

from .core_types import DOVelocityField
from .errors import ContractViolation


def reduce_order(ensemble, n_modes: int, device=None) -> DOVelocityField:
    """ensemble (n_realizations, nt, ny, nx, 2) -> DOVelocityField."""
    import torch
    from . import _lib
    _lib.load()   # fails loudly without a GPU: no CPU path
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    x = ensemble if isinstance(ensemble, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(ensemble))
    if x.dim() != 5 or x.shape[4] != 2:
        raise ContractViolation("ensemble must have shape (r, t, y, x, 2)")
    n_real, nt, ny, nx, _ = x.shape
    n_cells = ny * nx
    if not (0 <= n_modes <= min(n_real, 2 * n_cells)):
        raise ContractViolation(f"n_modes={n_modes} exceeds min(n_realizations, 2*N_c)={min(n_real, 2 * n_cells)}")
    X = x.to(device=dev, dtype=torch.float64).permute(1, 0, 2, 3, 4).reshape(nt, n_real, 2 * n_cells)
    mu = X.mean(dim=1)                                    # [nt, 2 N_c]
    mean = mu.reshape(nt, ny, nx, 2)
    if n_modes == 0:
        return DOVelocityField(mean=mean.cpu().numpy(), modes=np.zeros((0, nt, ny, nx, 2)),
                               coeffs=np.zeros((nt, n_real, 0)))
    centered = X - mu[:, None, :]
    _, _, vh = torch.linalg.svd(centered, full_matrices=False)   # batched over t
    basis = vh[:, :n_modes, :].clone()                         # [nt, n_modes, 2 N_c]
    peak = torch.gather(basis, 2, basis.abs().argmax(dim=2, keepdim=True))
    basis = torch.where(peak < 0, -basis, basis)               # largest-magnitude entry positive
    coeffs = centered @ basis.transpose(1, 2)                  # [nt, n_real, n_modes]
    modes = basis.reshape(nt, n_modes, ny, nx, 2).permute(1, 0, 2, 3, 4)
    return DOVelocityField(mean=mean.cpu().numpy(), modes=modes.contiguous().cpu().numpy(),
                           coeffs=coeffs.cpu().numpy())
