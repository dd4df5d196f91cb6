"""reduce_order on the GPU against the reference's
own outputs (tests/golden/reduce_order.npz, written by make_golden.py from
pkg/src/flowmdp/synthesis.py:reduce_order) and the reference's test
properties (test_synthesis.py:153-200).  The SVD differs from LAPACK's in
rounding, so comparisons use tolerances (stated per assertion)."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fm = pytest.importorskip("paper_2109_00857_b200")
from paper_2109_00857_b200.order import reduce_order  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reduce_order.npz")


def _reconstruct(field):
    out = np.broadcast_to(field.mean[None], (field.coeffs.shape[1],) + field.mean.shape).copy()
    for m in range(field.modes.shape[0]):
        out += field.coeffs[:, :, m][:, :, None, None, None].transpose(1, 0, 2, 3, 4) * field.modes[m][None]
    return out


def test_matches_reference_outputs():
    g = np.load(GOLD)
    f = reduce_order(g["ensemble"], 4)
    scale = np.abs(g["ensemble"]).max()
    assert np.abs(f.mean - g["mean"]).max() <= 1e-13 * scale            # ensemble mean
    assert np.abs(f.modes - g["modes"]).max() <= 1e-9                   # unit-norm modes, sign-fixed
    assert np.abs(f.coeffs - g["coeffs"]).max() <= 1e-9 * scale


def test_identical_members():
    rng = np.random.default_rng(21)
    snap = rng.normal(size=(3, 4, 5, 2))
    f = reduce_order(np.broadcast_to(snap, (6, 3, 4, 5, 2)).copy(), 2)
    assert np.allclose(f.mean, snap, atol=1e-12)
    assert np.abs(f.coeffs).max() <= 1e-9


def test_recovers_low_rank_exactly():
    rng = np.random.default_rng(23)
    basis = rng.normal(size=(5, 3, 4, 4, 2))
    weights = rng.normal(size=(16, 5))
    ens = np.einsum("rk,ktyxc->rtyxc", weights, basis)
    back = _reconstruct(reduce_order(ens, 5))
    assert np.abs(back - ens).max() <= 1e-9 * np.abs(ens).max()


def test_modes_orthonormal_and_sign_fixed():
    rng = np.random.default_rng(24)
    f = reduce_order(rng.normal(size=(10, 2, 3, 4, 2)), 4)
    for t in range(2):
        flat = f.modes[:, t].reshape(4, -1)
        assert np.allclose(flat @ flat.T, np.eye(4), atol=1e-9)
        assert (flat[np.arange(4), np.abs(flat).argmax(axis=1)] > 0).all()


def test_mode_limit():
    rng = np.random.default_rng(25)
    ens = rng.normal(size=(4, 2, 2, 2, 2))
    with pytest.raises(fm.ContractViolation):
        reduce_order(ens, 5)
    with pytest.raises(fm.ContractViolation):
        reduce_order(ens, -1)
