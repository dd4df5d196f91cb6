"""Digests shared by tests/golden/make_golden.py and the parity tests.

A digest is SHA-256 over (dtype, shape, bytes) of each array, so equal
digests mean bit-identical arrays."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLDEN_JSON = os.path.join(GOLDEN_DIR, "golden.json")


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def env_digest(env) -> str:
    f = env.field
    return sha(np.asarray(f.mean, np.float64), np.asarray(f.modes, np.float64),
               np.asarray(f.coeffs, np.float64), np.asarray(env.scalar.g_mean, np.float64),
               np.asarray(env.obstacles.mask).astype(np.uint8))


def _block_arrays(b):
    if isinstance(b, tuple):
        return b
    return b.rows, b.cols, b.vals


def model_digest(model) -> str:
    arrays = []
    for row in model.blocks:
        for b in row:
            r, c, v = _block_arrays(b)
            arrays += [np.asarray(r, np.uint32), np.asarray(c, np.uint32), np.asarray(v, np.float64)]
    arrays.append(np.asarray(model.rewards, np.float64))
    return sha(*arrays)


def load_golden() -> dict:
    with open(GOLDEN_JSON) as fh:
        return json.load(fh)


def rows_digest(ensemble) -> str:
    """Digest of every trajectory of a rollout ensemble: outcome fields and
    each row's values as repr (what the CSV writer prints)."""
    h = hashlib.sha256()
    for tr in ensemble.trajectories:
        h.update(f"{tr.realization}|{tr.status}|{tr.final_cause}|{tr.n_steps}|{tr.arrival_t}|{tr.cum_reward!r}\n"
                 .encode())
        for row in tr.rows:
            h.update(("|".join(repr(x) for x in row) + "\n").encode())
    return h.hexdigest()
