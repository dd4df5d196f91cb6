"""Stage files of the planner pipeline (the reference's io.py formats).

SURVEY.md 8(f) row 2: the model / policy writers that follow the hot path.
Layouts (all little-endian, reference io.py:1-26):

  environment container   manifest.json + mean/modes/coeffs/scalar f32 blobs
                          + mask u8 (io.py:121-170)
  model file   "MDPMODEL", u32 version / n_states / n_actions / nt, u64 nnz,
               u64 byte offset per (action, time) block + one for the
               rewards, per block rows u32 | cols u32 | vals f32, then
               rewards f32 [n_actions][N_g]                (io.py:213-244)
  policy file  "MDPOLICY", u32 version / n_states, values f32 [n_states],
               actions u16 [n_states - 1]                   (io.py:298-309)
  trajectories CSV with repr() floats, summary JSON (io.py:337-368)

``write_model`` of a device-resident model (``DeviceModel``) serialises in
HBM: ``fm_export_coo`` lays the canonical COO out in block order and
``k_model_image`` writes rows, columns and f32 probabilities / rewards into
the file image, which is copied to the host once.  A host ``SparseModel``
is written with numpy.  Both produce the reference's bytes.
"""

from __future__ import annotations

import csv
import json
import struct
from pathlib import Path

import numpy as np

from .core_types import CooBlock, DOVelocityField, Environment, GridSpec, ObstacleMask, ScalarMeanField, SparseModel
from .errors import InputOutputError

MODEL_MAGIC = b"MDPMODEL"
POLICY_MAGIC = b"MDPOLICY"
MODEL_VERSION = 1
POLICY_VERSION = 1
ENV_FORMAT, ENV_VERSION = "env-container", 1
TRAJECTORY_COLUMNS = ("realization", "step", "t", "x", "y", "action", "reward", "cum_reward", "status")


# ---------------------------------------------------------------------------
# environment container
# ---------------------------------------------------------------------------

def _blob(path: Path, dtype: str, shape: tuple) -> np.ndarray:
    try:
        data = path.read_bytes()
    except OSError as exc:
        raise InputOutputError(f"cannot read blob {path}: {exc}") from exc
    want = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if len(data) != want:
        raise InputOutputError(f"blob {path} has {len(data)} bytes, expected {want}")
    return np.frombuffer(data, dtype=dtype).reshape(shape)


def write_environment(path, env) -> None:
    """Reduced-order environment container (f32 payloads, u8 mask)."""
    root = Path(path)
    root.mkdir(parents=True, exist_ok=True)
    g, fld = env.grid, env.field
    manifest = {
        "format": ENV_FORMAT, "version": ENV_VERSION, "kind": "environment",
        "grid": {"nx": g.nx, "ny": g.ny, "nt": g.nt, "dx": g.dx, "dt": g.dt,
                 "origin": [g.origin[0], g.origin[1]]},
        "n_modes": int(fld.modes.shape[0]), "n_realizations": int(fld.coeffs.shape[1]),
        "blobs": {"mean": "mean.f32", "modes": "modes.f32", "coeffs": "coeffs.f32", "scalar": "scalar.f32",
                  "mask": "mask.u8"},
    }
    (root / "manifest.json").write_text(json.dumps(manifest, sort_keys=True, indent=2) + "\n")
    for name, arr, dt in (("mean.f32", fld.mean, "<f4"), ("modes.f32", fld.modes, "<f4"),
                          ("coeffs.f32", fld.coeffs, "<f4"), ("scalar.f32", env.scalar.g_mean, "<f4"),
                          ("mask.u8", env.obstacles.mask, "u1")):
        (root / name).write_bytes(np.ascontiguousarray(arr).astype(dt).tobytes())


def read_environment(path) -> Environment:
    """Load a container; f32 payloads widen to f64 (what the build consumes)."""
    root = Path(path)
    try:
        man = json.loads((root / "manifest.json").read_text())
    except (OSError, json.JSONDecodeError) as exc:
        raise InputOutputError(f"cannot read container {path}: {exc}") from exc
    if man.get("format") != ENV_FORMAT or man.get("kind") != "environment":
        raise InputOutputError(f"{path} is not an environment container")
    gm = man["grid"]
    g = GridSpec(nx=int(gm["nx"]), ny=int(gm["ny"]), nt=int(gm["nt"]), dx=float(gm["dx"]), dt=float(gm["dt"]),
                 origin=(float(gm["origin"][0]), float(gm["origin"][1])))
    nm, nr = int(man["n_modes"]), int(man["n_realizations"])
    return Environment(
        grid=g,
        field=DOVelocityField(mean=_blob(root / "mean.f32", "<f4", (g.nt, g.ny, g.nx, 2)).astype(np.float64),
                              modes=_blob(root / "modes.f32", "<f4", (nm, g.nt, g.ny, g.nx, 2)).astype(np.float64),
                              coeffs=_blob(root / "coeffs.f32", "<f4", (g.nt, nr, nm)).astype(np.float64)),
        scalar=ScalarMeanField(g_mean=_blob(root / "scalar.f32", "<f4", (g.nt, g.ny, g.nx)).astype(np.float64)),
        obstacles=ObstacleMask(mask=_blob(root / "mask.u8", "u1", (g.nt, g.ny, g.nx)).astype(bool)),
    )


def f32_round_trip(env) -> Environment:
    """The arrays a container write + read hands to the build (f32-rounded)."""
    fld = env.field
    return Environment(
        grid=env.grid,
        field=DOVelocityField(mean=fld.mean.astype(np.float32).astype(np.float64),
                              modes=fld.modes.astype(np.float32).astype(np.float64),
                              coeffs=fld.coeffs.astype(np.float32).astype(np.float64)),
        scalar=ScalarMeanField(g_mean=env.scalar.g_mean.astype(np.float32).astype(np.float64)),
        obstacles=ObstacleMask(mask=np.asarray(env.obstacles.mask, dtype=bool)),
    )


# ---------------------------------------------------------------------------
# model file
# ---------------------------------------------------------------------------

def _model_header(n_states: int, n_actions: int, nt: int, block_nnz: np.ndarray) -> bytes:
    n_blocks = n_actions * nt
    head = len(MODEL_MAGIC) + 16 + 8 + 8 * (n_blocks + 1)
    offs = np.empty(n_blocks + 1, dtype="<u8")
    offs[0] = head
    np.cumsum(block_nnz.astype(np.uint64) * np.uint64(12), out=offs[1:])
    offs[1:] += np.uint64(head)
    return (MODEL_MAGIC + struct.pack("<IIII", MODEL_VERSION, n_states, n_actions, nt)
            + struct.pack("<Q", int(block_nnz.sum())) + offs.tobytes())


def model_file_bytes(model) -> bytes:
    """Serialised model (reference io.write_model bytes)."""
    from .builder import DeviceModel
    if isinstance(model, DeviceModel):
        return _device_model_bytes(model)
    na, nt = model.n_actions, model.nt
    nnz = np.array([model.blocks[a][t].nnz for a in range(na) for t in range(nt)], dtype=np.int64)
    parts = [_model_header(model.n_states, na, nt, nnz)]
    for a in range(na):
        for t in range(nt):
            b = model.blocks[a][t]
            parts += [np.asarray(b.rows).astype("<u4").tobytes(), np.asarray(b.cols).astype("<u4").tobytes(),
                      np.asarray(b.vals).astype("<f4").tobytes()]
    parts.append(np.asarray(model.rewards).astype("<f4").tobytes())
    return b"".join(parts)


def _device_model_bytes(dm) -> bytes:
    import torch

    from . import _lib
    if dm.t_range != (0, dm.grid.nt) or dm.j_range != (0, dm.grid.ny):
        raise InputOutputError("a model file needs the full (unsharded) model")
    dm.check()
    block_off, rows, cols, vals, rewards = dm.export_device()
    nb = dm.n_actions * dm.grid.nt
    off_h = block_off.cpu().numpy().astype(np.int64)
    header = _model_header(dm.n_states, dm.n_actions, dm.grid.nt, np.diff(off_h))
    total = len(header) + 12 * dm.nnz + 4 * rewards.numel()
    img = torch.empty(total, dtype=torch.uint8, device=rewards.device)
    _lib.check(_lib.load().fm_model_image(block_off.data_ptr(), nb, rows.data_ptr(), cols.data_ptr(),
                                          vals.data_ptr(), dm.nnz, rewards.data_ptr(), rewards.numel(),
                                          len(header), img.data_ptr(), _lib.stream_ptr()), "fm_model_image")
    host = img.cpu().numpy()
    host[: len(header)] = np.frombuffer(header, dtype=np.uint8)
    return host.tobytes()


def write_model(path, model) -> None:
    """Model file of a SparseModel or a DeviceModel (io.py:213-244)."""
    out = Path(path)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_bytes(model_file_bytes(model))


def read_model(path) -> SparseModel:
    """Model file -> SparseModel; f32 vals / rewards widen to f64 (io.py:247-295)."""
    try:
        data = Path(path).read_bytes()
    except OSError as exc:
        raise InputOutputError(f"cannot read model file {path}: {exc}") from exc
    if len(data) < len(MODEL_MAGIC) + 24 or data[: len(MODEL_MAGIC)] != MODEL_MAGIC:
        raise InputOutputError(f"{path} is not a model file (bad magic)")
    pos = len(MODEL_MAGIC)
    version, n_states, na, nt = struct.unpack_from("<IIII", data, pos)
    if version != MODEL_VERSION:
        raise InputOutputError(f"unsupported model file version {version}")
    (nnz_total,) = struct.unpack_from("<Q", data, pos + 16)
    pos += 24
    offs = np.frombuffer(data, dtype="<u8", count=na * nt + 1, offset=pos).astype(np.int64)
    pos += 8 * (na * nt + 1)
    n_g = n_states - 1
    if int(offs[-1]) + 4 * na * n_g != len(data):
        raise InputOutputError(f"model file {path} is truncated or padded")
    blocks = [[None] * nt for _ in range(na)]
    seen = 0
    for a in range(na):
        for t in range(nt):
            lo, hi = int(offs[a * nt + t]), int(offs[a * nt + t + 1])
            if (hi - lo) % 12 or lo < pos or hi > offs[-1]:
                raise InputOutputError(f"model file {path} has a corrupt block table")
            n = (hi - lo) // 12
            blocks[a][t] = CooBlock(rows=np.frombuffer(data, "<u4", n, lo).astype(np.uint32),
                                    cols=np.frombuffer(data, "<u4", n, lo + 4 * n).astype(np.uint32),
                                    vals=np.frombuffer(data, "<f4", n, lo + 8 * n).astype(np.float64), nnz=n)
            seen += n
    if seen != nnz_total:
        raise InputOutputError(f"model file {path} nnz mismatch")
    rewards = np.frombuffer(data, "<f4", na * n_g, int(offs[-1])).astype(np.float64)
    return SparseModel(blocks=blocks, rewards=rewards, n_states=n_states, n_actions=na, nt=nt)


# ---------------------------------------------------------------------------
# policy file, trajectories, summary
# ---------------------------------------------------------------------------

def _host(x) -> np.ndarray:
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


def write_policy(path, values, actions) -> None:
    """values f64 [n_states] (incl. SINK) and actions [n_states - 1] (io.py:298-309)."""
    v, a = _host(values), _host(actions)
    if a.dtype == np.int16:
        a = a.view(np.uint16)
    if a.shape[0] != v.shape[0] - 1:
        raise InputOutputError("actions must cover exactly the non-sink states")
    out = Path(path)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_bytes(POLICY_MAGIC + struct.pack("<II", POLICY_VERSION, v.shape[0]) + v.astype("<f4").tobytes()
                    + a.astype("<u2").tobytes())


def read_policy(path) -> tuple:
    """Policy file -> (values f64, actions u16) (io.py:312-334)."""
    try:
        data = Path(path).read_bytes()
    except OSError as exc:
        raise InputOutputError(f"cannot read policy file {path}: {exc}") from exc
    if len(data) < len(POLICY_MAGIC) + 8 or data[: len(POLICY_MAGIC)] != POLICY_MAGIC:
        raise InputOutputError(f"{path} is not a policy file (bad magic)")
    pos = len(POLICY_MAGIC)
    version, n = struct.unpack_from("<II", data, pos)
    if version != POLICY_VERSION:
        raise InputOutputError(f"unsupported policy file version {version}")
    pos += 8
    if len(data) != pos + 4 * n + 2 * (n - 1):
        raise InputOutputError(f"policy file {path} is truncated or padded")
    return (np.frombuffer(data, "<f4", n, pos).astype(np.float64),
            np.frombuffer(data, "<u2", n - 1, pos + 4 * n).astype(np.uint16))


def write_trajectories_csv(path, ensemble) -> None:
    """One CSV row per trajectory step, floats as repr (io.py:337-362)."""
    out = Path(path)
    out.parent.mkdir(parents=True, exist_ok=True)
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(TRAJECTORY_COLUMNS)
        for tr in ensemble.trajectories:
            for step, t, x, y, action, reward, cum, status in tr.rows:
                w.writerow([tr.realization, step, t, repr(float(x)), repr(float(y)), action, repr(float(reward)),
                            repr(float(cum)), status])


def write_summary_json(path, summary: dict) -> None:
    out = Path(path)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps(summary, sort_keys=True, indent=2) + "\n")


def read_summary_json(path) -> dict:
    try:
        return json.loads(Path(path).read_text())
    except OSError as exc:
        raise InputOutputError(f"cannot read summary {path}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise InputOutputError(f"malformed summary {path}: {exc}") from exc
