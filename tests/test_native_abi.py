"""CPU-side checks of the native boundary: the sm_100a library loads and
exports every entry point include/flowmdp_b200.h declares, ctypes struct
layouts match the header, and the device hypot restatement is bit-exact
against glibc (what np.hypot calls)."""

from __future__ import annotations

import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2109_00857_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flowmdp_b200.h")


def _declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int32_t|int64_t|const char \*)\s*(fm_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_abi():
    names = _declared_functions()
    assert "fm_build" in names and "fm_solve_backward" in names and len(names) >= 12


def test_library_exports_every_declared_symbol():
    _lib.build_native()
    lib = _lib.load(require_gpu=False)
    declared = _declared_functions()
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"
    for name in declared:
        assert hasattr(lib, name), f"{name} not exported"
    assert lib.fm_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


_STRUCT_PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "flowmdp_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(fm_grid), sizeof(fm_env), sizeof(fm_action),
         sizeof(fm_reward), sizeof(fm_model), sizeof(fm_build_args), sizeof(fm_violation), sizeof(fm_csr));
  printf("%zu %zu %zu %zu\n", offsetof(fm_build_args, mask_sat), offsetof(fm_build_args, viol_flags),
         offsetof(fm_model, capacity), offsetof(fm_model, d_nnz));
  printf("%zu %zu %zu %zu\n", sizeof(fm_rollout_args), offsetof(fm_rollout_args, policy),
         offsetof(fm_rollout_args, n_traj), offsetof(fm_rollout_args, final_cell));
  printf("%zu %zu\n", offsetof(fm_build_args, h_actions), offsetof(fm_build_args, vmax_y));
  return 0;
}
"""


def test_ctypes_layout_matches_header():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "probe.c")
        exe = os.path.join(d, "probe")
        open(src, "w").write(_STRUCT_PROBE)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, src])
        lines = subprocess.check_output([exe], text=True).split("\n")
    sizes = [int(x) for x in lines[0].split()]
    offs = [int(x) for x in lines[1].split()]
    ours = [C.sizeof(s) for s in (_lib.FmGrid, _lib.FmEnv, _lib.FmAction, _lib.FmReward, _lib.FmModel,
                                   _lib.FmBuildArgs, _lib.FmViolation, _lib.FmCsr)]
    assert ours == sizes
    assert offs == [_lib.FmBuildArgs.mask_sat.offset, _lib.FmBuildArgs.viol_flags.offset,
                    _lib.FmModel.capacity.offset, _lib.FmModel.d_nnz.offset]
    R = _lib.FmRolloutArgs
    assert [int(x) for x in lines[2].split()] == [C.sizeof(R), R.policy.offset, R.n_traj.offset,
                                                  R.final_cell.offset]
    assert [int(x) for x in lines[3].split()] == [_lib.FmBuildArgs.h_actions.offset, _lib.FmBuildArgs.vmax_y.offset]


_HYPOT_PROBE = r"""
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include "fm_hypot.cuh"
static uint64_t s = 0x9E3779B97F4A7C15ULL;
static double u(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (double)(s >> 11) * 0x1p-53; }
int main(void) {
  long bad = 0, n = 0;
  const double scales[] = {1e-300, 1e-6, 1e-3, 0.5, 1.0, 3.0, 10.0, 1e3, 1e150, 1e300};
  for (long i = 0; i < 12000000; ++i) {
    double sc = scales[i % 10];
    double x = (2 * u() - 1) * sc, y = (2 * u() - 1) * sc;
    if (i % 3 == 0) { x = (25.5 + x) - 25.5; y = (12.5 + y) - 12.5; }   /* step-like deltas */
    if (i % 7 == 0) y = x * (u() * 1e-17);                              /* tiny ratio branch */
    double h = hypot(x, y), m = fm_hypot(x, y);
    ++n;
    if (h != m && !(h != h && m != m)) ++bad;
  }
  printf("%ld %ld\n", n, bad);
  return 0;
}
"""


def test_device_hypot_matches_glibc():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "h.c")
        exe = os.path.join(d, "h")
        open(src, "w").write(_HYPOT_PROBE)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "paper_2109_00857_b200",
                                                                                     "csrc"),
                               "-o", exe, src, "-lm"])
        n, bad = map(int, subprocess.check_output([exe], text=True).split())
    assert n == 12000000 and bad == 0


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2109_00857_b200.errors import NativeUnavailable
    with pytest.raises(NativeUnavailable):
        _lib.load(require_gpu=True)
