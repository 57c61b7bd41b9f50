"""The checked build (lib_checked.so, -DSG_CHECKED): device-side index and
protocol asserts over the parity suites.

compute-sanitizer is closed on this GPU pool (profiles/r02_sanitizer_closed.txt),
so memory safety of the hot kernels is checked by the kernels themselves: in
the checked build every shared-memory tile / blob / bin index of the big-tile
sweep, the joint sweep, the bucket scatter and the generic tally is asserted
against its allocation before use, the step tail's role ticket against the
grid, and the tail's spin-wait is bounded (a lost release is recorded instead
of hanging).  The normal build compiles every check to nothing (identical
SASS).
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1511_06416_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.gpu

# the suites whose kernels carry the checks: joint / packed sweeps and the merged
# step tail, big-tile and generic sweeps, bad-input validation, run() graphs
SUITES = ["tests/test_gpu_joint.py", "tests/test_gpu_small.py", "tests/test_gpu_large.py",
          "tests/test_gpu_parity.py", "tests/test_gpu_validation.py", "tests/test_gpu_run_graphs.py",
          "tests/test_gpu_configs.py"]


def _checked_env():
    if not _lib.CHECKED_LIB_PATH.exists():
        pytest.fail(f"{_lib.CHECKED_LIB_PATH} is not built: run __graft_entry__.build()")
    env = dict(os.environ)
    env["SAMEGIBBS_LIB"] = str(_lib.CHECKED_LIB_PATH)
    env["SG_CHECKED_RUN"] = "1"
    return env


def test_checked_build_records_a_failing_check():
    """The probe kernels fail their check on purpose: every unit reports the line, then clears."""
    code = ("from paper_1511_06416_b200 import _lib\n"
            "lib = _lib.load()\n"
            "assert _lib.LIB_PATH.name == 'lib_checked.so', _lib.LIB_PATH\n"
            "assert all(v == 0 for v in _lib.checked_lines(lib).values())\n"
            "hit = _lib.checked_lines(lib, probe=True)\n"
            "assert all(v > 0 for v in hit.values()), hit\n"
            "assert all(v == 0 for v in _lib.checked_lines(lib).values())\n"
            "print('probe', hit)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=_checked_env(), capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "probe" in r.stdout


def test_parity_suites_pass_under_device_asserts():
    """The parity suites, against the checked library: results unchanged and no
    device-side check fails after any test (conftest's SG_CHECKED_RUN hook)."""
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider", *SUITES],
                       cwd=ROOT, env=_checked_env(), capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    print("checked-build run:", r.stdout.strip().splitlines()[-1] if r.stdout.strip() else "")
    assert r.returncode == 0, tail
    assert " passed" in r.stdout, tail
