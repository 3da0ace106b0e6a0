"""The device counterpart of TfbState::validate (routing.cpp:116-137): an
invariant-checking build of the whole library (-DPAG_VALIDATE,
build/lib_validate.so: `make -C paper_2603_06660_b200/csrc variant-all
V=validate FLAGS=-DPAG_VALIDATE`) checks after every expansion and end_round
that W and both rings stay within b, z_max is the largest sq in W, no node
resides twice across W, R_F, R_T and the flushed R_L, and the final result
list is ordered; a violation fails the call with the reference's
logic_error text. Run on register (b <= 32) and array (b > 32) layouts, both
occupancy flavours, both distance modes and the construction search."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "build", "lib_validate.so")


@pytest.mark.gpu
def test_tfb_invariants_hold_on_device(built):
    if not os.path.exists(LIB):
        pytest.skip("build/lib_validate.so not built (make variant-all V=validate FLAGS=-DPAG_VALIDATE)")
    args = []
    for name in ("euc48", "deg64", "cos20", "pad30"):
        fx = built(name)
        args += [fx["index"], fx["q_path"]]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "validate_run.py"), *args],
                         env=dict(os.environ, PAG_GPU_LIB=LIB), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "validated" in out.stdout
