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


@pytest.mark.gpu
def test_acceptance_criterion_7_fuzz_on_device():
    """acceptance.cpp:360-426 ("search-state invariants under fuzz") with the
    invariant-checking build: the reference's index recipe, per-query K in
    [1, 64] and efS = K + U[0, 128); 1,500 queries here (the full 10,000 are
    recorded under profiles/): no violated invariant, every result
    bit-identical to the oracle in both distance modes, exact = seeds + passes."""
    import json
    if not os.path.exists(LIB):
        pytest.skip("build/lib_validate.so not built (make variant-all V=validate FLAGS=-DPAG_VALIDATE)")
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "pag_ref")):
        pytest.skip("oracle/_ref/pag_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "fuzz_criterion7.py"), "1500"],
                         env=dict(os.environ, PAG_GPU_LIB=LIB), capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["queries"] == 1500 and r["invariant_violations"] == 0, r
    for mode in ("reference_order", "warp_tree"):
        assert r[mode] == {"bit_identical_to_oracle": 1500, "exact_equals_seeds_plus_passes": 1500}, r
