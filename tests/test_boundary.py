"""The drop-in boundary compiled by its consumers, not only bound by ctypes.

CPU: a C99 program (tests/c/abi_consumer.c) compiled with -Werror -pedantic
against include/pag_gpu.h, linked to libpag_gpu.so, pins the struct layouts
and runs the host-only entry points; the C++ adapter include/pag_gpu.hpp
(the reference-side binding of INTEGRATION.md §2) compiles and links against
the reference's own headers and library (tests/cpp/adapter_check.cpp).
GPU: that C++ program checks, in one process, pag::search_batch on the GPU
against the reference library's pag::search, the construction search
against search_padded, a handle opened from the in-memory PagIndex
(pag_gpu_open_from_arrays) and refreshed from memory after insert_online
batches (pag_gpu_refresh_from_arrays), bit for bit, plus the exception
mapping."""
from __future__ import annotations

import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2603_06660_b200")
ADAPTER = os.path.join(ROOT, "oracle", "_ref", "adapter_check")
HAVE_REF_SRC = os.path.exists("/root/reference/proj/include/pag/routing.hpp")


def test_c_consumer_compiles_and_runs_host_calls(tmp_path):
    exe = str(tmp_path / "abi_consumer")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"),
                    "-o", exe, os.path.join(ROOT, "tests", "c", "abi_consumer.c"), "-L", LIBDIR, "-l:libpag_gpu.so",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)
    out = subprocess.run([exe, os.path.join(ROOT, "tests", "golden", "golden_index.pagidx")], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("ok n=")


@pytest.mark.skipif(not HAVE_REF_SRC, reason="needs the reference headers (/root/reference)")
def test_cpp_adapter_builds_against_reference():
    subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp"), "-s"], check=True)
    assert os.access(ADAPTER, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("name,K,efS", [("euc48", 10, 60), ("cos20", 5, 40), ("pad30", 20, 90), ("deg64", 64, 128)])
def test_cpp_adapter_equals_reference_in_process(built, name, K, efS):
    if not os.access(ADAPTER, os.X_OK):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    fx = built(name)
    out = subprocess.run([ADAPTER, fx["index"], fx["q_path"], str(K), str(efS)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["queries_equal"] == r["queries"] and r["nodes_equal"] == r["nodes"]
    # opened from the in-memory PagIndex; refreshed from memory after insert_online batches
    assert r["from_arrays_equal"] == r["queries"]
    assert r["after_refresh"] == 2 * r["queries"] and r["after_refresh_equal"] == r["after_refresh"]
    assert r["k_gt_efs_invalid_argument"] and r["open_runtime_error"]
