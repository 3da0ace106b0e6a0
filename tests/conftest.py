"""Shared fixtures: small indexes built by the UNMODIFIED reference
(oracle/_ref/pag_ref, compiled from the reference's own sources) so that the
oracle, the reference and the GPU all search the same PAGIDX01 file."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")


def _ensure_built():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=True)
    so = os.path.join(ROOT, "paper_2603_06660_b200", "libpag_gpu.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2603_06660_b200", "csrc"), "-s", "-j4"], check=True)


_ensure_built()

from oracle import oracle as O  # noqa: E402
from paper_2603_06660_b200.fvecs import gaussian_mixture, write_fvecs  # noqa: E402

# name -> (generator kwargs, build kwargs)
FIXTURES = {
    # d=48 euclidean, default degree cap 32 (M=16)
    "euc48": (dict(n=2500, d=48, centres=25, sigma=0.5, unit=False, metric="euclidean"),
              dict(M=16, efC=100, seed=3)),
    # cosine metric (queries normalised on the device), d=20 -> L=4
    "cos20": (dict(n=1500, d=20, centres=15, sigma=0.4, unit=False, metric="cosine"),
              dict(M=8, efC=80, seed=5)),
    # d=10 -> L=2, padded_dim 10 (not a multiple of 4: sq_dist tail path)
    "tail10": (dict(n=1200, d=10, centres=10, sigma=0.6, unit=False, metric="euclidean"),
               dict(M=8, efC=60, seed=7)),
    # degree cap 64 (two 32-edge groups per expansion)
    "deg64": (dict(n=3000, d=16, centres=20, sigma=0.5, unit=False, metric="euclidean"),
              dict(M=32, efC=120, seed=9)),
    # the benchmark shapes' compile-time distance kernels (padded_dim = 128 x NCH):
    # unit-normalised mixtures like cfg-2/3/4 at a few thousand points
    "unit256": (dict(n=1500, d=256, centres=16, sigma=0.4, unit=True, metric="euclidean"),
                dict(M=16, efC=100, seed=11)),
    "unit512": (dict(n=1200, d=512, centres=16, sigma=0.4, unit=True, metric="euclidean"),
                dict(M=16, efC=100, seed=13)),
    "unit768": (dict(n=1200, d=768, centres=16, sigma=0.4, unit=True, metric="euclidean"),
                dict(M=16, efC=100, seed=15)),
    "unit1024": (dict(n=1000, d=1024, centres=16, sigma=0.3, unit=True, metric="euclidean"),
                 dict(M=16, efC=100, seed=17)),
    # dim % L != 0: queries and rows zero-padded to padded_dim (routing.cpp:253-254)
    # d=30 -> L=4, padded 32 (dstride 32)
    "pad30": (dict(n=1800, d=30, centres=15, sigma=0.5, unit=False, metric="euclidean"),
              dict(M=12, efC=80, seed=19)),
    # d=9 -> L=2, padded 10, dstride 12; cosine (normalisation after padding)
    "pad9c": (dict(n=1400, d=9, centres=12, sigma=0.5, unit=False, metric="cosine"),
              dict(M=8, efC=60, seed=21)),
}


def build_fixture(tmpdir: str, name: str):
    gen, bp = FIXTURES[name]
    base = gaussian_mixture(gen["n"], gen["d"], gen["centres"], gen["sigma"], seed=100 + len(name),
                            centre_seed=7, unit=gen["unit"])
    queries = gaussian_mixture(60, gen["d"], gen["centres"], gen["sigma"], seed=200 + len(name),
                               centre_seed=7, unit=gen["unit"])
    bpath = os.path.join(tmpdir, f"{name}.base.fvecs")
    qpath = os.path.join(tmpdir, f"{name}.q.fvecs")
    ipath = os.path.join(tmpdir, f"{name}.pagidx")
    write_fvecs(bpath, base)
    write_fvecs(qpath, queries)
    O.ref_build(bpath, ipath, threads=1, metric=gen["metric"], **bp)
    return dict(name=name, base=base, queries=queries, base_path=bpath, q_path=qpath, index=ipath,
                metric=gen["metric"])


@pytest.fixture(scope="session")
def fixture_dir(tmp_path_factory):
    return str(tmp_path_factory.mktemp("pagfx"))


@pytest.fixture(scope="session")
def built(fixture_dir):
    if not O.have_ref():
        pytest.skip("oracle/_ref/pag_ref not built (needs /root/reference at build time)")
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = build_fixture(fixture_dir, name)
        return cache[name]

    return get


@pytest.fixture(scope="session")
def acceptance(fixture_dir):
    """The reference acceptance fixture (proj/tests/acceptance.cpp:613-633):
    gen_synthetic(gaussian, 10000, 128, 1), BuildParams{M=16, efC=200,
    seed=1} built single-threaded, 100 queries gen_synthetic(gaussian, 100,
    128, 2)."""
    if not O.have_ref():
        pytest.skip("oracle/_ref/pag_ref not built")
    b = os.path.join(fixture_dir, "acc.base.fvecs")
    q = os.path.join(fixture_dir, "acc.q.fvecs")
    i = os.path.join(fixture_dir, "acc.pagidx")
    if not os.path.exists(i):
        O.ref_gen_synthetic("gaussian", 10000, 128, 1, b)
        O.ref_gen_synthetic("gaussian", 100, 128, 2, q)
        O.ref_build(b, i, threads=1, M=16, efC=200, seed=1)
    from paper_2603_06660_b200.fvecs import read_fvecs
    return dict(base_path=b, q_path=q, index=i, base=read_fvecs(b), queries=read_fvecs(q))


def assert_same_results(a, b, what=""):
    """a, b: (ids, sq, n_out, stats) with identical semantics; bit-exact."""
    ids_a, sq_a, n_a, st_a = a
    ids_b, sq_b, n_b, st_b = b
    np.testing.assert_array_equal(n_a, n_b, err_msg=f"{what}: n_out")
    for i in range(len(n_a)):
        k = int(n_a[i])
        np.testing.assert_array_equal(ids_a[i, :k], ids_b[i, :k], err_msg=f"{what}: ids q{i}")
        np.testing.assert_array_equal(sq_a[i, :k].view(np.uint32), sq_b[i, :k].view(np.uint32),
                                      err_msg=f"{what}: sq q{i}")
    np.testing.assert_array_equal(st_a, st_b, err_msg=f"{what}: counters")
