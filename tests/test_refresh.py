"""Online-insert refresh (BASELINE config 5 shape):
the unmodified reference applies insert_online batches (oracle/_ref/pag_ref
insert, one PesSet across batches like insert-bench) and saves the index
after each; the GPU index is refreshed in place from each phase file and must
search exactly like the oracle on that file."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import assert_same_results
from oracle import oracle as O
from paper_2603_06660_b200.fvecs import gaussian_mixture, write_fvecs


@pytest.fixture(scope="module")
def phases(fixture_dir):
    if not O.have_ref():
        pytest.skip("oracle/_ref/pag_ref not built")
    base = gaussian_mixture(1500, 32, 12, 0.5, seed=41, centre_seed=7)
    ins = gaussian_mixture(450, 32, 12, 0.5, seed=42, centre_seed=7)
    q = gaussian_mixture(40, 32, 12, 0.5, seed=43, centre_seed=7)
    b, i, idx = (os.path.join(fixture_dir, f) for f in ("rf_base.fvecs", "rf_ins.fvecs", "rf.pagidx"))
    write_fvecs(b, base)
    write_fvecs(i, ins)
    O.ref_build(b, idx, threads=1, M=8, efC=60, seed=5)
    prefix = os.path.join(fixture_dir, "rf_phase")
    O.ref_run("insert", index=idx, data=i, batches=3, **{"out-prefix": prefix})
    return idx, [f"{prefix}.{k}.pagidx" for k in range(3)], q


def test_phase_files_extend_the_base(phases):
    idx, files, _ = phases
    sizes = [O.OracleIndex(p).n for p in [idx] + files]
    assert sizes == [1500, 1650, 1800, 1950]


@pytest.mark.gpu
def test_refresh_matches_oracle_each_phase(phases):
    import paper_2603_06660_b200 as pag
    idx, files, q = phases
    ix = pag.load_index(idx)
    try:
        # a reference-order search before the first refresh: the chain-interleaved
        # row copy exists already and every refresh has to extend it
        got = ix.search_batch(q, pag.SearchParams(K=10, efS=40))
        want = O.OracleIndex(idx).search(q, 10, 40)
        assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, idx)
        for path in files:
            st = ix.refresh(path)
            assert st["new_nodes"] == 150 and 150 <= st["changed_blocks"] < ix.n
            for K, efS in ((10, 40), (20, 80)):
                got = ix.search_batch(q, pag.SearchParams(K=K, efS=efS))
                want = O.OracleIndex(path).search(q, K, efS)
                assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, path)
            gi, gs = ix.ground_truth(q, 10)
            oi, os_ = O.ground_truth(O.OracleIndex(path).rows(), q, 10)
            assert np.array_equal(gi, oi)
        with pytest.raises(ValueError, match="not an extension"):
            ix.refresh(idx)  # shrinking is refused
    finally:
        ix.close()


@pytest.mark.gpu
def test_in_memory_source_equals_the_file_source(phases):
    """pag_gpu_open_from_arrays / pag_gpu_refresh_from_arrays: the reference's
    in-memory storage (IndexArrays, here restored from the phase files) as the
    source; searches, construction searches and ground truth equal the
    file-opened handle's and the oracle's, with and without cached norms."""
    import paper_2603_06660_b200 as pag
    idx, files, q = phases
    a0 = pag.IndexArrays.from_file(idx)
    mem = pag.PagIndex.from_arrays(a0)
    a0.norms = None
    mem2 = pag.PagIndex.from_arrays(a0, devices=(0, 0))  # norms recomputed; two replicas
    dsk = pag.load_index(idx)
    try:
        assert (mem.n, mem.dim, mem.L, mem.efC, mem.total_edges) == (dsk.n, dsk.dim, dsk.L, dsk.efC, dsk.total_edges)
        for path in [None] + files:
            if path is not None:
                st = mem.refresh_from_arrays(pag.IndexArrays.from_file(path))
                st2 = dsk.refresh(path)
                assert (st["new_nodes"], st["changed_blocks"]) == (st2["new_nodes"], st2["changed_blocks"])
                a = pag.IndexArrays.from_file(path)
                a.norms = None
                mem2.refresh_from_arrays(a)
            want = O.OracleIndex(path or idx).search(q, 10, 60)
            for ix in (mem, mem2, dsk):
                got = ix.search_batch(q, pag.SearchParams(K=10, efS=60))
                assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, str(path))
            gi, gs = dsk.ground_truth(q, 10)
            for ix in (mem, mem2):
                mi, ms = ix.ground_truth(q, 10)
                assert np.array_equal(mi, gi) and np.array_equal(ms.view(np.uint32), gs.view(np.uint32))
            nodes = np.arange(0, dsk.n, 37, dtype=np.uint32)
            c0, c1 = dsk.construction_search(nodes), mem.construction_search(nodes)
            assert np.array_equal(c0.ids, c1.ids) and np.array_equal(c0.pes_n, c1.pes_n)
        with pytest.raises(ValueError, match="not an extension"):
            mem.refresh_from_arrays(pag.IndexArrays.from_file(idx))
    finally:
        for ix in (mem, mem2, dsk):
            ix.close()


@pytest.mark.gpu
def test_in_memory_source_is_validated_like_a_file(phases):
    """load_index's checks (builder.cpp:434-492) hold for the in-memory source
    too: a degree over the cap, an edge target past n and a padded_dim that
    does not match L are refused with the file path's texts."""
    import paper_2603_06660_b200 as pag
    idx, _, _ = phases
    a = pag.IndexArrays.from_file(idx)
    bad = pag.IndexArrays(**{**a.__dict__, "degrees": a.degrees.copy()})
    bad.degrees[7] = 2 * a.M + 1
    with pytest.raises(RuntimeError, match="degree over cap"):
        pag.PagIndex.from_arrays(bad)
    bad = pag.IndexArrays(**{**a.__dict__, "targets": a.targets.copy()})
    bad.targets[3, 0] = a.n
    with pytest.raises(RuntimeError, match="edge target out of range"):
        pag.PagIndex.from_arrays(bad)
    bad = pag.IndexArrays(**{**a.__dict__, "padded_dim": a.padded_dim + 1})
    with pytest.raises(RuntimeError, match="padded_dim mismatch on load"):
        pag.PagIndex.from_arrays(bad)
    ok = pag.PagIndex.from_arrays(a)  # and the untouched arrays still load
    assert ok.n == a.n
    ok.close()
