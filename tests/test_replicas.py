"""Multi-replica handles (index replicated per GPU, queries
sharded, no collective) exercised on one GPU: pag_gpu_open_devices with a
repeated device ordinal gives several full replicas on cuda:0, each with its
own stream, scratch and persistent host worker. Every entry point must give
results bit-identical to a one-replica handle (and to the oracle), with
uneven shards and batches smaller than the replica count. Also the launch
ordering rules of one replica: launches on different streams, and the
per-ticket status of asynchronous batches."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import assert_same_results
from oracle import oracle as O

pytestmark = pytest.mark.gpu

REPLICAS = (0, 0, 0)


@pytest.fixture(scope="module")
def pag():
    import paper_2603_06660_b200 as pag
    return pag


def _same(a, b, what):
    assert_same_results((a.ids, a.sq, a.n_out, a.stats), (b.ids, b.sq, b.n_out, b.stats), what)


def test_open_devices_info_and_errors(pag, built):
    fx = built("euc48")
    ix = pag.load_index(fx["index"], devices=REPLICAS)
    try:
        assert ix.n_devices == 3
        assert ix.device_bytes > 0
    finally:
        ix.close()
    with pytest.raises(ValueError, match="missing GPU"):
        pag.load_index(fx["index"], devices=(0, 31))


@pytest.mark.parametrize("name,K,efS,nq", [("euc48", 10, 60, 61), ("euc48", 100, 300, 7), ("cos20", 10, 50, 2),
                                           ("deg64", 32, 96, 1), ("tail10", 10, 40, 60)])
def test_search_sharded_equals_single_replica(pag, built, name, K, efS, nq):
    fx = built(name)
    q = fx["queries"][:nq]
    one = pag.load_index(fx["index"])
    many = pag.load_index(fx["index"], devices=REPLICAS)
    try:
        for exact in (True, False):
            p = pag.SearchParams(K=K, efS=efS, exact_dist=exact)
            a = one.search_batch(q, p)
            b = many.search_batch(q, p)
            _same(a, b, f"{name} {K}/{efS} nq={nq} exact={exact}")
        want = O.OracleIndex(fx["index"]).search(q, K, efS)
        got = many.search_batch(q, pag.SearchParams(K=K, efS=efS))
        assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, f"{name} sharded vs oracle")
    finally:
        one.close()
        many.close()


def test_submit_wait_sharded(pag, built):
    import torch
    fx = built("euc48")
    many = pag.load_index(fx["index"], devices=REPLICAS)
    one = pag.load_index(fx["index"])
    try:
        p = pag.SearchParams(K=10, efS=50)
        pinned = torch.empty(fx["queries"].shape, dtype=torch.float32, pin_memory=True)
        pinned.numpy()[:] = fx["queries"]
        batches = [fx["queries"][: 60 - 7 * i] for i in range(6)]
        want = [one.search_batch(b, p) for b in batches]
        pend = [many.search_submit(pinned.numpy()[: len(b)] if i % 2 else b, p) for i, b in enumerate(batches)]
        for pb, w in zip(pend[::-1], want[::-1]):  # out of order; the ring (depth 4) wraps
            _same(pb.wait(), w, "sharded async")
    finally:
        many.close()
        one.close()


def test_construction_sharded(pag, built):
    fx = built("deg64")
    one = pag.load_index(fx["index"])
    many = pag.load_index(fx["index"], devices=REPLICAS)
    try:
        nodes = np.arange(0, one.n, 13, dtype=np.uint32)
        for params in (None, pag.SearchParams(K=64, efS=300, b_override=48)):
            a = one.construction_search(nodes, params)
            b = many.construction_search(nodes, params)
            _same(a, b, "construction")
            assert np.array_equal(a.pes_n, b.pes_n) and np.array_equal(a.pes, b.pes)
        pend = [many.construction_submit(nodes[: 90 - 11 * i]) for i in range(5)]
        for i, pb in enumerate(pend):
            r = pb.wait()
            w = one.construction_search(nodes[: 90 - 11 * i])
            _same(r, w, "construction async")
            assert np.array_equal(r.pes_n, w.pes_n) and np.array_equal(r.pes, w.pes)
        tiny = many.construction_search(nodes[:2])  # fewer nodes than replicas
        _same(tiny, one.construction_search(nodes[:2]), "construction nn < replicas")
    finally:
        one.close()
        many.close()


@pytest.mark.parametrize("k", [1, 10, 100])
def test_ground_truth_sharded(pag, built, monkeypatch, k):
    fx = built("euc48")
    many = pag.load_index(fx["index"], devices=REPLICAS)
    try:
        oix = O.OracleIndex(fx["index"])
        gi, gs = many.ground_truth(fx["queries"], k)
        oi, os_ = O.ground_truth(oix.rows(), fx["queries"], k)
        assert np.array_equal(gi, oi) and np.array_equal(gs.view(np.uint32), os_.view(np.uint32))
        gi2, _ = many.ground_truth(fx["queries"][:2], k)  # fewer queries than replicas
        assert np.array_equal(gi2, oi[:2])
    finally:
        many.close()


def test_refresh_sharded(pag, fixture_dir):
    from paper_2603_06660_b200.fvecs import gaussian_mixture, write_fvecs
    if not O.have_ref():
        pytest.skip("oracle/_ref/pag_ref not built")
    base = gaussian_mixture(1200, 24, 10, 0.5, seed=51, centre_seed=7)
    ins = gaussian_mixture(300, 24, 10, 0.5, seed=52, centre_seed=7)
    q = gaussian_mixture(31, 24, 10, 0.5, seed=53, centre_seed=7)
    b, i, idx = (os.path.join(fixture_dir, f) for f in ("rr_base.fvecs", "rr_ins.fvecs", "rr.pagidx"))
    write_fvecs(b, base)
    write_fvecs(i, ins)
    O.ref_build(b, idx, threads=1, M=8, efC=60, seed=5)
    prefix = os.path.join(fixture_dir, "rr_phase")
    O.ref_run("insert", index=idx, data=i, batches=2, **{"out-prefix": prefix})
    many = pag.load_index(idx, devices=REPLICAS)
    try:
        for k in range(2):
            path = f"{prefix}.{k}.pagidx"
            many.refresh(path)
            got = many.search_batch(q, pag.SearchParams(K=10, efS=40))
            want = O.OracleIndex(path).search(q, 10, 40)
            assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, f"refresh phase {k}")
    finally:
        many.close()


def test_launches_on_different_streams_keep_order(pag, built):
    """One replica, launches alternating between two caller streams and the
    handle's own stream (host calls), all writing the same output buffers:
    the scratch sets and claim counters alternate per launch, so a launch on
    another stream must not overlap its predecessor (pag_host.cpp run_search
    orders them by an event)."""
    import torch
    fx = built("deg64")
    ix = pag.load_index(fx["index"])
    try:
        p = pag.SearchParams(K=10, efS=200)
        qa = fx["queries"]
        qb = np.ascontiguousarray(qa[::-1] * 1.01, np.float32)
        want_a, want_b = ix.search_batch(qa, p), ix.search_batch(qb, p)
        nq = qa.shape[0]
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        da, db = torch.from_numpy(qa).cuda(), torch.from_numpy(qb).cuda()
        outs = [torch.zeros((nq, 10), dtype=torch.int32, device="cuda"),
                torch.zeros((nq, 10), dtype=torch.float32, device="cuda"),
                torch.zeros((nq,), dtype=torch.int32, device="cuda"),
                torch.zeros((nq, 8), dtype=torch.int32, device="cuda")]
        torch.cuda.synchronize()
        for rep in range(9):
            src, s = (da, s1) if rep % 3 == 0 else (db, s2) if rep % 3 == 1 else (da, s1)
            ix.search_device(src.data_ptr(), nq, p, *(t.data_ptr() for t in outs), s.cuda_stream)
            host = ix.search_batch(qb if rep % 2 else qa, p)  # the handle's stream in between
            _same(host, want_b if rep % 2 else want_a, f"host call {rep}")
        torch.cuda.synchronize()
        assert np.array_equal(outs[0].cpu().numpy().view(np.uint32), want_a.ids)
        assert np.array_equal(outs[1].cpu().numpy(), want_a.sq)
    finally:
        ix.close()


def test_async_error_reported_by_its_own_wait(pag, built):
    """A failing batch completed early by later submits (ring of 4) reports
    its error at its own wait; those submits and their waits succeed."""
    fx = built("cos20")
    ix = pag.load_index(fx["index"], devices=(0, 0))
    try:
        p = pag.SearchParams(K=5, efS=20)
        bad = np.zeros((3, 20), np.float32)
        good = fx["queries"]
        want = ix.search_batch(good, p)
        pb = ix.search_submit(bad, p)
        later = [ix.search_submit(good, p) for _ in range(5)]  # the 4th and 5th complete `pb`
        for x in later:
            _same(x.wait(), want, "later batch")
        with pytest.raises(ValueError, match="zero query under cosine metric"):
            pb.wait()
    finally:
        ix.close()
