"""GPU parity tests: the sm_100a search (through the C ABI) against the CPU
oracle on the same PAGIDX01 files and queries.

Default mode (exact_dist=1) must be BIT-IDENTICAL to the oracle (ids,
squared distances, n_out, and the counters exact/test/pass/visited plus
edges_scanned). The warp-tree distance mode is held to the north-star
tolerance: id sets equal on >= 99% of queries, sq within 1e-5 relative,
recall@K within 0.002.
"""
from __future__ import annotations

import os
import re

import numpy as np
import pytest

from conftest import assert_same_results
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pag():
    import paper_2603_06660_b200 as pag
    return pag


_open = {}


def gpu_index(pag, path):
    if path not in _open:
        _open[path] = pag.load_index(path)
    return _open[path]


def check_bitexact(pag, fx, K, efS, **kw):
    ix = gpu_index(pag, fx["index"])
    got = ix.search_batch(fx["queries"], pag.SearchParams(K=K, efS=efS, **kw))
    oix = O.OracleIndex(fx["index"])
    okw = {k: v for k, v in kw.items() if k in ("b_override", "use_prt", "use_tfb")}
    want = oix.search(fx["queries"], K, efS, **okw)
    assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, f"{fx['name']} K={K} efS={efS} {kw}")
    return got


CASES = [
    ("euc48", 10, 10), ("euc48", 10, 40), ("euc48", 10, 200), ("euc48", 1, 1), ("euc48", 32, 64),
    ("euc48", 10, 15), ("euc48", 100, 300), ("euc48", 250, 500), ("euc48", 0, 0), ("euc48", 0, 7),
    ("cos20", 10, 50), ("cos20", 5, 5), ("tail10", 10, 30), ("tail10", 40, 90),
    ("deg64", 10, 60), ("deg64", 64, 128), ("deg64", 10, 700),
]


@pytest.mark.parametrize("name,K,efS", CASES)
def test_search_bitexact_vs_oracle(pag, built, name, K, efS):
    check_bitexact(pag, built(name), K, efS)


@pytest.mark.parametrize("flags", [dict(use_prt=False), dict(use_tfb=False), dict(b_override=32),
                                   dict(b_override=7)])
def test_ablations_bitexact(pag, built, flags):
    got = check_bitexact(pag, built("euc48"), 10, 80, **flags)
    if "use_prt" in flags:
        assert np.array_equal(got.stats[:, 1], got.stats[:, 2])


def test_search_matches_reference_binary(pag, built, fixture_dir):
    """Directly against the unmodified reference (not only the oracle)."""
    fx = built("euc48")
    got = gpu_index(pag, fx["index"]).search_batch(fx["queries"], pag.SearchParams(K=10, efS=60))
    ids, sq, n_out, st, _ = O.ref_search(fx["index"], fx["q_path"], 10, 60,
                                         os.path.join(fixture_dir, "gref.bin"), no_warm=True)
    assert_same_results((got.ids, got.sq, got.n_out, got.stats[:, :4]), (ids, sq, n_out, st), "vs reference")


@pytest.mark.parametrize("hash_log2", ["4", "6"])
def test_visited_bitmap_spill_is_exact(pag, built, monkeypatch, hash_log2):
    """Force a tiny smem visited table so nearly every mark spills to the
    per-warp HBM bitmap (cleared between queries): results stay bit-identical,
    also across consecutive batches reusing the same bitmaps."""
    monkeypatch.setenv("PAG_GPU_HASH_LOG2", hash_log2)
    fx = built("deg64")
    ix = pag.load_index(fx["index"])
    try:
        for K, efS in ((10, 400), (32, 96), (10, 60)):
            got = ix.search_batch(fx["queries"], pag.SearchParams(K=K, efS=efS))
            want = O.OracleIndex(fx["index"]).search(fx["queries"], K, efS)
            assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, f"bitmap spill {K}/{efS}")
    finally:
        ix.close()


def test_fast_distance_mode_within_tolerance(pag, built):
    fx = built("euc48")
    ix = gpu_index(pag, fx["index"])
    gi, gs = O.ground_truth(fx["base"], fx["queries"], 10)
    for efS in (20, 60, 150):
        a = ix.search_batch(fx["queries"], pag.SearchParams(K=10, efS=efS, exact_dist=False))
        b = O.OracleIndex(fx["index"]).search(fx["queries"], 10, efS)
        same = np.mean([set(a.ids[i, :a.n_out[i]]) == set(b[0][i, :b[2][i]]) for i in range(len(a.n_out))])
        assert same >= 0.99
        for i in range(len(a.n_out)):
            for j in range(int(a.n_out[i])):
                if a.ids[i, j] == b[0][i, j]:
                    assert abs(a.sq[i, j] - b[1][i, j]) <= 1e-5 * max(1e-30, abs(b[1][i, j]))
        ra = pag.mean_recall(a.ids, a.n_out, gi, gs, 10)
        rb = pag.mean_recall(b[0], b[2], gi, gs, 10)
        assert abs(ra - rb) <= 0.002


def test_golden_acceptance_on_gpu(pag, acceptance):
    """proj/test_output.txt:8,12 reproduced by the GPU path, with the GPU
    ground-truth kernel bit-identical to the oracle's."""
    ix = gpu_index(pag, acceptance["index"])
    gi, gs = ix.ground_truth(acceptance["queries"], 100)
    oi, os_ = O.ground_truth(acceptance["base"], acceptance["queries"], 100)
    assert np.array_equal(gi, oi) and np.array_equal(gs.view(np.uint32), os_.view(np.uint32))
    golden = {(10, 200): (0.9560, 0.2052), (10, 400): (0.9930, 0.2202),
              (100, 500): (0.9594, 0.2550), (100, 800): (0.9813, 0.2651)}
    for (K, efS), (rec_w, gam_w) in golden.items():
        r = ix.search_batch(acceptance["queries"], pag.SearchParams(K=K, efS=efS))
        rec = np.mean([pag.recall_at_k(r.ids[i, :r.n_out[i]], gi[i], gs[i], K) for i in range(len(gi))])
        gam = np.mean(r.stats[:, 2] / r.stats[:, 1])
        assert round(rec, 4) == rec_w and round(gam, 4) == gam_w
        assert abs(pag.mean_recall(r.ids, r.n_out, gi, gs, K) - rec) < 1e-12


@pytest.mark.parametrize("name,k", [("euc48", 1), ("euc48", 10), ("euc48", 100), ("tail10", 50),
                                    ("deg64", 1000), ("cos20", 4000)])
def test_ground_truth_bitexact(pag, built, name, k):
    fx = built(name)
    ix = gpu_index(pag, fx["index"])
    oix = O.OracleIndex(fx["index"])
    q = np.zeros((fx["queries"].shape[0], oix.padded), np.float32)
    q[:, :oix.dim] = fx["queries"]
    gi, gs = ix.ground_truth(fx["queries"], k)
    oi, os_ = O.ground_truth(oix.rows(), q, k)
    assert gi.shape == oi.shape
    assert np.array_equal(gi, oi) and np.array_equal(gs.view(np.uint32), os_.view(np.uint32))


@pytest.mark.parametrize("name,k,pool", [("euc48", 1, False), ("euc48", 10, False), ("euc48", 32, False),
                                         ("tail10", 16, False), ("cos20", 8, False), ("deg64", 25, False),
                                         ("euc48", 100, False), ("deg64", 1000, False), ("pad30", 200, False),
                                         ("cos20", 64, False), ("unit512", 1000, False), ("euc48", 10, True),
                                         ("pad9c", 5, True), ("euc48", 1, True), ("cos20", 8, True),
                                         ("tail10", 16, True), ("deg64", 25, True)])
def test_tensor_core_ground_truth_equals_exact(pag, built, monkeypatch, name, k, pool):
    """tcgen05 TF32 GEMM ground truth gives the same ids and bits as the exact
    SIMT kernel and the oracle, with every query certified: by the per-query
    bound + pool path (the default for k <= 1000), and for k <= 32 also by the
    per-split top-C candidate lists + certificate (pool = False rows)."""
    fx = built(name)
    ix = gpu_index(pag, fx["index"])
    if not pool and k <= 32:
        monkeypatch.setenv("PAG_GPU_GT_LISTS", "1")
    before = ix.gt_uncertified()
    ti, ts = ix.ground_truth(fx["queries"], k)
    assert ix.gt_uncertified() == before, "tensor-core candidates not certified"
    monkeypatch.delenv("PAG_GPU_GT_LISTS", raising=False)
    monkeypatch.setenv("PAG_GPU_GT_EXACT", "1")
    ei, es = ix.ground_truth(fx["queries"], k)
    assert np.array_equal(ti, ei) and np.array_equal(ts.view(np.uint32), es.view(np.uint32))
    oix = O.OracleIndex(fx["index"])
    q = np.zeros((fx["queries"].shape[0], oix.padded), np.float32)
    q[:, :oix.dim] = fx["queries"]
    oi, _ = O.ground_truth(oix.rows(), q, k)
    assert np.array_equal(ti, oi)


def test_device_path_matches_host_path(pag, built):
    import torch
    fx = built("euc48")
    ix = gpu_index(pag, fx["index"])
    p = pag.SearchParams(K=10, efS=50)
    host = ix.search_batch(fx["queries"], p)
    nq = fx["queries"].shape[0]
    q = torch.from_numpy(fx["queries"]).cuda()
    ids = torch.empty((nq, 10), dtype=torch.int32, device="cuda")
    sq = torch.empty((nq, 10), dtype=torch.float32, device="cuda")
    n = torch.empty((nq,), dtype=torch.int32, device="cuda")
    st = torch.empty((nq, 8), dtype=torch.int32, device="cuda")
    ix.search_device(q.data_ptr(), nq, p, ids.data_ptr(), sq.data_ptr(), n.data_ptr(), st.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), host.ids)
    assert np.array_equal(sq.cpu().numpy(), host.sq)
    assert np.array_equal(st.cpu().numpy()[:, :5].astype(np.uint64), host.stats)


def test_errors_match_reference(pag, built):
    fx = built("euc48")
    ix = gpu_index(pag, fx["index"])
    with pytest.raises(ValueError, match="K > efS"):  # routing.cpp:209
        ix.search_batch(fx["queries"], pag.SearchParams(K=50, efS=10))
    with pytest.raises(ValueError, match="query dimension mismatch"):  # routing.cpp:252
        pag.search(ix, np.zeros(fx["queries"].shape[1] + 1, np.float32))
    with pytest.raises(RuntimeError, match=re.escape("cannot open index: /nonexistent/pag.bin")):
        pag.load_index("/nonexistent/pag.bin")
    cos = gpu_index(pag, built("cos20")["index"])
    with pytest.raises(ValueError, match="zero query under cosine metric"):  # routing.cpp:257
        pag.search(cos, np.zeros(20, np.float32))
    with pytest.raises(ValueError, match="missing GPU"):
        pag.load_index(fx["index"], devices=(31,))


def test_cosine_scale_invariance(pag, built):  # test_routing.cpp:372-396
    fx = built("cos20")
    ix = gpu_index(pag, fx["index"])
    p = pag.SearchParams(K=5, efS=50)
    a = ix.search_batch(fx["queries"], p)
    b = ix.search_batch(7.5 * fx["queries"], p)
    assert np.array_equal(a.ids, b.ids)


def test_single_query_api_and_empty_batch(pag, built):
    fx = built("euc48")
    ix = gpu_index(pag, fx["index"])
    r = pag.search(ix, fx["queries"][3], pag.SearchParams(K=10, efS=40))
    want = O.OracleIndex(fx["index"]).search(fx["queries"][3:4], 10, 40)
    assert [c[0] for c in r.results] == list(want[0][0]) and r.stats.exact_dist_count == int(want[3][0, 0])
    empty = ix.search_batch(np.zeros((0, fx["queries"].shape[1]), np.float32), pag.SearchParams())
    assert empty.ids.shape == (0, 10)
    # conservation (test_routing.cpp:221-241): exact = seeds + passes
    full = ix.search_batch(fx["queries"], pag.SearchParams(K=10, efS=80))
    seeds = min(O.OracleIndex(fx["index"]).n_entries, 10)
    assert np.all(full.stats[:, 0] == seeds + full.stats[:, 2])
    assert np.all(full.stats[:, 1] >= full.stats[:, 2])


CONSTRUCTION = [("euc48", {}), ("cos20", {}), ("deg64", {}), ("tail10", {}),
                ("euc48", dict(K=50, efS=90, b_override=16)), ("euc48", dict(collect_pes=False)),
                ("deg64", dict(K=64, efS=300, b_override=48)),
                ("deg64", dict(K=150, efS=400, b_override=160))]  # b > 128, efS > 200: 6-blocks/SM flavour


@pytest.mark.parametrize("name,kw", CONSTRUCTION)
def test_construction_search_bitexact(pag, built, name, kw):
    """§8(f) next-2: insert_with_state's search (builder.cpp:218-227) batched
    on the GPU — results, counters and pes_rejected lists (routing.cpp:190-199)
    bit-identical to the oracle (b <= 32 register and b > 32 memory layouts)."""
    fx = built(name)
    ix = gpu_index(pag, fx["index"])
    oix = O.OracleIndex(fx["index"])
    nodes = np.arange(0, oix.n, 5, dtype=np.uint32)
    params = None
    if "K" in kw:
        params = pag.SearchParams(K=kw["K"], efS=kw["efS"], b_override=kw["b_override"])
    got = ix.construction_search(nodes, params, collect_pes=kw.get("collect_pes"))
    want = oix.construction_search(nodes, **kw)
    assert_same_results((got.ids, got.sq, got.n_out, got.stats), want[:4], f"construction {name} {kw}")
    assert np.array_equal(got.pes_n, want[5])
    for i in range(len(nodes)):
        assert got.pes_rejected(i) == [int(x) for x in want[4][i, :int(want[5][i])]]
    assert (got.pes_n.sum() > 0) == kw.get("collect_pes", True)


def test_construction_search_vs_reference_binary_and_truncation(pag, built, fixture_dir):
    fx = built("euc48")
    ix = gpu_index(pag, fx["index"])
    count, stride = 60, 41
    ids, sq, n_out, st, pes, pes_n, _ = O.ref_build_search(fx["index"], count, stride,
                                                          os.path.join(fixture_dir, "gbs.bin"), no_warm=True)
    nodes = (np.arange(count, dtype=np.uint64) * stride % ix.n).astype(np.uint32)
    got = ix.construction_search(nodes)
    assert_same_results((got.ids, got.sq, got.n_out, got.stats[:, :4]), (ids, sq, n_out, st), "vs reference")
    assert np.array_equal(got.pes_n, pes_n)
    one = ix.construction_search(nodes, pes_cap=1)  # truncated lists keep the full count
    assert np.array_equal(one.pes_n, pes_n)
    has = pes_n > 0
    assert np.array_equal(one.pes[has, 0], pes[has, 0])
    with pytest.raises(ValueError, match="node id out of range"):
        ix.construction_search(np.array([ix.n], np.uint32))


def test_construction_device_path_matches_host_path(pag, built):
    import torch
    fx = built("deg64")
    ix = gpu_index(pag, fx["index"])
    nodes = np.arange(0, ix.n, 11, dtype=np.uint32)
    host = ix.construction_search(nodes)
    nn, K, cap = len(nodes), ix.efC, 256
    d = lambda *s, t=torch.int32: torch.zeros(s, dtype=t, device="cuda")  # noqa: E731
    nodes_d = torch.from_numpy(nodes.view(np.int32)).cuda()
    ids, sq, n, st, pes, pn = d(nn, K), d(nn, K, t=torch.float32), d(nn), d(nn, 8), d(nn, cap), d(nn)
    ix.construction_search_device(nodes_d.data_ptr(), nn, None, None, ids.data_ptr(), sq.data_ptr(), n.data_ptr(),
                                  st.data_ptr(), pes.data_ptr(), cap, pn.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), host.ids)
    assert np.array_equal(sq.cpu().numpy(), host.sq)
    assert np.array_equal(pn.cpu().numpy().view(np.uint32), host.pes_n)
    pes = pes.cpu().numpy().view(np.uint32)
    for i in range(nn):  # entries past pes_n are unspecified on the device path
        m = min(int(host.pes_n[i]), cap)
        assert np.array_equal(pes[i, :m], host.pes[i, :m])


def test_back_to_back_launches_keep_stream_order(pag, built):
    """Consecutive launches overlap (programmatic dependent launch): a batch
    written into the same output buffers right after another must still end
    with the later batch's results, across alternating counter/scratch sets
    and changing batch sizes."""
    import torch
    fx = built("deg64")
    ix = gpu_index(pag, fx["index"])
    p = pag.SearchParams(K=10, efS=60)
    qa = fx["queries"]
    qb = np.ascontiguousarray(qa[::-1] * 1.01, np.float32)
    want_a = ix.search_batch(qa, p)
    want_b = ix.search_batch(qb, p)
    nq = qa.shape[0]
    s = torch.cuda.Stream()
    da, db = torch.from_numpy(qa).cuda(), torch.from_numpy(qb).cuda()
    ids = torch.zeros((nq, 10), dtype=torch.int32, device="cuda")
    sq = torch.zeros((nq, 10), dtype=torch.float32, device="cuda")
    n = torch.zeros((nq,), dtype=torch.int32, device="cuda")
    st = torch.zeros((nq, 8), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    for rep in range(7):
        src, want, m = ((da, want_a, nq) if rep % 2 == 0 else (db, want_b, nq - 3 * rep))
        ix.search_device(src.data_ptr(), m, p, ids.data_ptr(), sq.data_ptr(), n.data_ptr(), st.data_ptr(),
                         s.cuda_stream)
    s.synchronize()
    # the last launch (rep 6, batch A, all queries) wins everywhere
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), want_a.ids)
    assert np.array_equal(sq.cpu().numpy(), want_a.sq)
    assert np.array_equal(st.cpu().numpy()[:, :5].astype(np.uint64), want_a.stats)
    for rep in range(3):  # B after A: B's rows win, rows past B's count keep A's
        ix.search_device(da.data_ptr(), nq, p, ids.data_ptr(), sq.data_ptr(), n.data_ptr(), st.data_ptr(),
                         s.cuda_stream)
        ix.search_device(db.data_ptr(), nq - 5, p, ids.data_ptr(), sq.data_ptr(), n.data_ptr(), st.data_ptr(),
                         s.cuda_stream)
    s.synchronize()
    got = ids.cpu().numpy().view(np.uint32)
    assert np.array_equal(got[:nq - 5], want_b.ids[:nq - 5])
    assert np.array_equal(got[nq - 5:], want_a.ids[nq - 5:])


def test_async_submit_wait_matches_sync(pag, built):
    """pag_gpu_search_submit / wait: results written by the kernel into pinned
    host memory, several batches in flight (more than the ring depth), pinned
    queries read in place and pageable ones copied."""
    import torch
    fx = built("euc48")
    ix = gpu_index(pag, fx["index"])
    p = pag.SearchParams(K=10, efS=50)
    want = ix.search_batch(fx["queries"], p)
    pinned = torch.empty(fx["queries"].shape, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = fx["queries"]
    pend = [ix.search_submit(pinned.numpy() if i % 2 else fx["queries"], p) for i in range(7)]
    for pb in pend[::-1]:  # out of order; the first ones were completed to free ring slots
        r = pb.wait()
        assert_same_results((r.ids, r.sq, r.n_out, r.stats), (want.ids, want.sq, want.n_out, want.stats), "async")
    with pytest.raises(ValueError, match="K > efS"):
        ix.search_submit(fx["queries"], pag.SearchParams(K=20, efS=10))
    cos = gpu_index(pag, built("cos20")["index"])
    bad = np.zeros((3, 20), np.float32)
    pb = cos.search_submit(bad, pag.SearchParams(K=5, efS=20))
    with pytest.raises(ValueError, match="zero query under cosine metric"):
        pb.wait()


@pytest.mark.parametrize("name", ["unit256", "unit512", "unit768", "unit1024"])
def test_benchmark_shapes_bitexact_and_fast(pag, built, name):
    """The compile-time distance kernels the benchmarks run (padded_dim =
    128 x NCH, NCH = 2/4/6/8): reference-order mode bit-exact against the
    oracle (register and memory TFB layouts, both occupancy flavours), and
    warp-tree mode within the north-star tolerance."""
    fx = built(name)
    for K, efS in ((10, 40), (10, 300), (100, 150)):
        check_bitexact(pag, fx, K, efS)
    ix = gpu_index(pag, fx["index"])
    gi, gs = O.ground_truth(fx["base"], fx["queries"], 10)
    a = ix.search_batch(fx["queries"], pag.SearchParams(K=10, efS=60, exact_dist=False))
    b = O.OracleIndex(fx["index"]).search(fx["queries"], 10, 60)
    same = np.mean([set(a.ids[i, :a.n_out[i]]) == set(b[0][i, :b[2][i]]) for i in range(len(a.n_out))])
    assert same >= 0.99
    both = a.ids == b[0]
    rel = np.abs(a.sq - b[1]) / np.maximum(np.abs(b[1]), 1e-30)
    assert rel[both].max() <= 1e-5
    assert abs(pag.mean_recall(a.ids, a.n_out, gi, gs, 10) - pag.mean_recall(b[0], b[2], gi, gs, 10)) <= 0.002


def test_working_set_off_chip_is_exact(pag, built, monkeypatch):
    """b > 32 with a per-warp smem budget too small for the working set: W,
    the rings, R_L and the merge buffer all live in the warp's HBM scratch.
    Bit-identical to the oracle, for queries and the construction search."""
    monkeypatch.setenv("PAG_GPU_SMEM_BUDGET", "2048")
    for name, K, efS, kw in (("euc48", 100, 300, {}), ("euc48", 250, 500, {}), ("deg64", 64, 128, {}),
                             ("deg64", 10, 700, dict(b_override=48)), ("cos20", 33, 70, {}),
                             ("deg64", 1000, 1000, {}),     # S = 32: deferred owner re-scan
                             ("deg64", 1100, 1300, {})):    # S = 35 > 32: plain re-scan
        fx = built(name)
        ix = pag.load_index(fx["index"])
        try:
            got = ix.search_batch(fx["queries"], pag.SearchParams(K=K, efS=efS, **kw))
            want = O.OracleIndex(fx["index"]).search(fx["queries"], K, efS, **kw)
            assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, f"off-chip {name} {K}/{efS} {kw}")
        finally:
            ix.close()
    fx = built("deg64")
    ix = pag.load_index(fx["index"])
    try:
        oix = O.OracleIndex(fx["index"])
        nodes = np.arange(0, oix.n, 7, dtype=np.uint32)
        kw = dict(K=64, efS=300, b_override=48)
        got = ix.construction_search(nodes, pag.SearchParams(**kw), collect_pes=True)
        want = oix.construction_search(nodes, collect_pes=True, **kw)
        assert_same_results((got.ids, got.sq, got.n_out, got.stats), want[:4], "off-chip construction")
        assert np.array_equal(got.pes_n, want[5])
    finally:
        ix.close()


def _with_duplicate_targets(src: str, dst: str, every: int = 7) -> int:
    """Copy a PAGIDX01 file, overwriting edge 2 of every `every`-th node with
    its edge 0 (same target, scalars and codes): targets repeated inside a
    32-edge group. Returns the number of patched nodes."""
    import struct
    data = bytearray(open(src, "rb").read())
    n = struct.unpack_from("<Q", data, 12)[0]
    L = struct.unpack_from("<I", data, 28)[0]
    n_entries = struct.unpack_from("<I", data, 62)[0]
    rec = 4 + (L + 1) // 2 + 12
    off = 66 + 4 * n_entries
    patched = 0
    for u in range(n):
        deg = struct.unpack_from("<I", data, off)[0]
        e0 = off + 4
        if u % every == 0 and deg >= 3:
            data[e0 + 2 * rec:e0 + 3 * rec] = data[e0:e0 + rec]
            patched += 1
        off = e0 + deg * rec
    open(dst, "wb").write(bytes(data))
    return patched


def test_duplicate_targets_in_group_bitexact(pag, built, tmp_path):
    """An index whose adjacency repeats targets inside a group (the loader
    accepts it; routing.cpp:160-183 skips a copy once an earlier one passed
    and was marked): the search takes its duplicate-resolution path and stays
    bit-identical to the oracle; a duplicate-free index reports 0 such nodes
    and takes the fast path."""
    fx = built("euc48")
    dup_path = str(tmp_path / "dup.pagidx")
    assert _with_duplicate_targets(fx["index"], dup_path) > 0
    clean = gpu_index(pag, fx["index"])
    assert clean.dup_nodes() == 0
    ix = pag.load_index(dup_path)
    try:
        assert ix.dup_nodes() > 0
        oix = O.OracleIndex(dup_path)
        for K, efS in ((10, 40), (10, 200), (100, 300)):
            got = ix.search_batch(fx["queries"], pag.SearchParams(K=K, efS=efS))
            want = oix.search(fx["queries"], K, efS)
            assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, f"duplicates {K}/{efS}")
    finally:
        ix.close()


def test_construction_search_reuses_out_arrays(pag, built):
    """construction_search(out=...) fills caller arrays (stale contents are
    overwritten, entries past each pes list are zero) and equals a fresh call."""
    fx = built("deg64")
    ix = gpu_index(pag, fx["index"])
    nodes = np.arange(3, ix.n, 13, dtype=np.uint32)
    fresh = ix.construction_search(nodes)
    nn, K, cap = len(nodes), ix.efC, 256
    out = pag.ConstructionResult(np.full((nn, K), 7, np.uint32), np.full((nn, K), 7, np.float32),
                                 np.full(nn, 7, np.uint32), np.zeros((nn, 5), np.uint64),
                                 np.full((nn, cap), 7, np.uint32), np.full(nn, 7, np.uint32))
    got = ix.construction_search(nodes, out=out)
    assert got is out
    for a, b in ((got.ids, fresh.ids), (got.sq, fresh.sq), (got.n_out, fresh.n_out), (got.stats, fresh.stats),
                 (got.pes, fresh.pes), (got.pes_n, fresh.pes_n)):
        assert np.array_equal(a, b)
    for i in range(nn):
        assert not got.pes[i, min(int(got.pes_n[i]), cap):].any()
    with pytest.raises(ValueError):
        ix.construction_search(nodes[:-1], out=out)


def test_construction_submit_wait_matches_blocking(pag, built):
    """pag_gpu_construction_submit: several batches in flight (the 4-slot ring
    wraps), each equal to the blocking construction_search, pes tails zero."""
    fx = built("deg64")
    ix = gpu_index(pag, fx["index"])
    batches = [np.arange(s, ix.n, 17, dtype=np.uint32)[:90] for s in range(6)]
    want = [ix.construction_search(b) for b in batches]
    pend = [ix.construction_submit(b) for b in batches]
    for p, w, b in zip(pend, want, batches):
        got = p.wait()
        for x, y in ((got.ids, w.ids), (got.sq, w.sq), (got.n_out, w.n_out), (got.stats, w.stats),
                     (got.pes_n, w.pes_n), (got.pes, w.pes)):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("name", ["euc48", "cos20", "tail10", "deg64", "pad9c", "unit256", "unit512", "unit768",
                                  "unit1024"])
def test_warp_tree_mode_bitexact_vs_oracle_same_order(pag, built, name):
    """exact_dist = 0 (warp-tree FMA partials + xor butterfly) is bit-identical
    to the oracle restating that summation order (pag_oracle.c
    warp_tree_sq_dist): the traversal is shared, so the mode's differences
    from the reference come from the summation order alone."""
    fx = built(name)
    ix = gpu_index(pag, fx["index"])
    oix = O.OracleIndex(fx["index"])
    for K, efS in ((10, 40), (10, 300), (100, 150)):
        got = ix.search_batch(fx["queries"], pag.SearchParams(K=K, efS=efS, exact_dist=False))
        want = oix.search(fx["queries"], K, efS, warp_tree=True)
        assert_same_results((got.ids, got.sq, got.n_out, got.stats), want, f"{name} warp-tree {K}/{efS}")
    nodes = np.arange(0, oix.n, 11, dtype=np.uint32)
    got = ix.construction_search(nodes, pag.SearchParams(K=ix.efC, efS=ix.efC, b_override=ix.b_build,
                                                         exact_dist=False))
    want = oix.construction_search(nodes, warp_tree=True)
    assert_same_results((got.ids, got.sq, got.n_out, got.stats), want[:4], f"{name} warp-tree construction")
    assert np.array_equal(got.pes_n, want[5])
