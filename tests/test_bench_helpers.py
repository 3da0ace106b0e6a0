"""CPU tests of the measurement code in bench.py: the algorithmic-bytes
formula, the readers of the reference binary's result files
(the checker of the full-size parity line), the fallback operating points and
the workload definitions against BASELINE.json."""
from __future__ import annotations

import json
import os

import numpy as np

import bench


def test_algorithmic_bytes_formula():
    # two queries: (exact, test, pass, visited, edges)
    st = np.array([[10, 50, 8, 5, 100], [0, 0, 0, 0, 0]], np.uint64)
    dpad, L, K = 768, 32, 10
    q0 = 4 * dpad + 4 * 5 + 100 * (16 + 16) + 10 * 4 * dpad + 8 * K
    q1 = 4 * dpad + 8 * K
    assert bench.algorithmic_bytes(st, dpad, L, K) == q0 + q1
    # odd subspace count: ceil(L/2) code bytes per edge
    assert bench.algorithmic_bytes(st[:1], 128, 15, 1) == 4 * 128 + 20 + 100 * (16 + 8) + 10 * 512 + 8


def test_reference_result_readers(tmp_path):
    nq, k = 3, 4
    ids = np.arange(nq * k, dtype=np.uint32).reshape(nq, k)
    sq = np.linspace(0, 1, nq * k, dtype=np.float32).reshape(nq, k)
    n_out = np.array([4, 2, 0], np.uint32)
    st = np.arange(nq * 4, dtype=np.uint64).reshape(nq, 4)
    p = tmp_path / "r.bin"
    with open(p, "wb") as f:
        f.write(np.array([nq, k], np.uint64).tobytes() + ids.tobytes() + sq.tobytes() + n_out.tobytes()
                + st.tobytes())
    r = bench.read_reference_results(str(p))
    for a, b in zip(r, (ids, sq, n_out, st)):
        assert np.array_equal(a, b)
    cap = 5
    pes_n = np.array([1, 7, 0], np.uint32)
    pes = np.arange(nq * cap, dtype=np.uint32).reshape(nq, cap)
    p2 = tmp_path / "c.bin"
    with open(p2, "wb") as f:
        f.write(np.array([nq, k, cap], np.uint64).tobytes() + ids.tobytes() + sq.tobytes() + n_out.tobytes()
                + st.tobytes() + pes_n.tobytes() + pes.tobytes())
    r2 = bench.read_reference_construction(str(p2))
    for a, b in zip(r2, (ids, sq, n_out, st, pes_n, pes)):
        assert np.array_equal(a, b)


def test_workloads_match_baseline_configs():
    base = json.load(open(os.path.join(bench.ROOT, "BASELINE.json")))
    cfgs = bench.CONFIGS
    # configs[1]: the headline workload (1M x 768, unit, 4096 centres, sigma 0.4, 10k queries, K = 10)
    c2 = cfgs["cfg2"]
    assert (c2["n"], c2["d"], c2["K"], c2["nq"], c2["centres"], c2["sigma"], c2["unit"]) == \
        (1_000_000, 768, 10, 10_000, 4096, 0.4, True)
    assert "1,000,000" in base["configs"][1] and "d=768" in base["configs"][1]
    assert (cfgs["cfg3"]["n"], cfgs["cfg3"]["d"], cfgs["cfg3"]["K"]) == (1_000_000, 1024, 100)
    assert (cfgs["cfg4"]["n"], cfgs["cfg4"]["d"], cfgs["cfg4"]["K"], cfgs["cfg4"]["nq"]) == (2_000_000, 512, 1000, 20_000)
    assert (cfgs["cfg1"]["n"], cfgs["cfg1"]["d"], cfgs["cfg1"]["K"]) == (20_000, 128, 10)


def test_reference_arm_fallback_operating_points(tmp_path):
    paths = {"index": str(tmp_path / "x.pagidx")}
    assert bench.default_efs(bench.CONFIGS["cfg2"], paths) == 70
    with open(tmp_path / "operating_point.json", "w") as f:
        json.dump({"efS": 80, "sweep": []}, f)
    assert bench.default_efs(bench.CONFIGS["cfg2"], paths) == 80


def _res(ids, sq, n=None, st=None):
    ids = np.asarray(ids, np.uint32)
    sq = np.asarray(sq, np.float32)
    n = np.full(ids.shape[0], ids.shape[1], np.uint32) if n is None else np.asarray(n, np.uint32)
    st = np.zeros((ids.shape[0], 4), np.uint64) if st is None else st
    return ids, sq, n, st


def test_compare_with_reference_bitexact_and_ties():
    r = _res([[1, 2, 3], [4, 5, 6]], [[0.1, 0.2, 0.3], [0.1, 0.2, 0.5]])
    c = bench.compare_with_reference(r, r, 3)
    assert c["ids_equal"] == c["sq_bit_equal"] == c["counters_equal"] == c["id_sets_equal"] == 1.0
    assert c["unexplained_diffs"] == 0 and c["max_rel_sq_diff"] == 0.0
    # query 0: id 3 swapped for id 9 at a distance tie with the K-th (explained);
    # query 1: id 5 (well inside the radius) missing (unexplained)
    g = _res([[1, 2, 9], [4, 6, 7]], [[0.1, 0.2, 0.3 * (1 + 2e-6)], [0.1, 0.5, 0.5]])
    c = bench.compare_with_reference(g, r, 3)
    assert c["id_sets_equal"] == 0.0 and c["unexplained_diffs"] == 1
    # recall against a ground truth, same tie policy as recall_at_k
    gt_ids = np.array([[1, 2, 3], [4, 5, 6]], np.uint32)
    gt_sq = np.array([[0.1, 0.2, 0.3], [0.1, 0.2, 0.5]], np.float32)
    c = bench.compare_with_reference(g, r, 3, gt_ids, gt_sq)
    assert c["reference_recall"] == 1.0 and abs(c["recall_delta"] - (4 / 6 - 1.0)) < 1e-5


def test_reference_arm_imports_no_native_library():
    """bench.py's reference arm must not map libpag_gpu.so (the driver checks
    which repo .so files the reference process loaded): the package exposes
    its API lazily and the measurement helpers are library-free."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import bench; import paper_2603_06660_b200 as p; "
            "from paper_2603_06660_b200 import fvecs, shard, recall; p.mean_recall; p.recall_at_k; "
            "bench.compare_with_reference; "
            "maps = open('/proc/self/maps').read(); assert 'libpag_gpu' not in maps, 'library loaded'; "
            "p.load_index; assert 'libpag_gpu' in open('/proc/self/maps').read(); print('ok')"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr


def test_source_hash_ignores_comments():
    a = "/* header\n note */\nint f() {\n  return 1;  // c\n}\n\n// trailing\n"
    b = "int f() {\n  return 1;\n}\n"
    assert bench._code_only(a) == bench._code_only(b)
    assert bench._code_only("X := 1\n# note\n", makefile=True) == "X := 1"
    assert len(bench.source_sha()) == 16
