"""ctypes front-end for the CPU ORACLE (test infrastructure only).

Wraps oracle/liboracle.so (the plain-C restatement of the reference query
path, oracle/pag_oracle.c) and drives oracle/_ref/pag_ref (the unmodified
reference compiled from its own sources). Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this module,
and only as the checker or the reported CPU baseline. The product
(paper_2603_06660_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_BIN = os.path.join(HERE, "_ref", "pag_ref")

_lib = None


def build(force: bool = False) -> None:
    """Compile liboracle.so (and _ref/pag_ref when /root/reference exists)."""
    args = ["make", "-C", HERE, "-s"]
    if force:
        args.append("-B")
    subprocess.run(args, check=True)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
    u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
    f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
    u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
    sig = {
        "pago_last_error": (C.c_char_p, []),
        "pago_sq_dist": (C.c_float, [f32p, f32p, C.c_size_t]),
        "pago_vec_norm": (C.c_float, [f32p, C.c_size_t]),
        "pago_default_subspace_count": (C.c_uint32, [C.c_uint32]),
        "pago_build_reference_set": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, f32p]),
        "pago_build_projection_table": (None, [f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32, f32p]),
        "pago_table_code_sum": (C.c_float, [f32p, C.c_uint32, C.c_uint32, u8p]),
        "pago_code_at": (C.c_uint32, [u8p, C.c_uint32]),
        "pago_set_code": (None, [u8p, C.c_uint32, C.c_uint32]),
        "pago_prt_test": (C.c_int, [C.c_float, C.c_float, C.c_float]),
        "pago_prt_threshold": (C.c_float, [C.c_float, C.c_float, C.c_float]),
        "pago_mt64_stream": (None, [C.c_uint64, u64p, C.c_size_t]),
        "pago_normal_stream": (None, [C.c_uint64, f64p, C.c_size_t]),
        "pago_load": (C.c_int, [C.c_char_p, C.POINTER(P)]),
        "pago_free": (None, [P]),
        "pago_info": (None, [P, u64p]),
        "pago_refs": (C.POINTER(C.c_float), [P]),
        "pago_entry_nodes": (C.POINTER(C.c_uint32), [P]),
        "pago_degree": (C.c_uint32, [P, C.c_uint32]),
        "pago_targets": (C.POINTER(C.c_uint32), [P, C.c_uint32]),
        "pago_scalars": (C.POINTER(C.c_float), [P, C.c_uint32]),
        "pago_codes": (C.POINTER(C.c_uint8), [P, C.c_uint32]),
        "pago_row": (C.POINTER(C.c_float), [P, C.c_uint32]),
        "pago_set_distance_mode": (None, [P, C.c_int]),
        "pago_search": (C.c_int, [P, f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.c_int, C.c_int, u32p, f32p, u32p, u64p]),
        "pago_query_table": (C.c_int, [P, f32p, f32p]),
        "pago_construction_search": (C.c_int, [P, u32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.c_int, u32p, f32p, u32p, u64p, u32p, C.c_uint32, u32p]),
        "pago_build_params": (None, [P, u32p]),
        "pago_ground_truth": (C.c_int, [f32p, C.c_uint64, f32p, C.c_uint64, C.c_uint32,
                                        C.c_uint32, u32p, f32p]),
        "pago_recall_at_k": (C.c_double, [u32p, C.c_size_t, u32p, f32p, C.c_size_t, C.c_uint32]),
        "pago_tfb_new": (P, [C.c_size_t, C.c_uint32, C.c_uint32]),
        "pago_tfb_free": (None, [P]),
        "pago_tfb_seed": (None, [P, C.c_uint32, C.c_float]),
        "pago_tfb_admit": (None, [P, C.c_uint32, C.c_float]),
        "pago_tfb_push_fp": (None, [P, C.c_uint32, C.c_float]),
        "pago_tfb_push_result": (None, [P, C.c_uint32, C.c_float]),
        "pago_tfb_end_round": (C.c_int, [P]),
        "pago_tfb_next_unvisited": (C.c_int64, [P]),
        "pago_tfb_set_visited": (None, [P, C.c_size_t, C.c_int]),
        "pago_tfb_admission_sq": (C.c_float, [P]),
        "pago_tfb_admission_dist": (C.c_float, [P]),
        "pago_tfb_dump": (C.c_size_t, [P, C.c_int, u32p, f32p, u8p, C.c_size_t]),
        "pago_tfb_validate": (C.c_int, [P]),
        "pago_ring_kat": (C.c_size_t, [C.c_uint32, u32p, f32p, C.c_size_t, u32p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _check(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc, lib().pago_last_error().decode())


class OracleIndex:
    """A PAGIDX01 file loaded by the oracle's restated loader."""

    def __init__(self, path: str):
        self._h = C.c_void_p()
        _check(lib().pago_load(path.encode(), C.byref(self._h)))
        info = np.zeros(10, np.uint64)
        lib().pago_info(self._h, info)
        (self.n, self.dim, self.padded, self.L, self.m, self.M, self.metric,
         self.n_entries, self.seed, self.total_edges) = (int(x) for x in info)
        self.sub_dim = self.padded // self.L
        bp = np.zeros(4, np.uint32)
        lib().pago_build_params(self._h, bp)
        self.efC, self.b_build, self.enable_pes, self.pes_flush = (int(x) for x in bp)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            lib().pago_free(h)
            self._h = C.c_void_p()

    def refs(self) -> np.ndarray:
        p = lib().pago_refs(self._h)
        return np.ctypeslib.as_array(p, (self.L * self.m * self.sub_dim,)).copy()

    def entry_nodes(self) -> np.ndarray:
        p = lib().pago_entry_nodes(self._h)
        return np.ctypeslib.as_array(p, (max(self.n_entries, 1),))[: self.n_entries].copy()

    def row(self, i: int) -> np.ndarray:
        return np.ctypeslib.as_array(lib().pago_row(self._h, i), (self.padded,)).copy()

    def rows(self) -> np.ndarray:
        p = lib().pago_row(self._h, 0)
        return np.ctypeslib.as_array(p, (self.n, self.padded)).copy()

    def degree(self, u: int) -> int:
        return int(lib().pago_degree(self._h, u))

    def set_warp_tree(self, on: bool) -> None:
        """Distances in the B200 library's warp-tree order (its exact_dist = 0
        mode) instead of the reference order, for the search and the
        construction search (pag_oracle.c warp_tree_sq_dist)."""
        lib().pago_set_distance_mode(self._h, int(bool(on)))

    def search(self, queries: np.ndarray, K: int, efS: int, b_override: int = 0,
               use_prt: bool = True, use_tfb: bool = True, warp_tree: bool = False):
        self.set_warp_tree(warp_tree)
        try:
            return self._search(queries, K, efS, b_override, use_prt, use_tfb)
        finally:
            self.set_warp_tree(False)

    def _search(self, queries, K, efS, b_override, use_prt, use_tfb):
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        nq = q.shape[0]
        ids = np.full((nq, max(K, 1)), 0xFFFFFFFF, np.uint32)
        sq = np.zeros((nq, max(K, 1)), np.float32)
        n_out = np.zeros(nq, np.uint32)
        stats = np.zeros((nq, 5), np.uint64)
        if K == 0:
            ids = np.zeros((nq, 0), np.uint32)
            sq = np.zeros((nq, 0), np.float32)
            ids_buf = np.zeros(1, np.uint32)
            sq_buf = np.zeros(1, np.float32)
            _check(lib().pago_search(self._h, q.reshape(-1) if nq else np.zeros(1, np.float32),
                                     nq, K, efS, b_override, int(use_prt), int(use_tfb),
                                     ids_buf, sq_buf, n_out, stats.reshape(-1)))
            return ids, sq, n_out, stats
        _check(lib().pago_search(self._h, q.reshape(-1) if nq else np.zeros(1, np.float32), nq,
                                 K, efS, b_override, int(use_prt), int(use_tfb),
                                 ids.reshape(-1), sq.reshape(-1), n_out, stats.reshape(-1)))
        return ids, sq, n_out, stats

    def construction_search(self, nodes, K=None, efS=None, b_override=None, collect_pes=None,
                            pes_cap: int = 256, warp_tree: bool = False):
        """insert_with_state's search (builder.cpp:218-227) for existing nodes:
        returns (ids, sq, n_out, stats[nn,5], pes[nn,pes_cap], pes_n)."""
        self.set_warp_tree(warp_tree)
        try:
            return self._construction_search(nodes, K, efS, b_override, collect_pes, pes_cap)
        finally:
            self.set_warp_tree(False)

    def _construction_search(self, nodes, K, efS, b_override, collect_pes, pes_cap):
        nodes = np.ascontiguousarray(nodes, np.uint32).reshape(-1)
        K = self.efC if K is None else K
        efS = self.efC if efS is None else efS
        b = self.b_build if b_override is None else b_override
        pes_on = bool(self.enable_pes) if collect_pes is None else bool(collect_pes)
        nn = len(nodes)
        ids = np.full((nn, max(K, 1)), 0xFFFFFFFF, np.uint32)
        sq = np.zeros((nn, max(K, 1)), np.float32)
        n_out = np.zeros(nn, np.uint32)
        stats = np.zeros((nn, 5), np.uint64)
        pes = np.zeros((nn, max(pes_cap, 1)), np.uint32)
        pes_n = np.zeros(nn, np.uint32)
        _check(lib().pago_construction_search(self._h, nodes if nn else np.zeros(1, np.uint32), nn, K, efS, b,
                                              int(pes_on), ids.reshape(-1), sq.reshape(-1), n_out,
                                              stats.reshape(-1), pes.reshape(-1), pes_cap, pes_n))
        return ids[:, :K], sq[:, :K], n_out, stats, pes[:, :pes_cap], pes_n

    def query_table(self, q: np.ndarray) -> np.ndarray:
        out = np.zeros(self.L * self.m, np.float32)
        _check(lib().pago_query_table(self._h, np.ascontiguousarray(q, np.float32), out))
        return out


def ground_truth(base: np.ndarray, queries: np.ndarray, k: int):
    base = np.ascontiguousarray(base, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    n, d = base.shape
    nq = queries.shape[0]
    ids = np.full((nq, k), 0xFFFFFFFF, np.uint32)
    sq = np.zeros((nq, k), np.float32)
    _check(lib().pago_ground_truth(base.reshape(-1), n, queries.reshape(-1), nq, d, k,
                                   ids.reshape(-1), sq.reshape(-1)))
    kk = min(k, n)
    return ids[:, :kk], sq[:, :kk]


def recall_at_k(result_ids: np.ndarray, truth_ids: np.ndarray, truth_sq: np.ndarray, K: int) -> float:
    r = np.ascontiguousarray(result_ids, np.uint32)
    t = np.ascontiguousarray(truth_ids, np.uint32)
    s = np.ascontiguousarray(truth_sq, np.float32)
    return float(lib().pago_recall_at_k(r, r.size, t, s, t.size, K))


# --------------------------------------------------------------------------
# the unmodified reference (oracle/_ref/pag_ref)
# --------------------------------------------------------------------------

def have_ref() -> bool:
    return os.path.exists(REF_BIN)


def ref_run(cmd: str, **kw) -> str:
    args = [REF_BIN, cmd]
    for k, v in kw.items():
        k = k.replace("_", "-") if k in ("no_prt", "no_tfb", "no_pes", "no_warm") else k
        if v is True:
            args.append(f"--{k}")
        elif v is False or v is None:
            continue
        else:
            args.append(f"--{k}={v}")
    out = subprocess.run(args, check=True, capture_output=True, text=True)
    return out.stdout


def ref_search(index: str, queries: str, K: int, efS: int, out: str, **kw):
    """Run the reference search; returns (ids, sq, n_out, stats[nq,4], timing)."""
    txt = ref_run("search", index=index, queries=queries, K=K, efS=efS, out=out, **kw)
    timing = json.loads(txt.strip().splitlines()[-1])
    with open(out, "rb") as f:
        nq, k = np.frombuffer(f.read(16), np.uint64)
        nq, k = int(nq), int(k)
        ids = np.frombuffer(f.read(nq * k * 4), np.uint32).reshape(nq, k)
        sq = np.frombuffer(f.read(nq * k * 4), np.float32).reshape(nq, k)
        n_out = np.frombuffer(f.read(nq * 4), np.uint32)
        stats = np.frombuffer(f.read(nq * 32), np.uint64).reshape(nq, 4)
    return ids, sq, n_out, stats, timing


def ref_build_search(index: str, count: int, stride: int, out: str, **kw):
    """The reference's construction search (search_padded with collect_pes) for
    nodes (i * stride) % n; returns (nodes, ids, sq, n_out, stats[nn,4], pes, pes_n, timing)."""
    txt = ref_run("build-search", index=index, count=count, stride=stride, out=out, **kw)
    timing = json.loads(txt.strip().splitlines()[-1])
    with open(out, "rb") as f:
        nn, k, cap = (int(x) for x in np.frombuffer(f.read(24), np.uint64))
        ids = np.frombuffer(f.read(nn * k * 4), np.uint32).reshape(nn, k)
        sq = np.frombuffer(f.read(nn * k * 4), np.float32).reshape(nn, k)
        n_out = np.frombuffer(f.read(nn * 4), np.uint32)
        stats = np.frombuffer(f.read(nn * 32), np.uint64).reshape(nn, 4)
        pes_n = np.frombuffer(f.read(nn * 4), np.uint32)
        pes = np.frombuffer(f.read(nn * cap * 4), np.uint32).reshape(nn, cap)
    return ids, sq, n_out, stats, pes, pes_n, timing


def ref_gt(base: str, queries: str, k: int, out: str, threads: int = 1):
    ref_run("gt", base=base, queries=queries, k=k, out=out, threads=threads)
    with open(out, "rb") as f:
        nq, kk = (int(x) for x in np.frombuffer(f.read(16), np.uint64))
        ids = np.frombuffer(f.read(nq * kk * 4), np.uint32).reshape(nq, kk)
        sq = np.frombuffer(f.read(nq * kk * 4), np.float32).reshape(nq, kk)
    return ids, sq


def ref_refs(index: str, out: str):
    ref_run("refs", index=index, out=out)
    with open(out, "rb") as f:
        L, m, sub, ne = (int(x) for x in np.frombuffer(f.read(32), np.uint64))
        refs = np.frombuffer(f.read(L * m * sub * 4), np.float32).copy()
        entries = np.frombuffer(f.read(ne * 4), np.uint32).copy()
    return refs, entries


def ref_tables(index: str, queries: str, out: str):
    ref_run("tables", index=index, queries=queries, out=out)
    with open(out, "rb") as f:
        nq, L, m = (int(x) for x in np.frombuffer(f.read(24), np.uint64))
        return np.frombuffer(f.read(nq * L * m * 4), np.float32).reshape(nq, L * m).copy()


def ref_build(data: str, out: str, threads: int = 1, **params) -> dict:
    txt = ref_run("build", data=data, out=out, threads=threads, **params)
    return json.loads(txt.strip().splitlines()[-1])


def ref_gen_synthetic(kind: str, n: int, d: int, seed: int, out: str, metric: str = "euclidean"):
    ref_run("gen-synthetic", kind=kind, n=n, d=d, seed=seed, out=out, metric=metric)
