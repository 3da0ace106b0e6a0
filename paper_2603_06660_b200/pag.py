"""Host-side mirror of the reference's search API over the B200 library.

Names, argument meaning and error behaviour follow the reference:
  SearchParams / SearchStats   proj/include/pag/routing.hpp:13-34
  SearchResult                 proj/include/pag/routing.hpp:173-177
  load_index                   proj/include/pag/builder.hpp:157
  search                       proj/include/pag/routing.hpp:181-188
  ground_truth / recall_at_k   proj/include/pag/bench.hpp:19-24
Reference exceptions map to Python ones: std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError (same message texts).

The compute path is libpag_gpu.so only (see _lib.py); nothing here computes
search results on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from ._lib import IndexArraysC, SearchParamsC, SearchStatsC, check, lib
from .recall import mean_recall, recall_at_k  # noqa: F401  (bench.hpp:22-24, re-exported)

Candidate = Tuple[int, float]  # (id, squared distance), builder.hpp:18-21


@dataclass
class SearchParams:
    """routing.hpp:13-22 (collect_pes is build-only and absent)."""
    K: int = 10
    efS: int = 100
    b_override: int = 0
    use_prt: bool = True
    use_tfb: bool = True
    exact_dist: bool = True  # reference-order fp32 distances (bit-identical results)

    def b(self) -> int:
        return self.b_override if self.b_override else max(10, self.K)

    def to_c(self) -> SearchParamsC:
        p = SearchParamsC()
        p.K, p.efS, p.b_override = int(self.K), int(self.efS), int(self.b_override)
        p.use_prt, p.use_tfb, p.exact_dist = int(self.use_prt), int(self.use_tfb), int(self.exact_dist)
        return p


@dataclass
class SearchStats:
    """routing.hpp:24-34, plus edges_scanned (sum of deg over expansions)."""
    exact_dist_count: int = 0
    test_count: int = 0
    pass_count: int = 0
    visited_count: int = 0
    edges_scanned: int = 0

    def gamma(self) -> float:
        return self.pass_count / self.test_count if self.test_count else 0.0


@dataclass
class SearchResult:
    """routing.hpp:173-177: K nearest (squared distances, ascending)."""
    results: List[Candidate] = field(default_factory=list)
    stats: SearchStats = field(default_factory=SearchStats)


@dataclass
class BatchResult:
    ids: np.ndarray      # nq x K uint32 (first n_out[i] valid)
    sq: np.ndarray       # nq x K float32
    n_out: np.ndarray    # nq uint32
    stats: np.ndarray    # nq x 5 uint64 {exact, test, pass, visited, edges_scanned}

    def result(self, i: int) -> SearchResult:
        k = int(self.n_out[i])
        s = self.stats[i]
        return SearchResult([(int(a), float(b)) for a, b in zip(self.ids[i, :k], self.sq[i, :k])],
                            SearchStats(*(int(x) for x in s)))


class PendingBatch:
    """An in-flight asynchronous batch (pag_gpu_search_submit); keeps the
    query and result arrays alive until wait()."""

    def __init__(self, index: "PagIndex", ticket: int, queries: np.ndarray, result: BatchResult):
        self._index, self.ticket, self._q, self._res = index, ticket, queries, result
        self._done = False

    def wait(self) -> BatchResult:
        if not self._done:
            self._done = True  # the slot is released even when the batch failed
            self._q = None
            check(lib.pag_gpu_search_wait(self._index.handle, self.ticket))
        return self._res

    def __del__(self):
        # the kernel writes into pinned memory that is unpacked into this
        # batch's arrays at completion: never drop them before that
        if not getattr(self, "_done", True):
            try:
                self.wait()
            except Exception:
                pass


@dataclass
class ConstructionResult(BatchResult):
    """BatchResult plus SearchResult.pes_rejected (routing.hpp:176) per node:
    pes[i, :min(pes_n[i], pes_cap)] in expansion order."""
    pes: np.ndarray = None     # nn x pes_cap uint32
    pes_n: np.ndarray = None   # nn uint32 (full count)

    def pes_rejected(self, i: int) -> List[int]:
        if int(self.pes_n[i]) > self.pes.shape[1]:
            raise RuntimeError("pes_rejected list truncated: raise pes_cap")
        return [int(x) for x in self.pes[i, :int(self.pes_n[i])]]


@dataclass
class IndexArrays:
    """The reference's in-memory PagIndex as host arrays (builder.hpp:62-132):
    the header parameters, and the fixed-stride storage the accessors
    targets(u) / scalars(u) / edge_codes(u, j) / vectors().row(i) expose.
    The source of PagIndex.from_arrays / refresh_from_arrays."""
    dim: int
    padded_dim: int
    L: int
    m: int
    M: int
    efC: int
    b_build: int
    pes_flush_interval: int
    seed: int
    metric: int            # 0 euclidean, 1 cosine
    enable_pes: bool
    entry_nodes: np.ndarray  # u32
    degrees: np.ndarray      # n u32
    targets: np.ndarray      # n x 2M u32
    scalars: np.ndarray      # n x 2M x 3 f32 {cos_beta, edge_norm, base_offset}
    codes: np.ndarray        # n x 2M x ceil(L/2) u8
    rows: np.ndarray         # n x padded_dim f32
    norms: Optional[np.ndarray] = None  # n f32 (None: computed from the rows)

    @property
    def n(self) -> int:
        return int(self.degrees.shape[0])

    @classmethod
    def from_file(cls, path: str) -> "IndexArrays":
        """load_index (builder.cpp:434-492) into host arrays: the PAGIDX01 v1
        records restored into the fixed-stride layout (restore_edge)."""
        buf = np.fromfile(path, np.uint8)
        hdr = np.frombuffer(buf[:66].tobytes(), np.dtype([
            ("magic", "<u8"), ("version", "<u4"), ("n", "<u8"), ("dim", "<u4"), ("padded", "<u4"), ("L", "<u4"),
            ("m", "<u4"), ("M", "<u4"), ("efC", "<u4"), ("b_build", "<u4"), ("pes", "<u4"), ("seed", "<u8"),
            ("metric", "u1"), ("enable_pes", "u1"), ("n_entries", "<u4")]))[0]
        if int(hdr["magic"]) != 0x5041474944583031:
            raise RuntimeError("bad index magic")
        if int(hdr["version"]) != 1:
            raise RuntimeError("unsupported index version")
        n, padded, M = int(hdr["n"]), int(hdr["padded"]), int(hdr["M"])
        L = int(hdr["L"]) or int(lib.pag_gpu_default_subspace_count(int(hdr["dim"])))
        cb, cap, ne = (L + 1) // 2, 2 * M, int(hdr["n_entries"])
        off = 66
        entries = np.frombuffer(buf[off:off + 4 * ne].tobytes(), "<u4").copy()
        off += 4 * ne
        deg = np.zeros(n, np.uint32)
        tg = np.zeros((n, cap), np.uint32)
        sc = np.zeros((n, cap, 3), np.float32)
        cd = np.zeros((n, cap, cb), np.uint8)
        rec = np.dtype([("t", "<u4"), ("codes", "u1", (cb,)), ("sc", "<f4", (3,))])
        for u in range(n):
            d = int(np.frombuffer(buf[off:off + 4].tobytes(), "<u4")[0])
            off += 4
            if d > cap:
                raise RuntimeError("degree over cap in file")
            r = np.frombuffer(buf[off:off + rec.itemsize * d].tobytes(), rec)
            off += rec.itemsize * d
            deg[u], tg[u, :d], cd[u, :d], sc[u, :d] = d, r["t"], r["codes"], r["sc"]
        rows = np.frombuffer(buf[off:off + 4 * n * padded].tobytes(), "<f4").reshape(n, padded).copy()
        off += 4 * n * padded
        norms = np.frombuffer(buf[off:off + 4 * n].tobytes(), "<f4").copy()
        if norms.shape[0] != n:
            raise RuntimeError("index read failed")
        return cls(int(hdr["dim"]), padded, L, int(hdr["m"]), M, int(hdr["efC"]), int(hdr["b_build"]),
                   int(hdr["pes"]), int(hdr["seed"]), int(hdr["metric"]), bool(hdr["enable_pes"]), entries, deg, tg,
                   sc, cd, rows, norms)

    def to_c(self):
        """(pag_index_arrays, the contiguous arrays it borrows)."""
        keep = [np.ascontiguousarray(self.entry_nodes, np.uint32), np.ascontiguousarray(self.degrees, np.uint32),
                np.ascontiguousarray(self.targets, np.uint32), np.ascontiguousarray(self.scalars, np.float32),
                np.ascontiguousarray(self.codes, np.uint8), np.ascontiguousarray(self.rows, np.float32),
                None if self.norms is None else np.ascontiguousarray(self.norms, np.float32)]
        a = IndexArraysC()
        a.n, a.dim, a.padded_dim, a.L, a.m, a.M = self.n, self.dim, self.padded_dim, self.L, self.m, self.M
        a.efC, a.b_build, a.pes_flush_interval, a.seed = self.efC, self.b_build, self.pes_flush_interval, self.seed
        a.metric, a.enable_pes, a.n_entries = self.metric, int(self.enable_pes), keep[0].shape[0]
        (a.entry_nodes, a.degrees, a.targets, a.scalars, a.codes, a.rows, a.norms) = (
            None if k is None else k.ctypes.data for k in keep)
        return a, keep


class PagIndex:
    """A PAGIDX01 index resident in HBM on one or more GPUs (move-only in the
    reference, builder.hpp:62-69; here a handle released by close())."""

    def __init__(self, path: Optional[str], devices: Sequence[int] = (0,), arrays: Optional[IndexArrays] = None):
        """One replica per entry of `devices` (CUDA device ordinals; an entry
        may repeat, giving several replicas on one GPU). Batches are split
        into contiguous shards, one per replica (pag_gpu_open_devices).
        With `arrays` the source is the in-memory index (pag_gpu_open_from_arrays)."""
        devs = [int(d) for d in devices] or [0]
        arr = (C.c_int * len(devs))(*devs)
        self._h = C.c_void_p()
        if arrays is not None:
            a, keep = arrays.to_c()
            check(lib.pag_gpu_open_from_arrays(C.byref(a), arr, len(devs), C.byref(self._h)))
            del keep
        else:
            check(lib.pag_gpu_open_devices(path.encode(), arr, len(devs), C.byref(self._h)))
        info = np.zeros(16, np.uint64)
        check(lib.pag_gpu_info(self._h, info, 16))
        (self.n, self.dim, self.padded_dim, self.L, self.m, self.M, metric, self.n_entries,
         self.seed, self.total_edges, self.n_devices, self.device_bytes, _, self.efC, self.b_build,
         enable_pes) = (int(x) for x in info)
        self.enable_pes = bool(enable_pes)
        self.metric = "cosine" if metric == 1 else "euclidean"
        self.path = path

    # reference accessors (builder.hpp:71-91)
    def size(self) -> int:
        return self.n

    def max_degree(self) -> int:
        return 2 * self.M

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            check(lib.pag_gpu_close(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def search_batch(self, queries: np.ndarray, params: SearchParams) -> BatchResult:
        q = np.ascontiguousarray(queries, np.float32)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        if q.shape[1] != self.dim:
            raise ValueError("query dimension mismatch")  # routing.cpp:252
        nq = q.shape[0]
        K = int(params.K)
        # entries past n_out[i] are unspecified (as the device path)
        ids = np.empty((nq, K), np.uint32)
        sq = np.empty((nq, K), np.float32)
        n_out = np.empty(nq, np.uint32)
        stats = np.empty((nq, 5), np.uint64)  # pag_search_stats rows (5 x u64)
        pc = params.to_c()
        check(lib.pag_gpu_search(self._h, q.ctypes.data if nq else None, nq, C.byref(pc),
                                 ids.ctypes.data if K and nq else None,
                                 sq.ctypes.data if K and nq else None,
                                 n_out.ctypes.data if nq else None, stats.ctypes.data if nq else None))
        return BatchResult(ids, sq, n_out, stats)

    def search_submit(self, queries: np.ndarray, params: SearchParams,
                      out: Optional[BatchResult] = None) -> "PendingBatch":
        """Asynchronous search_batch: returns at once; PendingBatch.wait()
        gives the BatchResult (written into `out` when given: reusing result
        arrays avoids first-touch page faults). Pinned query arrays are read
        in place by the kernel (keep them alive and unmodified until wait)."""
        q = np.ascontiguousarray(queries, np.float32)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        if q.shape[1] != self.dim:
            raise ValueError("query dimension mismatch")  # routing.cpp:252
        nq = q.shape[0]
        K = int(params.K)
        if out is not None:
            if (out.ids.shape != (nq, K) or out.sq.shape != (nq, K) or out.n_out.shape != (nq,)
                    or out.stats.shape != (nq, 5) or out.ids.dtype != np.uint32 or out.sq.dtype != np.float32
                    or out.n_out.dtype != np.uint32 or out.stats.dtype != np.uint64
                    or not all(a.flags.c_contiguous for a in (out.ids, out.sq, out.n_out, out.stats))):
                raise ValueError("out arrays do not match the batch")
            res = out
        else:
            res = BatchResult(np.empty((nq, K), np.uint32), np.empty((nq, K), np.float32),
                              np.empty(nq, np.uint32), np.empty((nq, 5), np.uint64))
        t = C.c_uint64(0)
        pc = params.to_c()
        check(lib.pag_gpu_search_submit(self._h, q.ctypes.data if nq else None, nq, C.byref(pc),
                                        res.ids.ctypes.data if K and nq else None,
                                        res.sq.ctypes.data if K and nq else None,
                                        res.n_out.ctypes.data if nq else None,
                                        res.stats.ctypes.data if nq else None, C.byref(t)))
        return PendingBatch(self, int(t.value), q, res)

    def construction_search(self, nodes, params: Optional[SearchParams] = None,
                            collect_pes: Optional[bool] = None, pes_cap: int = 256,
                            out: Optional[ConstructionResult] = None) -> ConstructionResult:
        """The search step of insert_with_state (builder.cpp:218-227) for
        nodes already in the index: query = the node's stored row, K = efS =
        efC, b = b_build, PES tracking per enable_pes (params / collect_pes
        override). Returns results, counters and pes_rejected lists; `out`
        (same shapes, C-contiguous) is filled instead of new arrays."""
        nodes = np.ascontiguousarray(nodes, np.uint32).reshape(-1)
        nn = len(nodes)
        K = int(params.K) if params is not None else self.efC
        if out is not None:
            ids, sq, n_out, pes, pes_n = out.ids, out.sq, out.n_out, out.pes, out.pes_n
            for a, shape, dt in ((ids, (nn, K), np.uint32), (sq, (nn, K), np.float32), (n_out, (nn,), np.uint32),
                                 (pes, (nn, pes_cap), np.uint32), (pes_n, (nn,), np.uint32)):
                if a.shape != shape or a.dtype != dt or not a.flags.c_contiguous:
                    raise ValueError("out arrays do not match the batch")
        else:
            ids = np.zeros((nn, K), np.uint32)
            sq = np.zeros((nn, K), np.float32)
            n_out = np.zeros(nn, np.uint32)
            pes = np.zeros((nn, pes_cap), np.uint32)
            pes_n = np.zeros(nn, np.uint32)
        st = (SearchStatsC * max(nn, 1))()
        pc = params.to_c() if params is not None else None
        cp = -1 if collect_pes is None else int(bool(collect_pes))
        check(lib.pag_gpu_construction_search(self._h, nodes.ctypes.data if nn else None, nn,
                                              C.byref(pc) if pc is not None else None, cp,
                                              ids.ctypes.data if K and nn else None,
                                              sq.ctypes.data if K and nn else None,
                                              n_out.ctypes.data if nn else None, st,
                                              pes.ctypes.data if pes_cap and nn else None, pes_cap,
                                              pes_n.ctypes.data if nn else None))
        stats = np.ctypeslib.as_array(C.cast(st, C.POINTER(C.c_uint64)), (max(nn, 1), 5))[:nn]
        if out is not None:
            out.stats[:] = stats
            return out
        return ConstructionResult(ids, sq, n_out, stats.copy(), pes, pes_n)

    def construction_submit(self, nodes, params: Optional[SearchParams] = None, collect_pes: Optional[bool] = None,
                            pes_cap: int = 256, out: Optional[ConstructionResult] = None) -> "PendingBatch":
        """Asynchronous construction_search (pag_gpu_construction_submit):
        returns at once; PendingBatch.wait() gives the ConstructionResult
        (written into `out` when given)."""
        nodes = np.ascontiguousarray(nodes, np.uint32).reshape(-1)
        nn = len(nodes)
        K = int(params.K) if params is not None else self.efC
        if out is not None:
            res = out
            for a, shape, dt in ((res.ids, (nn, K), np.uint32), (res.sq, (nn, K), np.float32),
                                 (res.n_out, (nn,), np.uint32), (res.stats, (nn, 5), np.uint64),
                                 (res.pes, (nn, pes_cap), np.uint32), (res.pes_n, (nn,), np.uint32)):
                if a.shape != shape or a.dtype != dt or not a.flags.c_contiguous:
                    raise ValueError("out arrays do not match the batch")
        else:
            res = ConstructionResult(np.empty((nn, K), np.uint32), np.empty((nn, K), np.float32),
                                     np.empty(nn, np.uint32), np.empty((nn, 5), np.uint64),
                                     np.empty((nn, pes_cap), np.uint32), np.empty(nn, np.uint32))
        pc = params.to_c() if params is not None else None
        cp = -1 if collect_pes is None else int(bool(collect_pes))
        t = C.c_uint64(0)
        check(lib.pag_gpu_construction_submit(self._h, nodes.ctypes.data if nn else None, nn,
                                              C.byref(pc) if pc is not None else None, cp,
                                              res.ids.ctypes.data if K and nn else None,
                                              res.sq.ctypes.data if K and nn else None,
                                              res.n_out.ctypes.data if nn else None,
                                              res.stats.ctypes.data if nn else None,
                                              res.pes.ctypes.data if pes_cap and nn else None, pes_cap,
                                              res.pes_n.ctypes.data if nn else None, C.byref(t)))
        return PendingBatch(self, int(t.value), nodes, res)

    def construction_search_device(self, nodes_ptr: int, nn: int, params: Optional[SearchParams],
                                   collect_pes: Optional[bool], ids_ptr: int, sq_ptr: int, n_out_ptr: int,
                                   stats_ptr: int, pes_ptr: int, pes_cap: int, pes_n_ptr: int,
                                   stream: int = 0) -> None:
        """Device-resident construction batch (async on `stream`)."""
        pc = params.to_c() if params is not None else None
        cp = -1 if collect_pes is None else int(bool(collect_pes))
        check(lib.pag_gpu_construction_search_device(self._h, nodes_ptr, nn, C.byref(pc) if pc is not None else None,
                                                     cp, ids_ptr, sq_ptr, n_out_ptr, stats_ptr, pes_ptr, pes_cap,
                                                     pes_n_ptr, stream or None))

    def search_device(self, q_ptr: int, nq: int, params: SearchParams, ids_ptr: int, sq_ptr: int,
                      n_out_ptr: int, stats_ptr: int, stream: int = 0) -> None:
        """Device-resident batch (pointers on the handle's first GPU); async
        on `stream`. Raw counters: nq x 8 uint32."""
        pc = params.to_c()
        check(lib.pag_gpu_search_device(self._h, q_ptr, nq, C.byref(pc), ids_ptr, sq_ptr,
                                        n_out_ptr, stats_ptr, stream or None))

    def refresh(self, path: str) -> dict:
        """Re-synchronise with a newer file of the same index (online inserts
        applied by the reference); uploads only what changed."""
        st = np.zeros(4, np.uint64)
        check(lib.pag_gpu_refresh(self._h, path.encode(), st))
        info = np.zeros(12, np.uint64)
        check(lib.pag_gpu_info(self._h, info, 12))
        self.n, self.total_edges, self.device_bytes = int(info[0]), int(info[9]), int(info[11])
        self.path = path
        return {"new_nodes": int(st[0]), "changed_blocks": int(st[1]), "bytes_uploaded": int(st[2]),
                "seconds": int(st[3]) / 1e6}

    @classmethod
    def from_arrays(cls, arrays: IndexArrays, devices: Sequence[int] = (0,)) -> "PagIndex":
        """The in-memory index as the source (no file round trip)."""
        return cls(None, devices, arrays=arrays)

    def refresh_from_arrays(self, arrays: IndexArrays) -> dict:
        """refresh() with the in-memory index as the newer state."""
        st = np.zeros(4, np.uint64)
        a, keep = arrays.to_c()
        check(lib.pag_gpu_refresh_from_arrays(self._h, C.byref(a), st))
        del keep
        info = np.zeros(12, np.uint64)
        check(lib.pag_gpu_info(self._h, info, 12))
        self.n, self.total_edges, self.device_bytes = int(info[0]), int(info[9]), int(info[11])
        return {"new_nodes": int(st[0]), "changed_blocks": int(st[1]), "bytes_uploaded": int(st[2]),
                "seconds": int(st[3]) / 1e6}

    def dup_nodes(self) -> int:
        """Nodes repeating a target inside one 32-edge group (0: the search
        skips its in-group duplicate resolution)."""
        info = np.zeros(17, np.uint64)
        check(lib.pag_gpu_info(self._h, info, 17))
        return int(info[16])

    def gt_uncertified(self) -> int:
        """Tensor-core ground-truth queries that failed the certificate and were re-run exactly."""
        info = np.zeros(13, np.uint64)
        check(lib.pag_gpu_info(self._h, info, 13))
        return int(info[12])

    def ground_truth(self, queries: np.ndarray, k: int) -> Tuple[np.ndarray, np.ndarray]:
        """bench.cpp:18-53 over the resident base rows: top-min(k, n) by (sq, id)."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        nq = q.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        sq = np.zeros((nq, k), np.float32)
        check(lib.pag_gpu_ground_truth(self._h, q.reshape(-1), nq, k, ids.reshape(-1), sq.reshape(-1)))
        kk = min(k, self.n)
        return ids[:, :kk], sq[:, :kk]


def load_index(path: str, devices: Sequence[int] = (0,)) -> PagIndex:
    """builder.hpp:157 load_index, onto the GPUs in `devices`."""
    return PagIndex(path, devices)


def search(index: PagIndex, q, params: Optional[SearchParams] = None) -> SearchResult:
    """routing.hpp:181-188: one query (dim() raw components)."""
    params = params or SearchParams()
    q = np.ascontiguousarray(q, np.float32).reshape(-1)
    if q.size != index.dim:
        raise ValueError("query dimension mismatch")
    return index.search_batch(q.reshape(1, -1), params).result(0)


def ground_truth(index: PagIndex, queries: np.ndarray, k_star: int):
    return index.ground_truth(queries, k_star)
