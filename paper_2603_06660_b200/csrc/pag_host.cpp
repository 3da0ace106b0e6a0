// pag_host.cpp — host side of the B200-native PAG query path: PAGIDX01
// ingest, reference-family regeneration, HBM residency per GPU, the batched
// search / ground-truth drivers and the C ABI declared in include/pag_gpu.h.
//
// Reference interfaces mirrored (paths relative to the reference root):
//   load_index            proj/src/builder.cpp:434-492 (+ PagIndex ctor :40-46)
//   build_reference_set   proj/src/projection.cpp:13-74
//   search                proj/src/routing.cpp:206-261
//   ground_truth          proj/src/bench.cpp:18-53
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <exception>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/pag_gpu.h"
#include "pag_device.h"

namespace {

thread_local std::string g_err;

struct PagError {
    int code;
    std::string msg;
};

[[noreturn]] void throw_err(int code, std::string msg) { throw PagError{code, std::move(msg)}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw_err(PAG_GPU_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Reference family (projection.cpp:13-74), regenerated bit-identically with
// the same libstdc++ engine and distribution: one mt19937_64 shared across
// subspaces in l-major order, a fresh normal_distribution per rotation,
// modified Gram-Schmidt in double, cast to float, vertices +e_1..+e_k then
// -e_1..-e_k scaled by 1/sqrt(L).
// ---------------------------------------------------------------------------
void haar_rotation(uint32_t k, std::mt19937_64& rng, std::vector<float>& out) {
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::vector<double> basis(static_cast<size_t>(k) * k, 0.0), v(k);
    for (uint32_t c = 0; c < k; ++c) {
        for (;;) {
            for (uint32_t r = 0; r < k; ++r) v[r] = gauss(rng);
            for (uint32_t p = 0; p < c; ++p) {
                const double* bp = &basis[static_cast<size_t>(p) * k];
                double dot = 0;
                for (uint32_t r = 0; r < k; ++r) dot += v[r] * bp[r];
                for (uint32_t r = 0; r < k; ++r) v[r] -= dot * bp[r];
            }
            double nn = 0;
            for (uint32_t r = 0; r < k; ++r) nn += v[r] * v[r];
            nn = std::sqrt(nn);
            if (nn > 1e-9) {
                for (uint32_t r = 0; r < k; ++r) basis[static_cast<size_t>(c) * k + r] = v[r] / nn;
                break;
            }
        }
    }
    out.resize(basis.size());
    for (size_t i = 0; i < basis.size(); ++i) out[i] = static_cast<float>(basis[i]);
}

std::vector<float> reference_family(uint32_t padded, uint32_t L, uint32_t m, uint64_t seed) {
    if (L == 0 || padded % L != 0) throw_err(PAG_GPU_EINVAL, "padded_dim not divisible by L");
    const uint32_t sub = padded / L;
    if (sub < 2) throw_err(PAG_GPU_EINVAL, "sub_dim < 2: cross-polytope degenerate");
    if (m == 0 || m > 16) throw_err(PAG_GPU_EINVAL, "m must be in [1, 16] (4-bit codes)");
    std::vector<float> refs(static_cast<size_t>(L) * m * sub, 0.0f);
    const float scale = 1.0f / std::sqrt(static_cast<float>(L));
    const uint32_t per_polytope = 2 * sub;
    const uint32_t polytopes = (m + per_polytope - 1) / per_polytope;
    std::mt19937_64 rng(seed);
    std::vector<float> rot;
    for (uint32_t l = 0; l < L; ++l) {
        uint32_t j = 0;
        for (uint32_t p = 0; p < polytopes && j < m; ++p) {
            haar_rotation(sub, rng, rot);
            for (uint32_t sgn = 0; sgn < 2 && j < m; ++sgn) {
                const float s = sgn == 0 ? scale : -scale;
                for (uint32_t c = 0; c < sub && j < m; ++c, ++j) {
                    float* dst = &refs[(static_cast<size_t>(l) * m + j) * sub];
                    for (uint32_t r = 0; r < sub; ++r) dst[r] = s * rot[static_cast<size_t>(c) * sub + r];
                }
            }
        }
    }
    return refs;
}

// projection.cpp:151-166
uint32_t default_L(uint32_t dim) {
    uint32_t p = 1;
    const double lim = std::sqrt(static_cast<double>(dim)) * std::sqrt(2.0);
    while (p * 2 <= lim && p * 2 <= dim) p *= 2;
    uint32_t hi = 1;
    while (hi * 2 <= dim / 8) hi *= 2;
    uint32_t lo = 8;
    if (hi < lo) {
        lo = hi = std::max(1u, hi);
        while (lo * 2 <= dim / 4) lo = hi = lo * 2;
    }
    return std::min(std::max(p, lo), hi);
}

// ---------------------------------------------------------------------------
// Read-only mapping of the index file
// ---------------------------------------------------------------------------
struct Mapped {
    const uint8_t* p = nullptr;
    size_t size = 0;
    int fd = -1;
    ~Mapped() {
        if (p && size) munmap(const_cast<uint8_t*>(p), size);
        if (fd >= 0) close(fd);
    }
};

struct Cursor {
    const uint8_t* p;
    size_t size, off = 0;
    template <typename T>
    T pod() {
        if (off + sizeof(T) > size) throw_err(PAG_GPU_ERUNTIME, "index read failed");
        T v;
        std::memcpy(&v, p + off, sizeof(T));
        off += sizeof(T);
        return v;
    }
    const uint8_t* take(size_t n) {
        if (off + n > size) throw_err(PAG_GPU_ERUNTIME, "index read failed");
        const uint8_t* r = p + off;
        off += n;
        return r;
    }
};

struct Replica {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    float* rows = nullptr;
    uint32_t* deg = nullptr;
    uint8_t* adj = nullptr;
    float* refsT = nullptr;
    uint32_t* entries = nullptr;
    float* bnorm = nullptr;  // squared row norms (from the file's cached norms), GT only
    // chain-interleaved copy of the rows (pag_device.h chain_positions), read
    // by the reference-order distances; built at the first such search and
    // extended after a refresh (rows are only ever appended)
    float* rows_x = nullptr;
    uint64_t rows_x_n = 0, rows_x_cap = 0;  // rows interleaved so far / allocated
    uint64_t cap_nodes = 0;  // allocated node capacity (refresh grows it)
    size_t bytes = 0;
    // search scratch
    uint32_t* gbm = nullptr;  // per-slot visited bitmaps
    uint32_t gbm_words = 0;
    size_t slots = 0;
    uint8_t* gscratch = nullptr;
    size_t gscratch_bytes = 0;
    uint32_t* qcounter = nullptr;  // two claim counters (launch parity), never reset
    uint32_t qbase[2] = {0, 0};    // their values at the next launch of each parity
    uint64_t seq = 0;              // search launches so far (parity of counters and scratch)
    // the stream of the last search launch: a launch on another stream first
    // waits for it (event), so launches of one replica never overlap across
    // streams (the two scratch sets / counters assume one launch order)
    cudaStream_t last_stream = nullptr;
    cudaEvent_t order_ev = nullptr;
    // batch I/O
    float* d_q = nullptr;
    size_t d_q_bytes = 0;
    uint8_t* d_out = nullptr;
    size_t d_out_bytes = 0;
    uint8_t* h_pin = nullptr;
    size_t h_pin_bytes = 0;
    // asynchronous batches (pag_gpu_search_submit): a ring of in-flight
    // requests whose kernels write results straight into pinned host memory
    struct AsyncSlot {
        uint8_t* h_res = nullptr;  // pinned, mapped: ids | sq | n_out | counters
        size_t h_bytes = 0;
        float* d_q = nullptr;      // device copy of pageable queries
        size_t d_q_bytes = 0;
        uint64_t ticket = 0;       // 0 = free
        uint64_t nq = 0;
        uint32_t K = 0;
        uint32_t* ids = nullptr;
        float* sq = nullptr;
        uint32_t* n_out = nullptr;
        pag_search_stats* stats = nullptr;
        // construction batches (pag_gpu_construction_submit)
        bool cons = false;
        uint32_t* pes = nullptr;
        uint32_t* pes_n = nullptr;
        uint32_t pes_cap = 0;
    };
    static constexpr int kAsyncDepth = 4;
    AsyncSlot aslot[kAsyncDepth];
    uint32_t* h_flags = nullptr;  // pinned, mapped: one completion word per slot
    uint32_t* d_done = nullptr;   // device: exited-warp counters per slot
    // persistent host worker of this replica (handles with more than one
    // replica): blocking searches, construction searches and ground truth of
    // all replicas run in parallel without spawning threads per call
    struct Worker;
    std::shared_ptr<Worker> worker;
};

// One host thread per replica, fed one job at a time by run_replicas().
struct Replica::Worker {
    std::mutex m;
    std::condition_variable cv;
    std::function<void()> job;
    bool stop = false, busy = false;
    std::exception_ptr err;
    std::thread th;
    Worker() {
        th = std::thread([this] {
            std::unique_lock<std::mutex> lk(m);
            for (;;) {
                cv.wait(lk, [this] { return stop || busy; });
                if (busy) {
                    std::function<void()> f = std::move(job);
                    lk.unlock();
                    std::exception_ptr e;
                    try {
                        f();
                    } catch (...) {
                        e = std::current_exception();
                    }
                    lk.lock();
                    err = e;
                    busy = false;
                    cv.notify_all();
                } else if (stop) {
                    return;
                }
            }
        });
    }
    void post(std::function<void()> f) {
        std::lock_guard<std::mutex> lk(m);
        job = std::move(f);
        err = nullptr;
        busy = true;
        cv.notify_all();
    }
    std::exception_ptr join_job() {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [this] { return !busy; });
        return err;
    }
    ~Worker() {
        {
            std::lock_guard<std::mutex> lk(m);
            stop = true;
            cv.notify_all();
        }
        if (th.joinable()) th.join();
    }
};

template <typename T>
void dev_alloc(T** p, size_t bytes) {
    cuda_check(cudaMalloc(reinterpret_cast<void**>(p), bytes ? bytes : 16), "cudaMalloc");
}

void dev_free(void* p) {
    if (p) cudaFree(p);
}

void grow_dev(void** p, size_t* cap, size_t need) {
    if (*cap >= need) return;
    dev_free(*p);
    *p = nullptr;
    size_t n = std::max(need, *cap + *cap / 2);
    cuda_check(cudaMalloc(p, n), "cudaMalloc");
    *cap = n;
}

}  // namespace

struct pag_gpu_index {
    uint64_t async_seq = 0;  // tickets issued by pag_gpu_search_submit
    uint64_t n = 0;
    uint32_t dim = 0, padded = 0, dstride = 0, L = 0, m = 0, M = 0, efC = 0, b_build = 0,
             pes_flush = 0;
    uint64_t seed = 0;
    uint8_t metric = 0, enable_pes = 0;
    std::vector<uint32_t> entries;
    uint32_t maxdeg = 0, cb = 0, cwp = 0, slot_stride = 0, block_bytes = 0, sub_dim = 0;
    uint64_t total_edges = 0;
    uint32_t dup_nodes = 1;        // nodes repeating a target inside a 32-edge group (0: fast path)
    float max_bnorm = 0.0f;        // max squared row norm
    uint64_t gt_uncertified = 0;   // tensor-core GT queries re-run exactly (diagnostic)
    // host mirror of the device adjacency + degrees (built at the first refresh)
    std::vector<uint8_t> mirror_adj;
    std::vector<uint32_t> mirror_deg;
    std::vector<float> refs;
    std::vector<Replica> reps;
    // status bits of asynchronous batches that a later submit completed to
    // free their ring slot, reported by their own wait (per ticket)
    std::unordered_map<uint64_t, uint32_t> early_status;
    std::mutex mu;

    pagdev::IndexView view(const Replica& r) const {
        pagdev::IndexView v{};
        v.rows = r.rows;
        v.rowsX = r.rows_x;
        v.xstride = pagdev::chain_xstride(padded);
        v.deg = r.deg;
        v.adj = r.adj;
        v.refsT = r.refsT;
        v.entries = r.entries;
        v.n = n;
        v.dim = dim;
        v.padded = padded;
        v.dstride = dstride;
        v.L = L;
        v.m = m;
        v.sub_dim = sub_dim;
        v.slot_stride = slot_stride;
        v.cwp = cwp;
        v.block_bytes = block_bytes;
        v.n_entries = static_cast<uint32_t>(entries.size());
        v.cosine = metric == 1;
        v.dup_free = dup_nodes == 0;
        return v;
    }
};

namespace {

void free_replica(Replica& r) {
    r.worker.reset();  // joins the replica's host thread
    cudaSetDevice(r.device);
    if (r.stream) cudaStreamSynchronize(r.stream);  // in-flight asynchronous batches
    // (launches on caller streams: cudaFree below waits for the device)
    if (r.order_ev) cudaEventDestroy(r.order_ev);
    for (void* p : {static_cast<void*>(r.rows), static_cast<void*>(r.deg), static_cast<void*>(r.adj),
                    static_cast<void*>(r.refsT), static_cast<void*>(r.entries),
                    static_cast<void*>(r.gbm),
                    static_cast<void*>(r.gscratch), static_cast<void*>(r.qcounter),
                    static_cast<void*>(r.d_q), static_cast<void*>(r.d_out), static_cast<void*>(r.bnorm),
                    static_cast<void*>(r.rows_x)})
        dev_free(p);
    if (r.h_pin) cudaFreeHost(r.h_pin);
    for (auto& a : r.aslot) {
        if (a.h_res) cudaFreeHost(a.h_res);
        dev_free(a.d_q);
    }
    if (r.h_flags) cudaFreeHost(r.h_flags);
    dev_free(r.d_done);
    if (r.stream) cudaStreamDestroy(r.stream);
    r = Replica{};
}

// One node's file records {target u32, codes[cb], cos_beta, edge_norm,
// base_offset} (builder.cpp:418-425) -> the device block (zeroed by caller).
void fill_block(uint8_t* blk, const uint8_t* e, uint32_t deg, uint64_t n, uint32_t S, uint32_t cb, uint32_t cwp) {
    const size_t rec = 4 + cb + 12;
    uint32_t* tg = reinterpret_cast<uint32_t*>(blk);
    float* en = reinterpret_cast<float*>(blk + 4u * S);
    float* cbeta = reinterpret_cast<float*>(blk + 8u * S);
    float* bo = reinterpret_cast<float*>(blk + 12u * S);
    uint8_t* codes = blk + 16u * S;
    for (uint32_t j = 0; j < deg; ++j, e += rec) {
        uint32_t t;
        std::memcpy(&t, e, 4);
        if (t >= n) throw_err(PAG_GPU_ERUNTIME, "edge target out of range in file");
        tg[j] = t;
        std::memcpy(codes + static_cast<size_t>(j) * 4 * cwp, e + 4, cb);
        std::memcpy(&cbeta[j], e + 4 + cb, 4);
        std::memcpy(&en[j], e + 8 + cb, 4);
        std::memcpy(&bo[j], e + 12 + cb, 4);
    }
}

// ---------------------------------------------------------------------------
// PAGIDX01 v1 ingest (builder.cpp:434-492) straight into the device layout
// ---------------------------------------------------------------------------
// dry = true: parse and validate the whole file on the host only (no GPU).
// devs: one replica per entry (a device may repeat: several replicas on one
// GPU, each with its own copy, stream and scratch)
// header fields -> validation (builder.cpp:434-446) and the derived device
// layout; regenerates the reference family
void init_layout(pag_gpu_index& ix) {
    if (ix.n >= 0xFFFFFFFFull) throw_err(PAG_GPU_ERUNTIME, "index too large for 32-bit ids");
    // PagIndex constructor: VectorSet(dim, padded) then repad(L) (builder.cpp:40-46)
    if (ix.padded < ix.dim) throw_err(PAG_GPU_EINVAL, "padded_dim < dim");
    if (ix.L == 0) ix.L = default_L(ix.dim);
    if (((ix.dim + ix.L - 1) / ix.L) * ix.L != ix.padded)
        throw_err(PAG_GPU_ERUNTIME, "padded_dim mismatch on load");
    ix.refs = reference_family(ix.padded, ix.L, ix.m, ix.seed);
    ix.sub_dim = ix.padded / ix.L;
    ix.dstride = (ix.padded + 3u) & ~3u;
    ix.maxdeg = 2 * ix.M;
    ix.cb = (ix.L + 1) / 2;
    ix.cwp = 1;
    while (ix.cwp * 4 < ix.cb) ix.cwp *= 2;
    ix.slot_stride = std::max(32u, (ix.maxdeg + 31u) & ~31u);
    ix.block_bytes = ix.slot_stride * (16u + 4u * ix.cwp);
}

// Where an index comes from: node(u, blk) fills node u's zeroed device block
// and returns its degree (called for u = 0 .. n-1 in order); rows() / norms()
// give the n x padded_dim rows and the n cached norms (norms may be null:
// computed from the rows), valid once every node has been read.
struct IndexSource {
    std::function<uint32_t(uint64_t, uint8_t*)> node;
    std::function<const uint8_t*()> rows;
    std::function<const uint8_t*()> norms;
};

// vecstore.cpp:97-108 (the cached norm of a stored row), for sources without norms
float host_vec_norm(const float* a, size_t padded) {
    float acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    size_t k = 0;
    for (; k + 4 <= padded; k += 4) {
        acc0 += a[k] * a[k];
        acc1 += a[k + 1] * a[k + 1];
        acc2 += a[k + 2] * a[k + 2];
        acc3 += a[k + 3] * a[k + 3];
    }
    for (; k < padded; ++k) acc0 += a[k] * a[k];
    return std::sqrt((acc0 + acc1) + (acc2 + acc3));
}

void upload_index(pag_gpu_index* ix, const std::vector<int>& devs, bool dry, const IndexSource& src);

std::unique_ptr<pag_gpu_index> open_index(const char* path, const std::vector<int>& devs, bool dry = false) {
    Mapped mp;
    mp.fd = ::open(path, O_RDONLY);
    if (mp.fd < 0) throw_err(PAG_GPU_ERUNTIME, std::string("cannot open index: ") + path);
    struct stat sb;
    if (fstat(mp.fd, &sb) != 0) throw_err(PAG_GPU_ERUNTIME, std::string("cannot open index: ") + path);
    mp.size = static_cast<size_t>(sb.st_size);
    if (mp.size) {
        void* p = mmap(nullptr, mp.size, PROT_READ, MAP_PRIVATE, mp.fd, 0);
        if (p == MAP_FAILED) throw_err(PAG_GPU_ERUNTIME, std::string("cannot open index: ") + path);
        madvise(p, mp.size, MADV_SEQUENTIAL);
        mp.p = static_cast<const uint8_t*>(p);
    }
    Cursor cur{mp.p, mp.size};
    auto ix = std::make_unique<pag_gpu_index>();
    if (cur.pod<uint64_t>() != 0x5041474944583031ull) throw_err(PAG_GPU_ERUNTIME, "bad index magic");
    if (cur.pod<uint32_t>() != 1u) throw_err(PAG_GPU_ERUNTIME, "unsupported index version");
    ix->n = cur.pod<uint64_t>();
    ix->dim = cur.pod<uint32_t>();
    ix->padded = cur.pod<uint32_t>();
    ix->L = cur.pod<uint32_t>();
    ix->m = cur.pod<uint32_t>();
    ix->M = cur.pod<uint32_t>();
    ix->efC = cur.pod<uint32_t>();
    ix->b_build = cur.pod<uint32_t>();
    ix->pes_flush = cur.pod<uint32_t>();
    ix->seed = cur.pod<uint64_t>();
    ix->metric = cur.pod<uint8_t>();
    ix->enable_pes = cur.pod<uint8_t>();
    const uint32_t n_entries = cur.pod<uint32_t>();
    ix->entries.resize(n_entries);
    if (n_entries) std::memcpy(ix->entries.data(), cur.take(4ull * n_entries), 4ull * n_entries);
    init_layout(*ix);
    // file records in node order, then the rows and the cached norms
    const uint64_t n = ix->n;
    const uint32_t S = ix->slot_stride, cb = ix->cb, cwp = ix->cwp, maxdeg = ix->maxdeg, padded = ix->padded;
    const size_t rec = 4 + cb + 12;
    const uint8_t* rows_p = nullptr;
    IndexSource src;
    src.node = [&](uint64_t, uint8_t* blk) {
        const uint32_t deg = cur.pod<uint32_t>();
        if (deg > maxdeg) throw_err(PAG_GPU_ERUNTIME, "degree over cap in file");
        fill_block(blk, cur.take(rec * deg), deg, n, S, cb, cwp);
        return deg;
    };
    src.rows = [&] {
        rows_p = cur.take(4ull * padded * n);
        cur.take(4ull * n);  // cached norms (presence checked here)
        return rows_p;
    };
    src.norms = [&] { return rows_p + 4ull * padded * n; };
    upload_index(ix.get(), devs, dry, src);
    return ix;
}

// source -> device layout on every replica of devs
// dry = true: parse and validate the whole source on the host only (no GPU).
// devs: one replica per entry (a device may repeat: several replicas on one
// GPU, each with its own copy, stream and scratch)
void upload_index(pag_gpu_index* ix, const std::vector<int>& devs, bool dry, const IndexSource& src) {
    const uint32_t n_entries = static_cast<uint32_t>(ix->entries.size());
    if (!dry) {
        if (devs.empty()) throw_err(PAG_GPU_EINVAL, "no device given");
        int ndev = 0;
        cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        for (int d : devs)
            if (d < 0 || d >= ndev) throw_err(PAG_GPU_EINVAL, "device list names a missing GPU");
    }

    const uint64_t n = ix->n;
    const size_t row_bytes = 4ull * ix->dstride;
    for (int d : (dry ? std::vector<int>{} : devs)) {
        Replica r;
        r.device = d;
        cuda_check(cudaSetDevice(d), "cudaSetDevice");
        cudaDeviceGetAttribute(&r.num_sms, cudaDevAttrMultiProcessorCount, d);
        cuda_check(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking), "cudaStreamCreate");
        dev_alloc(&r.rows, n * row_bytes);
        dev_alloc(&r.deg, 4ull * n);
        dev_alloc(&r.adj, static_cast<size_t>(n) * ix->block_bytes);
        dev_alloc(&r.refsT, 4ull * ix->refs.size());
        dev_alloc(&r.entries, 4ull * std::max<size_t>(1, n_entries));
        dev_alloc(&r.qcounter, 16);
        cuda_check(cudaMemset(r.qcounter, 0, 16), "memset");
        cuda_check(cudaEventCreateWithFlags(&r.order_ev, cudaEventDisableTiming), "cudaEventCreate");
        r.bytes = n * row_bytes + 4ull * n + static_cast<size_t>(n) * ix->block_bytes +
                  4ull * ix->refs.size();
        r.cap_nodes = n;
        ix->reps.push_back(r);
    }

    // refs transposed: refsT[(l*sub + c)*m + j] = refs[(l*m + j)*sub + c]
    {
        const uint32_t L = ix->L, m = ix->m, sub = ix->sub_dim;
        std::vector<float> rt(ix->refs.size());
        for (uint32_t l = 0; l < L; ++l)
            for (uint32_t j = 0; j < m; ++j)
                for (uint32_t c = 0; c < sub; ++c)
                    rt[(static_cast<size_t>(l) * sub + c) * m + j] =
                        ix->refs[(static_cast<size_t>(l) * m + j) * sub + c];
        for (auto& r : ix->reps) {
            cudaSetDevice(r.device);
            cuda_check(cudaMemcpy(r.refsT, rt.data(), 4 * rt.size(), cudaMemcpyHostToDevice), "H2D refs");
            if (n_entries)
                cuda_check(cudaMemcpy(r.entries, ix->entries.data(), 4ull * n_entries,
                                      cudaMemcpyHostToDevice),
                           "H2D entries");
        }
    }

    // adjacency: stream node blocks through two pinned staging buffers
    const size_t CH = 1u << 16;  // nodes per chunk
    const size_t chunk_bytes = CH * ix->block_bytes;
    uint8_t* stage[2] = {nullptr, nullptr};
    uint32_t* dstage[2] = {nullptr, nullptr};
    auto host_alloc = [dry](void** p, size_t bytes) {
        if (dry) {
            *p = std::malloc(bytes);
            if (!*p) throw std::bad_alloc();
        } else {
            cuda_check(cudaHostAlloc(p, bytes, 0), "cudaHostAlloc");
        }
    };
    host_alloc(reinterpret_cast<void**>(&stage[0]), chunk_bytes);
    host_alloc(reinterpret_cast<void**>(&stage[1]), chunk_bytes);
    host_alloc(reinterpret_cast<void**>(&dstage[0]), CH * 4);
    host_alloc(reinterpret_cast<void**>(&dstage[1]), CH * 4);
    struct Free {
        uint8_t** s;
        uint32_t** d;
        bool dry;
        ~Free() {
            for (int i = 0; i < 2; ++i) {
                if (dry) {
                    std::free(s[i]);
                    std::free(d[i]);
                } else {
                    if (s[i]) cudaFreeHost(s[i]);
                    if (d[i]) cudaFreeHost(d[i]);
                }
            }
        }
    } fr{stage, dstage, dry};
    int buf = 0;
    // the source streams through pinned staging into the first replica; the
    // others are then filled device to device (NVLink peer copies across
    // GPUs, or on-device copies), so the host link carries the index once
    Replica* r0 = ix->reps.empty() ? nullptr : &ix->reps[0];
    for (uint64_t u0 = 0; u0 < n; u0 += CH) {
        const uint64_t cnt = std::min<uint64_t>(CH, n - u0);
        if (r0) cudaStreamSynchronize(r0->stream);  // buffer reuse
        uint8_t* blk0 = stage[buf];
        uint32_t* dg = dstage[buf];
        std::memset(blk0, 0, cnt * ix->block_bytes);
        for (uint64_t i = 0; i < cnt; ++i) {
            const uint32_t deg = src.node(u0 + i, blk0 + i * ix->block_bytes);
            dg[i] = deg;
            ix->total_edges += deg;
        }
        if (r0) {
            cudaSetDevice(r0->device);
            cuda_check(cudaMemcpyAsync(r0->adj + u0 * ix->block_bytes, blk0, cnt * ix->block_bytes,
                                       cudaMemcpyHostToDevice, r0->stream),
                       "H2D adjacency");
            cuda_check(cudaMemcpyAsync(r0->deg + u0, dg, cnt * 4, cudaMemcpyHostToDevice, r0->stream),
                       "H2D degrees");
        }
        buf ^= 1;
    }
    if (r0) cuda_check(cudaStreamSynchronize(r0->stream), "adjacency upload");

    // rows (n x padded fp32), restrided to dstride with zero padding
    {
        const uint8_t* rows = src.rows();
        const uint8_t* norms = src.norms();
        const size_t RCH = std::max<size_t>(1, chunk_bytes / row_bytes);
        buf = 0;
        for (uint64_t i0 = 0; i0 < n; i0 += RCH) {
            const uint64_t cnt = std::min<uint64_t>(RCH, n - i0);
            if (r0) cudaStreamSynchronize(r0->stream);
            uint8_t* st = stage[buf];
            if (dry) {
                // host-only inspection: rows are validated for presence only
            } else if (ix->dstride == ix->padded) {
                std::memcpy(st, rows + i0 * row_bytes, cnt * row_bytes);
            } else {
                std::memset(st, 0, cnt * row_bytes);
                for (uint64_t i = 0; i < cnt; ++i)
                    std::memcpy(st + i * row_bytes, rows + (i0 + i) * 4ull * ix->padded, 4ull * ix->padded);
            }
            if (r0) {
                cudaSetDevice(r0->device);
                cuda_check(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(r0->rows) + i0 * row_bytes, st,
                                           cnt * row_bytes, cudaMemcpyHostToDevice, r0->stream),
                           "H2D rows");
            }
            buf ^= 1;
        }
        if (r0) cuda_check(cudaStreamSynchronize(r0->stream), "rows upload");
        for (size_t i = 1; i < ix->reps.size(); ++i) {  // replica i <- replica 0
            Replica& r = ix->reps[i];
            cudaSetDevice(r.device);
            cuda_check(cudaMemcpyPeerAsync(r.rows, r.device, r0->rows, r0->device, n * row_bytes, r.stream),
                       "peer copy rows");
            cuda_check(cudaMemcpyPeerAsync(r.adj, r.device, r0->adj, r0->device, n * ix->block_bytes, r.stream),
                       "peer copy adjacency");
            cuda_check(cudaMemcpyPeerAsync(r.deg, r.device, r0->deg, r0->device, 4ull * n, r.stream),
                       "peer copy degrees");
        }
        for (auto& r : ix->reps) cuda_check(cudaStreamSynchronize(r.stream), "replica copies");
        // squared norms for the tensor-core ground truth (cached norms are the
        // stored rows' vec_norm, builder.cpp:489-491)
        if (!ix->reps.empty()) {
            std::vector<float> bn(n);
            for (uint64_t i = 0; i < n; ++i) {
                float v;
                if (norms)
                    std::memcpy(&v, norms + 4 * i, 4);
                else
                    v = host_vec_norm(reinterpret_cast<const float*>(rows) + i * ix->padded, ix->padded);
                bn[i] = v * v;
                ix->max_bnorm = std::max(ix->max_bnorm, bn[i]);
            }
            for (auto& r : ix->reps) {
                cudaSetDevice(r.device);
                dev_alloc(&r.bnorm, 4ull * std::max<uint64_t>(1, n));
                cuda_check(cudaMemcpy(r.bnorm, bn.data(), 4ull * n, cudaMemcpyHostToDevice), "H2D norms");
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Search driver (routing.cpp:206-261 per query, batched)
// ---------------------------------------------------------------------------
struct Plan {
    pagdev::SearchLaunch L{};
    size_t gscratch_stride = 0;
    int grid = 0;
};

// Test / diagnostic knobs (PAG_GPU_*): warps per CTA, visited-table size and
// fill, per-warp smem budget, plan print. Read at every plan (a few getenv
// calls per batch) so that tests can change them between calls.
struct Knobs {
    int wpb = 4;
    int hash_log2 = -1, hash_fill = -1;
    int max_bps = 0;  // cap on resident blocks per SM (0: the occupancy limit)
    long long smem_budget = -1;
    bool debug = false;
    Knobs() {
        if (const char* e = std::getenv("PAG_GPU_WPB")) wpb = std::max(1, std::min(4, std::atoi(e)));
        if (const char* e = std::getenv("PAG_GPU_MAX_BPS")) max_bps = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("PAG_GPU_HASH_LOG2")) hash_log2 = std::atoi(e);
        if (const char* e = std::getenv("PAG_GPU_HASH_FILL")) hash_fill = std::max(1, std::min(90, std::atoi(e)));
        if (const char* e = std::getenv("PAG_GPU_SMEM_BUDGET")) smem_budget = std::atoll(e);
        debug = std::getenv("PAG_GPU_DEBUG") != nullptr;
    }
};
Knobs knobs() { return Knobs(); }

// warps (queries in flight) per CTA
int warps_per_block() { return knobs().wpb; }
#ifndef PAG_WARP_SMEM_BUDGET
#define PAG_WARP_SMEM_BUDGET (14 * 1024)
#endif
constexpr uint32_t kWarpSmemBudget = PAG_WARP_SMEM_BUDGET;

uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

Plan make_plan(const pag_gpu_index& ix, const Replica& r, const pag_search_params& p, uint32_t nq) {
    Plan pl;
    auto& L = pl.L;
    const uint32_t bdef = p.b_override ? p.b_override : std::max(10u, p.K);
    L.b = p.use_tfb ? bdef : std::max(p.efS, bdef);
    L.r_max = p.use_tfb ? (p.efS + L.b - 1) / L.b : 1u;
    L.K = p.K;
    L.efS = p.efS;
    L.use_prt = p.use_prt;
    L.exact_dist = p.exact_dist;
    L.nq = nq;
    L.ix = ix.view(r);
    const int kWarpsPerBlock = warps_per_block();
    L.warps_per_block = kWarpsPerBlock;
    const Knobs kn = knobs();
    // the visited table holds half its slots before spilling to the bitmap:
    // 512 marks cover efS <= 200 at K = 10; past that, with b > 32, the marks
    // outgrow any on-chip table and a small one keeps occupancy (with b <= 32
    // the full table stays faster at every efS: cfg-2 efS 300 8.2 vs 8.6 ms)
    L.hash_log2 = (p.efS <= 200 || L.b <= 32) ? 10 : 8;
    // reference-order searches past efS = 100 with the register working set:
    // the marks outgrow 768 slots (efS 200: construction search 7.73 -> 7.52 ms,
    // cfg-2 5.62 -> 5.52 ms with 2048 slots); that mode has no staging buffer,
    // so the larger table still leaves 4 blocks per SM
    if (p.exact_dist && L.b <= 32 && p.efS > 100 && 4 * ix.dstride + 4 * ix.L * 16 <= 5 * 1024) L.hash_log2 = 11;
    if (kn.hash_log2 >= 0) L.hash_log2 = static_cast<uint32_t>(kn.hash_log2);
    L.hash_log2 = std::max(3u, std::min(16u, L.hash_log2));  // >= 2 buckets of 4 slots
    {
        // percent of the slots filled before marks spill to the HBM bitmap:
        // 75 with b <= 32 (cfg-2 efS 150: 3.90 -> 3.66 ms, efS 70-300 +0.6-2.7%),
        // 50 otherwise (cfg-3: the longer probes cost more than the spills)
        uint32_t fill = L.b <= 32 ? 75 : 50;
        if (kn.hash_fill > 0) fill = static_cast<uint32_t>(kn.hash_fill);
        L.hash_limit = static_cast<uint32_t>((static_cast<uint64_t>(1u << L.hash_log2) * fill) / 100);
    }
    const uint32_t b = L.b;
    L.rl_cap = L.r_max * b + b;  // every W flush of a query (r_max - 1 end_rounds + the final flush)
    const uint32_t capr = L.rl_cap;
    const bool regs = pagdev::search_uses_registers(L);
    // fixed smem regions
    uint32_t off = 0;
    L.off_q = off;
    // (reference-order mode: the query is re-laid chain-interleaved in place)
    off = align16(off + 4 * (p.exact_dist ? std::max(ix.dstride, pagdev::chain_xstride(ix.padded)) : ix.dstride));
    off = (off + 63u) & ~63u;  // 64-B aligned table (code_sum ORs the code offset into the base)
    L.off_T = off;
    off = align16(off + 4 * ix.L * 16);  // T rows padded to 16 (m <= 16)
    L.off_hash = off;
    off = align16(off + (4u << L.hash_log2));
    L.off_sqbuf = off;
    off = align16(off + 256);
    // movable regions: W (12b), rings (24b), R_L (24 capr), merge (48b);
    // with b <= 32 the working set and R_T live in registers
    // (b <= 32: the rings region holds R_F only, 32 slots; R_T is in registers)
    const uint64_t szW = regs ? 0 : align16(12 * b), szR = regs ? 12 * 32 : align16(24 * b),
                   szRL = align16(24 * capr), szM = align16(48 * b);
    bool w_s = true, r_s = true, rl_s = true, m_s = true;
    auto total = [&]() {
        return off + (w_s ? szW : 0) + (r_s ? szR : 0) + (rl_s ? szRL : 0) + (m_s ? szM : 0);
    };
    // per-warp budget that keeps the kernel's resident-block bound (4 or 6
    // blocks of 4 warps in 228 KB) reachable
    uint64_t budget = pagdev::search_high_occupancy(L) ? std::min<uint32_t>(kWarpSmemBudget, 9 * 1024)
                                                       : kWarpSmemBudget;
    if (kn.smem_budget >= 0) budget = static_cast<uint64_t>(kn.smem_budget);  // tests
    if (total() > budget) rl_s = false;
    if (total() > budget) m_s = false;
    if (total() > budget) r_s = false;
    // W last: with the per-owner caches it is touched S = b/32 entries at a
    // time (L1-friendly), and occupancy (4 blocks/SM) hides more latency
    // than an on-chip W saves (cfg4 K=1000: +17%)
    if (total() > budget) w_s = false;
    uint64_t goff = 0;
    auto place = [&](bool in_smem, uint64_t sz, uint32_t* o, uint32_t* flag) {
        *flag = in_smem;
        if (in_smem) {
            *o = off;
            off = align16(static_cast<uint32_t>(off + sz));
        } else {
            *o = static_cast<uint32_t>(goff);
            goff = (goff + sz + 255) & ~255ull;
        }
    };
    place(w_s, szW, &L.off_W, &L.W_in_smem);
    place(r_s, szR, &L.off_rf, &L.rings_in_smem);
    L.off_rt = L.off_rf + 12 * b;
    place(rl_s, szRL, &L.off_rl, &L.rl_in_smem);
    place(m_s, szM, &L.off_merge, &L.merge_in_smem);
#ifdef PAG_VALIDATE
    {  // resident ids of W, both rings and R_L (debug check, HBM)
        uint32_t dbg_flag = 0;
        place(false, align16(4 * (capr + 3 * b)), &L.off_dbg, &dbg_flag);
    }
#endif
    L.warp_smem_bytes = (off + 63u) & ~63u;  // keeps every warp's table 64-B aligned
    pl.gscratch_stride = std::max<uint64_t>(256, goff);
    L.gscratch_stride = pl.gscratch_stride;
    // per-slot HBM visited bitmap (n bits, 16-B multiple)
    L.gbm_words = static_cast<uint32_t>(((ix.n + 127) / 128) * 4);
    int bps = 0;
    cuda_check(pagdev::search_occupancy(L, &bps), "occupancy");
    if (bps <= 0) throw_err(PAG_GPU_ERUNTIME, "search configuration does not fit on the GPU");
    if (kn.max_bps > 0) bps = std::min(bps, kn.max_bps);  // concurrency experiments
    const int want_blocks = static_cast<int>((nq + kWarpsPerBlock - 1) / kWarpsPerBlock);
    pl.grid = std::max(1, std::min(r.num_sms * bps, want_blocks));
    if (kn.debug)
        std::fprintf(stderr, "[pag_gpu] plan: b=%u warps/block=%d blocks/SM=%d grid=%d smem/warp=%u W/rings/RL/merge in smem %u%u%u%u\n",
                     L.b, L.warps_per_block, bps, pl.grid, L.warp_smem_bytes, L.W_in_smem, L.rings_in_smem,
                     L.rl_in_smem, L.merge_in_smem);
    return pl;
}

void ensure_scratch(Replica& r, Plan& pl) {
    auto& L = pl.L;
    const size_t slots = static_cast<size_t>(pl.grid) * pl.L.warps_per_block;
    // two scratch sets (launch parity): a launch may overlap its predecessor
    if (slots > r.slots || L.gbm_words > r.gbm_words) {
        const size_t ns = std::max(slots, r.slots);
        const uint32_t words = std::max(L.gbm_words, r.gbm_words);
        dev_free(r.gbm);  // (cudaFree waits for running kernels)
        r.gbm = nullptr;
        dev_alloc(&r.gbm, 2 * ns * words * 4ull);
        cuda_check(cudaMemset(r.gbm, 0, 2 * ns * words * 4ull), "memset");  // blocking: any stream may follow
        r.slots = ns;
        r.gbm_words = words;
    }
    L.gbm_words = r.gbm_words;
    grow_dev(reinterpret_cast<void**>(&r.gscratch), &r.gscratch_bytes, 2 * r.slots * pl.gscratch_stride);
    const uint32_t par = static_cast<uint32_t>(r.seq & 1u);
    L.gbm = r.gbm + par * r.slots * r.gbm_words;
    L.gscratch = r.gscratch + par * r.slots * pl.gscratch_stride;
    L.qcounter = r.qcounter + par;
    L.qbase = r.qbase[par];
}

// the chain-interleaved row copy of a replica, complete for the current n
// (first reference-order search, or the first one after a refresh); blocking,
// so that any stream may launch afterwards
void ensure_rows_x(pag_gpu_index& ix, Replica& r) {
    if (r.rows_x && r.rows_x_n == ix.n) return;
    const size_t xrow = 4ull * pagdev::chain_xstride(ix.padded);
    if (r.rows_x_cap < ix.n) {
        dev_free(r.rows_x);  // (cudaFree waits for running kernels)
        r.rows_x = nullptr;
        r.rows_x_n = r.rows_x_cap = 0;
        const uint64_t cap = std::max<uint64_t>(ix.n, r.cap_nodes);
        dev_alloc(&r.rows_x, cap * xrow);
        r.rows_x_cap = cap;
    }
    cuda_check(pagdev::launch_interleave_rows(r.rows, r.rows_x, r.rows_x_n, ix.n, ix.padded, ix.dstride, r.stream),
               "interleave rows");
    cuda_check(cudaStreamSynchronize(r.stream), "interleave rows");
    r.rows_x_n = ix.n;
}

void validate_params(const pag_gpu_index& ix, const pag_search_params& p) {
    if (ix.n == 0) throw_err(PAG_GPU_ERUNTIME, "search on empty index");  // routing.cpp:208
    if (p.K > p.efS) throw_err(PAG_GPU_EINVAL, "K > efS");                // routing.cpp:209
}

// asynchronous-batch completion signalling (see SearchLaunch::host_flag)
struct AsyncArgs {
    uint32_t* done_ctr = nullptr;
    uint32_t* host_flag = nullptr;  // device address of the pinned word
    uint32_t flag_value = 0;
};

// construction search (builder.cpp:218-227) device-side extras
struct ConstructionArgs {
    const uint32_t* nodes = nullptr;  // device: query i = stored row of nodes[i]
    uint32_t collect_pes = 0, pes_cap = 0;
    uint32_t* pes = nullptr;          // device: nq x pes_cap
    uint32_t* pes_n = nullptr;        // device: nq
};

// Runs nq queries already on the replica's device. Device buffers:
// q (nq x dim), ids/sq (nq x K), n_out (nq), stats (nq x 8).
void run_search(pag_gpu_index& ix, Replica& r, const pag_search_params& p, const float* q_dev,
                uint32_t nq, uint32_t* ids, float* sq, uint32_t* n_out, uint32_t* stats, cudaStream_t stream,
                const ConstructionArgs* ca = nullptr, const AsyncArgs* aa = nullptr) {
    if (nq == 0) return;
    if (p.exact_dist) ensure_rows_x(ix, r);
    Plan pl = make_plan(ix, r, p, nq);
    ensure_scratch(r, pl);
    // one launch order per replica: a launch on another stream than the last
    // one waits for everything before it there and does not overlap it
    bool pdl = true;
    if (r.seq && stream != r.last_stream) {
        cuda_check(cudaEventRecord(r.order_ev, r.last_stream), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(stream, r.order_ev, 0), "cudaStreamWaitEvent");
        pdl = false;
    }
    auto& L = pl.L;
    if (aa) {
        L.done_ctr = aa->done_ctr;
        L.host_flag = aa->host_flag;
        L.flag_value = aa->flag_value;
        L.n_warps = static_cast<uint32_t>(pl.grid) * L.warps_per_block;
    }
    L.queries = q_dev;
    L.pdl = pdl;
    if (ca) {
        L.qnodes = ca->nodes;
        L.collect_pes = ca->collect_pes;
        L.pes_cap = ca->pes_cap;
        L.out_pes = ca->pes;
        L.out_pes_n = ca->pes_n;
    }
    L.out_ids = ids;
    L.out_sq = sq;
    L.out_n = n_out;
    L.out_stats = stats;
    cuda_check(pagdev::launch_search(L, pl.grid, stream), "search kernel launch");
    // the launch advances its counter by nq + one failed claim per warp
    r.qbase[r.seq & 1u] += nq + static_cast<uint32_t>(pl.grid) * static_cast<uint32_t>(L.warps_per_block);
    r.last_stream = stream;
    ++r.seq;
}

static_assert(sizeof(pag_search_stats) == 40, "pag_search_stats is five packed u64 (bindings rely on it)");

// PAG_GPU_HOST_TRACE=1: per-call host phase times on stderr (diagnostic)
struct HostTrace {
    bool on = std::getenv("PAG_GPU_HOST_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    char buf[512];
    int len = 0;
    void mark(const char* what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        len += std::snprintf(buf + len, sizeof(buf) - len, " %s %.1fus", what,
                             std::chrono::duration<double, std::micro>(t - t0).count());
        t0 = t;
    }
    ~HostTrace() {
        if (on) std::fprintf(stderr, "[pag host]%s\n", buf);
    }
};

// host-side construction request: nodes (host ids) and PES outputs
struct ConstructionHost {
    const uint32_t* nodes;
    uint32_t collect_pes, pes_cap;
    uint32_t* pes;    // nq x pes_cap (may be null when pes_cap == 0)
    uint32_t* pes_n;  // nq
};

void search_on_replica(pag_gpu_index& ix, Replica& r, const pag_search_params& p, const float* q,
                       uint64_t nq, uint32_t* ids, float* sq, uint32_t* n_out,
                       pag_search_stats* stats, uint32_t* status_or, const ConstructionHost* ch = nullptr) {
    cuda_check(cudaSetDevice(r.device), "cudaSetDevice");
    if (nq == 0) return;
    HostTrace tr;
    const uint32_t K = p.K;
    const size_t qb = ch ? 4ull * nq : 4ull * nq * ix.dim;
    const size_t ob_ids = 4ull * nq * std::max(1u, K), ob_n = 4ull * nq,
                 ob_st = 4ull * nq * pagdev::kStatWords;
    const size_t ob_pes = ch ? 4ull * nq * ch->pes_cap : 0, ob_pn = ch ? 4ull * nq : 0;
    grow_dev(reinterpret_cast<void**>(&r.d_q), &r.d_q_bytes, qb);
    grow_dev(reinterpret_cast<void**>(&r.d_out), &r.d_out_bytes, 2 * ob_ids + ob_n + ob_st + ob_pes + ob_pn);
    uint32_t* d_ids = reinterpret_cast<uint32_t*>(r.d_out);
    float* d_sq = reinterpret_cast<float*>(r.d_out + ob_ids);
    uint32_t* d_n = reinterpret_cast<uint32_t*>(r.d_out + 2 * ob_ids);
    uint32_t* d_st = reinterpret_cast<uint32_t*>(r.d_out + 2 * ob_ids + ob_n);
    ConstructionArgs ca;
    if (ch) {
        ca.nodes = reinterpret_cast<const uint32_t*>(r.d_q);
        ca.collect_pes = ch->collect_pes;
        ca.pes_cap = ch->pes_cap;
        ca.pes = reinterpret_cast<uint32_t*>(r.d_out + 2 * ob_ids + ob_n + ob_st);
        ca.pes_n = reinterpret_cast<uint32_t*>(r.d_out + 2 * ob_ids + ob_n + ob_st + ob_pes);
    }
    const ConstructionArgs* cap = ch ? &ca : nullptr;
    // entries past each pes list are zero (the kernel writes min(n, cap))
    if (ch && ob_pes) cuda_check(cudaMemsetAsync(ca.pes, 0, ob_pes, r.stream), "memset pes");
    // queries in pinned (mapped) host memory are read by the kernel in place
    // over PCIe at each query's start (3 KB per query at d=768), which
    // overlaps the transfer with the search; pageable ones are copied first
    const float* q_src = r.d_q;
    if (!ch) {
        cudaPointerAttributes at{};
        if (!std::getenv("PAG_GPU_NO_ZEROCOPY") && cudaPointerGetAttributes(&at, q) == cudaSuccess &&
            at.type == cudaMemoryTypeHost && at.devicePointer)
            q_src = static_cast<const float*>(at.devicePointer);
        else
            (void)cudaGetLastError();
    }
    if (q_src == r.d_q)
        cuda_check(cudaMemcpyAsync(r.d_q, ch ? static_cast<const void*>(ch->nodes) : static_cast<const void*>(q), qb,
                                   cudaMemcpyHostToDevice, r.stream),
                   "H2D queries");
    tr.mark("prep");
    run_search(ix, r, p, q_src, static_cast<uint32_t>(nq), d_ids, d_sq, d_n, d_st, r.stream, cap);
    tr.mark("launch");
    // one D2H of the contiguous result block (ids | sq | n_out | counters)
    // into pinned staging
    const size_t ob_res = 2 * ob_ids + ob_n + ob_st;
    if (r.h_pin_bytes < ob_res) {
        if (r.h_pin) cudaFreeHost(r.h_pin);
        r.h_pin = nullptr;
        r.h_pin_bytes = 0;
        cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&r.h_pin), ob_res, 0), "cudaHostAlloc");
        r.h_pin_bytes = ob_res;
    }
    cuda_check(cudaMemcpyAsync(r.h_pin, r.d_out, ob_res, cudaMemcpyDeviceToHost, r.stream), "D2H results");
    cuda_check(cudaStreamSynchronize(r.stream), "search");
    tr.mark("kernel+d2h");
    const uint32_t* st = reinterpret_cast<const uint32_t*>(r.h_pin + 2 * ob_ids + ob_n);
    if (K) {
        std::memcpy(ids, r.h_pin, 4ull * nq * K);
        std::memcpy(sq, r.h_pin + ob_ids, 4ull * nq * K);
    }
    std::memcpy(n_out, r.h_pin + 2 * ob_ids, ob_n);
    if (ch) {
        if (ob_pes) cuda_check(cudaMemcpyAsync(ch->pes, ca.pes, ob_pes, cudaMemcpyDeviceToHost, r.stream), "D2H pes");
        cuda_check(cudaMemcpyAsync(ch->pes_n, ca.pes_n, ob_pn, cudaMemcpyDeviceToHost, r.stream), "D2H pes_n");
    }
    cuda_check(cudaStreamSynchronize(r.stream), "D2H");
    uint32_t so = 0;
    for (uint64_t i = 0; i < nq; ++i) {
        const uint32_t* s = &st[i * pagdev::kStatWords];
        so |= s[pagdev::kStatStatus];
        if (stats) {
            stats[i].exact_dist_count = s[pagdev::kStatExact];
            stats[i].test_count = s[pagdev::kStatTest];
            stats[i].pass_count = s[pagdev::kStatPass];
            stats[i].visited_count = s[pagdev::kStatVisited];
            stats[i].edges_scanned = s[pagdev::kStatEdges];
        }
    }
    *status_or = so;
    tr.mark("unpack");
}

// ---------------------------------------------------------------------------
// Ground truth driver
// ---------------------------------------------------------------------------
struct DevBuf {  // scoped device allocation
    void* p = nullptr;
    explicit DevBuf(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~DevBuf() { dev_free(p); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// exact SIMT ground truth (pag_gt.cu) for nq padded queries on the device
void exact_gt(const pag_gpu_index& ix, Replica& r, const float* d_q, uint32_t nq, uint32_t kk, uint32_t* d_ids,
              float* d_sq) {
    DevBuf scratch(4 * pagdev::gt_scratch_elems(ix.n, nq, kk));
    pagdev::GtLaunch g{};
    g.base = r.rows;
    g.n = ix.n;
    g.padded = ix.padded;
    g.dstride = ix.dstride;
    g.queries = d_q;
    g.nq = nq;
    g.k = kk;
    g.out_ids = d_ids;
    g.out_sq = d_sq;
    g.scratch_sq = scratch.as<float>();
    g.scratch_id = nullptr;
    cuda_check(pagdev::launch_ground_truth(g, r.stream), "ground truth kernels");
    cuda_check(cudaStreamSynchronize(r.stream), "ground truth");
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap tensor_map_rows(const float* base, uint64_t rows, uint32_t padded, uint32_t dstride, uint32_t box_rows) {
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr),
                   "cuTensorMapEncodeTiled lookup");
        if (!fn || qr != cudaDriverEntryPointSuccess) throw_err(PAG_GPU_ECUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    CUtensorMap m;
    const cuuint64_t dims[2] = {padded, rows};
    const cuuint64_t strides[1] = {4ull * dstride};
    const cuuint32_t box[2] = {pagdev::gt_tc_block_k(), box_rows};
    const cuuint32_t es[2] = {1, 1};
    if (encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        throw_err(PAG_GPU_ECUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

// bench.cpp:18-53. k <= 1000: tensor-core filter GEMM under a per-query bound
// + exact re-rank of the pool (or, on request, per-split candidate lists +
// certificate for k <= 32); queries not settled that way re-run exactly;
// k > 1000: exact SIMT.
// Returns the number of queries whose tensor-core candidates were not
// certified and were re-run exactly.
uint64_t ground_truth_on_replica(pag_gpu_index& ix, Replica& r, const float* q, uint64_t nq, uint32_t k,
                                 uint32_t* ids, float* sq) {
    cuda_check(cudaSetDevice(r.device), "cudaSetDevice");
    if (nq == 0 || k == 0) return 0;
    const uint32_t kk = static_cast<uint32_t>(std::min<uint64_t>(k, ix.n));
    const uint32_t nqu = static_cast<uint32_t>(nq);
    std::vector<float> qp(nq * ix.dstride, 0.0f);
    for (uint64_t i = 0; i < nq; ++i) std::memcpy(&qp[i * ix.dstride], q + i * ix.dim, 4ull * ix.dim);
    DevBuf d_q(4 * qp.size()), d_ids(4ull * nq * kk), d_sq(4ull * nq * kk);
    cuda_check(cudaMemcpy(d_q.p, qp.data(), 4 * qp.size(), cudaMemcpyHostToDevice), "H2D");
    const bool no_tc = !r.bnorm || std::getenv("PAG_GPU_GT_EXACT");
    // k <= 1000: per-query bound + pool (a graph search supplies the bound
    // rows); PAG_GPU_GT_LISTS: the per-split top-C lists for k <= 32 (needs no
    // search; cfg-2 k = 10: 0.154 s against the pool path's time in
    // profiles/); otherwise the exact SIMT kernel
    const bool lists = !no_tc && kk <= pagdev::gt_tc_cmax() / 2 && std::getenv("PAG_GPU_GT_LISTS");
    const bool pool = !no_tc && !lists && kk <= 1000;
    const bool tc = lists;
    std::vector<uint32_t> redo;
    if (pool) {
        // 1. k rows per query from a graph search of the raw query (ids only;
        //    any k distinct rows give the bound)
        pag_search_params sp;
        pag_gpu_default_params(&sp);
        sp.K = kk;
        sp.efS = std::max(kk, 64u);  // a few more expansions tighten the bound of a small k
        sp.exact_dist = 0;
        DevBuf rawq(4ull * nq * ix.dim), sids(4ull * nq * kk), ssq(4ull * nq * kk), sn(4ull * nq),
            sst(4ull * nq * pagdev::kStatWords);
        cuda_check(cudaMemcpyAsync(rawq.p, q, 4ull * nq * ix.dim, cudaMemcpyHostToDevice, r.stream), "H2D");
        run_search(ix, r, sp, rawq.as<float>(), nqu, sids.as<uint32_t>(), ssq.as<float>(), sn.as<uint32_t>(),
                   sst.as<uint32_t>(), r.stream);
        // 2. bound, filter GEMM into per-query pools, exact re-rank of the pools
        const uint32_t BN = pagdev::gt_tc_block_n();
        const uint32_t mt = (nqu + pagdev::gt_tc_block_m() - 1) / pagdev::gt_tc_block_m();
        const uint64_t ntile = (ix.n + BN - 1) / BN;
        uint32_t ns = std::max<uint32_t>(1, std::min<uint32_t>(64, (4u * r.num_sms + mt / 2) / mt));
        const uint64_t rps = ((ntile + ns - 1) / ns) * BN;
        ns = static_cast<uint32_t>((ix.n + rps - 1) / rps);
        // pool capacity: the rows within 2 delta above the bound can be many
        // more than k where the k-th neighbour lies in a dense shell (cfg-2
        // k = 100: 35 of 10k queries overflowed 2048); 8192 x 4 B per query
        const uint32_t cap = 8192;
        CUtensorMap tmA = tensor_map_rows(d_q.as<float>(), nq, ix.padded, ix.dstride, pagdev::gt_tc_block_m());
        CUtensorMap tmB = tensor_map_rows(r.rows, ix.n, ix.padded, ix.dstride, BN);
        DevBuf qn(4ull * nq), thr(4ull * nq), pcnt(4ull * nq), pid(4ull * nq * cap), unc(4ull * nq);
        pagdev::GtTcPoolLaunch g{};
        g.tmA = &tmA;
        g.tmB = &tmB;
        g.base = r.rows;
        g.n = ix.n;
        g.padded = ix.padded;
        g.dstride = ix.dstride;
        g.queries = d_q.as<float>();
        g.nq = nqu;
        g.k = kk;
        g.nsplit = ns;
        g.rows_per_split = rps;
        g.qnorm = qn.as<float>();
        g.bnorm = r.bnorm;
        g.max_bnorm = ix.max_bnorm;
        g.search_ids = sids.as<uint32_t>();
        g.search_n = sn.as<uint32_t>();
        g.thrx = thr.as<float>();
        g.pool_cnt = pcnt.as<uint32_t>();
        g.pool_id = pid.as<uint32_t>();
        g.pool_cap = cap;
        g.out_ids = d_ids.as<uint32_t>();
        g.out_sq = d_sq.as<float>();
        g.uncertified = unc.as<uint32_t>();
        cuda_check(pagdev::launch_gt_tc_pool(g, r.stream), "tensor-core ground truth (pool)");
        std::vector<uint32_t> flags(nq);
        cuda_check(cudaMemcpyAsync(flags.data(), unc.p, 4ull * nq, cudaMemcpyDeviceToHost, r.stream), "D2H");
        cuda_check(cudaStreamSynchronize(r.stream), "tensor-core ground truth (pool)");
        for (uint32_t i = 0; i < nqu; ++i)
            if (flags[i]) redo.push_back(i);
    } else if (tc) {
        const uint32_t C = pagdev::gt_tc_cmax(), BN = pagdev::gt_tc_block_n();
        const uint32_t mt = (nqu + pagdev::gt_tc_block_m() - 1) / pagdev::gt_tc_block_m();
        const uint64_t ntile = (ix.n + BN - 1) / BN;
        uint32_t ns = std::max<uint32_t>(1, std::min<uint32_t>(64, (4u * r.num_sms + mt / 2) / mt));
        const uint64_t rps = ((ntile + ns - 1) / ns) * BN;
        ns = static_cast<uint32_t>((ix.n + rps - 1) / rps);
        CUtensorMap tmA = tensor_map_rows(d_q.as<float>(), nq, ix.padded, ix.dstride, pagdev::gt_tc_block_m());
        CUtensorMap tmB = tensor_map_rows(r.rows, ix.n, ix.padded, ix.dstride, BN);
        DevBuf qn(4ull * nq), cd(4ull * nq * ns * C), cid(4ull * nq * ns * C), cthr(4ull * nq * ns), unc(4ull * nq);
        pagdev::GtTcLaunch g{};
        g.tmA = &tmA;
        g.tmB = &tmB;
        g.base = r.rows;
        g.n = ix.n;
        g.padded = ix.padded;
        g.dstride = ix.dstride;
        g.queries = d_q.as<float>();
        g.nq = nqu;
        g.k = kk;
        g.nsplit = ns;
        g.C = C;
        g.rows_per_split = rps;
        g.qnorm = qn.as<float>();
        g.bnorm = r.bnorm;
        g.max_bnorm = ix.max_bnorm;
        g.cand_d = cd.as<float>();
        g.cand_id = cid.as<uint32_t>();
        g.cand_thr = cthr.as<float>();
        g.out_ids = d_ids.as<uint32_t>();
        g.out_sq = d_sq.as<float>();
        g.uncertified = unc.as<uint32_t>();
        cuda_check(pagdev::launch_gt_tc(g, r.stream), "tensor-core ground truth");
        std::vector<uint32_t> flags(nq);
        cuda_check(cudaMemcpyAsync(flags.data(), unc.p, 4ull * nq, cudaMemcpyDeviceToHost, r.stream), "D2H");
        cuda_check(cudaStreamSynchronize(r.stream), "tensor-core ground truth");
        for (uint32_t i = 0; i < nqu; ++i)
            if (flags[i]) redo.push_back(i);

    } else {
        exact_gt(ix, r, d_q.as<float>(), nqu, kk, d_ids.as<uint32_t>(), d_sq.as<float>());
    }
    std::vector<uint32_t> hi(nq * kk);
    std::vector<float> hs(nq * kk);
    cuda_check(cudaMemcpy(hi.data(), d_ids.p, 4 * hi.size(), cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(hs.data(), d_sq.p, 4 * hs.size(), cudaMemcpyDeviceToHost), "D2H");
    if (!redo.empty()) {  // exact fallback for the uncertified queries
        const uint32_t nr = static_cast<uint32_t>(redo.size());
        std::vector<float> qr(static_cast<size_t>(nr) * ix.dstride);
        for (uint32_t i = 0; i < nr; ++i)
            std::memcpy(&qr[static_cast<size_t>(i) * ix.dstride], &qp[static_cast<size_t>(redo[i]) * ix.dstride],
                        4ull * ix.dstride);
        DevBuf rq(4 * qr.size()), rids(4ull * nr * kk), rsq(4ull * nr * kk);
        cuda_check(cudaMemcpy(rq.p, qr.data(), 4 * qr.size(), cudaMemcpyHostToDevice), "H2D");
        exact_gt(ix, r, rq.as<float>(), nr, kk, rids.as<uint32_t>(), rsq.as<float>());
        std::vector<uint32_t> ri(static_cast<size_t>(nr) * kk);
        std::vector<float> rs(static_cast<size_t>(nr) * kk);
        cuda_check(cudaMemcpy(ri.data(), rids.p, 4 * ri.size(), cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(rs.data(), rsq.p, 4 * rs.size(), cudaMemcpyDeviceToHost), "D2H");
        for (uint32_t i = 0; i < nr; ++i) {
            std::memcpy(&hi[static_cast<size_t>(redo[i]) * kk], &ri[static_cast<size_t>(i) * kk], 4ull * kk);
            std::memcpy(&hs[static_cast<size_t>(redo[i]) * kk], &rs[static_cast<size_t>(i) * kk], 4ull * kk);
        }
    }
    for (uint64_t i = 0; i < nq; ++i) {
        std::memcpy(ids + i * k, &hi[i * kk], 4ull * kk);
        std::memcpy(sq + i * k, &hs[i * kk], 4ull * kk);
    }
    return redo.size();
}

// Online-insert refresh: the reference appended
// rows (insert_online, builder.cpp:354-363) and rewired adjacency lists
// (rebuild_neighbors :92-124, append_edge :126-139, PES flush :250-279) and
// saved the index again. Only what changed travels: new rows and norms, and
// the node blocks whose bytes differ from the host mirror, scattered on the
// device by one kernel. stats: {new nodes, dirty blocks, bytes uploaded, us}.
void grow_replica(pag_gpu_index& ix, Replica& r, uint64_t need) {
    if (need <= r.cap_nodes) return;
    const uint64_t cap = std::max<uint64_t>(need, r.cap_nodes + r.cap_nodes / 4 + 1024);
    const size_t row_bytes = 4ull * ix.dstride;
    auto regrow = [&](auto** p, size_t old_bytes, size_t new_bytes) {
        void* q = nullptr;
        cuda_check(cudaMalloc(&q, new_bytes), "cudaMalloc");
        if (*p && old_bytes) cuda_check(cudaMemcpy(q, *p, old_bytes, cudaMemcpyDeviceToDevice), "D2D grow");
        dev_free(*p);
        *p = static_cast<std::remove_reference_t<decltype(**p)>*>(q);
    };
    regrow(&r.rows, ix.n * row_bytes, cap * row_bytes);
    regrow(&r.deg, ix.n * 4, cap * 4);
    regrow(&r.adj, ix.n * ix.block_bytes, cap * ix.block_bytes);
    regrow(&r.bnorm, ix.n * 4, cap * 4);
    r.cap_nodes = cap;
}

// A newer state of the loaded index: header fields to check, random-access
// node records (thread-safe: called from several host threads), rows, norms.
struct RefreshSource {
    uint64_t n_new = 0;
    uint32_t dim = 0, padded = 0, L = 0, m = 0, M = 0;
    uint64_t seed = 0;
    uint8_t metric = 0;
    const uint32_t* entries = nullptr;
    uint32_t n_entries = 0;
    std::function<uint32_t(uint64_t)> degree;              // deg(u)
    std::function<void(uint64_t, uint32_t, uint8_t*)> fill;  // node u with deg edges -> zeroed block
    const uint8_t* rows = nullptr;   // n_new x padded fp32
    const uint8_t* norms = nullptr;  // n_new cached norms, or null (computed)
};

void refresh_from(pag_gpu_index& ix, const RefreshSource& src, uint64_t* st) {
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t n_new = src.n_new;
    const uint32_t padded = src.padded;
    if (src.dim != ix.dim || padded != ix.padded || (src.L != ix.L && src.L != 0) || src.m != ix.m ||
        src.M != ix.M || src.seed != ix.seed || src.metric != ix.metric || n_new < ix.n ||
        src.n_entries != ix.entries.size() ||
        (src.n_entries && std::memcmp(src.entries, ix.entries.data(), 4ull * src.n_entries) != 0))
        throw_err(PAG_GPU_EINVAL, "refresh: index is not an extension of the loaded one");
    if (n_new >= 0xFFFFFFFFull) throw_err(PAG_GPU_ERUNTIME, "index too large for 32-bit ids");
    const uint64_t n_old = ix.n;
    const uint32_t BB = ix.block_bytes;
    Replica& r0 = ix.reps.at(0);
    cudaSetDevice(r0.device);
    if (ix.mirror_deg.size() != n_old) {  // first refresh: mirror the device state
        ix.mirror_adj.resize(n_old * BB);
        ix.mirror_deg.resize(n_old);
        cuda_check(cudaMemcpy(ix.mirror_adj.data(), r0.adj, n_old * BB, cudaMemcpyDeviceToHost), "D2H mirror");
        cuda_check(cudaMemcpy(ix.mirror_deg.data(), r0.deg, 4 * n_old, cudaMemcpyDeviceToHost), "D2H mirror");
    }
    ix.mirror_adj.resize(n_new * BB);
    ix.mirror_deg.resize(n_new);
    // host threads over node ranges: build each block, diff it against the
    // mirror and collect the changed ones (merged in node order)
    std::vector<uint32_t> degs(n_new);
    uint64_t edges = 0;
    for (uint64_t u = 0; u < n_new; ++u) {
        const uint32_t deg = src.degree(u);
        if (deg > ix.maxdeg) throw_err(PAG_GPU_ERUNTIME, "degree over cap in file");
        edges += deg;
        degs[u] = deg;
    }
    const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::vector<uint32_t>> dirty_t(nth);
    std::vector<std::string> err_t(nth);
    auto diff_range = [&](unsigned t) {
        const uint64_t u0 = n_new * t / nth, u1 = n_new * (t + 1) / nth;
        std::vector<uint8_t> blk(BB);
        try {
            for (uint64_t u = u0; u < u1; ++u) {
                std::fill(blk.begin(), blk.end(), 0);
                src.fill(u, degs[u], blk.data());
                uint8_t* mb = &ix.mirror_adj[u * BB];
                if (u >= n_old || ix.mirror_deg[u] != degs[u] || std::memcmp(mb, blk.data(), BB) != 0) {
                    std::memcpy(mb, blk.data(), BB);
                    ix.mirror_deg[u] = degs[u];
                    dirty_t[t].push_back(static_cast<uint32_t>(u));
                }
            }
        } catch (const PagError& e) {
            err_t[t] = e.msg;
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned t = 1; t < nth; ++t) th.emplace_back(diff_range, t);
        diff_range(0);
        for (auto& x : th) x.join();
    }
    for (const auto& e : err_t)
        if (!e.empty()) throw_err(PAG_GPU_ERUNTIME, e);
    std::vector<uint32_t> dirty;
    for (const auto& d : dirty_t) dirty.insert(dirty.end(), d.begin(), d.end());
    const uint8_t* rows = src.rows;
    const uint8_t* norms = src.norms;
    const size_t row_bytes = 4ull * ix.dstride;
    std::vector<uint8_t> newrows((n_new - n_old) * row_bytes, 0);
    std::vector<float> newbn(n_new - n_old);
    for (uint64_t i = n_old; i < n_new; ++i) {
        std::memcpy(&newrows[(i - n_old) * row_bytes], rows + i * 4ull * padded, 4ull * padded);
        float v;
        if (norms)
            std::memcpy(&v, norms + 4 * i, 4);
        else
            v = host_vec_norm(reinterpret_cast<const float*>(rows) + i * padded, padded);
        newbn[i - n_old] = v * v;
        ix.max_bnorm = std::max(ix.max_bnorm, newbn[i - n_old]);
    }
    std::vector<uint8_t> staging(dirty.size() * BB);
    for (size_t i = 0; i < dirty.size(); ++i)
        std::memcpy(&staging[i * BB], &ix.mirror_adj[static_cast<uint64_t>(dirty[i]) * BB], BB);
    uint64_t up = 0;
    for (auto& r : ix.reps) {
        cuda_check(cudaSetDevice(r.device), "cudaSetDevice");
        grow_replica(ix, r, n_new);
        DevBuf dst(staging.size()), did(4 * dirty.size());
        if (!dirty.empty()) {
            cuda_check(cudaMemcpy(dst.p, staging.data(), staging.size(), cudaMemcpyHostToDevice), "H2D blocks");
            cuda_check(cudaMemcpy(did.p, dirty.data(), 4 * dirty.size(), cudaMemcpyHostToDevice), "H2D ids");
            cuda_check(pagdev::scatter_blocks(dst.p, did.as<uint32_t>(), static_cast<uint32_t>(dirty.size()), r.adj,
                                              BB, r.stream),
                       "scatter blocks");
        }
        cuda_check(cudaMemcpyAsync(r.deg, ix.mirror_deg.data(), 4 * n_new, cudaMemcpyHostToDevice, r.stream), "H2D deg");
        if (n_new > n_old) {
            cuda_check(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(r.rows) + n_old * row_bytes, newrows.data(),
                                       newrows.size(), cudaMemcpyHostToDevice, r.stream),
                       "H2D rows");
            cuda_check(cudaMemcpyAsync(r.bnorm + n_old, newbn.data(), 4 * newbn.size(), cudaMemcpyHostToDevice,
                                       r.stream),
                       "H2D norms");
        }
        cuda_check(cudaStreamSynchronize(r.stream), "refresh");
        r.bytes = r.cap_nodes * (row_bytes + 4 + BB) + 4ull * ix.refs.size();
        up = staging.size() + 4 * dirty.size() + 4 * n_new + newrows.size() + 4 * newbn.size();
    }
    ix.n = n_new;
    ix.total_edges = edges;
    if (st) {
        st[0] = n_new - n_old;
        st[1] = dirty.size();
        st[2] = up;
        st[3] = static_cast<uint64_t>(
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
}

void refresh_index(pag_gpu_index& ix, const char* path, uint64_t* st) {
    Mapped mp;
    mp.fd = ::open(path, O_RDONLY);
    if (mp.fd < 0) throw_err(PAG_GPU_ERUNTIME, std::string("cannot open index: ") + path);
    struct stat sb;
    if (fstat(mp.fd, &sb) != 0 || sb.st_size == 0) throw_err(PAG_GPU_ERUNTIME, "index read failed");
    mp.size = static_cast<size_t>(sb.st_size);
    void* mm = mmap(nullptr, mp.size, PROT_READ, MAP_PRIVATE, mp.fd, 0);
    if (mm == MAP_FAILED) throw_err(PAG_GPU_ERUNTIME, std::string("cannot open index: ") + path);
    mp.p = static_cast<const uint8_t*>(mm);
    Cursor cur{mp.p, mp.size};
    if (cur.pod<uint64_t>() != 0x5041474944583031ull) throw_err(PAG_GPU_ERUNTIME, "bad index magic");
    if (cur.pod<uint32_t>() != 1u) throw_err(PAG_GPU_ERUNTIME, "unsupported index version");
    RefreshSource src;
    src.n_new = cur.pod<uint64_t>();
    src.dim = cur.pod<uint32_t>();
    src.padded = cur.pod<uint32_t>();
    src.L = cur.pod<uint32_t>();
    src.m = cur.pod<uint32_t>();
    src.M = cur.pod<uint32_t>();
    cur.pod<uint32_t>();  // efC
    cur.pod<uint32_t>();  // b_build
    cur.pod<uint32_t>();  // pes_flush_interval
    src.seed = cur.pod<uint64_t>();
    src.metric = cur.pod<uint8_t>();
    cur.pod<uint8_t>();
    src.n_entries = cur.pod<uint32_t>();
    src.entries = reinterpret_cast<const uint32_t*>(cur.take(4ull * src.n_entries));
    // the file is scanned once for record offsets and degrees
    const uint64_t n_new = src.n_new;
    if (n_new < ix.n || src.padded != ix.padded || src.M != ix.M || (src.L != ix.L && src.L != 0))
        throw_err(PAG_GPU_EINVAL, "refresh: index is not an extension of the loaded one");
    const uint32_t S = ix.slot_stride, cb = ix.cb, cwp = ix.cwp;
    const size_t rec = 4 + cb + 12;
    std::vector<uint64_t> recoff(n_new);
    std::vector<uint32_t> degs(n_new);
    for (uint64_t u = 0; u < n_new; ++u) {
        const uint32_t deg = cur.pod<uint32_t>();
        if (deg > ix.maxdeg) throw_err(PAG_GPU_ERUNTIME, "degree over cap in file");
        degs[u] = deg;
        recoff[u] = static_cast<uint64_t>(cur.take(rec * deg) - mp.p);
    }
    src.degree = [&](uint64_t u) { return degs[u]; };
    src.fill = [&](uint64_t u, uint32_t deg, uint8_t* blk) { fill_block(blk, mp.p + recoff[u], deg, n_new, S, cb, cwp); };
    src.rows = cur.take(4ull * src.padded * n_new);
    src.norms = cur.take(4ull * n_new);
    refresh_from(ix, src, st);
}

// ---------------------------------------------------------------------------
// The reference's in-memory PagIndex as the source (pag_index_arrays,
// builder.hpp:62-132): fixed-stride targets / scalars / codes, a copy of the
// degrees, the VectorSet's rows and norms. Same validation as the file path.
// ---------------------------------------------------------------------------
void check_arrays(const pag_index_arrays* a) {
    if (!a) throw_err(PAG_GPU_EINVAL, "null argument");
    if (a->n && (!a->degrees || !a->targets || !a->scalars || !a->codes || !a->rows))
        throw_err(PAG_GPU_EINVAL, "null argument");
    if (a->n_entries && !a->entry_nodes) throw_err(PAG_GPU_EINVAL, "null argument");
}

// node u of the arrays -> the device block (zeroed by the caller)
void fill_block_arrays(uint8_t* blk, const pag_index_arrays& a, uint64_t u, uint32_t deg, uint64_t n, uint32_t S,
                       uint32_t cb, uint32_t cwp) {
    const uint64_t stride = 2ull * a.M;  // PagIndex::max_degree (builder.hpp:72)
    const uint32_t* tg_in = a.targets + u * stride;
    const float* sc = a.scalars + 3ull * u * stride;  // EdgeScalars{cos_beta, edge_norm, base_offset}
    const uint8_t* cd = a.codes + u * stride * cb;
    uint32_t* tg = reinterpret_cast<uint32_t*>(blk);
    float* en = reinterpret_cast<float*>(blk + 4u * S);
    float* cbeta = reinterpret_cast<float*>(blk + 8u * S);
    float* bo = reinterpret_cast<float*>(blk + 12u * S);
    uint8_t* codes = blk + 16u * S;
    for (uint32_t j = 0; j < deg; ++j) {
        if (tg_in[j] >= n) throw_err(PAG_GPU_ERUNTIME, "edge target out of range in file");
        tg[j] = tg_in[j];
        std::memcpy(codes + static_cast<size_t>(j) * 4 * cwp, cd + static_cast<size_t>(j) * cb, cb);
        cbeta[j] = sc[3 * j];
        en[j] = sc[3 * j + 1];
        bo[j] = sc[3 * j + 2];
    }
}

std::unique_ptr<pag_gpu_index> open_arrays(const pag_index_arrays* a, const std::vector<int>& devs) {
    check_arrays(a);
    auto ix = std::make_unique<pag_gpu_index>();
    ix->n = a->n;
    ix->dim = a->dim;
    ix->padded = a->padded_dim;
    ix->L = a->L;
    ix->m = a->m;
    ix->M = a->M;
    ix->efC = a->efC;
    ix->b_build = a->b_build;
    ix->pes_flush = a->pes_flush_interval;
    ix->seed = a->seed;
    ix->metric = a->metric;
    ix->enable_pes = a->enable_pes;
    ix->entries.assign(a->entry_nodes, a->entry_nodes + a->n_entries);
    init_layout(*ix);
    const uint64_t n = ix->n;
    const uint32_t S = ix->slot_stride, cb = ix->cb, cwp = ix->cwp, maxdeg = ix->maxdeg;
    IndexSource src;
    src.node = [&](uint64_t u, uint8_t* blk) {
        const uint32_t deg = a->degrees[u];
        if (deg > maxdeg) throw_err(PAG_GPU_ERUNTIME, "degree over cap in file");
        fill_block_arrays(blk, *a, u, deg, n, S, cb, cwp);
        return deg;
    };
    src.rows = [&] { return reinterpret_cast<const uint8_t*>(a->rows); };
    src.norms = [&] { return reinterpret_cast<const uint8_t*>(a->norms); };
    upload_index(ix.get(), devs, false, src);
    return ix;
}

void refresh_arrays(pag_gpu_index& ix, const pag_index_arrays* a, uint64_t* st) {
    check_arrays(a);
    RefreshSource src;
    src.n_new = a->n;
    src.dim = a->dim;
    src.padded = a->padded_dim;
    src.L = a->L;
    src.m = a->m;
    src.M = a->M;
    src.seed = a->seed;
    src.metric = a->metric;
    src.entries = a->entry_nodes;
    src.n_entries = a->n_entries;
    const uint64_t n_new = a->n;
    const uint32_t S = ix.slot_stride, cb = ix.cb, cwp = ix.cwp;
    src.degree = [&](uint64_t u) { return a->degrees[u]; };
    src.fill = [&](uint64_t u, uint32_t deg, uint8_t* blk) { fill_block_arrays(blk, *a, u, deg, n_new, S, cb, cwp); };
    src.rows = reinterpret_cast<const uint8_t*>(a->rows);
    src.norms = reinterpret_cast<const uint8_t*>(a->norms);
    refresh_from(ix, src, st);
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return PAG_GPU_OK;
    } catch (const PagError& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return PAG_GPU_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PAG_GPU_ERUNTIME;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Asynchronous batches: submit returns after the launch; the kernel reads
// pinned queries (or construction node ids) in place, writes results into
// the slot's pinned block and raises the slot's completion word; wait spins
// on that word and unpacks. Consecutive submits keep the programmatic-
// dependent-launch overlap (no event or copy between the kernels).
// ---------------------------------------------------------------------------
namespace {

// completion word of a ticket: never the reset value 0
uint32_t flag_of(uint64_t ticket) { return static_cast<uint32_t>(ticket) | 0x80000000u; }

void async_complete(Replica& r, Replica::AsyncSlot& a, uint32_t* status_or) {
    const int si = static_cast<int>(&a - r.aslot);
    volatile uint32_t* flag = r.h_flags + si;
    const uint32_t want = flag_of(a.ticket);
    uint64_t spins = 0;
    while (*flag != want) {
        if ((++spins & 1023u) == 0) {
            const cudaError_t e = cudaStreamQuery(r.stream);
            if (e != cudaSuccess && e != cudaErrorNotReady) {
                a.ticket = 0;
                cuda_check(e, "asynchronous search");
            }
            if (e == cudaSuccess && *flag != want) {
                a.ticket = 0;
                throw_err(PAG_GPU_ECUDA, "asynchronous search: completion flag missing");
            }
            std::this_thread::yield();
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const uint64_t nq = a.nq;
    const uint32_t K = a.K;
    const size_t ob_ids = 4ull * nq * std::max(1u, K), ob_n = 4ull * nq;
    if (K) {
        std::memcpy(a.ids, a.h_res, 4ull * nq * K);
        std::memcpy(a.sq, a.h_res + ob_ids, 4ull * nq * K);
    }
    std::memcpy(a.n_out, a.h_res + 2 * ob_ids, ob_n);
    const uint32_t* st = reinterpret_cast<const uint32_t*>(a.h_res + 2 * ob_ids + ob_n);
    if (a.cons) {  // pes lists: the written prefix of each row, zeros past it
        const size_t ob_st = 4ull * nq * pagdev::kStatWords;
        const uint8_t* hp = a.h_res + 2 * ob_ids + ob_n + ob_st;
        const uint32_t* hpn = reinterpret_cast<const uint32_t*>(hp + 4ull * nq * a.pes_cap);
        std::memcpy(a.pes_n, hpn, 4ull * nq);
        if (a.pes_cap)
            for (uint64_t i = 0; i < nq; ++i) {
                const uint32_t m = std::min(hpn[i], a.pes_cap);
                uint32_t* row = a.pes + i * a.pes_cap;
                std::memcpy(row, hp + 4ull * i * a.pes_cap, 4ull * m);
                std::memset(row + m, 0, 4ull * (a.pes_cap - m));
            }
    }
    uint32_t so = 0;
    for (uint64_t i = 0; i < nq; ++i) {
        const uint32_t* w = st + i * pagdev::kStatWords;
        so |= w[pagdev::kStatStatus];
        if (a.stats) {
            a.stats[i].exact_dist_count = w[pagdev::kStatExact];
            a.stats[i].test_count = w[pagdev::kStatTest];
            a.stats[i].pass_count = w[pagdev::kStatPass];
            a.stats[i].visited_count = w[pagdev::kStatVisited];
            a.stats[i].edges_scanned = w[pagdev::kStatEdges];
        }
    }
    a.ticket = 0;
    *status_or |= so;
}

// frees the ring slot of `ticket` on replica r: an older batch still holding
// it is completed now and its status is kept for its own wait
void free_slot(pag_gpu_index& ix, Replica& r, uint64_t ticket) {
    Replica::AsyncSlot& a = r.aslot[ticket % Replica::kAsyncDepth];
    if (!a.ticket) return;
    const uint64_t old = a.ticket;
    uint32_t so = 0;
    async_complete(r, a, &so);
    if (so) ix.early_status[old] |= so;  // only failures need keeping (a later wait of an OK ticket returns OK)
}

void async_submit_replica(pag_gpu_index& ix, Replica& r, const pag_search_params& p, const float* q,
                          uint64_t nq, uint32_t* ids, float* sq, uint32_t* n_out, pag_search_stats* stats,
                          uint64_t ticket, const ConstructionHost* ch = nullptr) {
    cuda_check(cudaSetDevice(r.device), "cudaSetDevice");
    if (!r.h_flags) {
        cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&r.h_flags), 4 * Replica::kAsyncDepth, cudaHostAllocMapped),
                   "cudaHostAlloc");
        std::memset(r.h_flags, 0, 4 * Replica::kAsyncDepth);
        dev_alloc(&r.d_done, 4 * Replica::kAsyncDepth);
        cuda_check(cudaMemset(r.d_done, 0, 4 * Replica::kAsyncDepth), "memset");
    }
    const int si = static_cast<int>(ticket % Replica::kAsyncDepth);
    Replica::AsyncSlot& a = r.aslot[si];
    free_slot(ix, r, ticket);  // ring full: finish the oldest first
    if (nq == 0) return;
    const uint32_t K = p.K;
    const size_t ob_ids = 4ull * nq * std::max(1u, K), ob_n = 4ull * nq, ob_st = 4ull * nq * pagdev::kStatWords;
    const size_t ob_pes = ch ? 4ull * nq * ch->pes_cap : 0, ob_pn = ch ? 4ull * nq : 0;
    const size_t ob_nodes = ch ? 4ull * nq : 0;  // construction node ids, read by the kernel in place
    const size_t need = 2 * ob_ids + ob_n + ob_st + ob_pes + ob_pn + ob_nodes;
    if (a.h_bytes < need) {
        if (a.h_res) cudaFreeHost(a.h_res);
        a.h_res = nullptr;
        a.h_bytes = 0;
        cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&a.h_res), need, cudaHostAllocMapped), "cudaHostAlloc");
        a.h_bytes = need;
    }
    uint8_t* dres = nullptr;
    cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dres), a.h_res, 0), "cudaHostGetDevicePointer");
    uint32_t* dflags = nullptr;
    cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflags), r.h_flags, 0), "cudaHostGetDevicePointer");
    const float* q_src = nullptr;
    cudaPointerAttributes at{};
    ConstructionArgs ca;
    if (ch) {  // construction: node ids and pes lists in the pinned block (no copy between launches)
        const size_t off = 2 * ob_ids + ob_n + ob_st + ob_pes + ob_pn;
        std::memcpy(a.h_res + off, ch->nodes, ob_nodes);
        ca.nodes = reinterpret_cast<const uint32_t*>(dres + off);
        ca.collect_pes = ch->collect_pes;
        ca.pes_cap = ch->pes_cap;
        ca.pes = reinterpret_cast<uint32_t*>(dres + 2 * ob_ids + ob_n + ob_st);
        ca.pes_n = reinterpret_cast<uint32_t*>(dres + 2 * ob_ids + ob_n + ob_st + ob_pes);
    } else if (!std::getenv("PAG_GPU_NO_ZEROCOPY") && cudaPointerGetAttributes(&at, q) == cudaSuccess &&
               at.type == cudaMemoryTypeHost && at.devicePointer) {
        q_src = static_cast<const float*>(at.devicePointer);
    } else {
        (void)cudaGetLastError();
        grow_dev(reinterpret_cast<void**>(&a.d_q), &a.d_q_bytes, 4ull * nq * ix.dim);
        cuda_check(cudaMemcpyAsync(a.d_q, q, 4ull * nq * ix.dim, cudaMemcpyHostToDevice, r.stream), "H2D queries");
        q_src = a.d_q;
    }
    AsyncArgs aa;
    aa.done_ctr = r.d_done + si;
    aa.host_flag = dflags + si;
    aa.flag_value = flag_of(ticket);
    r.h_flags[si] = 0;
    a.nq = nq;
    a.K = K;
    a.ids = ids;
    a.sq = sq;
    a.n_out = n_out;
    a.stats = stats;
    a.cons = ch != nullptr;
    a.pes = ch ? ch->pes : nullptr;
    a.pes_n = ch ? ch->pes_n : nullptr;
    a.pes_cap = ch ? ch->pes_cap : 0;
    run_search(ix, r, p, q_src, static_cast<uint32_t>(nq), reinterpret_cast<uint32_t*>(dres),
               reinterpret_cast<float*>(dres + ob_ids), reinterpret_cast<uint32_t*>(dres + 2 * ob_ids),
               reinterpret_cast<uint32_t*>(dres + 2 * ob_ids + ob_n), r.stream, ch ? &ca : nullptr, &aa);
    a.ticket = ticket;  // only a launched batch holds the slot
}

// A submit over all replicas: every replica's shard is launched, or none
// holds caller pointers when the call fails (the shards already launched
// are completed before the error is returned; their status is dropped with
// the failed batch).
template <typename LaunchShard>
void submit_all(pag_gpu_index& ix, uint64_t t, LaunchShard&& launch) {
    const size_t nd = ix.reps.size();
    size_t d = 0;
    try {
        for (; d < nd; ++d) launch(d);
    } catch (...) {
        for (size_t e = 0; e < nd; ++e) {
            Replica& r = ix.reps[e];
            Replica::AsyncSlot& a = r.aslot[t % Replica::kAsyncDepth];
            if (a.ticket == t) {
                uint32_t so = 0;
                try {
                    cudaSetDevice(r.device);
                    async_complete(r, a, &so);
                } catch (...) {
                }
                a.ticket = 0;
            }
        }
        throw;
    }
}

void check_status(uint32_t so) {
    if (so & pagdev::kStatusZeroCosineQuery) throw_err(PAG_GPU_EINVAL, "zero query under cosine metric");
    // PAG_VALIDATE builds (routing.cpp:116-137 texts, std::logic_error)
    if (so & pagdev::kStatusTfbCapacity) throw_err(PAG_GPU_ELOGIC, "TFB: working set over capacity");
    if (so & pagdev::kStatusTfbZmax) throw_err(PAG_GPU_ELOGIC, "TFB: stale z_max");
    if (so & pagdev::kStatusTfbDuplicate) throw_err(PAG_GPU_ELOGIC, "TFB: duplicate node residence");
    if (so & pagdev::kStatusTfbOrder) throw_err(PAG_GPU_ELOGIC, "TFB: result list out of order");
}

// ix.dup_nodes from the first replica's adjacency (after load / refresh)
void update_dup_nodes(pag_gpu_index& ix) {
    if (ix.reps.empty()) return;
    Replica& r = ix.reps[0];
    cuda_check(cudaSetDevice(r.device), "cudaSetDevice");
    uint32_t* cnt = nullptr;
    dev_alloc(&cnt, 4);
    uint32_t h = 1;
    cudaError_t e = pagdev::count_dup_groups(r.adj, r.deg, ix.n, ix.block_bytes, cnt, r.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(r.stream);
    if (e == cudaSuccess) e = cudaMemcpy(&h, cnt, 4, cudaMemcpyDeviceToHost);
    dev_free(cnt);
    cuda_check(e, "duplicate-target check");
    ix.dup_nodes = h;
}

// Runs fn(d) for every replica d: inline for one replica, else on the
// replicas' persistent host workers in parallel (started on first use); the
// first error (in replica order) is rethrown after all have finished.
void run_replicas(pag_gpu_index& ix, const std::function<void(size_t)>& fn) {
    const size_t nd = ix.reps.size();
    if (nd == 1) {
        fn(0);
        return;
    }
    for (size_t d = 0; d < nd; ++d) {
        Replica& r = ix.reps[d];
        if (!r.worker) r.worker = std::make_shared<Replica::Worker>();
        r.worker->post([&fn, d] { fn(d); });
    }
    std::exception_ptr first;
    for (size_t d = 0; d < nd; ++d) {
        std::exception_ptr e = ix.reps[d].worker->join_job();
        if (e && !first) first = e;
    }
    if (first) std::rethrow_exception(first);
}

// query shard [q0, q1) of replica d (contiguous, the same bounds as the
// torchrun sharding in shard.py)
inline uint64_t shard_lo(uint64_t n, size_t d, size_t nd) { return n * d / nd; }

pag_search_params construction_params(const pag_gpu_index& ix, const pag_search_params* params) {
    pag_search_params p{};
    if (params) {
        p = *params;
    } else {  // insert_with_state (builder.cpp:220-224): K = efS = efC, b = b_build
        pag_gpu_default_params(&p);
        p.K = p.efS = ix.efC;
        p.b_override = ix.b_build;
    }
    return p;
}

std::unique_ptr<pag_gpu_index> open_checked(const char* index_path, const std::vector<int>& devs) {
    auto ix = open_index(index_path, devs);
    update_dup_nodes(*ix);
    return ix;
}

}  // namespace

extern "C" {

void pag_gpu_default_params(pag_search_params* p) {
    p->K = 10;
    p->efS = 100;
    p->b_override = 0;
    p->use_prt = 1;
    p->use_tfb = 1;
    p->exact_dist = 1;
    p->reserved = 0;
}

int pag_gpu_open(const char* index_path, uint32_t device_mask, pag_gpu_index** out) {
    return guarded([&] {
        if (!out || !index_path) throw_err(PAG_GPU_EINVAL, "null argument");
        *out = nullptr;
        if (device_mask == 0) device_mask = 1;
        std::vector<int> devs;
        for (int d = 0; d < 32; ++d)
            if (device_mask & (1u << d)) devs.push_back(d);
        *out = open_checked(index_path, devs).release();
    });
}

int pag_gpu_open_devices(const char* index_path, const int* devices, uint32_t n_devices, pag_gpu_index** out) {
    return guarded([&] {
        if (!out || !index_path || (n_devices && !devices)) throw_err(PAG_GPU_EINVAL, "null argument");
        *out = nullptr;
        std::vector<int> devs(devices, devices + n_devices);
        if (devs.empty()) devs.push_back(0);
        *out = open_checked(index_path, devs).release();
    });
}

int pag_gpu_open_from_arrays(const pag_index_arrays* a, const int* devices, uint32_t n_devices,
                             pag_gpu_index** out) {
    return guarded([&] {
        if (!out || (n_devices && !devices)) throw_err(PAG_GPU_EINVAL, "null argument");
        *out = nullptr;
        std::vector<int> devs(devices, devices + n_devices);
        if (devs.empty()) devs.push_back(0);
        auto ix = open_arrays(a, devs);
        update_dup_nodes(*ix);
        *out = ix.release();
    });
}

int pag_gpu_refresh_from_arrays(pag_gpu_index* ix, const pag_index_arrays* a, uint64_t* stats) {
    return guarded([&] {
        if (!ix) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        refresh_arrays(*ix, a, stats);
        update_dup_nodes(*ix);
    });
}

int pag_gpu_inspect(const char* index_path, uint64_t* info, size_t n_info) {
    return guarded([&] {
        if (!index_path || !info) throw_err(PAG_GPU_EINVAL, "null argument");
        auto ix = open_index(index_path, {}, true);
        const uint64_t v[12] = {ix->n, ix->dim, ix->padded, ix->L, ix->m, ix->M, ix->metric,
                                ix->entries.size(), ix->seed, ix->total_edges, 0, 0};
        for (size_t i = 0; i < n_info && i < 12; ++i) info[i] = v[i];
    });
}

int pag_gpu_reference_family(uint32_t padded_dim, uint32_t L, uint32_t m, uint64_t seed, float* out,
                             size_t n_out) {
    return guarded([&] {
        auto refs = reference_family(padded_dim, L, m, seed);
        if (!out || n_out < refs.size()) throw_err(PAG_GPU_EINVAL, "output buffer too small");
        std::memcpy(out, refs.data(), 4 * refs.size());
    });
}

uint32_t pag_gpu_default_subspace_count(uint32_t dim) { return default_L(dim); }

int pag_gpu_refresh(pag_gpu_index* ix, const char* index_path, uint64_t* stats) {
    return guarded([&] {
        if (!ix || !index_path) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        refresh_index(*ix, index_path, stats);
        update_dup_nodes(*ix);
    });
}

int pag_gpu_close(pag_gpu_index* ix) {
    return guarded([&] {
        if (!ix) return;
        for (auto& r : ix->reps) free_replica(r);
        delete ix;
    });
}

int pag_gpu_info(const pag_gpu_index* ix, uint64_t* info, size_t n_info) {
    return guarded([&] {
        if (!ix || !info) throw_err(PAG_GPU_EINVAL, "null argument");
        const uint64_t v[17] = {ix->n, ix->dim, ix->padded, ix->L, ix->m, ix->M, ix->metric,
                                ix->entries.size(), ix->seed, ix->total_edges, ix->reps.size(),
                                ix->reps.empty() ? 0
                                                 : ix->reps[0].bytes + ix->reps[0].rows_x_cap * 4ull *
                                                                           pagdev::chain_xstride(ix->padded),
                                ix->gt_uncertified,
                                ix->efC, ix->b_build, ix->enable_pes, ix->dup_nodes};
        for (size_t i = 0; i < n_info && i < 17; ++i) info[i] = v[i];
    });
}

int pag_gpu_search(pag_gpu_index* ix, const float* q, uint64_t nq, const pag_search_params* params,
                   uint32_t* ids, float* sq, uint32_t* n_out, pag_search_stats* stats) {
    return guarded([&] {
        if (!ix || !params) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        const pag_search_params p = *params;
        validate_params(*ix, p);
        if (nq == 0) return;
        if (!q || !n_out || (p.K && (!ids || !sq))) throw_err(PAG_GPU_EINVAL, "null argument");
        if (nq >= 0xFFFFFFFFull) throw_err(PAG_GPU_EINVAL, "batch too large");
        const size_t nd = ix->reps.size();
        std::vector<uint32_t> status(nd, 0);
        run_replicas(*ix, [&](size_t d) {
            const uint64_t q0 = shard_lo(nq, d, nd), q1 = shard_lo(nq, d + 1, nd);
            search_on_replica(*ix, ix->reps[d], p, q + q0 * ix->dim, q1 - q0, ids + q0 * p.K, sq + q0 * p.K,
                              n_out + q0, stats ? stats + q0 : nullptr, &status[d]);
        });
        uint32_t so = 0;
        for (auto s : status) so |= s;
        check_status(so);
    });
}

int pag_gpu_construction_search(pag_gpu_index* ix, const uint32_t* nodes, uint64_t nn,
                                const pag_search_params* params, int collect_pes, uint32_t* ids, float* sq,
                                uint32_t* n_out, pag_search_stats* stats, uint32_t* pes, uint32_t pes_cap,
                                uint32_t* pes_n) {
    return guarded([&] {
        if (!ix) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        // insert_with_state (builder.cpp:220-224): K = efS = efC, b = b_build,
        // collect_pes = enable_pes, unless the caller overrides
        const pag_search_params p = construction_params(*ix, params);
        const uint32_t pes_on = collect_pes < 0 ? ix->enable_pes : static_cast<uint32_t>(collect_pes != 0);
        validate_params(*ix, p);
        if (nn == 0) return;
        if (!nodes || !n_out || !pes_n || (p.K && (!ids || !sq)) || (pes_cap && !pes))
            throw_err(PAG_GPU_EINVAL, "null argument");
        if (nn >= 0xFFFFFFFFull) throw_err(PAG_GPU_EINVAL, "batch too large");
        for (uint64_t i = 0; i < nn; ++i)
            if (nodes[i] >= ix->n) throw_err(PAG_GPU_EINVAL, "node id out of range");
        const size_t nd = ix->reps.size();
        std::vector<uint32_t> status(nd, 0);
        run_replicas(*ix, [&](size_t d) {
            const uint64_t q0 = shard_lo(nn, d, nd), q1 = shard_lo(nn, d + 1, nd);
            ConstructionHost ch{nodes + q0, pes_on, pes_cap, pes ? pes + q0 * pes_cap : nullptr, pes_n + q0};
            search_on_replica(*ix, ix->reps[d], p, nullptr, q1 - q0, ids + q0 * p.K, sq + q0 * p.K, n_out + q0,
                              stats ? stats + q0 : nullptr, &status[d], &ch);
        });
        uint32_t so = 0;
        for (auto s : status) so |= s;
        check_status(so);
    });
}

int pag_gpu_construction_search_device(pag_gpu_index* ix, const uint32_t* nodes_dev, uint64_t nn,
                                       const pag_search_params* params, int collect_pes, uint32_t* ids_dev,
                                       float* sq_dev, uint32_t* n_out_dev, uint32_t* stats_dev,
                                       uint32_t* pes_dev, uint32_t pes_cap, uint32_t* pes_n_dev, void* stream) {
    return guarded([&] {
        if (!ix) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        const pag_search_params p = construction_params(*ix, params);
        validate_params(*ix, p);
        if (nn >= 0xFFFFFFFFull) throw_err(PAG_GPU_EINVAL, "batch too large");
        Replica& r = ix->reps[0];
        cuda_check(cudaSetDevice(r.device), "cudaSetDevice");
        ConstructionArgs ca;
        ca.nodes = nodes_dev;
        ca.collect_pes = collect_pes < 0 ? ix->enable_pes : static_cast<uint32_t>(collect_pes != 0);
        ca.pes_cap = pes_cap;
        ca.pes = pes_dev;
        ca.pes_n = pes_n_dev;
        run_search(*ix, r, p, nullptr, static_cast<uint32_t>(nn), ids_dev, sq_dev, n_out_dev, stats_dev,
                   static_cast<cudaStream_t>(stream), &ca);
    });
}

int pag_gpu_search_submit(pag_gpu_index* ix, const float* q, uint64_t nq, const pag_search_params* params,
                          uint32_t* ids, float* sq, uint32_t* n_out, pag_search_stats* stats, uint64_t* ticket) {
    return guarded([&] {
        if (!ix || !params || !ticket) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        const pag_search_params p = *params;
        validate_params(*ix, p);
        if (nq && (!q || !n_out || (p.K && (!ids || !sq)))) throw_err(PAG_GPU_EINVAL, "null argument");
        if (nq >= 0xFFFFFFFFull) throw_err(PAG_GPU_EINVAL, "batch too large");
        const uint64_t t = ++ix->async_seq;
        const size_t nd = ix->reps.size();
        submit_all(*ix, t, [&](size_t d) {
            const uint64_t q0 = shard_lo(nq, d, nd), q1 = shard_lo(nq, d + 1, nd);
            async_submit_replica(*ix, ix->reps[d], p, q + q0 * ix->dim, q1 - q0, ids + q0 * p.K, sq + q0 * p.K,
                                 n_out + q0, stats ? stats + q0 : nullptr, t);
        });
        *ticket = t;
    });
}

int pag_gpu_construction_submit(pag_gpu_index* ix, const uint32_t* nodes, uint64_t nn,
                                const pag_search_params* params, int collect_pes, uint32_t* ids, float* sq,
                                uint32_t* n_out, pag_search_stats* stats, uint32_t* pes, uint32_t pes_cap,
                                uint32_t* pes_n, uint64_t* ticket) {
    return guarded([&] {
        if (!ix || !ticket) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        const pag_search_params p = construction_params(*ix, params);
        const uint32_t pes_on = collect_pes < 0 ? ix->enable_pes : static_cast<uint32_t>(collect_pes != 0);
        validate_params(*ix, p);
        if (nn && (!nodes || !n_out || !pes_n || (p.K && (!ids || !sq)) || (pes_cap && !pes)))
            throw_err(PAG_GPU_EINVAL, "null argument");
        if (nn >= 0xFFFFFFFFull) throw_err(PAG_GPU_EINVAL, "batch too large");
        for (uint64_t i = 0; i < nn; ++i)
            if (nodes[i] >= ix->n) throw_err(PAG_GPU_EINVAL, "node id out of range");
        const uint64_t t = ++ix->async_seq;
        const size_t nd = ix->reps.size();
        submit_all(*ix, t, [&](size_t d) {
            const uint64_t q0 = shard_lo(nn, d, nd), q1 = shard_lo(nn, d + 1, nd);
            ConstructionHost ch{nodes + q0, pes_on, pes_cap, pes ? pes + q0 * pes_cap : nullptr, pes_n + q0};
            async_submit_replica(*ix, ix->reps[d], p, nullptr, q1 - q0, ids + q0 * p.K, sq + q0 * p.K, n_out + q0,
                                 stats ? stats + q0 : nullptr, t, &ch);
        });
        *ticket = t;
    });
}

int pag_gpu_search_wait(pag_gpu_index* ix, uint64_t ticket) {
    return guarded([&] {
        if (!ix) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        if (ticket == 0 || ticket > ix->async_seq) throw_err(PAG_GPU_EINVAL, "unknown ticket");
        uint32_t so = 0;
        auto it = ix->early_status.find(ticket);  // completed by a later submit
        if (it != ix->early_status.end()) {
            so |= it->second;
            ix->early_status.erase(it);
        }
        std::exception_ptr first;
        for (auto& r : ix->reps) {
            Replica::AsyncSlot& a = r.aslot[ticket % Replica::kAsyncDepth];
            if (a.ticket == ticket) {
                try {
                    cuda_check(cudaSetDevice(r.device), "cudaSetDevice");
                    async_complete(r, a, &so);
                } catch (...) {
                    if (!first) first = std::current_exception();
                }
            }
        }
        if (first) std::rethrow_exception(first);
        check_status(so);
    });
}

int pag_gpu_search_device(pag_gpu_index* ix, const float* q_dev, uint64_t nq,
                          const pag_search_params* params, uint32_t* ids_dev, float* sq_dev,
                          uint32_t* n_out_dev, uint32_t* stats_dev, void* stream) {
    return guarded([&] {
        if (!ix || !params) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        const pag_search_params p = *params;
        validate_params(*ix, p);
        Replica& r = ix->reps[0];
        cuda_check(cudaSetDevice(r.device), "cudaSetDevice");
        cudaStream_t s = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
        if (nq >= 0xFFFFFFFFull) throw_err(PAG_GPU_EINVAL, "batch too large");
        run_search(*ix, r, p, q_dev, static_cast<uint32_t>(nq), ids_dev, sq_dev, n_out_dev, stats_dev, s);
    });
}

int pag_gpu_ground_truth(pag_gpu_index* ix, const float* queries, uint64_t nq, uint32_t k,
                         uint32_t* ids, float* sq) {
    return guarded([&] {
        if (!ix) throw_err(PAG_GPU_EINVAL, "null argument");
        std::lock_guard<std::mutex> g(ix->mu);
        if (nq == 0 || k == 0) return;
        if (!queries || !ids || !sq) throw_err(PAG_GPU_EINVAL, "null argument");
        const size_t nd = ix->reps.size();
        std::vector<uint64_t> unc(nd, 0);
        run_replicas(*ix, [&](size_t d) {
            const uint64_t q0 = shard_lo(nq, d, nd), q1 = shard_lo(nq, d + 1, nd);
            unc[d] = ground_truth_on_replica(*ix, ix->reps[d], queries + q0 * ix->dim, q1 - q0, k, ids + q0 * k,
                                             sq + q0 * k);
        });
        for (auto u : unc) ix->gt_uncertified += u;
    });
}

const char* pag_gpu_last_error(void) { return g_err.c_str(); }

// diagnostic (PAG_PHASE_TIMING builds): per-phase summed warp cycles
void pag_gpu_phase_cycles(unsigned long long* out8, int reset) { pagdev::search_phase_cycles(out8, reset != 0); }

const char* pag_gpu_version(void) { return "pag_gpu 0.2 (sm_100a)"; }

}  // extern "C"
