// pag_gpu.hpp — header-only C++ adapter over the C ABI (pag_gpu.h) for the
// reference code base: the binding a maintainer of /root/reference/proj
// would add as proj/include/pag/gpu.hpp. It maps the
// reference's types onto the ABI:
//   SearchParams / SearchResult / Candidate   proj/include/pag/routing.hpp:13-34,173-177
//   PagIndex load_index(const std::string&)   proj/include/pag/builder.hpp:157
//   PagIndex (in memory, after build / insert_online)  builder.hpp:62-132
//   search(const PagIndex&, span, SearchParams, TfbState&)  routing.hpp:181-184
// and the ABI's status codes onto the reference's exception classes
// (std::invalid_argument / std::runtime_error, same message texts).
#pragma once
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "pag/routing.hpp"  // the reference's SearchParams, SearchResult, Candidate
#include "pag_gpu.h"

namespace pag {

inline void gpu_check(int rc) {
    if (rc == PAG_GPU_OK) return;
    std::string msg = pag_gpu_last_error();
    if (rc == PAG_GPU_EINVAL) throw std::invalid_argument(msg);
    if (rc == PAG_GPU_ELOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

// The reference's in-memory PagIndex as the ABI's borrowed arrays
// (pag_index_arrays): fixed-stride accessors of builder.hpp:74-85, a
// snapshot of the atomic degrees; norms are recomputed from the rows.
struct IndexArrays {
    pag_index_arrays a{};
    std::vector<uint32_t> degrees;
    explicit IndexArrays(const PagIndex& ix) : degrees(ix.size()) {
        static_assert(sizeof(EdgeScalars) == 3 * sizeof(float), "EdgeScalars is {cos_beta, edge_norm, base_offset}");
        for (uint32_t u = 0; u < ix.size(); ++u) degrees[u] = ix.degree(u);
        const BuildParams& bp = ix.params();
        a.n = ix.size();
        a.dim = static_cast<uint32_t>(ix.vectors().dim());
        a.padded_dim = static_cast<uint32_t>(ix.vectors().padded_dim());
        a.L = ix.refs().L;
        a.m = bp.m;
        a.M = bp.M;
        a.efC = bp.efC;
        a.b_build = bp.b_build;
        a.pes_flush_interval = bp.pes_flush_interval;
        a.seed = bp.seed;
        a.metric = static_cast<uint8_t>(ix.vectors().metric());
        a.enable_pes = bp.enable_pes ? 1 : 0;
        a.n_entries = static_cast<uint32_t>(ix.entry_nodes().size());
        a.entry_nodes = ix.entry_nodes().data();
        a.degrees = degrees.data();
        if (ix.size()) {
            a.targets = ix.targets(0);
            a.scalars = reinterpret_cast<const float*>(ix.scalars(0));
            a.codes = ix.edge_codes(0, 0);
            a.rows = ix.vectors().row(0);
        }
        a.norms = nullptr;
    }
};

// A PAG index resident on one or more GPUs (move-only, like PagIndex): from
// a PAGIDX01 file, or straight from the reference's in-memory PagIndex.
class GpuIndex {
public:
    explicit GpuIndex(const PagIndex& index, std::vector<int> devices = {0}) {
        const IndexArrays ia(index);
        gpu_check(pag_gpu_open_from_arrays(&ia.a, devices.data(), static_cast<uint32_t>(devices.size()), &h_));
        read_info();
    }
    explicit GpuIndex(const std::string& path, std::vector<int> devices = {0}) {
        gpu_check(pag_gpu_open_devices(path.c_str(), devices.data(), static_cast<uint32_t>(devices.size()), &h_));
        read_info();
    }
    // re-synchronise with the PagIndex after insert_online batches (only new
    // rows and changed adjacency blocks travel)
    void refresh(const PagIndex& index) {
        const IndexArrays ia(index);
        gpu_check(pag_gpu_refresh_from_arrays(h_, &ia.a, nullptr));
        read_info();
    }
    void refresh(const std::string& path) {
        gpu_check(pag_gpu_refresh(h_, path.c_str(), nullptr));
        read_info();
    }

private:
    void read_info() {
        uint64_t info[17];
        gpu_check(pag_gpu_info(h_, info, 17));
        n_ = info[0];
        dim_ = static_cast<uint32_t>(info[1]);
        efC_ = static_cast<uint32_t>(info[13]);
    }

public:
    GpuIndex(GpuIndex&& o) noexcept : h_(o.h_), n_(o.n_), dim_(o.dim_), efC_(o.efC_) { o.h_ = nullptr; }
    GpuIndex(const GpuIndex&) = delete;
    GpuIndex& operator=(const GpuIndex&) = delete;
    ~GpuIndex() {
        if (h_) pag_gpu_close(h_);
    }
    uint64_t size() const { return n_; }
    uint32_t dim() const { return dim_; }
    uint32_t efC() const { return efC_; }
    pag_gpu_index* handle() const { return h_; }

private:
    pag_gpu_index* h_ = nullptr;
    uint64_t n_ = 0;
    uint32_t dim_ = 0, efC_ = 0;
};

inline pag_search_params to_abi(const SearchParams& sp, bool exact_dist = true) {
    pag_search_params p;
    pag_gpu_default_params(&p);
    p.K = sp.K;
    p.efS = sp.efS;
    p.b_override = sp.b_override;
    p.use_prt = sp.use_prt;
    p.use_tfb = sp.use_tfb;
    p.exact_dist = exact_dist ? 1 : 0;
    return p;
}

// Batched drop-in for pag::search: queries is nq x dim row-major; one
// SearchResult per query, bit-identical to pag::search with exact_dist.
inline std::vector<SearchResult> search_batch(const GpuIndex& ix, std::span<const float> queries,
                                              const SearchParams& sp, bool exact_dist = true) {
    if (queries.size() % ix.dim() != 0) throw std::invalid_argument("query dimension mismatch");
    const uint64_t nq = queries.size() / ix.dim();
    const pag_search_params p = to_abi(sp, exact_dist);
    std::vector<uint32_t> ids(nq * sp.K), n_out(nq);
    std::vector<float> sq(nq * sp.K);
    std::vector<pag_search_stats> st(nq);
    gpu_check(pag_gpu_search(ix.handle(), queries.data(), nq, &p, ids.data(), sq.data(), n_out.data(), st.data()));
    std::vector<SearchResult> out(nq);
    for (uint64_t i = 0; i < nq; ++i) {
        for (uint32_t j = 0; j < n_out[i]; ++j) out[i].results.push_back({ids[i * sp.K + j], sq[i * sp.K + j]});
        out[i].stats.exact_dist_count = st[i].exact_dist_count;
        out[i].stats.test_count = st[i].test_count;
        out[i].stats.pass_count = st[i].pass_count;
        out[i].stats.visited_count = st[i].visited_count;
    }
    return out;
}

// The search step of insert_with_state (builder.cpp:218-227) for nodes already
// in the index, with the index's own efC / b_build / enable_pes; RobustPrune
// and the reverse edges stay on the CPU.
inline std::vector<SearchResult> construction_search(const GpuIndex& ix, std::span<const uint32_t> nodes,
                                                     uint32_t pes_cap = 256) {
    const uint64_t nn = nodes.size();
    const uint32_t efC = ix.efC();
    std::vector<uint32_t> ids(nn * efC), n_out(nn), pes(nn * pes_cap), pes_n(nn);
    std::vector<float> sq(nn * efC);
    std::vector<pag_search_stats> st(nn);
    gpu_check(pag_gpu_construction_search(ix.handle(), nodes.data(), nn, nullptr, -1, ids.data(), sq.data(),
                                          n_out.data(), st.data(), pes.data(), pes_cap, pes_n.data()));
    std::vector<SearchResult> out(nn);
    for (uint64_t i = 0; i < nn; ++i) {
        for (uint32_t j = 0; j < n_out[i]; ++j) out[i].results.push_back({ids[i * efC + j], sq[i * efC + j]});
        if (pes_n[i] > pes_cap) throw std::runtime_error("pes_rejected list truncated");
        out[i].pes_rejected.assign(pes.begin() + i * pes_cap, pes.begin() + i * pes_cap + pes_n[i]);
        out[i].stats.exact_dist_count = st[i].exact_dist_count;
        out[i].stats.test_count = st[i].test_count;
        out[i].stats.pass_count = st[i].pass_count;
        out[i].stats.visited_count = st[i].visited_count;
    }
    return out;
}

}  // namespace pag
