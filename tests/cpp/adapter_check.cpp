// adapter_check.cpp — TEST PROGRAM: a compiled C++ consumer of the drop-in
// boundary. It includes the adapter include/pag_gpu.hpp (which includes the
// reference's own headers, pag/routing.hpp) exactly as a maintainer of the
// reference would, and checks in one process, on the same PAGIDX01 file and
// queries, that pag::search_batch on the GPU equals the reference library's
// pag::search (proj/src/routing.cpp:249-261) bit for bit, that the
// construction search equals search_padded with the build parameters
// (builder.cpp:218-227), that a GpuIndex opened straight from the in-memory
// PagIndex (pag_gpu_open_from_arrays) searches like the one opened from the
// file, that after insert_online batches on the PagIndex a refresh from
// memory (pag_gpu_refresh_from_arrays) makes the GPU search equal the
// reference's search of the extended index, and that errors surface as the
// reference's exception classes. Built by tests/cpp/Makefile into oracle/_ref/ (it
// links the reference objects compiled from /root/reference/proj/src).
//
// usage: adapter_check <index.pagidx> <queries.fvecs> <K> <efS>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pag/builder.hpp"
#include "pag/routing.hpp"
#include "pag_gpu.hpp"

static std::vector<float> read_fvecs(const char* path, uint32_t* dim) {
    std::ifstream f(path, std::ios::binary);
    std::vector<float> out;
    int32_t d = 0;
    while (f.read(reinterpret_cast<char*>(&d), 4)) {
        const size_t o = out.size();
        out.resize(o + d);
        f.read(reinterpret_cast<char*>(out.data() + o), 4ull * d);
    }
    *dim = static_cast<uint32_t>(d);
    return out;
}

static bool same(const pag::SearchResult& a, const pag::SearchResult& b, bool pes) {
    if (a.results.size() != b.results.size()) return false;
    for (size_t i = 0; i < a.results.size(); ++i) {
        uint32_t x, y;
        std::memcpy(&x, &a.results[i].sq, 4);
        std::memcpy(&y, &b.results[i].sq, 4);
        if (a.results[i].id != b.results[i].id || x != y) return false;
    }
    if (a.stats.exact_dist_count != b.stats.exact_dist_count || a.stats.test_count != b.stats.test_count ||
        a.stats.pass_count != b.stats.pass_count || a.stats.visited_count != b.stats.visited_count)
        return false;
    return !pes || a.pes_rejected == b.pes_rejected;
}

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: adapter_check index queries K efS\n");
        return 2;
    }
    uint32_t d = 0;
    const std::vector<float> qs = read_fvecs(argv[2], &d);
    const size_t nq = qs.size() / d;
    pag::SearchParams sp;
    sp.K = static_cast<uint32_t>(std::stoul(argv[3]));
    sp.efS = static_cast<uint32_t>(std::stoul(argv[4]));

    const pag::PagIndex ref = pag::load_index(argv[1]);
    pag::GpuIndex gpu(argv[1]);
    // queries: GPU batch vs the reference's per-query search
    const auto got = pag::search_batch(gpu, qs, sp);
    size_t q_equal = 0;
    pag::TfbState state;
    for (size_t i = 0; i < nq; ++i)
        q_equal += same(got[i], pag::search(ref, std::span<const float>(qs.data() + i * d, d), sp, state), false);
    // construction: insert_with_state's search for every 7th node
    std::vector<uint32_t> nodes;
    for (uint32_t v = 0; v < ref.size(); v += 7) nodes.push_back(v);
    const auto cons = pag::construction_search(gpu, nodes);
    pag::SearchParams bp;
    bp.K = bp.efS = ref.params().efC;
    bp.b_override = ref.params().b_build;
    bp.collect_pes = ref.params().enable_pes;
    size_t c_equal = 0;
    for (size_t i = 0; i < nodes.size(); ++i)
        c_equal += same(cons[i], pag::search_padded(ref, ref.vectors().row(nodes[i]), bp, state), true);
    // the in-memory PagIndex as the source: same results as the file-based handle
    pag::PagIndex live = pag::load_index(argv[1]);
    pag::GpuIndex mem(live);
    const auto got_mem = pag::search_batch(mem, qs, sp);
    size_t a_equal = 0;
    for (size_t i = 0; i < nq; ++i) a_equal += same(got_mem[i], got[i], false);
    // online inserts on the PagIndex (builder.cpp:354-363), two batches, then a
    // refresh from memory; the GPU must search the extended index like the reference
    size_t r_equal = 0, r_total = 0;
    {
        pag::PesSet pes;
        const size_t per_batch = std::min<size_t>(nq / 2, 12);
        size_t next = 0;
        for (int batch = 0; batch < 2; ++batch) {
            for (size_t i = 0; i < per_batch; ++i, ++next) {
                std::vector<float> x(qs.begin() + next * d, qs.begin() + (next + 1) * d);
                for (auto& v : x) v = v * 0.75f + 0.01f * static_cast<float>(i + 1);  // not a duplicate of a query
                pag::insert_online(live, x, pes);
            }
            mem.refresh(live);
            const auto after = pag::search_batch(mem, qs, sp);
            for (size_t i = 0; i < nq; ++i, ++r_total)
                r_equal += same(after[i], pag::search(live, std::span<const float>(qs.data() + i * d, d), sp, state),
                                false);
        }
        if (mem.size() != live.size()) r_equal = 0;
    }
    // errors: the reference's exception classes and texts
    bool err_ok = false;
    try {
        pag::SearchParams bad = sp;
        bad.K = bad.efS + 1;
        pag::search_batch(gpu, std::span<const float>(qs.data(), d), bad);
    } catch (const std::invalid_argument& e) {
        err_ok = std::string(e.what()) == "K > efS";
    }
    bool open_ok = false;
    try {
        pag::GpuIndex missing("/nonexistent/pag.bin");
    } catch (const std::runtime_error& e) {
        open_ok = std::string(e.what()).find("cannot open index") == 0;
    }
    std::printf("{\"queries\": %zu, \"queries_equal\": %zu, \"nodes\": %zu, \"nodes_equal\": %zu, "
                "\"from_arrays_equal\": %zu, \"after_refresh\": %zu, \"after_refresh_equal\": %zu, "
                "\"k_gt_efs_invalid_argument\": %s, \"open_runtime_error\": %s}\n",
                nq, q_equal, nodes.size(), c_equal, a_equal, r_total, r_equal, err_ok ? "true" : "false",
                open_ok ? "true" : "false");
    return (q_equal == nq && c_equal == nodes.size() && a_equal == nq && r_equal == r_total && err_ok && open_ok)
               ? 0
               : 1;
}
