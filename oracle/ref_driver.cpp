// ref_driver.cpp — TEST INFRASTRUCTURE. A small command-line driver around
// the UNMODIFIED reference library, compiled from its own sources under
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/pag_ref.
// The reference's own CLI (proj/tools/pag_cli.cpp) cannot build here
// (CLI11.hpp is absent), so this plays the roles of its gen / build /
// search / ground-truth subcommands (pag_cli.cpp:200-300) and of
// run_benchmark's timing protocol (bench.cpp:151-190).
//
// Only tests/, __graft_entry__ and bench.py (cpu_baseline / --impl reference)
// execute this binary, and only as the checker or the reported CPU baseline.

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pag/bench.hpp"
#include "pag/builder.hpp"
#include "pag/projection.hpp"
#include "pag/routing.hpp"
#include "pag/vecstore.hpp"

using namespace pag;
using clk = std::chrono::steady_clock;

namespace {

struct Args {
    std::vector<std::string> pos;
    std::vector<std::pair<std::string, std::string>> kv;
    std::string get(const std::string& k, const std::string& def = "") const {
        for (auto& p : kv)
            if (p.first == k) return p.second;
        return def;
    }
    bool has(const std::string& k) const {
        for (auto& p : kv)
            if (p.first == k) return true;
        return false;
    }
};

Args parse(int argc, char** argv, int start) {
    Args a;
    for (int i = start; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) == 0) {
            std::string k = s.substr(2), v = "1";
            auto eq = k.find('=');
            if (eq != std::string::npos) {
                v = k.substr(eq + 1);
                k = k.substr(0, eq);
            }
            a.kv.emplace_back(k, v);
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

// raw fvecs rows (no normalisation: search() applies the reference's own
// query preparation, routing.cpp:249-261)
std::vector<float> read_fvecs_raw(const std::string& path, uint32_t* dim, size_t* n) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open " + path);
    std::vector<float> out;
    int32_t d = 0;
    size_t rows = 0;
    while (true) {
        int32_t dd;
        if (std::fread(&dd, 4, 1, f) != 1) break;
        if (rows == 0) d = dd;
        if (dd != d || dd <= 0) throw std::runtime_error("bad fvecs record");
        size_t off = out.size();
        out.resize(off + static_cast<size_t>(d));
        if (std::fread(out.data() + off, 4, static_cast<size_t>(d), f) != static_cast<size_t>(d))
            throw std::runtime_error("truncated fvecs");
        ++rows;
    }
    std::fclose(f);
    *dim = static_cast<uint32_t>(d);
    *n = rows;
    return out;
}

MetricKind metric_of(const std::string& s) {
    return s == "cosine" ? MetricKind::cosine : MetricKind::euclidean;
}

void write_all(std::FILE* f, const void* p, size_t n) {
    if (std::fwrite(p, 1, n, f) != n) throw std::runtime_error("write failed");
}

int cmd_gen_synthetic(const Args& a) {
    // pag gen (pag_cli.cpp:200-204)
    SyntheticKind kind =
        a.get("kind", "gaussian") == "clustered" ? SyntheticKind::clustered : SyntheticKind::gaussian;
    size_t n = std::stoull(a.get("n"));
    uint32_t d = static_cast<uint32_t>(std::stoul(a.get("d")));
    uint64_t seed = std::stoull(a.get("seed", "42"));
    VectorSet vs = gen_synthetic(kind, n, d, seed, metric_of(a.get("metric", "euclidean")));
    save_fvecs(a.get("out"), vs);
    return 0;
}

int cmd_build(const Args& a) {
    // pag build (pag_cli.cpp:206-218)
    VectorSet vs =
        load_vectors(a.get("data"), VecFormat::fvecs, metric_of(a.get("metric", "euclidean")));
    BuildParams bp;
    if (a.has("M")) bp.M = std::stoul(a.get("M"));
    if (a.has("efC")) bp.efC = std::stoul(a.get("efC"));
    if (a.has("L")) bp.L = std::stoul(a.get("L"));
    if (a.has("m")) bp.m = std::stoul(a.get("m"));
    if (a.has("b_build")) bp.b_build = std::stoul(a.get("b_build"));
    if (a.has("seed")) bp.seed = std::stoull(a.get("seed"));
    if (a.has("no-pes")) bp.enable_pes = false;
    unsigned threads = static_cast<unsigned>(std::stoul(a.get("threads", "1")));
    auto t0 = clk::now();
    PagIndex index = build(std::move(vs), bp, threads);
    double s = std::chrono::duration<double>(clk::now() - t0).count();
    save_index(index, a.get("out"));
    size_t edges = 0;
    for (uint32_t u = 0; u < index.size(); ++u) edges += index.degree(u);
    std::printf("{\"build_seconds\": %.3f, \"nodes\": %u, \"edges\": %zu, \"threads\": %u}\n", s,
                index.size(), edges, threads);
    return 0;
}

// search over a query file (the roles of pag_cli.cpp:244-266 and
// run_benchmark's timing, bench.cpp:151-190). --efS takes a comma list; per
// efS: one untimed warm sweep, `reps` timed sweeps with `threads` threads
// (one TfbState per thread, atomic query counter), optionally a 1-thread
// warm + timed sweep over the first `single-limit` queries, and with --out
// the results (suffix ".efS<e>" when several efS are given; --single-efS
// restricts the 1-thread timing to one of them). One JSON line per efS.
int cmd_search(const Args& a) {
    PagIndex index = load_index(a.get("index"));
    uint32_t d;
    size_t nq;
    std::vector<float> qs = read_fvecs_raw(a.get("queries"), &d, &nq);
    if (a.has("limit")) nq = std::min<size_t>(nq, std::stoull(a.get("limit")));
    std::vector<uint32_t> efs_list;
    {
        std::string e = a.get("efS", "100");
        size_t p = 0;
        while (p <= e.size()) {
            size_t c = e.find(',', p);
            if (c == std::string::npos) c = e.size();
            if (c > p) efs_list.push_back(static_cast<uint32_t>(std::stoul(e.substr(p, c - p))));
            p = c + 1;
        }
    }
    SearchParams sp;
    sp.K = std::stoul(a.get("K", "10"));
    if (a.has("b")) sp.b_override = std::stoul(a.get("b"));
    sp.use_prt = !a.has("no-prt");
    sp.use_tfb = !a.has("no-tfb");
    unsigned threads = static_cast<unsigned>(std::stoul(a.get("threads", "1")));
    int reps = std::stoi(a.get("reps", "1"));
    const size_t single = a.has("single-limit") ? std::min<size_t>(nq, std::stoull(a.get("single-limit"))) : 0;
    const uint32_t K = sp.K;

    std::vector<uint32_t> ids(nq * K, 0xFFFFFFFFu);
    std::vector<float> sq(nq * K, 0.0f);
    std::vector<uint32_t> nout(nq, 0);
    std::vector<uint64_t> st(nq * 4, 0);

    auto run_one = [&](size_t qi, TfbState& state) {
        std::span<const float> q(qs.data() + qi * d, d);
        SearchResult r = search(index, q, sp, state);
        nout[qi] = static_cast<uint32_t>(r.results.size());
        for (size_t i = 0; i < r.results.size(); ++i) {
            ids[qi * K + i] = r.results[i].id;
            sq[qi * K + i] = r.results[i].sq;
        }
        st[qi * 4 + 0] = r.stats.exact_dist_count;
        st[qi * 4 + 1] = r.stats.test_count;
        st[qi * 4 + 2] = r.stats.pass_count;
        st[qi * 4 + 3] = r.stats.visited_count;
    };
    auto sweep = [&](unsigned nth, size_t count) {
        if (nth <= 1) {
            TfbState state;
            for (size_t qi = 0; qi < count; ++qi) run_one(qi, state);
        } else {
            std::atomic<size_t> next{0};
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < nth; ++t)
                pool.emplace_back([&] {
                    TfbState state;
                    size_t qi;
                    while ((qi = next.fetch_add(1)) < count) run_one(qi, state);
                });
            for (auto& th : pool) th.join();
        }
    };
    auto timed = [&](unsigned nth, size_t count) {
        auto t0 = clk::now();
        sweep(nth, count);
        return std::chrono::duration<double>(clk::now() - t0).count();
    };
    for (uint32_t efS : efs_list) {
        sp.efS = efS;
        // one untimed warm sweep, then timed sweeps (bench.cpp:161-188)
        if (!a.has("no-warm")) sweep(threads, nq);
        double best = 1e30, total = 0;
        for (int r = 0; r < reps; ++r) {
            const double s = timed(threads, nq);
            total += s;
            best = std::min(best, s);
        }
        if (a.has("out")) {
            std::string path = a.get("out");
            if (efs_list.size() > 1) path += ".efS" + std::to_string(efS);
            std::FILE* f = std::fopen(path.c_str(), "wb");
            if (!f) throw std::runtime_error("cannot open output");
            uint64_t hdr[2] = {nq, K};
            write_all(f, hdr, sizeof hdr);
            write_all(f, ids.data(), ids.size() * 4);
            write_all(f, sq.data(), sq.size() * 4);
            write_all(f, nout.data(), nout.size() * 4);
            write_all(f, st.data(), st.size() * 8);
            std::fclose(f);
        }
        double s1 = 0;
        const bool single_here = single && (!a.has("single-efS") || std::stoul(a.get("single-efS")) == efS);
        if (single_here) {
            sweep(1, single);  // warm
            s1 = timed(1, single);
        }
        std::printf(
            "{\"efS\": %u, \"queries\": %zu, \"threads\": %u, \"reps\": %d, \"seconds_mean\": %.6f, "
            "\"seconds_best\": %.6f, \"qps\": %.3f, \"single_queries\": %zu, \"single_qps\": %.3f}\n",
            efS, nq, threads, reps, total / std::max(1, reps), best, reps ? nq / (total / reps) : 0.0,
            single_here ? single : 0, single_here ? single / s1 : 0.0);
        std::fflush(stdout);
    }
    return 0;
}

// insert_with_state's search (builder.cpp:218-227) over a saved index: the
// query of node v is its stored padded row, K = efS = efC, b = b_build,
// collect_pes = enable_pes (each overridable). Nodes are (i * stride) % n.
int cmd_build_search(const Args& a) {
    PagIndex index = load_index(a.get("index"));
    const BuildParams& bp = index.params();
    const size_t n = index.size();
    const size_t count = std::stoull(a.get("count", "100"));
    const size_t stride = std::stoull(a.get("stride", "1"));
    SearchParams sp;
    sp.K = std::stoul(a.get("K", std::to_string(bp.efC)));
    sp.efS = std::stoul(a.get("efS", std::to_string(bp.efC)));
    sp.b_override = std::stoul(a.get("b", std::to_string(bp.b_build)));
    sp.collect_pes = a.has("pes") ? a.get("pes") == "1" : bp.enable_pes;
    const uint32_t pes_cap = std::stoul(a.get("pes-cap", "256"));
    unsigned threads = static_cast<unsigned>(std::stoul(a.get("threads", "1")));
    int reps = std::stoi(a.get("reps", "1"));
    const uint32_t K = sp.K;
    std::vector<uint32_t> nodes(count);
    for (size_t i = 0; i < count; ++i) nodes[i] = static_cast<uint32_t>((i * stride) % n);
    std::vector<uint32_t> ids(count * K, 0xFFFFFFFFu), nout(count, 0), pes(count * pes_cap, 0), pes_n(count, 0);
    std::vector<float> sq(count * K, 0.0f);
    std::vector<uint64_t> st(count * 4, 0);
    auto run_one = [&](size_t i, TfbState& state) {
        SearchResult r = search_padded(index, index.vectors().row(nodes[i]), sp, state);
        nout[i] = static_cast<uint32_t>(r.results.size());
        for (size_t j = 0; j < r.results.size(); ++j) {
            ids[i * K + j] = r.results[j].id;
            sq[i * K + j] = r.results[j].sq;
        }
        st[i * 4 + 0] = r.stats.exact_dist_count;
        st[i * 4 + 1] = r.stats.test_count;
        st[i * 4 + 2] = r.stats.pass_count;
        st[i * 4 + 3] = r.stats.visited_count;
        pes_n[i] = static_cast<uint32_t>(r.pes_rejected.size());
        for (size_t j = 0; j < r.pes_rejected.size() && j < pes_cap; ++j) pes[i * pes_cap + j] = r.pes_rejected[j];
    };
    auto sweep = [&]() {
        std::atomic<size_t> next{0};
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < std::max(1u, threads); ++t)
            pool.emplace_back([&] {
                TfbState state;
                size_t i;
                while ((i = next.fetch_add(1)) < count) run_one(i, state);
            });
        for (auto& th : pool) th.join();
    };
    if (!a.has("no-warm")) sweep();
    double total = 0;
    for (int r = 0; r < reps; ++r) {
        auto t0 = clk::now();
        sweep();
        total += std::chrono::duration<double>(clk::now() - t0).count();
    }
    if (a.has("out")) {
        std::FILE* f = std::fopen(a.get("out").c_str(), "wb");
        if (!f) throw std::runtime_error("cannot open output");
        uint64_t hdr[3] = {count, K, pes_cap};
        write_all(f, hdr, sizeof hdr);
        write_all(f, ids.data(), ids.size() * 4);
        write_all(f, sq.data(), sq.size() * 4);
        write_all(f, nout.data(), nout.size() * 4);
        write_all(f, st.data(), st.size() * 8);
        write_all(f, pes_n.data(), pes_n.size() * 4);
        write_all(f, pes.data(), pes.size() * 4);
        std::fclose(f);
    }
    std::printf("{\"nodes\": %zu, \"threads\": %u, \"reps\": %d, \"seconds_mean\": %.6f, \"qps\": %.3f}\n",
                count, threads, reps, total / std::max(1, reps), reps ? count / (total / reps) : 0.0);
    return 0;
}

int cmd_gt(const Args& a) {
    MetricKind metric = metric_of(a.get("metric", "euclidean"));
    VectorSet base = load_vectors(a.get("base"), VecFormat::fvecs, metric);
    VectorSet queries = load_vectors(a.get("queries"), VecFormat::fvecs, metric);
    uint32_t k = std::stoul(a.get("k", "10"));
    unsigned threads = static_cast<unsigned>(std::stoul(a.get("threads", "1")));
    GroundTruth gt = ground_truth(base, queries, k, threads);
    std::FILE* f = std::fopen(a.get("out").c_str(), "wb");
    if (!f) throw std::runtime_error("cannot open output");
    uint64_t hdr[2] = {gt.rows.size(), gt.k_star};
    write_all(f, hdr, sizeof hdr);
    for (auto& row : gt.rows)
        for (auto& c : row) write_all(f, &c.id, 4);
    for (auto& row : gt.rows)
        for (auto& c : row) write_all(f, &c.sq, 4);
    std::fclose(f);
    return 0;
}

int cmd_refs(const Args& a) {
    PagIndex index = load_index(a.get("index"));
    const ReferenceSet& rs = index.refs();
    std::FILE* f = std::fopen(a.get("out").c_str(), "wb");
    if (!f) throw std::runtime_error("cannot open output");
    uint64_t hdr[4] = {rs.L, rs.m, rs.sub_dim, index.entry_nodes().size()};
    write_all(f, hdr, sizeof hdr);
    write_all(f, rs.refs.data(), rs.refs.size() * 4);
    write_all(f, index.entry_nodes().data(), index.entry_nodes().size() * 4);
    std::fclose(f);
    return 0;
}

int cmd_tables(const Args& a) {
    // per-query projection tables after the search() query preparation
    PagIndex index = load_index(a.get("index"));
    uint32_t d;
    size_t nq;
    std::vector<float> qs = read_fvecs_raw(a.get("queries"), &d, &nq);
    const VectorSet& vs = index.vectors();
    std::FILE* f = std::fopen(a.get("out").c_str(), "wb");
    if (!f) throw std::runtime_error("cannot open output");
    uint64_t hdr[3] = {nq, index.refs().L, index.refs().m};
    write_all(f, hdr, sizeof hdr);
    std::vector<float> qbuf;
    for (size_t qi = 0; qi < nq; ++qi) {
        qbuf.assign(vs.padded_dim(), 0.0f);
        std::memcpy(qbuf.data(), qs.data() + qi * d, d * 4);
        if (vs.metric() == MetricKind::cosine) {
            float nrm = vec_norm(qbuf.data(), vs.padded_dim());
            for (auto& x : qbuf) x /= nrm;
        }
        ProjectionTable t = build_projection_table(qbuf.data(), index.refs());
        write_all(f, t.entries.data(), t.entries.size() * 4);
    }
    std::fclose(f);
    return 0;
}

int cmd_insert(const Args& a) {
    // online insertion phases (the insert-bench loop, pag_cli.cpp:327-366):
    // one PesSet across batches; after each batch the index is saved as
    // <out-prefix>.<b>.pagidx (written to a temp name, then renamed) so a
    // reader can refresh from it while the next batch is being inserted.
    PagIndex index = load_index(a.get("index"));
    uint32_t d;
    size_t n_ins;
    std::vector<float> xs = read_fvecs_raw(a.get("data"), &d, &n_ins);
    if (d != index.vectors().dim()) throw std::runtime_error("insert dimension mismatch");
    const uint32_t batches = std::stoul(a.get("batches", "1"));
    const size_t per_batch = n_ins / batches;
    const std::string prefix = a.get("out-prefix");
    index.reserve(index.size() + per_batch * batches);
    PesSet pes;
    for (uint32_t b = 0; b < batches; ++b) {
        auto t0 = clk::now();
        for (size_t i = b * per_batch; i < (b + 1) * per_batch; ++i)
            insert_online(index, std::span<const float>(xs.data() + i * d, d), pes);
        const double ins_s = std::chrono::duration<double>(clk::now() - t0).count();
        const std::string path = prefix + "." + std::to_string(b) + ".pagidx";
        save_index(index, path + ".tmp");
        std::rename((path + ".tmp").c_str(), path.c_str());
        std::printf("{\"batch\": %u, \"n_indexed\": %u, \"insert_seconds\": %.3f, \"path\": \"%s\"}\n", b,
                    index.size(), ins_s, path.c_str());
        std::fflush(stdout);
    }
    return 0;
}

int cmd_sqdist(const Args& a) {
    // sq_dist of query rows against listed base rows, for the distance KATs
    PagIndex index = load_index(a.get("index"));
    uint32_t d;
    size_t nq;
    std::vector<float> qs = read_fvecs_raw(a.get("queries"), &d, &nq);
    const VectorSet& vs = index.vectors();
    std::FILE* f = std::fopen(a.get("out").c_str(), "wb");
    std::vector<float> qbuf(vs.padded_dim());
    for (size_t qi = 0; qi < nq; ++qi) {
        std::fill(qbuf.begin(), qbuf.end(), 0.0f);
        std::memcpy(qbuf.data(), qs.data() + qi * d, d * 4);
        for (uint32_t i = 0; i < index.size(); ++i) {
            float s = sq_dist(vs.row(i), qbuf.data(), vs.padded_dim());
            write_all(f, &s, 4);
        }
    }
    std::fclose(f);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr,
                     "usage: pag_ref {gen-synthetic|build|search|build-search|gt|refs|tables|sqdist|insert} "
                     "--key=value ...\n");
        return 2;
    }
    std::string cmd = argv[1];
    Args a = parse(argc, argv, 2);
    try {
        if (cmd == "gen-synthetic") return cmd_gen_synthetic(a);
        if (cmd == "build") return cmd_build(a);
        if (cmd == "search") return cmd_search(a);
        if (cmd == "gt") return cmd_gt(a);
        if (cmd == "refs") return cmd_refs(a);
        if (cmd == "tables") return cmd_tables(a);
        if (cmd == "sqdist") return cmd_sqdist(a);
        if (cmd == "insert") return cmd_insert(a);
        if (cmd == "build-search") return cmd_build_search(a);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
}
