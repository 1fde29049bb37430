// ref_driver.cpp -- C entry points over the UNMODIFIED reference (featdrive)
// headers, compiled from /root/reference/proj/include into oracle/_ref/libfdref.so
// by oracle/Makefile.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by tests/ to pin the C
// restatement (fd_oracle.c) and to produce tests/golden/, and by bench.py's
// cpu_baseline and --impl reference legs to time the reference's own CPU code.
// No reference source is copied here; this file only calls the reference API.
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <optional>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "featdrive/common.hpp"
#include "featdrive/extract/extractor.hpp"
#include "featdrive/featbuf/buffer_manager.hpp"
#include "featdrive/featbuf/device_region.hpp"
#include "featdrive/graph/sampling.hpp"
#include "featdrive/graph/topology.hpp"
#include "featdrive/pipeline/pipeline.hpp"
#include <system_error>

#include "featdrive/storage/feature_file.hpp"
#include "featdrive/storage/generator.hpp"

using namespace featdrive;

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;  // exception category of the last failure (fdref_last_error_kind)
thread_local int g_sys_errno = 0;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// 1 std::system_error (errno in g_sys_errno), 2 other std::runtime_error, 3 std::invalid_argument,
// 4 std::out_of_range, 5 other std::logic_error, 9 anything else.
void record(const std::exception& e) {
    g_err = e.what();
    g_sys_errno = 0;
    if (auto* se = dynamic_cast<const std::system_error*>(&e)) {
        g_kind = 1;
        g_sys_errno = se->code().value();
    } else if (dynamic_cast<const std::runtime_error*>(&e)) {
        g_kind = 2;
    } else if (dynamic_cast<const std::invalid_argument*>(&e)) {
        g_kind = 3;
    } else if (dynamic_cast<const std::out_of_range*>(&e)) {
        g_kind = 4;
    } else if (dynamic_cast<const std::logic_error*>(&e)) {
        g_kind = 5;
    } else {
        g_kind = 9;
    }
}

// Map the reference's exception types onto the status codes used by the C ABI.
template <typename Fn>
int guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const std::out_of_range& e) {
        return fail(1, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(2, e.what());
    } catch (const InvariantViolation& e) {
        return fail(3, e.what());
    } catch (const featbuf::StandbyTimeout& e) {
        return fail(6, e.what());
    } catch (const std::exception& e) {
        return fail(9, e.what());
    }
}

struct ExtractHandle {
    std::unique_ptr<storage::FeatureTable> table;
    std::unique_ptr<featbuf::BufferManager> buffer;
    std::unique_ptr<featbuf::StagingArena> staging;
    std::unique_ptr<featbuf::FeatureRegion> region;
    std::unique_ptr<featbuf::CopyEngine> copies;
    pipeline::StageCounters counters;
    extract::TestHooks hooks;
    std::unique_ptr<extract::Extractor> extractor;
};

}  // namespace

extern "C" {

const char* fdref_last_error() { return g_err.c_str(); }
int fdref_last_error_kind() { return g_kind; }
int fdref_last_errno() { return g_sys_errno; }

// storage::FeatureTable(path) alone (feature_file.hpp:27-51): 0 on success, else the
// exception is recorded (fdref_last_error / _kind / _errno).
int fdref_feature_table_check(const char* path) {
    try {
        storage::FeatureTable t(path);
        return 0;
    } catch (const std::exception& e) {
        record(e);
        return 9;
    }
}

uint64_t fdref_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t fdref_hash_combine(uint64_t a, uint64_t b) { return hash_combine(a, b); }
uint64_t fdref_hash_bytes64(const void* p, uint64_t n) {
    return hash_bytes64(std::span<const std::byte>(static_cast<const std::byte*>(p), n));
}
uint64_t fdref_batch_seed(uint64_t seed, uint64_t epoch, uint64_t b) {
    return pipeline::PipelineSession::batch_seed(seed, epoch, b);
}

// Engine words exactly as sample_khop seeds them (sampling.hpp:78).
void fdref_mt_stream(uint64_t rng_seed, uint64_t n, uint64_t* out) {
    std::mt19937_64 rng(splitmix64(rng_seed));
    for (uint64_t i = 0; i < n; ++i) out[i] = rng();
}

// Sequence of uniform_int_distribution<u64>(0, js[i]) draws on that engine.
void fdref_uniform_seq(uint64_t rng_seed, const uint64_t* js, uint64_t n, uint64_t* out) {
    std::mt19937_64 rng(splitmix64(rng_seed));
    for (uint64_t i = 0; i < n; ++i) out[i] = std::uniform_int_distribution<std::uint64_t>(0, js[i])(rng);
}

// ---- generator (storage/generator.hpp) -------------------------------------
void fdref_synthetic_row(uint64_t seed, uint64_t node, uint32_t dim, void* out) {
    storage::synthetic_row(seed, node, dim, std::span<std::byte>(static_cast<std::byte*>(out), dim * 4u));
}
uint64_t fdref_synthetic_in_degree(uint64_t seed, uint64_t node, uint32_t avg, uint64_t n) {
    return storage::synthetic_in_degree(seed, node, avg, n);
}
uint64_t fdref_synthetic_in_neighbors(uint64_t seed, uint64_t node, uint32_t avg, uint64_t n, uint64_t* out) {
    auto v = storage::synthetic_in_neighbors(seed, node, avg, n);
    std::memcpy(out, v.data(), v.size() * 8);
    return v.size();
}
int fdref_generate_dataset(const char* dir, uint64_t num_nodes, uint32_t dim, uint32_t avg, uint64_t seed,
                           uint64_t* num_edges) {
    return guarded([&] {
        storage::GeneratorParams p;
        p.num_nodes = num_nodes;
        p.dim = dim;
        p.avg_degree = avg;
        p.seed = seed;
        p.out_dir = dir;
        auto m = storage::create_synthetic_dataset(p);
        *num_edges = m.num_edges;
        return 0;
    });
}

// Multi-threaded driver over the reference's per-node generator functions (all
// pure functions of (seed, node), generator.hpp:65-121), filling caller memory
// (e.g. numpy memmaps of indptr.bin / indices.bin in /dev/shm). Byte-identical to
// create_synthetic_dataset's files; used to stage Papers-scale CPU baselines.
extern "C++" template <typename Fn>
void parallel_nodes(uint64_t n, uint32_t threads, Fn&& fn) {
    std::vector<std::thread> pool;
    std::atomic<uint64_t> next{0};
    const uint64_t chunk = 1 << 14;
    for (uint32_t t = 0; t < std::max<uint32_t>(threads, 1); ++t)
        pool.emplace_back([&] {
            for (;;) {
                uint64_t lo = next.fetch_add(chunk);
                if (lo >= n) return;
                uint64_t hi = std::min(n, lo + chunk);
                for (uint64_t v = lo; v < hi; ++v) fn(v);
            }
        });
    for (auto& th : pool) th.join();
}

void fdref_gen_indptr(uint64_t seed, uint64_t n, uint32_t avg, uint32_t threads, uint64_t* indptr) {
    parallel_nodes(n, threads, [&](uint64_t v) { indptr[v + 1] = storage::synthetic_in_degree(seed, v, avg, n); });
    indptr[0] = 0;
    for (uint64_t v = 0; v < n; ++v) indptr[v + 1] += indptr[v];
}

void fdref_gen_indices(uint64_t seed, uint64_t n, uint32_t avg, uint32_t threads, const uint64_t* indptr,
                       uint64_t* indices) {
    parallel_nodes(n, threads, [&](uint64_t v) {
        auto nb = storage::synthetic_in_neighbors(seed, v, avg, n);
        std::memcpy(indices + indptr[v], nb.data(), nb.size() * 8);
    });
}

void fdref_gen_features(uint64_t seed, uint64_t n, uint32_t dim, uint32_t threads, void* out) {
    parallel_nodes(n, threads, [&](uint64_t v) {
        storage::synthetic_row(seed, v, dim,
                               std::span<std::byte>(static_cast<std::byte*>(out) + v * dim * 4ull, dim * 4ull));
    });
}

// ---- graph (graph/topology.hpp, graph/sampling.hpp) ------------------------
void* fdref_topology_open(const char* dir) {
    try {
        return new graph::Topology(dir);
    } catch (const std::exception& e) {
        record(e);
        return nullptr;
    }
}
void fdref_topology_close(void* t) { delete static_cast<graph::Topology*>(t); }
uint64_t fdref_topology_num_nodes(void* t) { return static_cast<graph::Topology*>(t)->num_nodes(); }
uint64_t fdref_topology_num_edges(void* t) { return static_cast<graph::Topology*>(t)->num_edges(); }

int fdref_sample_khop(void* topo, const uint64_t* seeds, uint64_t n_seeds, const uint32_t* fanouts,
                      uint32_t n_layers, uint64_t rng_seed, uint64_t* nodes, uint64_t nodes_cap,
                      uint32_t* edges, uint64_t edges_cap, uint64_t* n_nodes, uint64_t* n_edges) {
    return guarded([&] {
        graph::Fanouts f;
        f.per_layer.assign(fanouts, fanouts + n_layers);
        auto b = graph::sample_khop(*static_cast<graph::Topology*>(topo),
                                    std::span<const NodeId>(seeds, n_seeds), f, rng_seed);
        *n_nodes = b.nodes.size();
        *n_edges = b.edges.size();
        if (b.nodes.size() > nodes_cap || b.edges.size() > edges_cap) return fail(4, "capacity");
        std::memcpy(nodes, b.nodes.data(), b.nodes.size() * 8);
        for (std::size_t i = 0; i < b.edges.size(); ++i) {
            edges[2 * i] = b.edges[i].src;
            edges[2 * i + 1] = b.edges[i].dst;
        }
        return 0;
    });
}

// partition_epoch (sampling.hpp:57-70), flattened: out[i] = i-th id in shuffled order.
int fdref_partition_epoch(const uint64_t* ids, uint64_t n, uint64_t batch_size, uint64_t shuffle_seed,
                          uint64_t* out) {
    return guarded([&] {
        auto chunks = graph::partition_epoch(std::vector<NodeId>(ids, ids + n), batch_size, shuffle_seed);
        uint64_t k = 0;
        for (auto& c : chunks)
            for (auto v : c) out[k++] = v;
        return 0;
    });
}

// ---- buffer manager (featbuf/buffer_manager.hpp) ---------------------------
// Deterministic single-extractor schedule of the metadata protocol run by
// Extractor::run_ticket (extractor.hpp:146-151, 391-394).
void* fdref_bm_create(uint64_t num_nodes, uint64_t slots, uint64_t min_reserved, int mapping) {
    try {
        featbuf::BufferConfig c;
        c.num_nodes = num_nodes;
        c.slot_count = slots;
        c.min_reserved = min_reserved;
        c.mapping = mapping == 1 ? featbuf::MappingKind::Dense
                    : mapping == 2 ? featbuf::MappingKind::Sparse
                                   : featbuf::MappingKind::Auto;
        c.standby_timeout = std::chrono::milliseconds(10);
        return new featbuf::BufferManager(c);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void fdref_bm_destroy(void* bm) { delete static_cast<featbuf::BufferManager*>(bm); }

int fdref_bm_extract(void* h, const uint64_t* nodes, uint64_t n, int64_t* alias) {
    return guarded([&] {
        auto& bm = *static_cast<featbuf::BufferManager*>(h);
        auto plan = bm.acquire_for_batch(std::span<const NodeId>(nodes, n));
        for (auto pos : plan.to_load) {
            SlotId s = bm.get_standby_slot();
            bm.bind_slot(nodes[pos], s);
            plan.alias[pos] = s;
        }
        for (auto pos : plan.to_load) bm.publish_valid(nodes[pos]);
        if (!plan.waits.empty()) return fail(3, "waits under a sequential schedule");
        std::memcpy(alias, plan.alias.data(), n * 8);
        return 0;
    });
}
int fdref_bm_release(void* h, const uint64_t* nodes, uint64_t n) {
    return guarded([&] {
        static_cast<featbuf::BufferManager*>(h)->release_batch(std::span<const NodeId>(nodes, n));
        return 0;
    });
}
void fdref_bm_stats(void* h, uint64_t* out) {
    auto s = static_cast<featbuf::BufferManager*>(h)->stats();
    out[0] = s.hits; out[1] = s.loads; out[2] = s.waits; out[3] = s.evictions;
    out[4] = s.takeovers; out[5] = s.releases; out[6] = s.standby_len;
}
void fdref_bm_entry(void* h, uint64_t node, int64_t* slot, uint32_t* ref, uint32_t* valid) {
    auto e = static_cast<featbuf::BufferManager*>(h)->mapping_entry(node);
    *slot = e.slot_index; *ref = e.ref_count; *valid = e.valid;
}
int64_t fdref_bm_reverse(void* h, uint64_t slot) {
    auto n = static_cast<featbuf::BufferManager*>(h)->reverse_mapping(SlotId(slot));
    return n == ~NodeId(0) ? -1 : int64_t(n);
}
int64_t fdref_bm_standby_mru(void* h) { return static_cast<featbuf::BufferManager*>(h)->standby_mru(); }
int fdref_bm_validate(void* h) {
    return guarded([&] { static_cast<featbuf::BufferManager*>(h)->validate(); return 0; });
}

// ---- real Extractor over an on-disk dataset (extract/extractor.hpp) --------
void* fdref_extractor_open(const char* dir, uint64_t slots, uint64_t min_reserved, int mapping) {
    try {
        auto h = std::make_unique<ExtractHandle>();
        h->table = std::make_unique<storage::FeatureTable>(std::string(dir) + "/features.bin");
        const auto& hd = h->table->header();
        featbuf::BufferConfig c;
        c.num_nodes = hd.num_nodes;
        c.slot_count = slots;
        c.row_bytes = hd.row_bytes;
        c.min_reserved = min_reserved;
        c.mapping = mapping == 1 ? featbuf::MappingKind::Dense
                    : mapping == 2 ? featbuf::MappingKind::Sparse
                                   : featbuf::MappingKind::Auto;
        c.standby_timeout = std::chrono::milliseconds(200);
        h->buffer = std::make_unique<featbuf::BufferManager>(c);
        h->staging = std::make_unique<featbuf::StagingArena>(
            std::max<uint64_t>(slots, 1), hd.aligned_row_bytes(), std::vector<uint64_t>{std::max<uint64_t>(slots, 1)});
        h->region = std::make_unique<featbuf::FeatureRegion>(slots, hd.row_bytes);
        h->copies = std::make_unique<featbuf::CopyEngine>();
        extract::ExtractorEnv env;
        env.table = h->table.get();
        env.buffer = h->buffer.get();
        env.staging = h->staging.get();
        env.region = h->region.get();
        env.copies = h->copies.get();
        env.counters = &h->counters;
        env.hooks = &h->hooks;
        extract::ExtractorConfig ec;
        ec.engine = storage::EngineKind::Threads;
        h->extractor = std::make_unique<extract::Extractor>(env, ec);
        return h.release();
    } catch (const std::exception& e) {
        record(e);
        return nullptr;
    }
}
void fdref_extractor_close(void* h) { delete static_cast<ExtractHandle*>(h); }

// extract_batch + the trainer_step checksum; rows (nullable) receives
// region.slot(alias[i]) for every i, i.e. the mini-batch as the trainer sees it.
int fdref_extractor_extract(void* hv, const uint64_t* nodes, uint64_t n, int64_t* alias, void* rows,
                            uint64_t* checksum) {
    return guarded([&] {
        auto& h = *static_cast<ExtractHandle*>(hv);
        graph::SampledBatch b;
        b.nodes.assign(nodes, nodes + n);
        auto a = h.extractor->extract_batch(b);
        std::memcpy(alias, a.data(), n * 8);
        uint32_t rb = h.table->row_bytes();
        if (rows)
            for (uint64_t i = 0; i < n; ++i)
                std::memcpy(static_cast<std::byte*>(rows) + i * rb, h.region->slot(a[i]).data(), rb);
        pipeline::TrainTicket t{std::move(b), std::move(a)};
        *checksum = pipeline::trainer_step(t, *h.region, h.table.get());
        return 0;
    });
}
int fdref_extractor_release(void* hv, const uint64_t* nodes, uint64_t n) {
    return guarded([&] {
        static_cast<ExtractHandle*>(hv)->buffer->release_batch(std::span<const NodeId>(nodes, n));
        return 0;
    });
}
void fdref_extractor_stats(void* hv, uint64_t* out) {
    auto s = static_cast<ExtractHandle*>(hv)->buffer->stats();
    out[0] = s.hits; out[1] = s.loads; out[2] = s.waits; out[3] = s.evictions;
    out[4] = s.takeovers; out[5] = s.releases; out[6] = s.standby_len;
}

// ---- pipeline (pipeline/pipeline.hpp) --------------------------------------
// run_sync_reference (261-293) or run_epoch (async, 175-257); per-batch records
// out[4*k..] = {batch_id, seed_count, node_count, checksum}. Returns #records.
int64_t fdref_run_epoch(const char* dir, const uint64_t* train_ids, uint64_t n_ids, uint64_t epoch,
                        uint64_t seed, uint64_t batch_size, const uint32_t* fanouts, uint32_t n_layers,
                        int sync_reference, uint32_t samplers, uint32_t extractors, uint64_t* out,
                        uint64_t out_cap, uint64_t* buffer_stats) {
    try {
        pipeline::PipelineConfig cfg;
        cfg.batch_size = batch_size;
        cfg.fanouts.per_layer.assign(fanouts, fanouts + n_layers);
        cfg.num_samplers = samplers;
        cfg.num_extractors = extractors;
        cfg.engine = storage::EngineKind::Threads;
        cfg.verify = true;
        pipeline::PipelineSession s(dir, cfg);
        auto st = sync_reference ? s.run_sync_reference(std::span<const NodeId>(train_ids, n_ids), epoch, seed)
                                 : s.run_epoch(std::span<const NodeId>(train_ids, n_ids), epoch, seed);
        uint64_t k = 0;
        for (auto& r : st.batch_records) {
            if (k >= out_cap) break;
            out[4 * k] = r.batch_id;
            out[4 * k + 1] = r.seed_count;
            out[4 * k + 2] = r.node_count;
            out[4 * k + 3] = r.checksum;
            ++k;
        }
        if (buffer_stats) {
            buffer_stats[0] = st.buffer.hits; buffer_stats[1] = st.buffer.loads;
            buffer_stats[2] = st.buffer.waits; buffer_stats[3] = st.buffer.evictions;
        }
        return int64_t(k);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// ---- CPU baseline: the reference's sample -> extract -> train-checksum path --
// `threads` workers each take whole batches (as the reference's samplers do,
// pipeline.hpp:419-440): graph::sample_khop on the shared read-only Topology,
// then every row is copied into the worker's batch region (the CopyEngine /
// FeatureRegion byte movement, device_region.hpp:60-64) from the host-resident
// table, then hash_bytes64 per row (trainer_step, pipeline.hpp:103-124).
// seeds: n_batches * batch_size ids (chunked as partition_epoch does).
// Returns wall seconds; checksums[b] and node_counts[b] per batch.
double fdref_bench_sample_extract(void* topo, const void* table, uint32_t row_bytes, const uint64_t* seeds,
                                  uint64_t n_batches, uint64_t batch_size, const uint32_t* fanouts,
                                  uint32_t n_layers, uint64_t seed, uint64_t epoch, uint64_t first_batch,
                                  uint32_t threads, uint64_t* checksums, uint64_t* node_counts) {
    auto& t = *static_cast<graph::Topology*>(topo);
    graph::Fanouts f;
    f.per_layer.assign(fanouts, fanouts + n_layers);
    std::atomic<uint64_t> next{0};
    std::atomic<bool> failed{false};
    auto t0 = std::chrono::steady_clock::now();
    auto worker = [&] {
        std::vector<std::byte> region;
        try {
            while (true) {
                uint64_t b = next.fetch_add(1);
                if (b >= n_batches) return;
                auto batch = graph::sample_khop(
                    t, std::span<const NodeId>(seeds + b * batch_size, batch_size), f,
                    pipeline::PipelineSession::batch_seed(seed, epoch, first_batch + b));
                region.resize(batch.nodes.size() * row_bytes);
                uint64_t sum = 0;
                for (std::size_t i = 0; i < batch.nodes.size(); ++i) {
                    const std::byte* src = static_cast<const std::byte*>(table) + batch.nodes[i] * uint64_t(row_bytes);
                    std::memcpy(region.data() + i * row_bytes, src, row_bytes);
                }
                for (std::size_t i = 0; i < batch.nodes.size(); ++i)
                    sum += hash_bytes64(std::span<const std::byte>(region.data() + i * row_bytes, row_bytes));
                checksums[b] = sum;
                node_counts[b] = batch.nodes.size();
            }
        } catch (const std::exception& e) {
            g_err = e.what();
            failed = true;
        }
    };
    std::vector<std::thread> pool;
    for (uint32_t i = 0; i < threads; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return failed ? -1.0 : s;
}

// Config 3 on the CPU: the same sampling fan-out, then the batches in order through ONE
// reference BufferManager (its single mutex serialises these operations in the reference
// anyway): acquire_for_batch, get_standby_slot + bind_slot per miss, the miss rows copied
// table -> region slot, publish_valid, trainer_step's hash over region[alias], and the
// lag-1 release_batch -- the GPU runner's buffer-manager path with the full table as the
// miss source. `bm` (fdref_bm_create) persists across calls, so a warm-up call warms it;
// `region` is slots x row_bytes bytes. Batches are sampled by `threads - 1` workers at
// most 2 x threads ahead of the extraction; `prev_*` carry the unreleased last batch.
double fdref_bench_sample_extract_bm(void* topo, const void* table, uint32_t row_bytes, const uint64_t* seeds,
                                     uint64_t n_batches, uint64_t batch_size, const uint32_t* fanouts,
                                     uint32_t n_layers, uint64_t seed, uint64_t epoch, uint64_t first_batch,
                                     uint32_t threads, void* bm, void* region, uint64_t* checksums,
                                     uint64_t* node_counts) {
    auto& t = *static_cast<graph::Topology*>(topo);
    auto& mgr = *static_cast<featbuf::BufferManager*>(bm);
    static thread_local std::vector<NodeId> held;  // the last extracted batch, released by the next call
    static thread_local void* held_bm = nullptr;
    if (held_bm != bm) {  // a different buffer manager: nothing of it is held
        held.clear();
        held_bm = bm;
    }
    graph::Fanouts f;
    f.per_layer.assign(fanouts, fanouts + n_layers);
    const uint64_t window = 2 * uint64_t(std::max<uint32_t>(threads, 2));
    std::vector<std::optional<graph::SampledBatch>> ready(n_batches);
    std::mutex mu;
    std::condition_variable cv;
    std::atomic<uint64_t> next{0}, consumed{0};
    std::atomic<bool> failed{false};
    auto t0 = std::chrono::steady_clock::now();
    auto sampler = [&] {
        try {
            while (!failed) {
                const uint64_t b = next.fetch_add(1);
                if (b >= n_batches) return;
                {
                    std::unique_lock lk(mu);
                    cv.wait(lk, [&] { return b < consumed + window || failed; });
                }
                auto batch = graph::sample_khop(
                    t, std::span<const NodeId>(seeds + b * batch_size, batch_size), f,
                    pipeline::PipelineSession::batch_seed(seed, epoch, first_batch + b));
                {
                    std::lock_guard lk(mu);
                    ready[b] = std::move(batch);
                }
                cv.notify_all();
            }
        } catch (const std::exception& e) {
            g_err = e.what();
            failed = true;
            cv.notify_all();
        }
    };
    std::vector<std::thread> pool;
    for (uint32_t i = 0; i + 1 < std::max<uint32_t>(threads, 2); ++i) pool.emplace_back(sampler);
    const auto* tab = static_cast<const std::byte*>(table);
    auto* reg = static_cast<std::byte*>(region);
    try {
        for (uint64_t b = 0; b < n_batches && !failed; ++b) {
            graph::SampledBatch batch;
            {
                std::unique_lock lk(mu);
                cv.wait(lk, [&] { return ready[b].has_value() || failed; });
                if (failed) break;
                batch = std::move(*ready[b]);
                ready[b].reset();
                consumed = b + 1;
            }
            cv.notify_all();
            const auto& nodes = batch.nodes;
            auto plan = mgr.acquire_for_batch(std::span<const NodeId>(nodes.data(), nodes.size()));
            for (auto pos : plan.to_load) {
                const SlotId s = mgr.get_standby_slot();
                mgr.bind_slot(nodes[pos], s);
                plan.alias[pos] = s;
                std::memcpy(reg + uint64_t(s) * row_bytes, tab + nodes[pos] * uint64_t(row_bytes), row_bytes);
            }
            for (auto pos : plan.to_load) mgr.publish_valid(nodes[pos]);
            if (!plan.waits.empty()) throw std::runtime_error("waits under a sequential schedule");
            uint64_t sum = 0;
            for (std::size_t i = 0; i < nodes.size(); ++i)
                sum += hash_bytes64(std::span<const std::byte>(reg + uint64_t(plan.alias[i]) * row_bytes, row_bytes));
            checksums[b] = sum;
            node_counts[b] = nodes.size();
            if (!held.empty()) mgr.release_batch(std::span<const NodeId>(held.data(), held.size()));
            held = nodes;
        }
    } catch (const std::exception& e) {
        g_err = e.what();
        failed = true;
        cv.notify_all();
    }
    for (auto& th : pool) th.join();
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return failed ? -1.0 : secs;
}

}  // extern "C"
