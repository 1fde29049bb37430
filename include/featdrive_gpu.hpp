// featdrive_gpu.hpp -- header-only C++ mirror of the reference's sample -> extract
// API (/root/reference/proj/include/featdrive), implemented over the C ABI in
// fdg.h (libfdg.so, B200 / sm_100a). Same names, argument meaning and exception
// types, so the reference's SET loop (pipeline.hpp:419-543) can call it:
//
//   featdrive::graph::Topology           -> featdrive_gpu::graph::Topology (device CSC + table)
//   featdrive::graph::sample_khop        -> featdrive_gpu::graph::sample_khop     (bit-exact)
//   featdrive::graph::partition_epoch    -> featdrive_gpu::graph::partition_epoch (same libstdc++)
//   featdrive::featbuf::BufferManager    -> featdrive_gpu::featbuf::BufferManager (GPU metadata)
//   featdrive::extract::Extractor        -> featdrive_gpu::extract::Extractor
//   featdrive::pipeline::trainer_step    -> featdrive_gpu::pipeline::trainer_step (GPU checksum)
//   PipelineSession::batch_seed          -> featdrive_gpu::pipeline::batch_seed
//   pipeline::PipelineSession / EpochStats -> featdrive_gpu::pipeline::PipelineSession / EpochStats
//                                            (run_epoch, run_epoch_multi, run_sync_reference,
//                                             the same per-epoch JSON document, stats.hpp:96-146)
//
// Exceptions: FDG_OUT_OF_RANGE -> std::out_of_range, FDG_INVALID_ARG ->
// std::invalid_argument, FDG_INVARIANT -> InvariantViolation (std::logic_error),
// FDG_CAPACITY -> StandbyTimeout (std::runtime_error), FDG_IO_ERROR -> std::system_error
// (errno set) or std::runtime_error (dataset format), anything else -> std::runtime_error.
// Link with -lfdg (paper_2406_13984_b200/libfdg.so).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <exception>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <system_error>
#include <thread>
#include <vector>

#include "fdg.h"

namespace featdrive_gpu {

using NodeId = std::uint64_t;
using SlotId = std::int64_t;

class InvariantViolation : public std::logic_error {
public:
    explicit InvariantViolation(const std::string& w) : std::logic_error(w) {}
};
class StandbyTimeout : public std::runtime_error {
public:
    explicit StandbyTimeout(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
    if (rc == FDG_OK) return;
    std::string msg = fdg_last_error();
    switch (rc) {
        case FDG_OUT_OF_RANGE: throw std::out_of_range(msg);
        case FDG_INVALID_ARG: throw std::invalid_argument(msg);
        case FDG_INVARIANT: throw InvariantViolation(msg);
        case FDG_CAPACITY: throw StandbyTimeout(msg);
        case FDG_IO_ERROR:  // dataset files: throw_errno (common.hpp:67-69) or a format runtime_error
            if (const int e = fdg_last_errno()) throw std::system_error(e, std::generic_category(), msg);
            throw std::runtime_error(msg);
        default: throw std::runtime_error(msg);
    }
}

namespace graph {

/// graph::Topology (topology.hpp:33-193) + the feature table, HBM-resident.
class Topology {
public:
    /// Loads indptr.bin / indices.bin / features.bin of a reference dataset dir.
    explicit Topology(const std::string& dataset_dir, int device = 0) {
        check(fdg_ctx_create(device, &ctx_));
        check(fdg_ctx_load_topology_files(ctx_, dataset_dir.c_str()));
        check(fdg_ctx_load_features_file(ctx_, (dataset_dir + "/features.bin").c_str()));
    }
    /// Bit-exact GPU generation of storage::create_synthetic_dataset's content.
    static std::unique_ptr<Topology> generate(std::uint64_t num_nodes, std::uint32_t dim, std::uint32_t avg_degree,
                                              std::uint64_t seed, int device = 0) {
        std::unique_ptr<Topology> t(new Topology(device));
        check(fdg_ctx_generate_topology(t->ctx_, seed, num_nodes, avg_degree));
        check(fdg_ctx_generate_features(t->ctx_, seed, num_nodes, dim, 0, 1));
        return t;
    }
    ~Topology() { fdg_ctx_destroy(ctx_); }
    Topology(const Topology&) = delete;
    Topology& operator=(const Topology&) = delete;

    /// Out-of-core tier: the feature table moves to pinned host memory mapped into the
    /// device; gathers and buffer-manager misses read it over PCIe (put a BufferManager
    /// in front of it).
    void features_to_host() { check(fdg_ctx_features_to_host(ctx_)); }
    bool features_on_host() const { return fdg_ctx_features_on_host(ctx_) != 0; }

    std::uint64_t num_nodes() const { return info().num_nodes; }
    std::uint64_t num_edges() const { return info().num_edges; }
    std::uint32_t row_bytes() const { return info().row_bytes; }
    fdg_ctx* handle() const { return ctx_; }

private:
    explicit Topology(int device) { check(fdg_ctx_create(device, &ctx_)); }
    fdg_ctx_info info() const {
        fdg_ctx_info i;
        check(fdg_ctx_info_get(ctx_, &i));
        return i;
    }
    fdg_ctx* ctx_ = nullptr;
};

/// graph::Fanouts (sampling.hpp:21-41)
struct Fanouts {
    std::vector<std::uint32_t> per_layer;
    void validate() const {
        if (per_layer.empty()) throw std::invalid_argument("fanouts: need at least one layer");
        for (auto f : per_layer)
            if (f < 1) throw std::invalid_argument("fanouts: every entry must be >= 1");
    }
    std::uint64_t max_batch_nodes(std::uint64_t batch_size) const {
        std::uint64_t total = 1, layer = 1;
        for (auto f : per_layer) {
            layer *= f;
            total += layer;
        }
        return batch_size * total;
    }
};

struct LocalEdge {  // sampling.hpp:43-46
    std::uint32_t src = 0;
    std::uint32_t dst = 0;
};

struct SampledBatch {  // sampling.hpp:48-54
    std::uint64_t batch_id = 0;
    std::uint64_t epoch = 0;
    std::vector<NodeId> seeds;
    std::vector<NodeId> nodes;
    std::vector<LocalEdge> edges;
    // extension (not in the reference): nodes before each hop's new nodes, [1] = unique
    // seeds -- the block structure the train stage consumes
    std::vector<std::uint64_t> layer_nodes;
};

/// graph::sample_khop (sampling.hpp:72-134), executed on the GPU, bit-exact.
/// One sampler workspace per (topology, fanouts, seed count) is reused.
inline SampledBatch sample_khop(const Topology& topo, std::span<const NodeId> seeds, const Fanouts& fanouts,
                                std::uint64_t rng_seed) {
    fanouts.validate();
    fdg_sampler* s = nullptr;
    check(fdg_sampler_create(topo.handle(), std::uint32_t(std::max<std::size_t>(seeds.size(), 1)),
                             fanouts.per_layer.data(), std::uint32_t(fanouts.per_layer.size()), &s));
    std::unique_ptr<fdg_sampler, int (*)(fdg_sampler*)> guard(s, fdg_sampler_destroy);
    std::uint64_t max_nodes = 0, max_edges = 0;
    check(fdg_sampler_capacity(s, &max_nodes, &max_edges));
    const std::uint64_t cap = std::max<std::uint64_t>({max_nodes, max_edges, 1});
    SampledBatch b;
    b.seeds.assign(seeds.begin(), seeds.end());
    b.nodes.resize(cap);
    std::vector<std::uint32_t> e(2 * cap);
    std::uint64_t nn = 0, ne = 0;
    b.layer_nodes.assign(fanouts.per_layer.size() + 2, 0);
    check(fdg_sample_khop_host(s, seeds.data(), std::uint32_t(seeds.size()), rng_seed, b.nodes.data(), e.data(), cap,
                               &nn, &ne, b.layer_nodes.data(), nullptr));
    b.nodes.resize(nn);
    b.edges.resize(ne);
    for (std::uint64_t i = 0; i < ne; ++i) b.edges[i] = LocalEdge{e[2 * i], e[2 * i + 1]};
    return b;
}

/// graph::partition_epoch (sampling.hpp:57-70)
inline std::vector<std::vector<NodeId>> partition_epoch(std::vector<NodeId> train_ids, std::uint64_t batch_size,
                                                        std::uint64_t shuffle_seed) {
    std::vector<NodeId> order(train_ids.size());
    check(fdg_partition_epoch(train_ids.data(), train_ids.size(), batch_size, shuffle_seed, order.data()));
    std::vector<std::vector<NodeId>> chunks;
    for (std::size_t at = 0; at < order.size(); at += batch_size)
        chunks.emplace_back(order.begin() + at, order.begin() + std::min(order.size(), at + batch_size));
    return chunks;
}

}  // namespace graph

namespace train {

/// The train stage (fdg_sage_*): GraphSAGE forward + softmax cross-entropy over a
/// sampled batch's blocks. The reference's trainer is the checksum trainer_step
/// (pipeline.hpp:103-124); the paper's model is a 3-layer GraphSAGE.
class GraphSAGE {
public:
    /// dims: L + 1 widths (dims[0] = feature width), one layer per sampling hop.
    GraphSAGE(const graph::Topology& topo, std::vector<std::uint32_t> dims, const graph::Fanouts& fanouts,
              std::uint32_t max_seeds)
        : topo_(topo), dims_(std::move(dims)) {
        if (dims_.size() != fanouts.per_layer.size() + 1)
            throw std::invalid_argument("GraphSAGE: one layer per sampling hop");
        check(fdg_sage_create(topo.handle(), dims_.data(), std::uint32_t(fanouts.per_layer.size()),
                              fanouts.per_layer.data(), max_seeds, &m_));
    }
    ~GraphSAGE() { fdg_sage_destroy(m_); }
    GraphSAGE(const GraphSAGE&) = delete;
    GraphSAGE& operator=(const GraphSAGE&) = delete;

    /// w_neigh, w_self: [dims[l]][dims[l+1]] row-major (out = in . W); bias: [dims[l+1]].
    void set_layer(std::uint32_t layer, const std::vector<float>& w_neigh, const std::vector<float>& w_self,
                   const std::vector<float>& bias) {
        check(fdg_sage_set_layer(m_, layer, w_neigh.data(), w_self.data(), bias.data()));
    }

    /// Mean loss over the batch's unique seeds, label(v) = splitmix64(v ^ label_seed) % C.
    float forward(const graph::SampledBatch& b, std::uint64_t label_seed) const {
        const std::uint64_t n = b.nodes.size(), e = b.edges.size();
        fdg_batch_counts c{};
        c.n_nodes = std::uint32_t(n);
        c.n_edges = std::uint32_t(e);
        c.n_layers = std::uint32_t(dims_.size() - 1);
        for (std::size_t i = 0; i < b.layer_nodes.size() && i < FDG_MAX_LAYERS + 2; ++i)
            c.layer_nodes[i] = std::uint32_t(b.layer_nodes[i]);
        void *nd = nullptr, *ed = nullptr, *x = nullptr, *cd = nullptr, *ld = nullptr;
        auto guard = [](void* p) { fdg_free(p); };
        check(fdg_malloc(&nd, std::max<std::uint64_t>(n, 1) * 8));
        std::unique_ptr<void, decltype(guard)> g1(nd, guard);
        check(fdg_malloc(&ed, std::max<std::uint64_t>(e, 1) * 8));
        std::unique_ptr<void, decltype(guard)> g2(ed, guard);
        check(fdg_malloc(&x, std::max<std::uint64_t>(n, 1) * topo_.row_bytes()));
        std::unique_ptr<void, decltype(guard)> g3(x, guard);
        check(fdg_malloc(&cd, sizeof(c)));
        std::unique_ptr<void, decltype(guard)> g4(cd, guard);
        check(fdg_malloc(&ld, sizeof(float)));
        std::unique_ptr<void, decltype(guard)> g5(ld, guard);
        check(fdg_memcpy_h2d(nd, b.nodes.data(), n * 8, nullptr));
        check(fdg_memcpy_h2d(ed, b.edges.data(), e * 8, nullptr));
        check(fdg_memcpy_h2d(cd, &c, sizeof(c), nullptr));
        if (n) check(fdg_gather(topo_.handle(), nullptr, static_cast<const std::uint64_t*>(nd), nullptr, n, x, nullptr));
        check(fdg_sage_forward(m_, nullptr, x, static_cast<const std::uint64_t*>(nd), static_cast<const std::uint32_t*>(ed),
                               static_cast<const fdg_batch_counts*>(cd), label_seed, static_cast<float*>(ld), nullptr));
        float loss = 0.f;
        check(fdg_memcpy_d2h(&loss, ld, sizeof(float), nullptr));
        check(fdg_device_sync());
        return loss;
    }
    fdg_sage* handle() const { return m_; }

private:
    const graph::Topology& topo_;
    std::vector<std::uint32_t> dims_;
    fdg_sage* m_ = nullptr;
};

}  // namespace train

namespace featbuf {

struct BufferStats {  // buffer_manager.hpp:192-200
    std::uint64_t hits = 0, loads = 0, waits = 0, evictions = 0, takeovers = 0, releases = 0, standby_len = 0;
};

/// featbuf::BufferManager + FeatureRegion, GPU-resident; operations are batch-wide.
class BufferManager {
public:
    BufferManager(const graph::Topology& topo, std::uint64_t slot_count, std::uint64_t min_reserved,
                  std::uint32_t max_batch_nodes)
        : topo_(topo) {
        check(fdg_bm_create(topo.handle(), slot_count, min_reserved, max_batch_nodes, &bm_));
    }
    ~BufferManager() { fdg_bm_destroy(bm_); }
    BufferManager(const BufferManager&) = delete;
    BufferManager& operator=(const BufferManager&) = delete;

    /// acquire_for_batch + get_standby_slot/bind_slot per miss + row copies + publish_valid.
    std::vector<SlotId> extract(std::span<const NodeId> nodes) {
        std::vector<SlotId> alias(nodes.size());
        DeviceVec<NodeId> nd(nodes.size());
        DeviceVec<SlotId> al(nodes.size());
        check(fdg_memcpy_h2d(nd.p, nodes.data(), nodes.size() * 8, nullptr));
        check(fdg_bm_extract(bm_, nullptr, nd.p, nullptr, nodes.size(), al.p, nullptr, nullptr));
        status();
        check(fdg_memcpy_d2h(alias.data(), al.p, alias.size() * 8, nullptr));
        check(fdg_stream_sync(nullptr));
        return alias;
    }
    /// release_batch (buffer_manager.hpp:352-364)
    void release_batch(std::span<const NodeId> nodes) {
        DeviceVec<NodeId> nd(nodes.size());
        check(fdg_memcpy_h2d(nd.p, nodes.data(), nodes.size() * 8, nullptr));
        check(fdg_bm_release(bm_, nullptr, nd.p, nullptr, nodes.size()));
        status();
    }
    BufferStats stats() const {
        fdg_bm_stats s;
        check(fdg_bm_stats_get(bm_, &s));
        return BufferStats{s.hits, s.loads, s.waits, s.evictions, s.takeovers, s.releases, s.standby_len};
    }
    void validate() const { check(fdg_bm_validate(bm_)); }
    fdg_bm* handle() const { return bm_; }
    const graph::Topology& topology() const { return topo_; }

private:
    template <typename T>
    struct DeviceVec {
        explicit DeviceVec(std::size_t n) { check(fdg_malloc(reinterpret_cast<void**>(&p), std::max<std::size_t>(n, 1) * sizeof(T))); }
        ~DeviceVec() { fdg_free(p); }
        T* p = nullptr;
    };
    void status() const {
        int rc = fdg_bm_status(bm_);
        if (rc == FDG_CAPACITY) throw StandbyTimeout("get_standby_slot: standby list exhausted; feature buffer is undersized");
        check(rc);
    }
    const graph::Topology& topo_;
    fdg_bm* bm_ = nullptr;
};

}  // namespace featbuf

namespace extract {

using NodeAliasList = std::vector<SlotId>;  // extractor.hpp:73

/// extract::Extractor (extractor.hpp:75-113)
class Extractor {
public:
    explicit Extractor(featbuf::BufferManager& buffer) : buffer_(buffer) {}
    NodeAliasList extract_batch(const graph::SampledBatch& batch) { return buffer_.extract(batch.nodes); }

private:
    featbuf::BufferManager& buffer_;
};

}  // namespace extract

namespace pipeline {

/// PipelineSession::batch_seed (pipeline.hpp:295-298)
inline std::uint64_t batch_seed(std::uint64_t seed, std::uint64_t epoch, std::uint64_t global_batch) {
    return fdg_batch_seed(seed, epoch, global_batch);
}

/// trainer_step (pipeline.hpp:103-124): sum of hash_bytes64 over each node's row,
/// read through its alias slot in the GPU feature region.
inline std::uint64_t trainer_step(const graph::SampledBatch& batch, const extract::NodeAliasList& alias,
                                  const featbuf::BufferManager& buffer) {
    if (alias.size() != batch.nodes.size()) throw InvariantViolation("alias list length != batch nodes");
    for (SlotId a : alias)
        if (a < 0) throw InvariantViolation("trainer saw an unassigned alias");
    void* ad = nullptr;
    void* cs = nullptr;
    check(fdg_malloc(&ad, std::max<std::size_t>(alias.size(), 1) * 8));
    check(fdg_malloc(&cs, 8));
    check(fdg_memset(cs, 0, 8, nullptr));
    check(fdg_memcpy_h2d(ad, alias.data(), alias.size() * 8, nullptr));
    check(fdg_checksum_alias(buffer.topology().handle(), nullptr, fdg_bm_region(buffer.handle()),
                             static_cast<const int64_t*>(ad), nullptr, alias.size(), static_cast<uint64_t*>(cs)));
    std::uint64_t sum = 0;
    check(fdg_memcpy_d2h(&sum, cs, 8, nullptr));
    check(fdg_stream_sync(nullptr));
    fdg_free(ad);
    fdg_free(cs);
    return sum;
}
// ------------------------------------------------------------------ session ----
// PipelineSession (pipeline.hpp:127-299) on the GPU runner (fdg_pipeline_*): one
// persistent pipeline (sampler streams + extraction + optional buffer manager) per
// worker segment, reused across epochs like the reference's per-worker buffer.

inline std::uint64_t splitmix64(std::uint64_t x) {  // common.hpp:77-82
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
inline std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b) {  // common.hpp:84-86
    return splitmix64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}

enum class RunMode { Async, SyncReference };

/// pipeline.hpp:30-76. GPU meaning: num_samplers = concurrent sampler streams;
/// num_extractors (N_e) only sizes the default slot count N_e * M_b, as in the
/// reference; slots = kNoBuffer extracts by direct gather (no buffer manager).
struct PipelineConfig {
    static constexpr std::uint64_t kNoBuffer = ~0ull;
    std::uint32_t num_samplers = 6;
    std::uint32_t num_extractors = 4;
    std::uint64_t batch_size = 1000;
    graph::Fanouts fanouts{{10, 10, 10}};
    std::uint64_t slots = 0;  // per-worker feature-buffer slots; 0 = N_e * M_b
    RunMode mode = RunMode::Async;
    std::uint32_t workers = 1;  // segments (concurrent pipelines on the topology's GPU)
    std::uint32_t group_batches = 1;
    bool verify = false;  // re-derive every batch on the non-pipelined path and compare

    void validate() const {
        if (num_samplers < 1 || num_extractors < 1)
            throw std::invalid_argument("config: need at least one sampler and one extractor");
        if (batch_size < 1) throw std::invalid_argument("config: batch_size must be >= 1");
        if (workers < 1) throw std::invalid_argument("config: workers must be >= 1");
        fanouts.validate();
    }
    std::uint64_t max_batch_nodes(std::uint64_t num_nodes) const {
        return std::min(fanouts.max_batch_nodes(batch_size), num_nodes);
    }
};

struct BatchRecord {  // stats.hpp:21-27
    std::uint64_t batch_id = 0, seed_count = 0, node_count = 0, checksum = 0;
    bool failed = false;
};

class PipelineError : public std::runtime_error {  // pipeline.hpp:84-93
public:
    PipelineError(std::string stage, const std::string& what)
        : std::runtime_error("[" + stage + "] " + what), stage_(std::move(stage)) {}
    const std::string& stage() const { return stage_; }

private:
    std::string stage_;
};

/// stats.hpp:47-146, same JSON document. Stage times: sample_busy = sampler-stream
/// busy time, extract_busy = extraction (gather / buffer manager + fused trainer
/// checksum) time, both from CUDA events; the GPU runner has no blocking queues, so
/// the *_block and train/release fields are 0 (training is fused into extraction).
struct EpochStats {
    std::uint64_t epoch = 0;
    std::uint32_t worker = 0;
    std::string mode;
    double wall_time_s = 0;
    std::uint64_t batches_sampled = 0, batches_trained = 0, batches_failed = 0, batches_released = 0;
    double sample_busy_s = 0, sample_block_s = 0;
    double extract_busy_s = 0, extract_block_s = 0, extract_io_wait_s = 0;
    double train_busy_s = 0, train_block_s = 0;
    double release_busy_s = 0, release_block_s = 0;
    std::uint64_t bytes_useful = 0, bytes_redundant = 0, bytes_requested = 0;
    std::uint64_t read_requests = 0, nodes_loaded = 0, staging_hits = 0;
    featbuf::BufferStats buffer;
    std::uint64_t feature_buffer_bytes = 0, staging_bytes = 0, slot_count = 0;
    std::uint64_t staging_borrows = 0, staging_cross_hits = 0;
    std::vector<BatchRecord> batch_records;

    std::string to_json() const {
        std::string o;
        auto num = [&](const char* k, double v, bool comma = true) {
            char b[64];
            std::snprintf(b, sizeof b, "\"%s\":%.17g%s", k, v, comma ? "," : "");
            o += b;
        };
        auto u = [&](const char* k, std::uint64_t v, bool comma = true) {
            o += "\"" + std::string(k) + "\":" + std::to_string(v) + (comma ? "," : "");
        };
        o += "{";
        u("epoch", epoch);
        u("worker", worker);
        o += "\"mode\":\"" + mode + "\",";
        num("wall_time_s", wall_time_s);
        o += "\"batches\":{";
        u("sampled", batches_sampled);
        u("trained", batches_trained);
        u("failed", batches_failed);
        u("released", batches_released, false);
        o += "},\"stage_time_s\":{";
        num("sample_busy", sample_busy_s);
        num("sample_block", sample_block_s);
        num("extract_busy", extract_busy_s);
        num("extract_block", extract_block_s);
        num("extract_io_wait", extract_io_wait_s);
        num("train_busy", train_busy_s);
        num("train_block", train_block_s);
        num("release_busy", release_busy_s);
        num("release_block", release_block_s, false);
        o += "},\"bytes\":{";
        u("useful", bytes_useful);
        u("redundant", bytes_redundant);
        u("requested", bytes_requested, false);
        o += "},\"reads\":{";
        u("requests", read_requests);
        u("nodes_loaded", nodes_loaded);
        u("staging_hits", staging_hits, false);
        o += "},\"buffer\":{";
        u("hits", buffer.hits);
        u("loads", buffer.loads);
        u("waits", buffer.waits);
        u("evictions", buffer.evictions);
        u("takeovers", buffer.takeovers);
        u("standby_len", buffer.standby_len, false);
        o += "},\"memory\":{";
        u("feature_buffer_bytes", feature_buffer_bytes);
        u("staging_bytes", staging_bytes);
        u("slot_count", slot_count);
        u("staging_borrows", staging_borrows);
        u("staging_cross_hits", staging_cross_hits, false);
        o += "},\"batch_checksums\":[";
        for (std::size_t i = 0; i < batch_records.size(); ++i) {
            const auto& b = batch_records[i];
            o += i ? ",{" : "{";
            u("batch", b.batch_id);
            u("seeds", b.seed_count);
            u("nodes", b.node_count);
            u("checksum", b.checksum);
            o += std::string("\"failed\":") + (b.failed ? "true" : "false") + "}";
        }
        o += "]}";
        return o;
    }
};

class PipelineSession {
public:
    PipelineSession(const graph::Topology& topo, PipelineConfig cfg) : topo_(topo), cfg_(std::move(cfg)) {
        cfg_.validate();
        mb_ = cfg_.max_batch_nodes(topo_.num_nodes());
        slots_ = cfg_.slots == PipelineConfig::kNoBuffer ? 0
                 : cfg_.slots                            ? cfg_.slots
                                                         : std::uint64_t(cfg_.num_extractors) * mb_;
        // pipeline.hpp:137-141 refuses slots below its N_e * M_b reservation; the GPU
        // runner holds at most two batches (the one extracted + the lag-1 release), so
        // its reservation is 2 * M_b.
        if (slots_ && slots_ < 2 * mb_)
            throw std::invalid_argument("config: slots " + std::to_string(slots_) +
                                        " below the deadlock reservation 2*M_b = " + std::to_string(2 * mb_));
        for (std::uint32_t w = 0; w < cfg_.workers; ++w) {
            fdg_pipeline_config pc{};
            pc.batch_size = std::uint32_t(cfg_.batch_size);
            pc.n_samplers = cfg_.num_samplers;
            pc.use_buffer_manager = slots_ ? 1 : 0;
            pc.buffer_slots = slots_;
            pc.write_x = 1;
            pc.checksum = 1;
            pc.group_batches = cfg_.group_batches;
            fdg_pipeline* p = nullptr;
            check(fdg_pipeline_create(topo_.handle(), cfg_.fanouts.per_layer.data(),
                                      std::uint32_t(cfg_.fanouts.per_layer.size()), &pc, &p));
            pipes_.push_back(p);
        }
    }
    ~PipelineSession() {
        for (auto p : pipes_) fdg_pipeline_destroy(p);
        if (sampler_) fdg_sampler_destroy(sampler_);
    }
    PipelineSession(const PipelineSession&) = delete;
    PipelineSession& operator=(const PipelineSession&) = delete;

    std::uint64_t max_batch_nodes() const { return mb_; }
    std::uint64_t slots_per_worker() const { return slots_; }
    const PipelineConfig& config() const { return cfg_; }

    static std::uint64_t batch_seed(std::uint64_t seed, std::uint64_t epoch, std::uint64_t global_batch) {
        return hash_combine(hash_combine(seed, epoch), global_batch);  // pipeline.hpp:295-298
    }

    EpochStats run_epoch(std::span<const NodeId> train_ids, std::uint64_t epoch, std::uint64_t seed) {
        auto all = run_epoch_multi(train_ids, epoch, seed);
        return std::move(all.front());
    }

    /// pipeline.hpp:185-259: contiguous chunk ranges per worker (sizes differ by at
    /// most one), all workers concurrently; the root-cause error is rethrown.
    std::vector<EpochStats> run_epoch_multi(std::span<const NodeId> train_ids, std::uint64_t epoch,
                                            std::uint64_t seed) {
        auto chunks = graph::partition_epoch({train_ids.begin(), train_ids.end()}, cfg_.batch_size,
                                             hash_combine(seed, epoch));
        const std::uint64_t total = chunks.size(), W = cfg_.workers;
        std::vector<EpochStats> out(W);
        std::vector<std::exception_ptr> err(W);
        auto work = [&](std::uint32_t w) {
            try {
                const std::uint64_t base = total / W, rem = total % W;
                const std::uint64_t lo = w * base + std::min<std::uint64_t>(w, rem);
                const std::uint64_t hi = lo + base + (w < rem ? 1 : 0);
                out[w] = run_segment(w, chunks, lo, hi, epoch, seed);
            } catch (...) {
                err[w] = std::current_exception();
            }
        };
        if (W == 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            for (std::uint32_t w = 0; w < W; ++w) th.emplace_back(work, w);
            for (auto& t : th) t.join();
        }
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
        return out;
    }

    /// pipeline.hpp:263-293: sample -> extract (gather + checksum) one batch at a time,
    /// synchronously, with no feature buffer.
    EpochStats run_sync_reference(std::span<const NodeId> train_ids, std::uint64_t epoch, std::uint64_t seed) {
        auto chunks = graph::partition_epoch({train_ids.begin(), train_ids.end()}, cfg_.batch_size,
                                             hash_combine(seed, epoch));
        EpochStats st;
        st.epoch = epoch;
        st.mode = "sync-reference";
        const auto t0 = std::chrono::steady_clock::now();
        const std::uint32_t rb = topo_.row_bytes();
        for (std::uint64_t b = 0; b < chunks.size(); ++b) {
            auto r = sync_batch(chunks[b], batch_seed(seed, epoch, b));
            ++st.batches_sampled;
            st.batch_records.push_back({b, chunks[b].size(), r.first, r.second, false});
            st.bytes_useful += r.first * rb;
            st.bytes_requested += r.first * rb;
            st.read_requests += r.first;
            st.nodes_loaded += r.first;
            ++st.batches_trained;
            ++st.batches_released;
        }
        st.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return st;
    }

private:
    // one batch on the non-pipelined path: (node count, trainer checksum)
    std::pair<std::uint64_t, std::uint64_t> sync_batch(std::span<const NodeId> seeds, std::uint64_t rng_seed) {
        std::lock_guard<std::mutex> lk(sync_mu_);  // one sync workspace, shared by verifying workers
        if (!sampler_) {
            check(fdg_sampler_create(topo_.handle(), std::uint32_t(cfg_.batch_size), cfg_.fanouts.per_layer.data(),
                                     std::uint32_t(cfg_.fanouts.per_layer.size()), &sampler_));
            std::uint64_t mn = 0, me = 0;
            check(fdg_sampler_capacity(sampler_, &mn, &me));
            cap_ = std::max<std::uint64_t>({mn, me, 1});
            sbuf_ = std::make_unique<Dev>((8 + 8 + 8 + std::uint64_t(topo_.row_bytes())) * cap_ + 8 * cfg_.batch_size +
                                          sizeof(fdg_batch_counts) + 512);
        }
        char* base = static_cast<char*>(sbuf_->p);
        auto* seeds_d = reinterpret_cast<std::uint64_t*>(base);
        auto* nodes_d = seeds_d + cfg_.batch_size;
        auto* edges_d = reinterpret_cast<std::uint32_t*>(nodes_d + cap_);
        auto* cs_d = reinterpret_cast<std::uint64_t*>(edges_d + 2 * cap_);
        auto* cnt_d = reinterpret_cast<fdg_batch_counts*>(cs_d + 1);
        void* x_d = reinterpret_cast<void*>((reinterpret_cast<std::uintptr_t>(cnt_d + 1) + 255) & ~std::uintptr_t(255));
        check(fdg_memcpy_h2d(seeds_d, seeds.data(), seeds.size() * 8, nullptr));
        check(fdg_sample_khop(sampler_, nullptr, seeds_d, std::uint32_t(seeds.size()), rng_seed, nodes_d, edges_d, cap_,
                              cnt_d));
        check(fdg_memset(cs_d, 0, 8, nullptr));
        check(fdg_gather(topo_.handle(), nullptr, nodes_d, &cnt_d->n_nodes, cap_, x_d, cs_d));
        fdg_batch_counts c{};
        std::uint64_t cs = 0;
        check(fdg_memcpy_d2h(&c, cnt_d, sizeof c, nullptr));
        check(fdg_memcpy_d2h(&cs, cs_d, 8, nullptr));
        check(fdg_stream_sync(nullptr));
        if (c.status == FDG_OUT_OF_RANGE) throw std::out_of_range("sample_khop: seed out of range");
        if (c.status) check(int(c.status));
        return {c.n_nodes, cs};
    }

    EpochStats run_segment(std::uint32_t w, const std::vector<std::vector<NodeId>>& chunks, std::uint64_t lo,
                           std::uint64_t hi, std::uint64_t epoch, std::uint64_t seed) {
        EpochStats st;
        st.epoch = epoch;
        st.worker = w;
        st.mode = "async";
        const std::uint32_t rb = topo_.row_bytes();
        st.slot_count = slots_;
        st.feature_buffer_bytes = slots_ * rb;
        const std::uint64_t n = hi - lo;
        if (n == 0) return st;
        fdg_pipeline* p = pipes_[w];
        std::vector<NodeId> seeds;
        std::vector<std::uint64_t> rng(n);
        for (std::uint64_t b = lo; b < hi; ++b) {
            if (b + 1 < hi && chunks[b].size() != cfg_.batch_size)
                throw PipelineError("sample", "only the last chunk of an epoch may be short");
            seeds.insert(seeds.end(), chunks[b].begin(), chunks[b].end());
            rng[b - lo] = batch_seed(seed, epoch, b);
        }
        featbuf::BufferStats before = buffer_stats(w);
        Dev sd(seeds.size() * 8);
        check(fdg_memcpy_h2d(sd.p, seeds.data(), seeds.size() * 8, nullptr));
        check(fdg_stream_sync(nullptr));
        std::vector<float> xms(n);
        float ms = 0;
        const auto t0 = std::chrono::steady_clock::now();
        check(fdg_pipeline_run_ragged(p, static_cast<const std::uint64_t*>(sd.p), 0, seeds.size(), rng.data(), n,
                                      nullptr, xms.data(), &ms));
        st.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::vector<fdg_batch_counts> recs(n);
        check(fdg_pipeline_records(p, 0, n, recs.data()));
        float sample_ms = 0;
        check(fdg_pipeline_sample_times(p, nullptr, &sample_ms));
        st.sample_busy_s = sample_ms / 1e3;
        for (float x : xms) st.extract_busy_s += x / 1e3;
        std::uint64_t nodes_total = 0;
        for (std::uint64_t j = 0; j < n; ++j) {
            const auto& c = recs[j];
            const bool failed = c.status != 0;
            st.batch_records.push_back({lo + j, chunks[lo + j].size(), c.n_nodes, failed ? 0 : c.checksum, failed});
            ++st.batches_sampled;
            if (failed) {
                ++st.batches_failed;
            } else {
                ++st.batches_trained;
                nodes_total += c.n_nodes;
            }
            ++st.batches_released;
            if (cfg_.verify && !failed) {
                auto ref = sync_batch(chunks[lo + j], rng[j]);
                if (ref.first != c.n_nodes || ref.second != c.checksum)
                    throw PipelineError("train", "batch " + std::to_string(lo + j) +
                                                     " differs from the synchronous path (nodes " +
                                                     std::to_string(c.n_nodes) + " vs " + std::to_string(ref.first) +
                                                     ")");
            }
        }
        featbuf::BufferStats after = buffer_stats(w);
        if (slots_) {
            st.buffer = {after.hits - before.hits,     after.loads - before.loads,
                         after.waits - before.waits,   after.evictions - before.evictions,
                         after.takeovers - before.takeovers, after.releases - before.releases,
                         after.standby_len};
            st.nodes_loaded = st.buffer.loads;
        } else {
            st.nodes_loaded = nodes_total;  // direct gather: every row is read
        }
        st.read_requests = st.nodes_loaded;
        st.bytes_useful = st.bytes_requested = st.nodes_loaded * rb;
        return st;
    }

    featbuf::BufferStats buffer_stats(std::uint32_t w) const {
        if (!slots_) return {};
        fdg_bm_stats s{};
        check(fdg_pipeline_bm_stats(pipes_[w], &s));
        return {s.hits, s.loads, s.waits, s.evictions, s.takeovers, s.releases, s.standby_len};
    }

    struct Dev {
        explicit Dev(std::uint64_t bytes) { check(fdg_malloc(&p, std::max<std::uint64_t>(bytes, 8))); }
        ~Dev() { fdg_free(p); }
        void* p = nullptr;
    };

    const graph::Topology& topo_;
    PipelineConfig cfg_;
    std::uint64_t mb_ = 0, slots_ = 0, cap_ = 0;
    std::vector<fdg_pipeline*> pipes_;
    fdg_sampler* sampler_ = nullptr;
    std::unique_ptr<Dev> sbuf_;
    std::mutex sync_mu_;
};

  }  // namespace pipeline
}  // namespace featdrive_gpu
