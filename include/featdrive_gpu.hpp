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
//
// Exceptions: FDG_OUT_OF_RANGE -> std::out_of_range, FDG_INVALID_ARG ->
// std::invalid_argument, FDG_INVARIANT -> InvariantViolation (std::logic_error),
// FDG_CAPACITY -> StandbyTimeout (std::runtime_error), anything else ->
// std::runtime_error. Link with -lfdg (paper_2406_13984_b200/libfdg.so).
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
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
    check(fdg_sample_khop_host(s, seeds.data(), std::uint32_t(seeds.size()), rng_seed, b.nodes.data(), e.data(), cap,
                               &nn, &ne, nullptr, nullptr));
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

}  // namespace pipeline
}  // namespace featdrive_gpu
