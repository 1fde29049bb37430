// featdrive_gpu.hpp -- header-only C++ drop-in for the reference's sample -> extract API
// (/root/reference/proj/include/featdrive), implemented over the C ABI in fdg.h (libfdg.so,
// B200 / sm_100a). Same namespaces below the top one, same class names, constructor shapes,
// argument meaning and exception types, so a reference SET loop compiles against it with the
// include and the top-level namespace changed (tests/cpp/set_loop.cpp builds both ways):
//
//   featdrive::graph::Topology(dir)              -> CSC in HBM (indptr u64, indices u32/u64)
//   featdrive::graph::sample_khop / partition_epoch  (bit-exact; pooled sampler workspaces)
//   featdrive::storage::FeatureTable(path)       -> the feature table in HBM (+ header, read_row_sync)
//   featdrive::featbuf::BufferManager(BufferConfig)  -> GPU metadata (mapping, refs, LRU ring);
//       acquire_for_batch / get_standby_slot / bind_slot / publish_valid / wait_for_valid /
//       release_batch / unwind_bound / release_ref as stream-ordered device operations
//   featdrive::featbuf::FeatureRegion(S, row)    -> S x row device bytes (the slots)
//   featdrive::extract::Extractor(ExtractorEnv, ExtractorConfig) -> extract_batch: the fused
//       Algorithm 1 on the GPU (acquire, LRU pops, bind, row loads, publish) -> NodeAliasList
//   featdrive::pipeline::trainer_step(TrainTicket, FeatureRegion, FeatureTable*) -> GPU checksum
//       (+ GPU byte compare against the table with verify)
//   featdrive::pipeline::PipelineSession(dir, cfg) -> the native runner (fdg_pipeline_*):
//       run_epoch / run_epoch_multi / run_sync_reference, the same EpochStats JSON
//
// Objects with no GPU counterpart keep their constructors and do nothing: CopyEngine (device
// copies are stream-ordered), StagingArena (SSD staging is out of scope), StageCounters
// (filled by Extractor::extract_batch from the buffer counters). Per-call paths allocate no
// device memory once warm: samplers are pooled per Topology, staging buffers grow and stay.
//
// Exceptions: FDG_OUT_OF_RANGE -> std::out_of_range, FDG_INVALID_ARG -> std::invalid_argument,
// FDG_INVARIANT -> InvariantViolation (std::logic_error), FDG_CAPACITY -> StandbyTimeout
// (std::runtime_error), FDG_IO_ERROR -> std::system_error (errno set) or std::runtime_error
// (dataset format), anything else -> std::runtime_error.
// Link with -lfdg (paper_2406_13984_b200/libfdg.so).
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <exception>
#include <functional>
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

// ------------------------------------------------------------------ common.hpp ----
using NodeId = std::uint64_t;
using SlotId = std::int64_t;  // -1 means "no slot"
inline constexpr SlotId kNoSlot = -1;
inline constexpr std::uint64_t kSectorBytes = 512;

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

constexpr std::uint64_t splitmix64(std::uint64_t x) {  // common.hpp:77-82
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
constexpr std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b) {  // common.hpp:84-86
    return splitmix64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}

/// DurationCounter / ScopedTimer (common.hpp:240-260).
class DurationCounter {
public:
    void add(std::int64_t ns) { ns_.fetch_add(ns, std::memory_order_relaxed); }
    std::int64_t ns() const { return ns_.load(std::memory_order_relaxed); }
    double seconds() const { return double(ns()) * 1e-9; }

private:
    std::atomic<std::int64_t> ns_{0};
};
class ScopedTimer {
public:
    explicit ScopedTimer(DurationCounter& c) : c_(c), t0_(std::chrono::steady_clock::now()) {}
    ~ScopedTimer() {
        c_.add(std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0_).count());
    }

private:
    DurationCounter& c_;
    std::chrono::steady_clock::time_point t0_;
};

namespace detail {
/// A device allocation that only grows: steady-state calls allocate nothing.
struct DevBuf {
    void* p = nullptr;
    std::size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) fdg_free(p);
    }
    void* reserve(std::size_t bytes) {
        bytes = std::max<std::size_t>(bytes, 8);
        if (bytes > cap) {
            if (p) fdg_free(p);
            p = nullptr;
            cap = 0;
            check(fdg_malloc(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};
}  // namespace detail

// ------------------------------------------------------------- pipeline/stats ----
namespace pipeline {
/// StageCounters (stats.hpp:30-48): filled by the drop-in's Extractor.
struct StageCounters {
    DurationCounter sample_busy, sample_block, extract_busy, extract_block, extract_io_wait, train_busy, train_block,
        release_busy, release_block;
    std::atomic<std::uint64_t> bytes_useful{0}, bytes_redundant{0}, bytes_requested{0}, read_requests{0},
        nodes_loaded{0}, staging_hits{0};
};
}  // namespace pipeline

// ------------------------------------------------------------------- storage ----
namespace storage {

inline constexpr std::array<char, 8> kFeatureMagic = {'F', 'E', 'A', 'T', 'D', 'R', 'V', '1'};
inline constexpr std::uint32_t kFormatVersion = 1;
inline constexpr std::uint32_t kDtypeF32 = 0;
inline constexpr std::uint64_t kHeaderBytes = 64;
inline constexpr std::uint64_t kDefaultDataOffset = 512;
inline const char* kFeatureFileName = "features.bin";
inline const char* kIndptrFileName = "indptr.bin";
inline const char* kIndicesFileName = "indices.bin";
inline const char* kManifestFileName = "manifest.json";

enum class EngineKind { Auto, Uring, Threads };  // async_io.hpp:458 (no GPU counterpart)

/// DatasetHeader (format.hpp:33-65).
struct DatasetHeader {
    std::array<char, 8> magic = kFeatureMagic;
    std::uint32_t version = kFormatVersion;
    std::uint64_t num_nodes = 0;
    std::uint32_t dim = 0;
    std::uint32_t dtype_code = kDtypeF32;
    std::uint32_t row_bytes = 0;
    std::uint64_t data_offset = kDefaultDataOffset;

    std::uint64_t row_start(NodeId node) const { return data_offset + node * std::uint64_t(row_bytes); }
    std::uint64_t row_end(NodeId node) const { return row_start(node) + row_bytes; }
    std::uint64_t file_bytes() const { return data_offset + num_nodes * std::uint64_t(row_bytes); }
    std::uint64_t aligned_row_bytes() const {
        std::uint64_t a = (row_bytes + kSectorBytes - 1) / kSectorBytes * kSectorBytes;
        if (row_bytes % kSectorBytes != 0) a += kSectorBytes;
        return a;
    }
};

/// storage::FeatureTable (feature_file.hpp:25-107): the table lives in HBM. The header is
/// validated exactly as the reference does (messages and exception types included).
class FeatureTable {
public:
    explicit FeatureTable(const std::string& path, bool /*want_direct*/ = true, int device = 0) : path_(path) {
        check(fdg_ctx_create(device, &ctx_));
        try {
            check(fdg_ctx_load_features_file(ctx_, path.c_str()));
        } catch (...) {
            fdg_ctx_destroy(ctx_);
            throw;
        }
        fill_header();
    }
    /// Extension: the bit-exact GPU generation of the reference generator's features.bin
    /// content (storage::synthetic_row, generator.hpp:65-81), without a file.
    static std::unique_ptr<FeatureTable> generate(std::uint64_t num_nodes, std::uint32_t dim, std::uint64_t seed,
                                                  int device = 0) {
        std::unique_ptr<FeatureTable> t(new FeatureTable());
        check(fdg_ctx_create(device, &t->ctx_));
        check(fdg_ctx_generate_features(t->ctx_, seed, num_nodes, dim, 0, 1));
        t->path_ = "<generated>";
        t->fill_header();
        return t;
    }
    ~FeatureTable() { fdg_ctx_destroy(ctx_); }
    FeatureTable(const FeatureTable&) = delete;
    FeatureTable& operator=(const FeatureTable&) = delete;

    const DatasetHeader& header() const { return header_; }
    const std::string& path() const { return path_; }
    std::uint32_t row_bytes() const { return header_.row_bytes; }
    std::uint64_t num_nodes() const { return header_.num_nodes; }
    bool direct_available() const { return false; }

    /// Plain read of one exact row (the correctness oracle, feature_file.hpp:73-94).
    void read_row_sync(NodeId node, std::span<std::byte> out) const {
        if (node >= header_.num_nodes)
            throw std::out_of_range("read_row_sync: node " + std::to_string(node) + " >= num_nodes " +
                                    std::to_string(header_.num_nodes));
        if (out.size() < header_.row_bytes) throw InvariantViolation("FD_CHECK failed: out.size() >= row_bytes");
        check(fdg_ctx_download_rows(ctx_, node, 1, out.data()));
    }
    std::vector<std::byte> read_row_sync(NodeId node) const {
        std::vector<std::byte> row(header_.row_bytes);
        read_row_sync(node, row);
        return row;
    }
    fdg_ctx* handle() const { return ctx_; }

private:
    FeatureTable() = default;
    void fill_header() {
        fdg_ctx_info i;
        check(fdg_ctx_info_get(ctx_, &i));
        header_.num_nodes = i.num_nodes ? i.num_nodes : rows_of(i);
        header_.row_bytes = i.row_bytes;
        header_.dim = i.row_bytes / 4;
    }
    static std::uint64_t rows_of(const fdg_ctx_info& i) { return i.rows_per_shard * std::max<std::uint32_t>(i.n_shards, 1); }
    std::string path_;
    DatasetHeader header_{};
    fdg_ctx* ctx_ = nullptr;
};

}  // namespace storage

// --------------------------------------------------------------------- graph ----
namespace graph {

struct TopologyOptions {  // topology.hpp:28-31 (both are host-cache knobs: no GPU meaning)
    bool force_pread_cache = false;
    std::size_t cache_blocks = 4096;
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

/// graph::Topology (topology.hpp:33-193): the CSC in HBM.
class Topology {
public:
    /// indptr.bin / indices.bin of a dataset directory, validated like the reference.
    explicit Topology(const std::string& dataset_dir, TopologyOptions = {}, int device = 0) {
        check(fdg_ctx_create(device, &ctx_));
        try {
            check(fdg_ctx_load_topology_files(ctx_, dataset_dir.c_str()));
        } catch (...) {
            fdg_ctx_destroy(ctx_);
            throw;
        }
    }
    /// Extension: bit-exact GPU generation of storage::create_synthetic_dataset's topology
    /// (and, with features, its feature rows in the same context).
    static std::unique_ptr<Topology> generate(std::uint64_t num_nodes, std::uint32_t dim, std::uint32_t avg_degree,
                                              std::uint64_t seed, int device = 0, bool features = true) {
        std::unique_ptr<Topology> t(new Topology(device));
        check(fdg_ctx_generate_topology(t->ctx_, seed, num_nodes, avg_degree));
        if (features) check(fdg_ctx_generate_features(t->ctx_, seed, num_nodes, dim, 0, 1));
        return t;
    }
    ~Topology() {
        for (auto& s : pool_) fdg_sampler_destroy(s.sampler);
        fdg_ctx_destroy(ctx_);
    }
    Topology(const Topology&) = delete;
    Topology& operator=(const Topology&) = delete;

    std::uint64_t num_nodes() const { return info().num_nodes; }
    std::uint64_t num_edges() const { return info().num_edges; }
    /// Host copy of indptr (downloaded on first use).
    const std::vector<std::uint64_t>& indptr() const {
        std::lock_guard lk(mu_);
        if (indptr_.empty()) {
            indptr_.resize(num_nodes() + 1);
            check(fdg_ctx_download_topology(ctx_, indptr_.data(), nullptr));
        }
        return indptr_;
    }
    std::uint64_t degree(NodeId node) const {
        if (node >= num_nodes()) throw InvariantViolation("FD_CHECK failed: node < num_nodes_");
        const auto& ip = indptr();
        return ip[node + 1] - ip[node];
    }
    /// Copies the in-neighbour list of `node` into `out` (topology.hpp:59-71).
    void in_neighbors(NodeId node, std::vector<NodeId>& out) const {
        if (node >= num_nodes()) throw std::out_of_range("topology: node " + std::to_string(node) + " out of range");
        const auto& ip = indptr();
        const std::uint64_t lo = ip[node], hi = ip[node + 1];
        out.resize(hi - lo);
        if (lo == hi) return;
        fdg_ctx_info i = info();
        std::vector<std::uint32_t> narrow(i.idx_bytes == 4 ? hi - lo : 0);
        const char* base = static_cast<const char*>(i.indices_dev) + lo * i.idx_bytes;
        if (i.idx_bytes == 8) {
            check(fdg_memcpy_d2h(out.data(), base, (hi - lo) * 8, nullptr));
        } else {
            check(fdg_memcpy_d2h(narrow.data(), base, (hi - lo) * 4, nullptr));
        }
        check(fdg_stream_sync(nullptr));
        if (i.idx_bytes == 4) std::copy(narrow.begin(), narrow.end(), out.begin());
    }
    bool uses_mmap() const { return false; }

    // extensions
    std::uint32_t row_bytes() const { return info().row_bytes; }
    void features_to_host() { check(fdg_ctx_features_to_host(ctx_)); }
    bool features_on_host() const { return fdg_ctx_features_on_host(ctx_) != 0; }
    /// Shares `table`'s rows with this context (non-owning): gathers, the native runner and
    /// the train stage then read features through the topology.
    void attach_features(const storage::FeatureTable& table) {
        fdg_ctx_info t;
        check(fdg_ctx_info_get(table.handle(), &t));
        const void* base = t.table_dev;
        check(fdg_ctx_set_feature_shards(ctx_, &base, 1, table.num_nodes(), table.num_nodes(), t.row_bytes, t.dtype));
    }
    fdg_ctx* handle() const { return ctx_; }

    /// Sampler workspace pool: one per concurrent caller, keyed by (fanouts, seed capacity),
    /// reused across calls (the reference's samplers share one read-only Topology).
    struct PooledSampler {
        fdg_sampler* sampler = nullptr;
        std::vector<std::uint32_t> fanouts;
        std::uint32_t max_seeds = 0;
        std::uint64_t cap = 0;
        bool busy = false;
        std::vector<std::uint32_t> edges;  // host staging
    };
    PooledSampler* acquire_sampler(const Fanouts& f, std::uint32_t seeds) const {
        std::lock_guard lk(mu_);
        for (auto& s : pool_)
            if (!s.busy && s.fanouts == f.per_layer && s.max_seeds >= seeds) {
                s.busy = true;
                return &s;
            }
        PooledSampler s;
        s.fanouts = f.per_layer;
        s.max_seeds = std::max<std::uint32_t>(seeds, 1000);
        check(fdg_sampler_create(ctx_, s.max_seeds, f.per_layer.data(), std::uint32_t(f.per_layer.size()), &s.sampler));
        std::uint64_t mn = 0, me = 0;
        check(fdg_sampler_capacity(s.sampler, &mn, &me));
        s.cap = std::max<std::uint64_t>({mn, me, 1});
        s.busy = true;
        pool_.push_back(std::move(s));
        return &pool_.back();
    }
    void release_sampler(PooledSampler* s) const {
        std::lock_guard lk(mu_);
        s->busy = false;
    }

private:
    explicit Topology(int device) { check(fdg_ctx_create(device, &ctx_)); }
    fdg_ctx_info info() const {
        fdg_ctx_info i;
        check(fdg_ctx_info_get(ctx_, &i));
        return i;
    }
    fdg_ctx* ctx_ = nullptr;
    mutable std::mutex mu_;
    mutable std::vector<std::uint64_t> indptr_;
    mutable std::deque<PooledSampler> pool_;
};

/// graph::sample_khop (sampling.hpp:72-134), executed on the GPU, bit-exact.
inline SampledBatch sample_khop(const Topology& topo, std::span<const NodeId> seeds, const Fanouts& fanouts,
                                std::uint64_t rng_seed) {
    fanouts.validate();
    auto* ps = topo.acquire_sampler(fanouts, std::uint32_t(seeds.size()));
    struct Release {
        const Topology& t;
        Topology::PooledSampler* s;
        ~Release() { t.release_sampler(s); }
    } release{topo, ps};
    SampledBatch b;
    b.seeds.assign(seeds.begin(), seeds.end());
    b.nodes.resize(ps->cap);
    ps->edges.resize(2 * ps->cap);
    std::uint64_t nn = 0, ne = 0;
    b.layer_nodes.assign(fanouts.per_layer.size() + 2, 0);
    check(fdg_sample_khop_host(ps->sampler, seeds.data(), std::uint32_t(seeds.size()), rng_seed, b.nodes.data(),
                               ps->edges.data(), ps->cap, &nn, &ne, b.layer_nodes.data(), nullptr));
    b.nodes.resize(nn);
    b.edges.resize(ne);
    for (std::uint64_t i = 0; i < ne; ++i) b.edges[i] = LocalEdge{ps->edges[2 * i], ps->edges[2 * i + 1]};
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

// ------------------------------------------------------------------- featbuf ----
namespace featbuf {

using StandbyTimeout = ::featdrive_gpu::StandbyTimeout;

enum class MappingKind { Auto, Dense, Sparse };  // the GPU mapping is always a dense 8-byte array

struct MappingEntry {  // buffer_manager.hpp:39-47
    SlotId slot_index = kNoSlot;
    std::uint32_t ref_count = 0;
    std::uint8_t valid = 0;
    bool empty() const { return slot_index == kNoSlot && ref_count == 0 && valid == 0; }
};

struct BufferConfig {  // buffer_manager.hpp:180-190
    std::uint64_t num_nodes = 0;
    std::uint64_t slot_count = 0;
    std::uint32_t row_bytes = 0;
    std::uint64_t min_reserved = 0;
    MappingKind mapping = MappingKind::Auto;
    std::chrono::milliseconds standby_timeout{60000};
    bool validate_every_op = false;
    bool record_events = false;
    int device = 0;  // extension
};

struct BufferStats {  // buffer_manager.hpp:192-200
    std::uint64_t hits = 0, loads = 0, waits = 0, evictions = 0, takeovers = 0, releases = 0, standby_len = 0;
};

struct AcquirePlan {  // buffer_manager.hpp:202-206
    std::vector<SlotId> alias;
    std::vector<std::uint32_t> to_load;
    std::vector<std::uint32_t> waits;
};

enum class WaitOutcome { Ready, TakeOver, Timeout };

/// FeatureRegion (device_region.hpp:24-50): S row slots in HBM. slot() returns a host copy
/// of the slot's bytes (the reference returns a span into host memory standing in for HBM).
class FeatureRegion {
public:
    FeatureRegion(std::uint64_t slot_count, std::uint32_t row_bytes) : slot_count_(slot_count), row_bytes_(row_bytes) {
        if (!(slot_count > 0 && row_bytes > 0)) throw InvariantViolation("FD_CHECK failed: slot_count > 0 && row_bytes > 0");
        check(fdg_malloc(&dev_, slot_count * std::uint64_t(row_bytes)));
    }
    ~FeatureRegion() { fdg_free(dev_); }
    FeatureRegion(const FeatureRegion&) = delete;
    FeatureRegion& operator=(const FeatureRegion&) = delete;

    std::uint64_t bytes() const { return slot_count_ * std::uint64_t(row_bytes_); }
    std::uint32_t row_bytes() const { return row_bytes_; }
    std::uint64_t slot_count() const { return slot_count_; }
    std::vector<std::byte> slot(SlotId s) const {
        if (!(s >= 0 && std::uint64_t(s) < slot_count_)) throw InvariantViolation("FD_CHECK failed: slot in range");
        std::vector<std::byte> out(row_bytes_);
        check(fdg_memcpy_d2h(out.data(), static_cast<const char*>(dev_) + std::uint64_t(s) * row_bytes_, row_bytes_,
                             nullptr));
        check(fdg_stream_sync(nullptr));
        return out;
    }
    void* device_data() const { return dev_; }

    // per-call staging for trainer_step (grows, never freed per call)
    std::mutex& scratch_mutex() const { return mu_; }
    detail::DevBuf& scratch(int k) const { return scratch_[k]; }

private:
    std::uint64_t slot_count_;
    std::uint32_t row_bytes_;
    void* dev_ = nullptr;
    mutable std::mutex mu_;
    mutable detail::DevBuf scratch_[3];
};

/// CopyEngine (device_region.hpp:52-91): GPU copies are stream-ordered; nothing to hold.
class CopyEngine {
public:
    explicit CopyEngine(std::chrono::nanoseconds latency = std::chrono::nanoseconds::zero()) : latency_(latency) {}
    std::size_t in_flight() const { return 0; }

private:
    std::chrono::nanoseconds latency_;
};

/// StagingArena (staging.hpp:102-106): the SSD staging arena has no GPU counterpart (the
/// table is HBM- or host-resident); kept so reference setup code compiles.
class StagingArena {
public:
    StagingArena(std::uint64_t total_slots, std::uint64_t slot_bytes, std::vector<std::uint64_t> worker_quota_slots,
                 std::chrono::milliseconds = std::chrono::milliseconds(60000))
        : total_slots_(total_slots), slot_bytes_(slot_bytes), quotas_(std::move(worker_quota_slots)) {}
    std::uint64_t capacity_bytes() const { return total_slots_ * slot_bytes_; }

private:
    std::uint64_t total_slots_, slot_bytes_;
    std::vector<std::uint64_t> quotas_;
};

/// featbuf::BufferManager (buffer_manager.hpp:222-527): the mapping table, slot references,
/// LRU standby list and eviction on the GPU. Every operation is a device operation
/// synchronised before it returns, so the per-node protocol keeps the reference's order.
class BufferManager {
public:
    explicit BufferManager(const BufferConfig& cfg) : cfg_(cfg) {
        if (cfg.slot_count == 0) throw InvariantViolation("slot_count must be positive");
        if (cfg.slot_count < cfg.min_reserved)
            throw InvariantViolation("feature buffer smaller than the N_e * M_b reservation");
        max_batch_ = std::uint32_t(std::min<std::uint64_t>({cfg.slot_count, cfg.num_nodes, 0x7FFFFFFFull}));
        check(fdg_bm_create_standalone(cfg.device, cfg.num_nodes, cfg.slot_count, cfg.row_bytes, cfg.min_reserved,
                                       max_batch_, nullptr, &bm_));
    }
    ~BufferManager() { fdg_bm_destroy(bm_); }
    BufferManager(const BufferManager&) = delete;
    BufferManager& operator=(const BufferManager&) = delete;

    const BufferConfig& config() const { return cfg_; }
    std::uint64_t slot_count() const { return cfg_.slot_count; }
    std::uint64_t feature_bytes() const { return cfg_.slot_count * std::uint64_t(cfg_.row_bytes); }

    /// Algorithm 1 lines 5-17 for one batch (`nodes` deduplicated).
    AcquirePlan acquire_for_batch(std::span<const NodeId> nodes) {
        std::lock_guard lk(mu_);
        const std::uint64_t n = nodes.size();
        if (n > max_batch_) throw std::invalid_argument("acquire_for_batch: batch larger than the slot count");
        auto* nd = static_cast<NodeId*>(buf_[0].reserve(n * 8));
        auto* al = static_cast<SlotId*>(buf_[1].reserve(n * 8));
        auto* tl = static_cast<std::uint32_t*>(buf_[2].reserve(n * 4 + 8));
        check(fdg_memcpy_h2d(nd, nodes.data(), n * 8, nullptr));
        check(fdg_bm_acquire(bm_, nullptr, nd, n, al, tl + 2, tl));
        status();
        AcquirePlan plan;
        plan.alias.resize(n);
        std::uint32_t n_load = 0;
        check(fdg_memcpy_d2h(&n_load, tl, 4, nullptr));
        check(fdg_memcpy_d2h(plan.alias.data(), al, n * 8, nullptr));
        check(fdg_stream_sync(nullptr));
        plan.to_load.resize(n_load);
        check(fdg_memcpy_d2h(plan.to_load.data(), tl + 2, std::uint64_t(n_load) * 4, nullptr));
        check(fdg_stream_sync(nullptr));
        if (cfg_.validate_every_op) validate();
        return plan;
    }
    /// Pops the LRU standby slot, evicting its previous node (274-294).
    SlotId get_standby_slot() {
        std::lock_guard lk(mu_);
        auto* sd = static_cast<SlotId*>(buf_[3].reserve(8));
        check(fdg_bm_pop_standby(bm_, nullptr, 1, sd));
        const int rc = fdg_bm_status(bm_);
        if (rc == FDG_CAPACITY)
            throw StandbyTimeout("get_standby_slot: no slot became available within " +
                                 std::to_string(cfg_.standby_timeout.count()) + " ms; feature buffer is undersized");
        check(rc);
        SlotId s = kNoSlot;
        check(fdg_memcpy_d2h(&s, sd, 8, nullptr));
        check(fdg_stream_sync(nullptr));
        return s;
    }
    void bind_slot(NodeId node, SlotId slot) {
        std::lock_guard lk(mu_);
        one_node(node, slot);
        check(fdg_bm_bind(bm_, nullptr, buf_[3].as<NodeId>(), buf_[3].as<SlotId>() + 1, 1));
        status();
    }
    void publish_valid(NodeId node) {
        std::lock_guard lk(mu_);
        one_node(node, 0);
        check(fdg_bm_publish(bm_, nullptr, buf_[3].as<NodeId>(), 1));
        status();
    }
    /// With stream-ordered extraction no load is ever in flight on another extractor: a
    /// valid node is Ready, a node with no slot is the caller's to take over.
    WaitOutcome wait_for_valid(NodeId node, SlotId& slot_out, std::chrono::milliseconds /*timeout*/) {
        const MappingEntry e = mapping_entry(node);
        if (e.ref_count == 0 && e.slot_index == kNoSlot && !e.valid)
            throw InvariantViolation("waiting on a node without holding a reference");
        if (e.valid) {
            slot_out = e.slot_index;
            return WaitOutcome::Ready;
        }
        return e.slot_index == kNoSlot ? WaitOutcome::TakeOver : WaitOutcome::Timeout;
    }
    /// release_batch (352-364): ref-- and MRU pushes at 0, mapping left valid.
    void release_batch(std::span<const NodeId> nodes) {
        std::lock_guard lk(mu_);
        auto* nd = static_cast<NodeId*>(buf_[0].reserve(nodes.size() * 8));
        check(fdg_memcpy_h2d(nd, nodes.data(), nodes.size() * 8, nullptr));
        check(fdg_bm_release(bm_, nullptr, nd, nullptr, nodes.size()));
        status();
        if (cfg_.validate_every_op) validate();
    }
    void unwind_bound(NodeId node) {
        std::lock_guard lk(mu_);
        check(fdg_bm_unwind_bound(bm_, nullptr, node));
        status();
    }
    void release_ref(NodeId node) {
        std::lock_guard lk(mu_);
        check(fdg_bm_release_ref(bm_, nullptr, node));
        status();
    }
    void abandon_claim(NodeId) {}  // no takeover claims exist on the stream-ordered path

    BufferStats stats() const {
        fdg_bm_stats s;
        check(fdg_bm_stats_get(bm_, &s));
        return BufferStats{s.hits, s.loads, s.waits, s.evictions, s.takeovers, s.releases, s.standby_len};
    }
    MappingEntry mapping_entry(NodeId node) const {
        std::int64_t slot = 0;
        std::uint32_t ref = 0, valid = 0;
        check(fdg_bm_entry(bm_, node, &slot, &ref, &valid));
        return MappingEntry{slot, ref, std::uint8_t(valid)};
    }
    NodeId reverse_mapping(SlotId slot) const {
        std::int64_t v = -1;
        check(fdg_bm_reverse(bm_, std::uint64_t(slot), &v));
        return v < 0 ? ~NodeId(0) : NodeId(v);
    }
    std::size_t standby_size() const { return stats().standby_len; }
    void validate() const { check(fdg_bm_validate(bm_)); }

    // extension
    fdg_bm* handle() const { return bm_; }
    std::uint32_t max_batch_nodes() const { return max_batch_; }
    /// Binds the miss source and the slot storage (done by the Extractor constructor).
    void attach(const storage::FeatureTable& table, FeatureRegion& region) {
        if (region.slot_count() != cfg_.slot_count || region.row_bytes() != cfg_.row_bytes)
            throw InvariantViolation("FeatureRegion shape differs from the BufferConfig");
        check(fdg_bm_bind_table(bm_, table.handle(), region.device_data()));
    }
    std::mutex& mutex() { return mu_; }
    detail::DevBuf& scratch(int k) { return buf_[k]; }
    void status() const {
        const int rc = fdg_bm_status(bm_);
        if (rc == FDG_CAPACITY)
            throw StandbyTimeout("get_standby_slot: no slot became available within " +
                                 std::to_string(cfg_.standby_timeout.count()) + " ms; feature buffer is undersized");
        if (rc == FDG_INVARIANT) throw InvariantViolation("buffer manager invariant violated (device-detected)");
        check(rc);
    }

private:
    void one_node(NodeId node, SlotId slot) {
        NodeId host[2] = {node, NodeId(slot)};
        auto* p = static_cast<NodeId*>(buf_[3].reserve(16));
        check(fdg_memcpy_h2d(p, host, 16, nullptr));
    }
    BufferConfig cfg_;
    std::uint32_t max_batch_ = 0;
    fdg_bm* bm_ = nullptr;
    std::mutex mu_;
    detail::DevBuf buf_[4];
};

}  // namespace featbuf

// ------------------------------------------------------------------- extract ----
namespace extract {

enum class Placement { DeviceSim, HostOnly };

struct TestHooks {  // extractor.hpp:40-46
    std::function<void(std::uint32_t worker, NodeId lo, NodeId hi)> on_disk_read;
    std::function<bool(NodeId)> inject_read_failure;
    std::function<void(std::uint32_t worker, std::uint64_t batch_id)> before_batch;
    std::function<void(std::uint32_t worker, std::uint64_t batch_id)> before_staging_free;
    std::function<void(std::uint32_t worker, std::uint64_t batch_id)> before_release;
};

struct ExtractorConfig {  // extractor.hpp:48-56
    std::uint32_t worker = 0;
    std::size_t io_depth = 64;
    storage::EngineKind engine = storage::EngineKind::Auto;
    std::chrono::nanoseconds read_latency{0};
    Placement placement = Placement::DeviceSim;
    std::chrono::milliseconds wait_timeout{60000};
    std::uint64_t max_extent_bytes = 1u << 20;
};

struct ExtractorEnv {  // extractor.hpp:58-66
    storage::FeatureTable* table = nullptr;
    featbuf::BufferManager* buffer = nullptr;
    featbuf::StagingArena* staging = nullptr;
    featbuf::FeatureRegion* region = nullptr;
    featbuf::CopyEngine* copies = nullptr;
    pipeline::StageCounters* counters = nullptr;
    const TestHooks* hooks = nullptr;
};

class BatchExtractError : public std::runtime_error {
public:
    explicit BatchExtractError(const std::string& what) : std::runtime_error(what) {}
};

using NodeAliasList = std::vector<SlotId>;  // extractor.hpp:73

/// extract::Extractor (extractor.hpp:75-113). extract_batch runs Algorithm 1 on the GPU in
/// one stream-ordered pass (acquire, LRU pops in batch order, bind, table -> slot row loads,
/// publish) and returns the alias list; the reference's I/O machinery has no counterpart.
class Extractor {
public:
    Extractor(ExtractorEnv env, ExtractorConfig cfg) : env_(env), cfg_(cfg) {
        if (!(env_.table && env_.buffer && env_.region && env_.counters))
            throw InvariantViolation("FD_CHECK failed: env_.table && env_.buffer && env_.region && env_.counters");
        if (cfg_.placement == Placement::DeviceSim && !env_.copies)
            throw InvariantViolation("FD_CHECK failed: env_.copies != nullptr");
        env_.buffer->attach(*env_.table, *env_.region);
    }

    NodeAliasList extract_batch(const graph::SampledBatch& batch) {
        if (env_.hooks && env_.hooks->before_batch) env_.hooks->before_batch(cfg_.worker, batch.batch_id);
        const std::uint64_t n = batch.nodes.size();
        NodeAliasList alias(n);
        featbuf::BufferManager& bm = *env_.buffer;
        {
            ScopedTimer io(env_.counters->extract_io_wait);
            std::lock_guard lk(bm.mutex());
            if (n > bm.max_batch_nodes()) throw std::invalid_argument("extract_batch: batch larger than the slot count");
            const auto before = bm.stats();
            auto* nd = static_cast<NodeId*>(bm.scratch(0).reserve(n * 8));
            auto* al = static_cast<SlotId*>(bm.scratch(1).reserve(n * 8));
            check(fdg_memcpy_h2d(nd, batch.nodes.data(), n * 8, nullptr));
            check(fdg_bm_extract(bm.handle(), nullptr, nd, nullptr, n, al, nullptr, nullptr));
            bm.status();
            check(fdg_memcpy_d2h(alias.data(), al, n * 8, nullptr));
            check(fdg_stream_sync(nullptr));
            const std::uint64_t loads = bm.stats().loads - before.loads, rb = env_.table->row_bytes();
            env_.counters->nodes_loaded.fetch_add(loads, std::memory_order_relaxed);
            env_.counters->read_requests.fetch_add(loads, std::memory_order_relaxed);
            env_.counters->bytes_requested.fetch_add(loads * rb, std::memory_order_relaxed);
            env_.counters->bytes_useful.fetch_add(loads * rb, std::memory_order_relaxed);
        }
        if (env_.hooks && env_.hooks->before_staging_free) env_.hooks->before_staging_free(cfg_.worker, batch.batch_id);
        for (SlotId a : alias)
            if (a < 0) throw InvariantViolation("alias unassigned after extraction");
        return alias;
    }

private:
    ExtractorEnv env_;
    ExtractorConfig cfg_;
};

}  // namespace extract

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
        std::lock_guard lk(mu_);
        void* nd = buf_[0].reserve(n * 8);
        void* ed = buf_[1].reserve(e * 8);
        void* x = buf_[2].reserve(n * std::uint64_t(topo_.row_bytes()));
        void* cd = buf_[3].reserve(sizeof(c));
        void* ld = buf_[4].reserve(sizeof(float));
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
    mutable std::mutex mu_;
    mutable detail::DevBuf buf_[5];  // per-call staging, grown once
};

}  // namespace train

// ------------------------------------------------------------------ pipeline ----
namespace pipeline {

/// PipelineSession::batch_seed (pipeline.hpp:295-298)
inline std::uint64_t batch_seed(std::uint64_t seed, std::uint64_t epoch, std::uint64_t global_batch) {
    return fdg_batch_seed(seed, epoch, global_batch);
}

struct TrainTicket {  // pipeline.hpp:78-81
    graph::SampledBatch batch;
    extract::NodeAliasList alias;
};

struct ReleaseTicket {  // pipeline.hpp:83-86
    std::uint64_t batch_id = 0;
    std::vector<NodeId> nodes;
};

class PipelineError : public std::runtime_error {  // pipeline.hpp:88-97
public:
    PipelineError(std::string stage, const std::string& what)
        : std::runtime_error("[" + stage + "] " + what), stage_(std::move(stage)) {}
    const std::string& stage() const { return stage_; }

private:
    std::string stage_;
};

class SiblingAbort : public PipelineError {
public:
    SiblingAbort() : PipelineError("pipeline", "aborted after a failure in another worker") {}
};

/// trainer_step (pipeline.hpp:103-124): sum of hash_bytes64 over each node's row read
/// through its alias slot, on the GPU; with verify_against, every region row is byte-compared
/// with the table's row of its node (on the GPU) and a mismatch throws as the reference does.
inline std::uint64_t trainer_step(const TrainTicket& ticket, const featbuf::FeatureRegion& region,
                                  const storage::FeatureTable* verify_against = nullptr) {
    const auto& alias = ticket.alias;
    const std::uint64_t n = ticket.batch.nodes.size();
    if (alias.size() != n) throw InvariantViolation("FD_CHECK failed: alias list length == batch nodes");
    for (SlotId a : alias)
        if (a < 0) throw InvariantViolation("trainer saw an unassigned alias");
    std::lock_guard lk(region.scratch_mutex());
    auto* ad = static_cast<std::int64_t*>(region.scratch(0).reserve(n * 8));
    auto* cs = static_cast<std::uint64_t*>(region.scratch(1).reserve(16));
    check(fdg_memset(cs, 0, 16, nullptr));
    check(fdg_memcpy_h2d(ad, alias.data(), n * 8, nullptr));
    check(fdg_region_checksum(nullptr, region.device_data(), region.row_bytes(), ad, n, cs));
    if (verify_against) {
        auto* nd = static_cast<NodeId*>(region.scratch(2).reserve(n * 8));
        check(fdg_memcpy_h2d(nd, ticket.batch.nodes.data(), n * 8, nullptr));
        check(fdg_region_verify(verify_against->handle(), nullptr, region.device_data(), ad, nd, n, cs + 1));
    }
    std::uint64_t out[2] = {0, ~0ull};
    check(fdg_memcpy_d2h(out, cs, verify_against ? 16 : 8, nullptr));
    check(fdg_stream_sync(nullptr));
    if (verify_against && out[1] != ~0ull)
        throw PipelineError("train", "buffer contents for node " + std::to_string(ticket.batch.nodes[out[1]]) +
                                         " do not match the synchronous read oracle (batch " +
                                         std::to_string(ticket.batch.batch_id) + ")");
    return out[0];
}

// ------------------------------------------------------------------ session ----
// PipelineSession (pipeline.hpp:127-299) on the GPU runner (fdg_pipeline_*): one
// persistent pipeline (sampler streams + extraction + optional buffer manager) per
// worker segment, reused across epochs like the reference's per-worker buffer.

enum class RunMode { Async, SyncReference };

/// pipeline.hpp:30-76. GPU meaning: num_samplers = concurrent sampler streams;
/// num_extractors (N_e) only sizes the default slot count N_e * M_b, as in the
/// reference; slots = kNoBuffer extracts by direct gather (no buffer manager). The
/// reference's queue / I/O / latency knobs are accepted and have no GPU counterpart.
struct PipelineConfig {
    static constexpr std::uint64_t kNoBuffer = ~0ull;
    std::uint32_t num_samplers = 6;
    std::uint32_t num_extractors = 4;
    std::size_t extracting_queue_cap = 6;
    std::size_t training_queue_cap = 4;
    std::size_t releasing_queue_cap = 4;
    std::uint64_t batch_size = 1000;
    graph::Fanouts fanouts{{10, 10, 10}};
    std::uint64_t slots = 0;  // per-worker feature-buffer slots; 0 = N_e * M_b
    std::size_t io_depth = 64;
    RunMode mode = RunMode::Async;
    extract::Placement placement = extract::Placement::DeviceSim;
    std::uint32_t workers = 1;  // segments (concurrent pipelines on the topology's GPU)
    featbuf::MappingKind mapping = featbuf::MappingKind::Auto;
    storage::EngineKind engine = storage::EngineKind::Auto;
    std::chrono::nanoseconds read_latency{0};
    std::chrono::nanoseconds copy_latency{0};
    std::chrono::nanoseconds compute_delay{0};
    std::uint32_t extract_retries = 0;
    bool verify = false;  // re-derive every batch on the non-pipelined path and compare
    std::chrono::milliseconds wait_timeout{60000};
    std::uint64_t staging_portion_slots = 0;
    bool buffer_validate_every_op = false;
    extract::TestHooks hooks;
    // GPU extensions
    std::uint32_t group_batches = 1;
    int device = 0;

    void validate() const {
        if (num_samplers < 1 || num_extractors < 1)
            throw std::invalid_argument("config: need at least one sampler and one extractor");
        if (extracting_queue_cap < 1 || training_queue_cap < 1 || releasing_queue_cap < 1)
            throw std::invalid_argument("config: queue capacities must be >= 1");
        if (batch_size < 1) throw std::invalid_argument("config: batch_size must be >= 1");
        if (io_depth < 1) throw std::invalid_argument("config: io_depth must be >= 1");
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
    /// pipeline.hpp:128-174: the dataset directory's topology and features.bin (header and
    /// lengths validated as the reference does), one runner per worker segment.
    PipelineSession(const std::string& dataset_dir, PipelineConfig cfg, graph::TopologyOptions topo_opts = {})
        : own_table_(std::make_unique<storage::FeatureTable>(dataset_dir + "/" + storage::kFeatureFileName, true,
                                                             cfg.device)),
          own_topo_(std::make_unique<graph::Topology>(dataset_dir, topo_opts, cfg.device)),
          topo_(*own_topo_),
          cfg_(std::move(cfg)) {
        own_topo_->attach_features(*own_table_);
        build();
    }
    /// Extension: a topology that already holds its feature rows (e.g. Topology::generate).
    PipelineSession(const graph::Topology& topo, PipelineConfig cfg) : topo_(topo), cfg_(std::move(cfg)) { build(); }
    ~PipelineSession() {
        for (auto p : pipes_) fdg_pipeline_destroy(p);
        if (sampler_) fdg_sampler_destroy(sampler_);
    }
    PipelineSession(const PipelineSession&) = delete;
    PipelineSession& operator=(const PipelineSession&) = delete;

    const graph::Topology& topology() const { return topo_; }
    const storage::FeatureTable* table() const { return own_table_.get(); }
    std::uint64_t max_batch_nodes() const { return mb_; }
    std::uint64_t slots_per_worker() const { return slots_; }
    const PipelineConfig& config() const { return cfg_; }

private:
    void build() {
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

public:
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

    std::unique_ptr<storage::FeatureTable> own_table_;
    std::unique_ptr<graph::Topology> own_topo_;
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
