// set_loop.cpp -- the reference's SET loop for one worker (pipeline.hpp:419-543: the calls
// the sampler / extractor / trainer / releaser threads make), run sequentially on a dataset
// directory, written against the reference's API. It builds against either header; only
// the include and the top-level namespace differ:
//
//   g++ -DFEATDRIVE_REFERENCE -I/root/reference/proj/include ...  -> the reference (CPU)
//   g++ -Iinclude ... -lfdg                                          -> featdrive_gpu (B200)
//
//   set_loop DATASET_DIR SLOTS [BATCHES]
//     prints, per batch: "batch nodes edges checksum hits loads evictions", then one batch
//     driven through the per-node protocol (acquire_for_batch, get_standby_slot, bind_slot,
//     publish_valid) and the reference's error behaviour for an out-of-range seed.
//   set_loop --generate N:DIM:AVG:SEED SLOTS BATCHES     (featdrive_gpu only)
//     the same loop at batch 1000 / fanout (10,10,10) on a dataset generated in HBM (the
//     bench's Papers shape); prints "per_call <batches/s>".
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <string>

#ifdef FEATDRIVE_REFERENCE
#include "featdrive/extract/extractor.hpp"
#include "featdrive/graph/sampling.hpp"
#include "featdrive/graph/topology.hpp"
#include "featdrive/pipeline/pipeline.hpp"
#include "featdrive/storage/feature_file.hpp"
namespace fd = featdrive;
#else
#include "featdrive_gpu.hpp"
namespace fd = featdrive_gpu;
#endif

using namespace fd;

namespace {

struct LoopResult {
    double seconds = 0;
    std::uint64_t batches = 0;
};

// One worker's stages, in order, per batch: sample_khop -> extract_batch -> trainer_step ->
// release_batch, with the reference's objects (buffer, region, copy engine, staging, counters).
LoopResult set_loop(const graph::Topology& topo, storage::FeatureTable& table, std::uint64_t slots,
                    std::uint64_t n_batches, bool print, std::uint64_t batch_size = 20,
                    std::vector<std::uint32_t> fanouts = {3, 3}) {
    pipeline::PipelineConfig cfg;
    cfg.batch_size = batch_size;
    cfg.fanouts = graph::Fanouts{fanouts};
    const std::uint64_t seed = 0, epoch = 0;
    const auto& h = table.header();
    const std::uint64_t mb = cfg.max_batch_nodes(h.num_nodes);
    featbuf::BufferConfig bc;
    bc.num_nodes = h.num_nodes;
    bc.slot_count = slots;
    bc.row_bytes = h.row_bytes;
    bc.min_reserved = mb;
    featbuf::BufferManager buffer(bc);
    featbuf::FeatureRegion region(slots, h.row_bytes);
    featbuf::CopyEngine copies;
    featbuf::StagingArena staging(mb, h.aligned_row_bytes(), std::vector<std::uint64_t>{mb});
    pipeline::StageCounters counters;
    extract::ExtractorEnv env;
    env.table = &table;
    env.buffer = &buffer;
    env.staging = &staging;
    env.region = &region;
    env.copies = &copies;
    env.counters = &counters;
    extract::ExtractorConfig ec;
    ec.engine = storage::EngineKind::Threads;
    extract::Extractor extractor(env, ec);

    std::vector<NodeId> train(cfg.batch_size * n_batches);
    std::iota(train.begin(), train.end(), NodeId(0));
    auto chunks = graph::partition_epoch(train, cfg.batch_size, hash_combine(seed, epoch));
    const auto t0 = std::chrono::steady_clock::now();
    for (std::uint64_t b = 0; b < chunks.size(); ++b) {
        auto batch = graph::sample_khop(topo, chunks[b], cfg.fanouts, pipeline::PipelineSession::batch_seed(seed, epoch, b));
        batch.batch_id = b;
        batch.epoch = epoch;
        auto alias = extractor.extract_batch(batch);
        pipeline::TrainTicket ticket{std::move(batch), std::move(alias)};
        const std::uint64_t checksum = pipeline::trainer_step(ticket, region, print && b % 2 ? &table : nullptr);
        buffer.release_batch(ticket.batch.nodes);
        if (print) {
            const auto st = buffer.stats();
            std::printf("%llu %zu %zu %llu %llu %llu %llu\n", (unsigned long long)b, ticket.batch.nodes.size(),
                        ticket.batch.edges.size(), (unsigned long long)checksum, (unsigned long long)st.hits,
                        (unsigned long long)st.loads, (unsigned long long)st.evictions);
        }
    }
    LoopResult r;
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r.batches = chunks.size();
    if (!print) return r;
    buffer.validate();

    // The per-node protocol of one more batch (Extractor::run_ticket's metadata order,
    // extractor.hpp:142-151, 391-394): pops in batch order, bind, publish.
    auto extra = graph::sample_khop(topo, chunks[0], graph::Fanouts{{4, 2}}, 12345);
    auto plan = buffer.acquire_for_batch(extra.nodes);
    for (auto pos : plan.to_load) {
        const SlotId s = buffer.get_standby_slot();
        buffer.bind_slot(extra.nodes[pos], s);
        plan.alias[pos] = s;
    }
    for (auto pos : plan.to_load) buffer.publish_valid(extra.nodes[pos]);
    unsigned long long acc = 0;
    for (std::size_t i = 0; i < plan.alias.size(); ++i) acc = acc * 1000003ull + std::uint64_t(plan.alias[i]);
    const auto st = buffer.stats();
    std::printf("protocol %zu %zu %llu %llu %llu %llu\n", extra.nodes.size(), plan.to_load.size(), acc,
                (unsigned long long)st.hits, (unsigned long long)st.loads, (unsigned long long)st.evictions);
    buffer.release_batch(extra.nodes);
    const auto e = buffer.mapping_entry(extra.nodes[0]);
    std::printf("entry %lld %u %u standby %zu\n", (long long)e.slot_index, e.ref_count, unsigned(e.valid),
                buffer.standby_size());
    buffer.validate();

    // reference error behaviour: an out-of-range seed throws std::out_of_range
    std::vector<NodeId> bad{1, h.num_nodes + 5};
    try {
        graph::sample_khop(topo, bad, cfg.fanouts, 1);
        std::printf("no exception\n");
    } catch (const std::out_of_range&) {
        std::printf("out_of_range ok\n");
    }
    return r;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: set_loop DATASET_DIR SLOTS [BATCHES]\n");
        return 2;
    }
    try {
        if (std::string(argv[1]) == "--generate") {
#ifdef FEATDRIVE_REFERENCE
            std::fprintf(stderr, "--generate is a featdrive_gpu extension\n");
            return 2;
#else
            // per-call throughput of this loop on a dataset generated in HBM (bench.py per_call)
            unsigned long long n = 0, dim = 0, avg = 0, seed = 0;
            if (std::sscanf(argv[2], "%llu:%llu:%llu:%llu", &n, &dim, &avg, &seed) != 4) return 2;
            const std::uint64_t gslots = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 0;
            const std::uint64_t batches = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 100;
            auto topo = graph::Topology::generate(n, std::uint32_t(dim), std::uint32_t(avg), seed, 0, false);
            auto table = storage::FeatureTable::generate(n, std::uint32_t(dim), seed);
            set_loop(*topo, *table, gslots, 4, false, 1000, {10, 10, 10});  // warm-up (pools, staging)
            const auto r = set_loop(*topo, *table, gslots, batches, false, 1000, {10, 10, 10});
            std::printf("per_call %.3f batches/s (%llu batches, %.3f s)\n", double(r.batches) / r.seconds,
                        (unsigned long long)r.batches, r.seconds);
            return 0;
#endif
        }
        const std::uint64_t slots = std::strtoull(argv[2], nullptr, 10);
        const std::uint64_t n_batches = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 8;
        const std::string dir = argv[1];
        graph::Topology topo(dir);
        storage::FeatureTable table(dir + "/" + storage::kFeatureFileName);
        set_loop(topo, table, slots, n_batches, true);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
