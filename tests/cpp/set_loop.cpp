// set_loop.cpp -- the reference's SET loop shape (pipeline.hpp:419-543, run
// sequentially: sample -> extract -> train -> release with lag 1) written against
// include/featdrive_gpu.hpp, i.e. the drop-in boundary a featdrive user calls.
// Prints one line per batch: "batch nodes edges checksum hits loads evictions".
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "featdrive_gpu.hpp"

using namespace featdrive_gpu;

int main(int argc, char** argv) {
    const std::uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 5000;
    const std::uint32_t dim = argc > 2 ? std::uint32_t(std::atoi(argv[2])) : 16;
    const std::uint32_t avg = argc > 3 ? std::uint32_t(std::atoi(argv[3])) : 12;
    const std::uint64_t slots = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 900;
    const std::uint64_t batch = 20, n_batches = 8;
    try {
        auto topo = graph::Topology::generate(n, dim, avg, 7);
        std::vector<NodeId> train(batch * n_batches);
        std::iota(train.begin(), train.end(), 0);
        auto chunks = graph::partition_epoch(train, batch, 0x1234);
        graph::Fanouts fan{{3, 3}};
        featbuf::BufferManager buffer(*topo, slots, 0, std::uint32_t(fan.max_batch_nodes(batch)));
        extract::Extractor ex(buffer);
        std::vector<NodeId> prev;
        for (std::uint64_t b = 0; b < chunks.size(); ++b) {
            auto sb = graph::sample_khop(*topo, chunks[b], fan, pipeline::batch_seed(0, 0, b));
            auto alias = ex.extract_batch(sb);
            std::uint64_t cs = pipeline::trainer_step(sb, alias, buffer);
            if (!prev.empty()) buffer.release_batch(prev);
            prev = sb.nodes;
            auto st = buffer.stats();
            std::printf("%llu %zu %zu %llu %llu %llu %llu\n", (unsigned long long)b, sb.nodes.size(),
                        sb.edges.size(), (unsigned long long)cs, (unsigned long long)st.hits,
                        (unsigned long long)st.loads, (unsigned long long)st.evictions);
        }
        buffer.validate();
        // reference error behaviour: an out-of-range seed throws std::out_of_range
        std::vector<NodeId> bad{1, n + 5};
        try {
            graph::sample_khop(*topo, bad, fan, 1);
            std::printf("no exception\n");
            return 2;
        } catch (const std::out_of_range&) {
            std::printf("out_of_range ok\n");
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
