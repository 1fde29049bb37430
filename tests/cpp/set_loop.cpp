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
        // the train stage on the same blocks (extension: GraphSAGE forward + loss)
        {
            train::GraphSAGE model(*topo, {dim, 8, 4}, fan, std::uint32_t(batch));
            const std::uint32_t d[3] = {dim, 8, 4};
            for (std::uint32_t l = 0; l < 2; ++l) {
                std::vector<float> wn(d[l] * d[l + 1]), ws(d[l] * d[l + 1]), bias(d[l + 1]);
                for (std::uint32_t k = 0; k < d[l]; ++k)
                    for (std::uint32_t c = 0; c < d[l + 1]; ++c) {
                        wn[k * d[l + 1] + c] = float(int((k * 7 + c * 3) % 11) - 5) * 0.05f;
                        ws[k * d[l + 1] + c] = float(int((k * 5 + c * 2) % 13) - 6) * 0.04f;
                    }
                for (std::uint32_t c = 0; c < d[l + 1]; ++c) bias[c] = float(int(c % 3) - 1) * 0.1f;
                model.set_layer(l, wn, ws, bias);
            }
            for (std::uint64_t b = 0; b < 2; ++b) {
                auto sb = graph::sample_khop(*topo, chunks[b], fan, pipeline::batch_seed(0, 0, b));
                std::printf("loss %llu %.9g\n", (unsigned long long)b, double(model.forward(sb, 77)));
            }
        }
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
