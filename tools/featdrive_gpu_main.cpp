// featdrive_gpu_main.cpp -- `featdrive-gpu run`: the reference CLI's `run`
// subcommand (tools/featdrive_main.cpp:126-208, options 303-326) on the B200
// runtime. Same options where they carry over, same exit codes (0 ok, 2 config,
// 3 runtime), one JSON document per epoch on stdout (EpochStats::to_json plus a
// "manifest" object), progress on stderr.
//
//   featdrive-gpu run --dataset DIR [--batch-size N] [--fanout 10,10,10]
//                     [--samplers N] [--extractors N] [--slots auto|none|N]
//                     [--mode async|sync] [--epochs N] [--seed S] [--train-count N]
//                     [--workers N] [--verify] [--device D]
//   featdrive-gpu run --generate NODES:DIM:AVG_DEGREE[:SEED] ...   (dataset generated in HBM,
//                     bit-identical to the reference generator)
//
// Options of the reference that configure its CPU/SSD machinery (--eq-cap, --tq-cap,
// --rq-cap, --io-depth, --placement, --read/copy-latency-us, --retries, --mapping)
// are accepted and reported in the manifest but have no GPU counterpart.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <numeric>
#include <string>

#include "featdrive_gpu.hpp"

namespace {

constexpr int kExitOk = 0, kExitConfig = 2, kExitRuntime = 3;

featdrive_gpu::graph::Fanouts parse_fanouts(const std::string& text) {
    featdrive_gpu::graph::Fanouts f;
    std::size_t at = 0;
    while (at < text.size()) {
        std::size_t comma = text.find(',', at);
        if (comma == std::string::npos) comma = text.size();
        f.per_layer.push_back(std::uint32_t(std::stoul(text.substr(at, comma - at))));
        at = comma + 1;
    }
    f.validate();
    return f;
}

std::string jstr(const std::string& s) { return "\"" + s + "\""; }

int usage() {
    std::fprintf(stderr,
                 "usage: featdrive-gpu run (--dataset DIR | --generate N:DIM:AVG[:SEED]) [--batch-size N] "
                 "[--fanout a,b,c] [--samplers N] [--extractors N] [--slots auto|none|N] [--mode async|sync] "
                 "[--epochs N] [--seed S] [--train-count N] [--workers N] [--verify] [--device D]\n");
    return kExitConfig;
}

}  // namespace

int main(int argc, char** argv) {
    using namespace featdrive_gpu;
    if (argc < 2 || std::string(argv[1]) != "run") return usage();
    std::map<std::string, std::string> opt = {
        {"batch-size", "1000"}, {"fanout", "10,10,10"}, {"samplers", "6"}, {"extractors", "4"},
        {"slots", "auto"},      {"mode", "async"},      {"epochs", "1"},   {"seed", "0"},
        {"train-count", "10000"}, {"workers", "1"},     {"device", "0"}};
    bool verify = false;
    static const char* ignored[] = {"eq-cap", "tq-cap", "rq-cap", "io-depth", "placement", "read-latency-us",
                                    "copy-latency-us", "compute-delay-ms", "retries", "mapping"};
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--", 0) != 0) return usage();
        a = a.substr(2);
        if (a == "verify") {
            verify = true;
            continue;
        }
        if (i + 1 >= argc) return usage();
        bool known = opt.count(a) || a == "dataset" || a == "generate";
        for (const char* k : ignored) known |= a == k;
        if (!known) {
            std::fprintf(stderr, "featdrive-gpu: unknown option --%s\n", a.c_str());
            return kExitConfig;
        }
        opt[a] = argv[++i];
    }
    try {
        pipeline::PipelineConfig cfg;
        cfg.batch_size = std::stoull(opt["batch-size"]);
        cfg.fanouts = parse_fanouts(opt["fanout"]);
        cfg.num_samplers = std::uint32_t(std::stoul(opt["samplers"]));
        cfg.num_extractors = std::uint32_t(std::stoul(opt["extractors"]));
        cfg.workers = std::uint32_t(std::stoul(opt["workers"]));
        cfg.verify = verify;
        if (opt["mode"] == "async")
            cfg.mode = pipeline::RunMode::Async;
        else if (opt["mode"] == "sync")
            cfg.mode = pipeline::RunMode::SyncReference;
        else
            throw std::invalid_argument("--mode must be async or sync");
        if (opt["slots"] == "none")
            cfg.slots = pipeline::PipelineConfig::kNoBuffer;
        else if (opt["slots"] != "auto")
            cfg.slots = std::stoull(opt["slots"]);
        cfg.validate();
        const int device = std::stoi(opt["device"]);
        const std::uint32_t epochs = std::uint32_t(std::stoul(opt["epochs"]));
        const std::uint64_t seed = std::stoull(opt["seed"]);

        cfg.device = device;
        std::unique_ptr<graph::Topology> topo;  // --generate: dataset in HBM (features in the same context)
        std::unique_ptr<pipeline::PipelineSession> session_ptr;
        std::string dataset_desc;
        if (opt.count("generate")) {
            std::string g = opt["generate"];
            std::vector<std::uint64_t> v;
            std::size_t at = 0;
            while (at <= g.size()) {
                std::size_t c = g.find(':', at);
                if (c == std::string::npos) c = g.size();
                v.push_back(std::stoull(g.substr(at, c - at)));
                at = c + 1;
            }
            if (v.size() < 3) throw std::invalid_argument("--generate wants NODES:DIM:AVG_DEGREE[:SEED]");
            topo = graph::Topology::generate(v[0], std::uint32_t(v[1]), std::uint32_t(v[2]), v.size() > 3 ? v[3] : 0,
                                             device);
            dataset_desc = "{\"generated\":{\"nodes\":" + std::to_string(v[0]) + ",\"dim\":" + std::to_string(v[1]) +
                           ",\"avg_degree\":" + std::to_string(v[2]) +
                           ",\"seed\":" + std::to_string(v.size() > 3 ? v[3] : 0) + "}}";
            session_ptr = std::make_unique<pipeline::PipelineSession>(*topo, cfg);
        } else if (opt.count("dataset")) {
            // PipelineSession(dataset_dir, cfg) as the reference CLI (pipeline.hpp:128-174)
            session_ptr = std::make_unique<pipeline::PipelineSession>(opt["dataset"], cfg);
            dataset_desc = jstr(opt["dataset"]);
        } else {
            return usage();
        }
        pipeline::PipelineSession& session = *session_ptr;
        const graph::Topology& topo_ref = session.topology();
        const std::uint64_t num_nodes = topo_ref.num_nodes();
        const std::uint64_t train_count = std::min<std::uint64_t>(std::stoull(opt["train-count"]), num_nodes);
        std::vector<NodeId> train_ids(train_count);
        std::iota(train_ids.begin(), train_ids.end(), NodeId(0));

        const auto now = std::chrono::system_clock::now().time_since_epoch();
        std::string manifest =
            "{\"build\":\"featdrive-gpu-1.0 (sm_100a)\",\"started_unix_ms\":" +
            std::to_string(std::chrono::duration_cast<std::chrono::milliseconds>(now).count()) +
            ",\"dataset\":" + dataset_desc + ",\"config\":{\"batch_size\":" + std::to_string(cfg.batch_size) +
            ",\"fanout\":" + jstr(opt["fanout"]) + ",\"samplers\":" + std::to_string(cfg.num_samplers) +
            ",\"extractors\":" + std::to_string(cfg.num_extractors) +
            ",\"slots\":" + std::to_string(session.slots_per_worker()) +
            ",\"max_batch_nodes\":" + std::to_string(session.max_batch_nodes()) + ",\"mode\":" + jstr(opt["mode"]) +
            ",\"workers\":" + std::to_string(cfg.workers) + ",\"epochs\":" + std::to_string(epochs) +
            ",\"seed\":" + std::to_string(seed) + ",\"train_count\":" + std::to_string(train_count) +
            ",\"verify\":" + (cfg.verify ? "true" : "false") + ",\"device\":" + std::to_string(device) + "}}";
        std::fprintf(stderr, "featdrive-gpu run: %llu nodes, %llu train ids, %u worker(s), mode %s\n",
                     (unsigned long long)num_nodes, (unsigned long long)train_count, cfg.workers, opt["mode"].c_str());
        std::fprintf(stderr, "  M_b=%llu  slots/worker=%llu  feature buffer %.2f MB\n",
                     (unsigned long long)session.max_batch_nodes(), (unsigned long long)session.slots_per_worker(),
                     double(session.slots_per_worker()) * topo_ref.row_bytes() / 1e6);
        std::uint64_t failed = 0;
        for (std::uint32_t epoch = 0; epoch < epochs; ++epoch) {
            std::string out;
            if (cfg.mode == pipeline::RunMode::SyncReference) {
                auto st = session.run_sync_reference(train_ids, epoch, seed);
                failed += st.batches_failed;
                out = st.to_json();
                std::fprintf(stderr, "  epoch %u [sync]: %.3f s, %llu batches\n", epoch, st.wall_time_s,
                             (unsigned long long)st.batches_trained);
            } else if (cfg.workers == 1) {
                auto st = session.run_epoch(train_ids, epoch, seed);
                failed += st.batches_failed;
                out = st.to_json();
                std::fprintf(stderr, "  epoch %u: %.3f s, %llu batches, hits %llu, loads %llu, read %.2f MB\n", epoch,
                             st.wall_time_s, (unsigned long long)st.batches_trained,
                             (unsigned long long)st.buffer.hits, (unsigned long long)st.buffer.loads,
                             double(st.bytes_requested) / 1e6);
            } else {
                auto all = session.run_epoch_multi(train_ids, epoch, seed);
                out = "{\"epoch\":" + std::to_string(epoch) + ",\"workers\":[";
                double wall = 0;
                for (std::size_t w = 0; w < all.size(); ++w) {
                    failed += all[w].batches_failed;
                    wall = std::max(wall, all[w].wall_time_s);
                    out += (w ? "," : "") + all[w].to_json();
                }
                out += "]}";
                std::fprintf(stderr, "  epoch %u: %.3f s across %u workers\n", epoch, wall, cfg.workers);
            }
            out.insert(out.size() - 1, ",\"manifest\":" + manifest);
            std::printf("%s\n", out.c_str());
            std::fflush(stdout);
        }
        if (failed) {
            std::fprintf(stderr, "featdrive-gpu run: %llu batch(es) failed extraction\n", (unsigned long long)failed);
            return kExitRuntime;
        }
        return kExitOk;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "featdrive-gpu: %s\n", e.what());
        return kExitConfig;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "featdrive-gpu: %s\n", e.what());
        return kExitRuntime;
    }
}
