// fdg_pipeline.cu -- native SET-loop runner: the B200 counterpart of
// PipelineSession's sampler / extractor / trainer / releaser stages
// (pipeline.hpp:325-543) for one worker (= one GPU).
//
// Reference: 4 sampler threads, 4 extractor threads, 1 trainer, 1 releaser and
// bounded queues (pipeline.hpp:356-377). Here the "queues" are CUDA events
// between streams:
//   mt stream       : MT19937-64 streams for upcoming batches of each sampler,
//                     one CTA per batch, generated far ahead of use
//   S sampler streams: groups of G consecutive batches, round-robin over the
//                     samplers; one launch chain samples a whole group
//   extract stream  : per batch, the gather (or buffer-manager extract + lag-1
//                     release) into the mini-batch tensor, the optional fused
//                     trainer checksum and the optional D2H of the batch record
// so groups g+1..g+S are sampled while group g is extracted. Batch j is keyed
// exactly as the reference (rng seed = batch_seed(seed, epoch, global id)).
#include <cuda.h>
#include <cuda_profiler_api.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <vector>

#include "fdg_internal.cuh"

namespace fdg {
struct Sampler;
int sampler_create(Ctx* ctx, uint32_t max_seeds, const uint32_t* fanouts, uint32_t n_layers, Sampler** out,
                   uint32_t group);
void sampler_destroy(Sampler* s);
int sampler_prefetch(Sampler* s, cudaStream_t st, const uint64_t* rng_seeds, uint32_t n);
int sampler_reserve_ring(Sampler* s, uint32_t n);
int sampler_debug_zero_word(Sampler* s, cudaStream_t st, uint64_t rng_seed, uint64_t pos);
void sampler_debug_reject(Sampler* s, int lane);
int sampler_sample_group(Sampler* s, cudaStream_t st, uint32_t n, const uint64_t* const* seeds, const uint32_t* n_seeds,
                         const uint64_t* rng_seeds, uint64_t* const* nodes, uint32_t* const* edges, uint64_t cap,
                         fdg_batch_counts* const* cnt);
void sampler_capacity(const Sampler* s, uint64_t* max_nodes, uint64_t* max_edges);
void sampler_hash_region(const Sampler* s, void** base, uint64_t* bytes);
int bm_status_to(fdg_bm* b, cudaStream_t st, uint32_t* dst);
void sampler_set_lean(Sampler* s, bool lean);
int bm_extract_meta(fdg_bm* b, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                    int64_t* alias, uint32_t parity, cudaEvent_t after_acquire = nullptr);
int bm_extract_move(fdg_bm* b, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                    const int64_t* alias, void* out, uint64_t* checksum, uint32_t parity, int mode = 0);
int bm_release(fdg_bm* b, cudaStream_t st, const uint64_t* nodes, const int64_t* alias, const uint32_t* n_dev,
               uint64_t n_host);
}  // namespace fdg

struct fdg_pipeline {
    fdg::Ctx* ctx = nullptr;
    fdg_pipeline_config cfg{};
    std::vector<fdg::Sampler*> samplers;
    std::vector<cudaStream_t> sstream;
    std::vector<cudaStream_t> mstream;   // per-sampler MT prefetch streams
    cudaStream_t xstream = nullptr;
    cudaStream_t tstream = nullptr;      // train stage (plain extraction): batch j's model step overlaps
    cudaEvent_t gathered[2] = {}, trained[2] = {};  // the next gathers; per X parity
    CUgreenCtx green_s = nullptr;        // SM partitions (option sampler_sms): samplers + MT streams
    CUgreenCtx green_x = nullptr;        // ... and everything on the extraction streams
    cudaStream_t xstream2 = nullptr;     // second extraction stream (plain gathers alternate; with the
                                         // buffer manager: the row-move stream)
    cudaStream_t dstream = nullptr;      // option records_stream: batch records' D2H off the extraction streams
    std::vector<cudaEvent_t> rec_ev;     // ... one event per in-flight record
    cudaEvent_t bound[2] = {nullptr, nullptr};  // buffer manager: batch parity's metadata half done
    cudaEvent_t moved[2] = {nullptr, nullptr};  // buffer manager: batch parity's row move done
    cudaEvent_t acquired[2] = {nullptr, nullptr};  // buffer manager, split move: batch parity's acquire done
    uint64_t cap = 0, max_nodes = 0;
    uint32_t nslots = 0;             // per-batch output slots (2 * S * G)
    std::vector<uint64_t*> nodes;
    std::vector<uint32_t*> edges;
    std::vector<uint64_t*> seeds;    // per-slot staging for host seeds
    std::vector<int64_t*> alias;
    std::vector<void*> X;
    std::vector<cudaEvent_t> extracted;  // per slot
    std::vector<cudaEvent_t> sampled;    // per group slot (2 * S)
    fdg_batch_counts* counts = nullptr;  // device, one per batch of the current run
    uint64_t counts_cap = 0;
    std::vector<cudaEvent_t> tev;        // per-batch extract timing events (2 per batch)
    std::vector<cudaEvent_t> sev;        // per-group sampling timing events (2 per group)
    uint64_t timed_groups = 0;
    fdg_bm* bm = nullptr;
    bool l2_persist = false;             // this pipeline set aside persisting L2 (undone on destroy)
    fdg_sage* model = nullptr;           // optional train stage after each extraction
    uint64_t label_seed = 0;
    float lr = 0.f;                      // != 0: backward + SGD after every forward
    float* losses = nullptr;             // device, one per batch of the current run
    uint64_t losses_cap = 0;
    uint64_t loss_batches = 0;           // batches of the last run with a loss
    cudaEvent_t t0 = nullptr;            // start of the last run (timing base)
    uint64_t timed_batches = 0;          // batches of the last run with extraction events
};

using namespace fdg;

int64_t fdg::g_bm_overlap = 1;
int64_t fdg::g_bm_meta_prio = 0;
int64_t fdg::g_bm_move_early = 0;
int64_t fdg::g_extract_prio = 2;
int64_t fdg::g_records_stream = 1;
int64_t fdg::g_pipe_slots = 0;
int64_t fdg::g_bm_split_move = 0;  // e2e 5286 / 5256 -> 5300 / 5349 batches/s (Papers bench, 2 runs each)
int64_t fdg::g_sampler_sms = 0;
int64_t fdg::g_prefetch_upfront = 0;    // A/B: all samplers' first MT chunks before any sampling
int64_t fdg::g_debug_zero_word = -1;     // (batch of the run << 24) | word position; -1 = off
int64_t fdg::g_debug_reject_batch = -1;  // batch of the run flagged as rejected; -1 = off

namespace {

// Green contexts (driver API, CUDA 12.4+) through cudaGetDriverEntryPoint: the runtime's own
// launches and events work on their streams (scripts/probes/green_ctx_probe.cu).
struct GreenApi {
    CUresult (*dev_get)(CUdevice*, int) = nullptr;
    CUresult (*get_res)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                      unsigned int) = nullptr;
    CUresult (*gen_desc)(CUdevResourceDesc*, CUdevResource*, unsigned int) = nullptr;
    CUresult (*create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
    CUresult (*destroy)(CUgreenCtx) = nullptr;
    CUresult (*stream)(CUstream*, CUgreenCtx, unsigned int, int) = nullptr;
    bool ok = false;
};

const GreenApi& green_api() {
    static GreenApi g = [] {
        GreenApi a;
        auto get = [](const char* name, auto& fn) {
            void* ptr = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(ptr);
            return fn != nullptr;
        };
        a.ok = get("cuDeviceGet", a.dev_get) && get("cuDeviceGetDevResource", a.get_res) &&
               get("cuDevSmResourceSplitByCount", a.split) && get("cuDevResourceGenerateDesc", a.gen_desc) &&
               get("cuGreenCtxCreate", a.create) && get("cuGreenCtxDestroy", a.destroy) &&
               get("cuGreenCtxStreamCreate", a.stream);
        cudaGetLastError();
        return a;
    }();
    return g;
}

// Splits the device's SMs: `want` (rounded by the driver's partition granularity) for the
// samplers, the rest for extraction.
int make_partitions(int device, uint32_t want, CUgreenCtx* gs, CUgreenCtx* gx) {
    const GreenApi& g = green_api();
    if (!g.ok) return fail(FDG_CUDA_ERROR, "sampler_sms: green contexts unavailable in this driver");
    CUdevice dev;
    CUdevResource all, grp, rest;
    unsigned int ng = 1;
    if (g.dev_get(&dev, device) != CUDA_SUCCESS || g.get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
        g.split(&grp, &ng, &all, &rest, 0, want) != CUDA_SUCCESS || ng != 1 || rest.sm.smCount == 0)
        return fail(FDG_INVALID_ARG, "sampler_sms: cannot split the device's SMs into " + std::to_string(want) +
                                         " + rest");
    CUdevResourceDesc d1, d2;
    if (g.gen_desc(&d1, &grp, 1) != CUDA_SUCCESS || g.gen_desc(&d2, &rest, 1) != CUDA_SUCCESS ||
        g.create(gs, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        g.create(gx, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
        return fail(FDG_CUDA_ERROR, "sampler_sms: green context creation failed");
    return FDG_OK;
}

// A non-blocking stream with priority `prio`, inside green context `gc` when given.
int make_stream(cudaStream_t* st, CUgreenCtx gc, int prio) {
    if (!gc) {
        FDG_CUDA(cudaStreamCreateWithPriority(st, cudaStreamNonBlocking, prio));
        return FDG_OK;
    }
    CUstream s;
    if (green_api().stream(&s, gc, CU_STREAM_NON_BLOCKING, prio) != CUDA_SUCCESS)
        return fail(FDG_CUDA_ERROR, "cuGreenCtxStreamCreate failed");
    *st = reinterpret_cast<cudaStream_t>(s);
    return FDG_OK;
}

void destroy(fdg_pipeline* p) {
    if (!p) return;
    cudaDeviceSynchronize();
    if (p->l2_persist) {  // the set-aside is device-wide: give it back
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
        cudaGetLastError();
    }
    for (auto s : p->samplers) sampler_destroy(s);
    for (auto s : p->sstream) cudaStreamDestroy(s);
    if (p->xstream) cudaStreamDestroy(p->xstream);
    if (p->xstream2) cudaStreamDestroy(p->xstream2);
    if (p->dstream) cudaStreamDestroy(p->dstream);
    for (auto e : p->acquired)
        if (e) cudaEventDestroy(e);
    for (auto e : p->rec_ev) cudaEventDestroy(e);
    if (p->tstream) cudaStreamDestroy(p->tstream);
    for (int i = 0; i < 2; ++i) {
        if (p->gathered[i]) cudaEventDestroy(p->gathered[i]);
        if (p->trained[i]) cudaEventDestroy(p->trained[i]);
    }
    for (auto s : p->mstream) cudaStreamDestroy(s);
    if (p->green_s) green_api().destroy(p->green_s);
    if (p->green_x) green_api().destroy(p->green_x);
    for (auto v : p->nodes) cudaFree(v);
    for (auto v : p->edges) cudaFree(v);
    for (auto v : p->seeds) cudaFree(v);
    for (auto v : p->alias) cudaFree(v);
    for (auto v : p->X) cudaFree(v);
    for (auto e : p->sampled) cudaEventDestroy(e);
    for (auto e : p->extracted) cudaEventDestroy(e);
    for (auto e : p->tev) cudaEventDestroy(e);
    for (auto e : p->sev) cudaEventDestroy(e);
    for (auto e : p->bound) if (e) cudaEventDestroy(e);
    for (auto e : p->moved) if (e) cudaEventDestroy(e);
    if (p->counts) cudaFree(p->counts);
    if (p->losses) cudaFree(p->losses);
    if (p->t0) cudaEventDestroy(p->t0);
    if (p->bm) fdg_bm_destroy(p->bm);
    delete p;
}

// Per-batch records and timing events for runs of up to n batches, grown geometrically
// (the pipeline reserves kReserveBatches at creation, so ordinary runs allocate nothing:
// cudaFree would synchronise the device inside the caller's timed region).
constexpr uint64_t kReserveBatches = 1024;
int reserve_batches(fdg_pipeline* p, uint64_t n, bool events) {
    if (p->counts_cap < n) {
        const uint64_t cap = std::max<uint64_t>(n, 2 * p->counts_cap);
        if (p->counts) cudaFree(p->counts);
        p->counts = nullptr;
        p->counts_cap = 0;
        FDG_CUDA(cudaMalloc(&p->counts, cap * sizeof(fdg_batch_counts)));
        p->counts_cap = cap;
    }
    if (!events) return FDG_OK;
    const uint64_t G = std::max<uint32_t>(p->cfg.group_batches, 1);
    const uint64_t have = p->tev.size() / 2;
    if (have >= n) return FDG_OK;
    const uint64_t want = std::max<uint64_t>(n, 2 * have);
    for (size_t i = p->tev.size(); i < 2 * want; ++i) {
        cudaEvent_t e;
        FDG_CUDA(cudaEventCreate(&e));
        p->tev.push_back(e);
    }
    for (size_t i = p->sev.size(); i < 2 * ((want + G - 1) / G); ++i) {
        cudaEvent_t e;
        FDG_CUDA(cudaEventCreate(&e));
        p->sev.push_back(e);
    }
    return FDG_OK;
}

// Builds everything of `p`; on failure the caller destroys the partial pipeline.
int pipeline_build(fdg_pipeline* p, fdg_ctx* ctx, const uint32_t* fanouts, uint32_t n_layers,
                   const fdg_pipeline_config* cfg) {
    p->ctx = ctx;
    p->cfg = *cfg;
    if (p->cfg.n_samplers == 0) p->cfg.n_samplers = 8;  // measured on B200: Papers flat at 6-10, products best from 8
    if (p->cfg.prefetch_group == 0) p->cfg.prefetch_group = 16;
    if (p->cfg.group_batches == 0) p->cfg.group_batches = 1;
    p->cfg.group_batches = std::min<uint32_t>(p->cfg.group_batches, 8);
    // the MT ring (2 prefetch chunks) must never recycle a slot of the group being sampled
    p->cfg.prefetch_group = std::max<uint32_t>(p->cfg.prefetch_group, 2 * p->cfg.group_batches);
    const uint32_t S = p->cfg.n_samplers, G = p->cfg.group_batches;
    // Sampler streams get the highest priority: their short latency-bound kernels
    // should take free SM slots ahead of the bandwidth-bound extraction.
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    const bool prio = !(p->cfg.flags & FDG_PIPE_NO_PRIORITY);
    // Optional SM partitioning: the latency-bound sampler chains on their own SMs, the
    // bandwidth-bound extraction on the rest (no buffer manager: its k_compact assumes a
    // device-wide co-resident grid).
    if (g_sampler_sms > 0 && !cfg->use_buffer_manager) {
        const int rc = make_partitions(ctx->device, uint32_t(g_sampler_sms), &p->green_s, &p->green_x);
        if (rc) return rc;
    }
    for (uint32_t i = 0; i < S; ++i) {
        Sampler* s = nullptr;
        int rc = sampler_create(ctx, cfg->batch_size, fanouts, n_layers, &s, G);
        if (rc) return rc;
        sampler_set_lean(s, g_intern_lean == 1 || (g_intern_lean == 2 && !cfg->checksum));
        p->samplers.push_back(s);
        // the MT prefetch ring (2 chunks) is sized here: a run never allocates or synchronises
        FDG_TRY(sampler_reserve_ring(s, 2 * p->cfg.prefetch_group));
        cudaStream_t st;
        FDG_TRY(make_stream(&st, p->green_s, prio ? prio_hi : prio_lo));
        p->sstream.push_back(st);
    }
    // Optional: keep the samplers' batch hash tables L2-resident (persisting window).
    if (!(p->cfg.flags & FDG_PIPE_NO_L2_PERSIST) && g_l2_persist_mb > 0) {
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
        uint64_t want = 0;
        for (auto s : p->samplers) {
            void* b;
            uint64_t n;
            sampler_hash_region(s, &b, &n);
            want += n;
        }
        if (max_persist > 0 && max_window > 0) {
            const uint64_t persist =
                std::min<uint64_t>(std::min<uint64_t>(want, uint64_t(max_persist)), uint64_t(g_l2_persist_mb) << 20);
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist);
            p->l2_persist = true;
            for (uint32_t i = 0; i < S; ++i) {
                void* b;
                uint64_t n;
                sampler_hash_region(p->samplers[i], &b, &n);
                cudaStreamAttrValue a{};
                a.accessPolicyWindow.base_ptr = b;
                a.accessPolicyWindow.num_bytes = std::min<uint64_t>(n, uint64_t(max_window));
                a.accessPolicyWindow.hitRatio = float(std::min(1.0, double(persist) / double(want)));
                a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                cudaStreamSetAttribute(p->sstream[i], cudaStreamAttributeAccessPolicyWindow, &a);
            }
            cudaGetLastError();  // an optimisation only; ignore unsupported configurations
        }
    }
    uint64_t mn, me;
    sampler_capacity(p->samplers[0], &mn, &me);
    p->max_nodes = mn;
    p->cap = std::max<uint64_t>(std::max(mn, me), 1);
    // With the buffer manager the metadata chain (latency-bound, on the critical path of every
    // batch) can run at the samplers' priority, ahead of the DRAM-bound row move (option).
    // option extract_prio: the extraction streams at the highest priority and the samplers at the
    // lowest (pending gather CTAs are placed before pending sampler CTAs): 1 always, 2 (default)
    // with the buffer manager only. Papers 181.7 -> 188.0 us per batch with plain gathers, but
    // config 3 523.4 -> 514.5 (its metadata chain is the critical path there).
    const bool xprio = (g_extract_prio == 1 || (g_extract_prio == 2 && cfg->use_buffer_manager)) && prio;
    if (xprio)
        for (auto& st : p->sstream) {
            cudaStreamDestroy(st);
            FDG_TRY(make_stream(&st, p->green_s, prio_lo));
        }
    FDG_TRY(make_stream(&p->xstream, p->green_x,
                        xprio || (cfg->use_buffer_manager && g_bm_meta_prio && prio) ? prio_hi : prio_lo));
    // Plain gathers of consecutive batches alternate between two streams so the tail
    // of one overlaps the head of the next (the buffer-manager path is stateful and
    // stays on one stream).
    // With the buffer manager the row moves get their own stream: batch j's move
    // overlaps batch j+1's acquire / select / bind (the metadata chain stays in order).
    if (cfg->use_buffer_manager || g_extract_streams > 1)
        FDG_TRY(make_stream(&p->xstream2, p->green_x, xprio ? prio_hi : prio_lo));
    if (cfg->use_buffer_manager)
        for (int i = 0; i < 2; ++i) {
            FDG_CUDA(cudaEventCreateWithFlags(&p->bound[i], cudaEventDisableTiming));
            FDG_CUDA(cudaEventCreateWithFlags(&p->moved[i], cudaEventDisableTiming));
            FDG_CUDA(cudaEventCreateWithFlags(&p->acquired[i], cudaEventDisableTiming));
        }
    // one MT stream per sampler: prefetch launches of different samplers overlap
    for (uint32_t i = 0; i < S; ++i) {
        cudaStream_t st;
        FDG_TRY(make_stream(&st, p->green_s, 0));
        p->mstream.push_back(st);
    }
    // per-batch output slots: how far the samplers may run ahead of the extraction (option
    // pipe_slots overrides 2 * S * G; at least G + 1)
    p->nslots = g_pipe_slots > 0 ? std::max<uint32_t>(uint32_t(g_pipe_slots), G + 1) : 2 * S * G;
    for (uint32_t i = 0; i < p->nslots; ++i) {
        uint64_t* n;
        uint32_t* e;
        uint64_t* sd;
        FDG_CUDA(cudaMalloc(&n, p->cap * 8));
        FDG_CUDA(cudaMalloc(&e, p->cap * 8));
        FDG_CUDA(cudaMalloc(&sd, uint64_t(cfg->batch_size) * 8));
        p->nodes.push_back(n);
        p->edges.push_back(e);
        p->seeds.push_back(sd);
        cudaEvent_t b;
        FDG_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        p->extracted.push_back(b);
        FDG_CUDA(cudaEventRecord(b, p->xstream));
    }
    for (uint32_t i = 0; i < 2 * S; ++i) {
        cudaEvent_t a;
        FDG_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        p->sampled.push_back(a);
    }
    if (!cfg->use_buffer_manager) p->cfg.write_x = 1;  // the gather's product is X itself
    for (uint32_t i = 0; i < 2; ++i) {
        void* x = nullptr;
        if (p->cfg.write_x) FDG_CUDA(cudaMalloc(&x, p->cap * ctx->row_bytes));
        p->X.push_back(x);
        int64_t* a = nullptr;
        if (cfg->use_buffer_manager) FDG_CUDA(cudaMalloc(&a, p->cap * 8));
        p->alias.push_back(a);
    }
    if (cfg->use_buffer_manager) {
        int rc = fdg_bm_create(ctx, cfg->buffer_slots, 0, uint32_t(p->max_nodes), &p->bm);
        if (rc) return rc;
    }
    FDG_TRY(reserve_batches(p, kReserveBatches, true));
    return FDG_OK;
}

}  // namespace

extern "C" {

int fdg_pipeline_create(fdg_ctx* ctx, const uint32_t* fanouts, uint32_t n_layers, const fdg_pipeline_config* cfg,
                        fdg_pipeline** out) {
    if (cfg->batch_size == 0) return fail(FDG_INVALID_ARG, "config: batch_size must be >= 1");
    if (ctx->row_bytes == 0) return fail(FDG_NOT_LOADED, "pipeline: no feature table loaded");
    cudaSetDevice(ctx->device);
    auto p = new fdg_pipeline();
    const int rc = pipeline_build(p, ctx, fanouts, n_layers, cfg);
    if (rc) {
        destroy(p);  // everything built so far
        return rc;
    }
    *out = p;
    return FDG_OK;
}

int fdg_pipeline_destroy(fdg_pipeline* p) {
    destroy(p);
    return FDG_OK;
}

int fdg_pipeline_run(fdg_pipeline* p, const uint64_t* seeds, int seeds_on_host, const uint64_t* rng_seeds,
                     uint64_t n_batches, fdg_batch_counts* records_host, float* extract_ms, float* elapsed_ms) {
    return fdg_pipeline_run_ragged(p, seeds, seeds_on_host, n_batches * p->cfg.batch_size, rng_seeds, n_batches,
                                   records_host, extract_ms, elapsed_ms);
}

int fdg_pipeline_run_ragged(fdg_pipeline* p, const uint64_t* seeds, int seeds_on_host, uint64_t n_seeds_total,
                            const uint64_t* rng_seeds, uint64_t n_batches, fdg_batch_counts* records_host,
                            float* extract_ms, float* elapsed_ms) {
    cudaSetDevice(p->ctx->device);
    const uint32_t S = p->cfg.n_samplers, PG = p->cfg.prefetch_group, B = p->cfg.batch_size;
    const uint32_t G = p->cfg.group_batches;
    if (n_batches == 0) return FDG_OK;
    if (n_seeds_total > n_batches * uint64_t(B) || n_seeds_total <= (n_batches - 1) * uint64_t(B))
        return fail(FDG_INVALID_ARG, "pipeline_run: every batch but the last must hold batch_size seeds");
    // seeds of batch j: [j*B, min((j+1)*B, n_seeds_total)) (the last chunk of partition_epoch may be short)
    auto seeds_of = [&](uint64_t j) { return uint32_t(std::min<uint64_t>(B, n_seeds_total - j * B)); };
    FDG_TRY(reserve_batches(p, n_batches, extract_ms != nullptr));
    const bool sample_only = p->cfg.flags & FDG_PIPE_SAMPLE_ONLY;
    const bool train = p->model != nullptr && !sample_only;
    if (train && p->losses_cap < n_batches) {
        if (p->losses) cudaFree(p->losses);
        FDG_CUDA(cudaMalloc(&p->losses, n_batches * sizeof(float)));
        p->losses_cap = n_batches;
    }
    p->loss_batches = 0;
    const bool extract_only = p->cfg.flags & FDG_PIPE_EXTRACT_ONLY;
    const uint64_t n_groups = (n_batches + G - 1) / G;
    const uint64_t sampled_groups = extract_only ? std::min<uint64_t>(n_groups, 2 * S) : n_groups;
    // per-sampler batch lists (in sampling order) and their MT prefetch in chunks of PG
    std::vector<std::vector<uint64_t>> mine(S);
    for (uint64_t g = 0; g < sampled_groups; ++g)
        for (uint64_t j = g * G; j < std::min<uint64_t>((g + 1) * G, n_batches); ++j) mine[g % S].push_back(j);
    std::vector<uint64_t> fetched(S, 0);  // batches of mine[s] whose streams were requested
    std::vector<uint64_t> consumed(S, 0);
    // The sampler's ring holds 2 * PG streams (sized by the first, full chunk). A chunk is
    // clipped so that at most 2 * PG streams are outstanding (fetched, not yet consumed):
    // the slot a new stream takes then always belongs to a batch already sampled, for any
    // group size G <= PG / 2 (a whole-chunk rule let G = 3, 5, 6, 7 overwrite streams of
    // the group about to be sampled).
    auto prefetch_upto = [&](uint32_t s, uint64_t upto) -> int {
        upto = std::min<uint64_t>(std::min<uint64_t>(upto, mine[s].size()), consumed[s] + 2 * uint64_t(PG));
        while (fetched[s] < upto) {
            std::vector<uint64_t> r;
            const uint64_t end = std::min<uint64_t>(fetched[s] + PG, upto);
            for (uint64_t k = fetched[s]; k < end; ++k) r.push_back(rng_seeds[mine[s][k]]);
            FDG_TRY(sampler_prefetch(p->samplers[s], p->mstream[s], r.data(), uint32_t(r.size())));
            fetched[s] += r.size();
        }
        return FDG_OK;
    };
    // FDG_PROFILE_RANGE=1: bracket the run for ncu range replay (concurrent kernels
    // profiled together: --replay-mode app-range --profile-from-start off)
    static const bool prof_range = std::getenv("FDG_PROFILE_RANGE") != nullptr;
    if (prof_range) {
        FDG_CUDA(cudaDeviceSynchronize());
        cudaProfilerStart();
    }
    cudaEvent_t t1;
    if (!p->t0) FDG_CUDA(cudaEventCreate(&p->t0));
    cudaEvent_t t0 = p->t0;
    p->timed_batches = 0;
    p->timed_groups = 0;
    FDG_CUDA(cudaEventCreate(&t1));
    // Everything of the run -- the first MT prefetch included -- is ordered after t0.
    auto h0 = std::chrono::steady_clock::now();
    FDG_CUDA(cudaEventRecord(t0, p->xstream));
    for (uint32_t s = 0; s < S; ++s) {
        FDG_CUDA(cudaStreamWaitEvent(p->sstream[s], t0, 0));
        FDG_CUDA(cudaStreamWaitEvent(p->mstream[s], t0, 0));
    }
    if (p->xstream2) FDG_CUDA(cudaStreamWaitEvent(p->xstream2, t0, 0));
    // The first chunk of each sampler's streams is requested right before that sampler's first
    // group (in the loop below), so batch 0's chain is enqueued behind one prefetch, not S.
    if (g_prefetch_upfront)
        for (uint32_t s = 0; s < S; ++s) FDG_TRY(prefetch_upto(s, PG));
    for (uint64_t g = 0; g < n_groups; ++g) {
        const uint64_t j0 = g * G, j1 = std::min<uint64_t>(j0 + G, n_batches);
        const uint32_t n = uint32_t(j1 - j0);
        const uint32_t s = uint32_t(g % S);
        const bool do_sample = g < sampled_groups;
        const uint32_t gslot = uint32_t(g % (2 * S));
        if (do_sample) {
            // keep the MT ring ~1.5 prefetch chunks ahead of this sampler's consumption
            FDG_TRY(prefetch_upto(s, consumed[s] + n + PG));
            cudaStream_t ss = p->sstream[s];
            const uint64_t* sd[8];
            uint32_t ns[8];
            uint64_t rs[8];
            uint64_t* nd[8];
            uint32_t* ed[8];
            fdg_batch_counts* cn[8];
            for (uint32_t i = 0; i < n; ++i) {
                const uint64_t j = j0 + i;
                const uint32_t slot = uint32_t(j % p->nslots);
                FDG_CUDA(cudaStreamWaitEvent(ss, p->extracted[slot], 0));
                sd[i] = seeds + j * B;
                ns[i] = seeds_of(j);
                if (seeds_on_host) {  // host -> device copy of this batch's seeds (pinned for async)
                    FDG_CUDA(cudaMemcpyAsync(p->seeds[slot], sd[i], uint64_t(ns[i]) * 8, cudaMemcpyHostToDevice, ss));
                    sd[i] = p->seeds[slot];
                }
                rs[i] = rng_seeds[j];
                nd[i] = p->nodes[slot];
                ed[i] = p->edges[slot];
                cn[i] = p->counts + j;
            }
            if (g_debug_zero_word >= 0) {  // test hook: a genuine Lemire rejection in batch jz
                const uint64_t jz = uint64_t(g_debug_zero_word) >> 24;
                if (jz >= j0 && jz < j1)
                    FDG_TRY(sampler_debug_zero_word(p->samplers[s], p->mstream[s], rng_seeds[jz],
                                                    uint64_t(g_debug_zero_word) & 0xFFFFFFu));
            }
            if (g_debug_reject_batch >= 0 && uint64_t(g_debug_reject_batch) >= j0 &&
                uint64_t(g_debug_reject_batch) < j1)
                sampler_debug_reject(p->samplers[s], int(uint64_t(g_debug_reject_batch) - j0));
            if (extract_ms) FDG_CUDA(cudaEventRecord(p->sev[2 * g], ss));
            FDG_TRY(sampler_sample_group(p->samplers[s], ss, n, sd, ns, rs, nd, ed, p->cap, cn));
            if (extract_ms) FDG_CUDA(cudaEventRecord(p->sev[2 * g + 1], ss));
            consumed[s] += n;
            FDG_CUDA(cudaEventRecord(p->sampled[gslot], ss));
            FDG_CUDA(cudaStreamWaitEvent(p->xstream, p->sampled[gslot], 0));
            if (p->xstream2) FDG_CUDA(cudaStreamWaitEvent(p->xstream2, p->sampled[gslot], 0));
        }
        for (uint64_t j = j0; j < j1; ++j) {
            const uint32_t slot = uint32_t(j % p->nslots);
            // extract-only diagnostics re-extract the batches sampled in the first groups
            const uint64_t src_j = do_sample ? j : (j % (sampled_groups * G));
            fdg_batch_counts* cnt = p->counts + src_j;
            // plain gathers alternate between the two extraction streams; with a model the train
            // stage (one model workspace) runs in batch order on its own stream behind them
            cudaStream_t xs = (!p->bm && p->xstream2 && (j & 1)) ? p->xstream2 : p->xstream;
            const bool tsplit = train && !p->bm;
            // stream on which the batch's work ends
            cudaStream_t xe = (p->bm && g_bm_overlap) ? p->xstream2 : tsplit ? p->tstream : xs;
            if (sample_only) {
                FDG_CUDA(cudaEventRecord(p->extracted[slot], xs));
                continue;
            }
            FDG_TRACE("extract", xs);
            // extraction window: the gather (plain), or the row move alone (buffer manager: the
            // metadata chain runs before it on the other stream)
            if (extract_ms && !p->bm) FDG_CUDA(cudaEventRecord(p->tev[2 * j], xs));
            const uint32_t* n_dev = &cnt->n_nodes;
            uint64_t* cs = p->cfg.checksum ? &cnt->checksum : nullptr;
            void* X = p->X[j & 1];
            const uint32_t nslot = uint32_t(src_j % p->nslots);
            if (!p->bm) {
                const uint32_t par = uint32_t(j & 1);
                // X[par] was last read by batch j-2's train stage
                if (tsplit && j >= 2) FDG_CUDA(cudaStreamWaitEvent(xs, p->trained[par], 0));
                FDG_TRY(launch_gather_bound(*p->ctx, xs, p->nodes[nslot], n_dev, p->cap, p->cap, X, cs,
                                            &cnt->status, true));
                if (tsplit) {
                    FDG_CUDA(cudaEventRecord(p->gathered[par], xs));
                    FDG_CUDA(cudaStreamWaitEvent(p->tstream, p->gathered[par], 0));
                    FDG_TRY(fdg_sage_forward(p->model, p->tstream, X, p->nodes[nslot], p->edges[nslot], cnt,
                                             p->label_seed, p->losses + j, nullptr));
                    if (p->lr != 0.f) {
                        FDG_TRY(fdg_sage_backward(p->model, p->tstream, p->nodes[nslot], p->edges[nslot], cnt,
                                                  p->label_seed));
                        FDG_TRY(fdg_sage_sgd(p->model, p->tstream, p->lr));
                    }
                    FDG_CUDA(cudaEventRecord(p->trained[par], p->tstream));
                }
            } else {
                const uint32_t par = uint32_t(j & 1);
                // alias[par], is_load[par] and X[par] were last used by batch j-2's move
                if (j >= 2) FDG_CUDA(cudaStreamWaitEvent(p->xstream, p->moved[par], 0));
                // option bm_split_move: X rows move right after the acquire (hits read their pinned
                // slots, misses the table), the misses' slot fills after the bind
                const bool split = g_bm_split_move && !cs && !p->ctx->host_table &&
                                   (p->ctx->row_bytes == 400 || p->ctx->row_bytes == 512 || p->ctx->row_bytes == 1024);
                FDG_TRY(bm_extract_meta(p->bm, p->xstream, p->nodes[nslot], n_dev, p->cap, p->alias[par], par,
                                        split ? p->acquired[par] : nullptr));
                if (split) {
                    FDG_CUDA(cudaStreamWaitEvent(xe, p->acquired[par], 0));
                    FDG_TRY(bm_extract_move(p->bm, xe, p->nodes[nslot], n_dev, p->cap, p->alias[par], X, nullptr, par, 1));
                }
                // option bm_move_early: batch j's move may start right after its bind, next to release j-1
                // (measured 517 -> 538 us per Papers batch: off)
                if (g_bm_move_early) FDG_CUDA(cudaEventRecord(p->bound[par], p->xstream));
                if (j > 0) {  // lag-1 release (the releaser stage, pipeline.hpp:525-543)
                    const uint64_t pj = do_sample ? j - 1 : ((j - 1) % (sampled_groups * G));
                    // batch j-1's move reads its node list: the list is free once both are done
                    FDG_CUDA(cudaStreamWaitEvent(p->xstream, p->moved[par ^ 1], 0));
                    // (batch j-1's alias list is alias[par ^ 1]: the release needs no mapping-table reads)
                    FDG_TRY(bm_release(p->bm, p->xstream, p->nodes[pj % p->nslots], p->alias[par ^ 1],
                                       &p->counts[pj].n_nodes, p->cap));
                    FDG_CUDA(cudaEventRecord(p->extracted[(j - 1) % p->nslots], p->xstream));
                }
                // Batch j's row move starts after release j-1, not right after bind j: the
                // release (alias-list walk, latency-bound) then runs without the move saturating
                // DRAM next to it, and the move overlaps batch j+1's acquire / select / bind.
                if (!g_bm_move_early) FDG_CUDA(cudaEventRecord(p->bound[par], p->xstream));
                FDG_CUDA(cudaStreamWaitEvent(xe, p->bound[par], 0));
                if (extract_ms) FDG_CUDA(cudaEventRecord(p->tev[2 * j], xe));
                FDG_TRY(bm_extract_move(p->bm, xe, p->nodes[nslot], n_dev, p->cap, p->alias[par], X, cs, par,
                                        split ? 2 : 0));
                if (extract_ms) FDG_CUDA(cudaEventRecord(p->tev[2 * j + 1], xe));
                FDG_TRY(bm_status_to(p->bm, xe, &cnt->status));  // e.g. CAPACITY = StandbyTimeout
                if (train) {  // the trainer consumes X (and the batch's blocks) before they are reused
                    FDG_TRY(fdg_sage_forward(p->model, xe, X, p->nodes[nslot], p->edges[nslot], cnt, p->label_seed,
                                             p->losses + j, nullptr));
                    if (p->lr != 0.f) {
                        FDG_TRY(fdg_sage_backward(p->model, xe, p->nodes[nslot], p->edges[nslot], cnt, p->label_seed));
                        FDG_TRY(fdg_sage_sgd(p->model, xe, p->lr));
                    }
                }
                FDG_CUDA(cudaEventRecord(p->moved[par], xe));
            }
            if (extract_ms && !p->bm) FDG_CUDA(cudaEventRecord(p->tev[2 * j + 1], tsplit ? xs : xe));
            if (records_host) {  // device -> host read of the batch record (counts + checksum)
                if (g_records_stream) {  // on its own stream: the next gather on xe does not queue behind it
                    if (!p->dstream) {
                        FDG_CUDA(cudaStreamCreateWithFlags(&p->dstream, cudaStreamNonBlocking));
                        p->rec_ev.resize(64);
                        for (auto& e : p->rec_ev) FDG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    }
                    cudaEvent_t e = p->rec_ev[j % p->rec_ev.size()];
                    FDG_CUDA(cudaEventRecord(e, xe));
                    FDG_CUDA(cudaStreamWaitEvent(p->dstream, e, 0));
                    FDG_CUDA(cudaMemcpyAsync(records_host + j, cnt, sizeof(fdg_batch_counts), cudaMemcpyDeviceToHost,
                                             p->dstream));
                } else {
                    FDG_CUDA(cudaMemcpyAsync(records_host + j, cnt, sizeof(fdg_batch_counts), cudaMemcpyDeviceToHost,
                                             xe));
                }
            }
            if (!p->bm) FDG_CUDA(cudaEventRecord(p->extracted[slot], xe));  // the node / edge lists are free
        }
    }
    if (p->bm && !sample_only) {  // drain: release the last batch
        const uint64_t lj = extract_only ? (n_batches - 1) % (sampled_groups * G) : n_batches - 1;
        FDG_CUDA(cudaStreamWaitEvent(p->xstream, p->moved[(n_batches - 1) & 1], 0));
        FDG_TRY(bm_release(p->bm, p->xstream, p->nodes[lj % p->nslots], p->alias[(n_batches - 1) & 1],
                           &p->counts[lj].n_nodes, p->cap));
        FDG_CUDA(cudaEventRecord(p->extracted[(n_batches - 1) % p->nslots], p->xstream));
    }
    for (uint32_t s = 0; s <= S + 2; ++s) {  // join the sampler, second extraction, train and record streams
        cudaStream_t js = s < S ? p->sstream[s] : s == S ? p->xstream2 : s == S + 1 ? p->tstream : p->dstream;
        if (!js) continue;
        cudaEvent_t e;
        FDG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        FDG_CUDA(cudaEventRecord(e, js));
        FDG_CUDA(cudaStreamWaitEvent(p->xstream, e, 0));
        cudaEventDestroy(e);
    }
    FDG_CUDA(cudaEventRecord(t1, p->xstream));
    p->cfg.host_enqueue_ms =
        std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - h0).count();
    FDG_CUDA(cudaEventSynchronize(t1));
    FDG_CUDA(cudaDeviceSynchronize());
    if (prof_range) cudaProfilerStop();
    float ms = 0;
    FDG_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    if (elapsed_ms) *elapsed_ms = ms;
    if (extract_ms && !sample_only)
        for (uint64_t j = 0; j < n_batches; ++j)
            FDG_CUDA(cudaEventElapsedTime(extract_ms + j, p->tev[2 * j], p->tev[2 * j + 1]));
    cudaEventDestroy(t1);
    if (extract_ms && !sample_only) p->timed_batches = n_batches;
    if (train) p->loss_batches = n_batches;
    if (extract_ms) p->timed_groups = sampled_groups;
    return FDG_OK;
}

int fdg_pipeline_extract_times(fdg_pipeline* p, uint64_t first, uint64_t n, float* start_ms, float* end_ms) {
    if (first + n > p->timed_batches)
        return fail(FDG_INVALID_ARG, "pipeline_extract_times: range beyond the last run's timed batches");
    for (uint64_t j = first; j < first + n; ++j) {
        FDG_CUDA(cudaEventElapsedTime(start_ms + (j - first), p->t0, p->tev[2 * j]));
        FDG_CUDA(cudaEventElapsedTime(end_ms + (j - first), p->t0, p->tev[2 * j + 1]));
    }
    return FDG_OK;
}

int fdg_pipeline_bm_stats(fdg_pipeline* p, fdg_bm_stats* out) {
    if (!p->bm) return fail(FDG_NOT_LOADED, "pipeline_bm_stats: pipeline has no buffer manager");
    return fdg_bm_stats_get(p->bm, out);
}

int fdg_pipeline_sample_times(fdg_pipeline* p, uint64_t* n_groups, float* busy_ms) {
    float tot = 0;
    for (uint64_t g = 0; g < p->timed_groups; ++g) {
        float ms = 0;
        FDG_CUDA(cudaEventElapsedTime(&ms, p->sev[2 * g], p->sev[2 * g + 1]));
        tot += ms;
    }
    if (n_groups) *n_groups = p->timed_groups;
    if (busy_ms) *busy_ms = tot;
    return FDG_OK;
}

int fdg_pipeline_set_model(fdg_pipeline* p, fdg_sage* m, uint64_t label_seed) {
    if (m && !p->cfg.write_x) return fail(FDG_INVALID_ARG, "pipeline_set_model: the train stage needs X (write_x)");
    p->model = m;
    p->label_seed = label_seed;
    if (m && !p->tstream) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        FDG_TRY(make_stream(&p->tstream, p->green_x, lo));
        for (int i = 0; i < 2; ++i) {
            FDG_CUDA(cudaEventCreateWithFlags(&p->gathered[i], cudaEventDisableTiming));
            FDG_CUDA(cudaEventCreateWithFlags(&p->trained[i], cudaEventDisableTiming));
        }
    }
    return FDG_OK;
}

int fdg_pipeline_set_training(fdg_pipeline* p, float lr) {
    p->lr = lr;
    return FDG_OK;
}

int fdg_pipeline_losses(fdg_pipeline* p, uint64_t first, uint64_t n, float* out) {
    if (first + n > p->loss_batches) return fail(FDG_INVALID_ARG, "pipeline_losses: range beyond the last run's batches");
    FDG_CUDA(cudaMemcpy(out, p->losses + first, n * sizeof(float), cudaMemcpyDeviceToHost));
    return FDG_OK;
}

int fdg_pipeline_get_config(const fdg_pipeline* p, fdg_pipeline_config* out) {
    *out = p->cfg;
    return FDG_OK;
}

int fdg_pipeline_records(fdg_pipeline* p, uint64_t first, uint64_t n, fdg_batch_counts* out) {
    if (first + n > p->counts_cap) return fail(FDG_INVALID_ARG, "pipeline_records: range beyond last run");
    FDG_CUDA(cudaMemcpy(out, p->counts + first, n * sizeof(fdg_batch_counts), cudaMemcpyDeviceToHost));
    return FDG_OK;
}

}  // extern "C"
