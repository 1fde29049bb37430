// fdg_api.cu -- the extern "C" boundary (include/fdg.h).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "fdg_internal.cuh"

namespace fdg {

int64_t g_host_tier_thp = 0;
int64_t g_force_idx64 = 0;
static thread_local std::string g_error;
static thread_local int g_errno = 0;

void set_error(const std::string& msg) { g_error = msg; }
int fail(int code, const std::string& msg) {
    g_error = msg;
    g_errno = 0;
    return code;
}
// Dataset-file errors: the reference throws std::runtime_error, or std::system_error (errno,
// generic_category, context) through throw_errno (common.hpp:67-69) when a call failed.
int io_fail(const std::string& msg, int err) {
    fail(FDG_IO_ERROR, msg);
    g_errno = err;
    return FDG_IO_ERROR;
}
int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    g_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what +
              " at " + file + ":" + std::to_string(line);
    return FDG_CUDA_ERROR;
}

struct Sampler;
int sampler_create(Ctx* ctx, uint32_t max_seeds, const uint32_t* fanouts, uint32_t n_layers, Sampler** out);
void sampler_destroy(Sampler* s);
int sampler_prefetch(Sampler* s, cudaStream_t st, const uint64_t* rng_seeds, uint32_t n);
int sampler_sample(Sampler* s, cudaStream_t st, const uint64_t* seeds, uint32_t n_seeds, uint64_t rng_seed,
                   uint64_t* nodes, uint32_t* edges, uint64_t cap, fdg_batch_counts* cnt);
int sampler_sample_host(Sampler* s, const uint64_t* seeds, uint32_t n_seeds, uint64_t rng_seed,
                        const uint64_t* ext_words, uint64_t n_ext_words, uint64_t* nodes, uint32_t* edges,
                        uint64_t cap, uint64_t* n_nodes, uint64_t* n_edges, uint64_t* layer_nodes,
                        uint64_t* layer_edges, uint64_t* words_used);
void sampler_capacity(const Sampler* s, uint64_t* max_nodes, uint64_t* max_edges);

namespace {

// An open file descriptor closed on scope exit.
struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

// Opens `path` read-only; `what` is the throw_errno context of the reference ("open " + path).
int open_file(const std::string& path, const std::string& what, Fd& f, int64_t* size) {
    f.fd = ::open(path.c_str(), O_RDONLY);
    if (f.fd < 0) return io_fail(what, errno);
    struct stat st {};
    if (::fstat(f.fd, &st) != 0) return io_fail("stat " + path, errno);
    *size = st.st_size;
    return FDG_OK;
}

int read_at(const Fd& f, const std::string& path, uint64_t offset, uint64_t bytes, void* dst) {
    uint64_t got = 0;
    while (got < bytes) {
        ssize_t n = ::pread(f.fd, static_cast<char*>(dst) + got, std::min<uint64_t>(bytes - got, 1ull << 30),
                            offset + got);
        if (n < 0 && errno == EINTR) continue;
        if (n < 0) return io_fail("read " + path, errno);
        if (n == 0) return io_fail("read " + path + ": unexpected EOF", 0);
        got += uint64_t(n);
    }
    return FDG_OK;
}

}  // namespace
// Counter pair for one dynamically scheduled launch on this context: a per-context ring on
// its own device, so launches in flight on different streams (up to kDynRing - 1 later
// launches) never share a pair and contexts on different devices never touch each other's.
uint32_t* dyn_counter(const Ctx& c) {
    if (!c.dyn_ring) return nullptr;
    const uint32_t k = __atomic_fetch_add(&c.dyn_next, 1u, __ATOMIC_RELAXED);
    return c.dyn_ring + 2 * (k % kDynRing);
}

}  // namespace fdg

using namespace fdg;

namespace {
// The runner drives up to 19 streams (8 samplers, 8 MT prefetch, 2 extraction, train). With the
// default 8 hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS) streams share queues and a kernel
// can wait behind another stream's blocked work: 32 queues measured sample-only 80.8 -> 72.8 us
// per Papers batch, products 182.8 -> 174.3 us, Papers with the checksum 202.8 -> 199.0 us. Read
// once at CUDA context creation, so it is set when the library loads (a value the process already
// set wins).
__attribute__((constructor)) void fdg_env_defaults() { setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0); }
}  // namespace

extern "C" {

int fdg_last_errno(void) { return g_errno; }

const char* fdg_last_error(void) { return g_error.c_str(); }
int fdg_version(void) { return 1; }

// ---- plumbing -----------------------------------------------------------------
int fdg_device_count(int* n) { FDG_CUDA(cudaGetDeviceCount(n)); return FDG_OK; }
int fdg_set_device(int d) { FDG_CUDA(cudaSetDevice(d)); return FDG_OK; }
int fdg_enable_peer_access(int device, int peer) {
    int can = 0;
    FDG_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
    if (!can) return fail(FDG_INVALID_ARG, "enable_peer_access: device cannot access the peer");
    FDG_CUDA(cudaSetDevice(device));
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return FDG_OK;
    }
    FDG_CUDA(e);
    return FDG_OK;
}
int fdg_malloc(void** p, uint64_t b) { FDG_CUDA(cudaMalloc(p, std::max<uint64_t>(b, 1))); return FDG_OK; }
int fdg_free(void* p) { FDG_CUDA(cudaFree(p)); return FDG_OK; }
int fdg_host_alloc(void** p, uint64_t b) { FDG_CUDA(cudaMallocHost(p, std::max<uint64_t>(b, 1))); return FDG_OK; }
int fdg_host_free(void* p) { FDG_CUDA(cudaFreeHost(p)); return FDG_OK; }
int fdg_memcpy_h2d(void* d, const void* s, uint64_t b, void* st) {
    FDG_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyHostToDevice, (cudaStream_t)st));
    return FDG_OK;
}
int fdg_memcpy_d2h(void* d, const void* s, uint64_t b, void* st) {
    FDG_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToHost, (cudaStream_t)st));
    return FDG_OK;
}
int fdg_memcpy_d2d(void* d, const void* s, uint64_t b, void* st) {
    FDG_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToDevice, (cudaStream_t)st));
    return FDG_OK;
}
int fdg_memset(void* d, int v, uint64_t b, void* st) {
    FDG_CUDA(cudaMemsetAsync(d, v, b, (cudaStream_t)st));
    return FDG_OK;
}
int fdg_stream_create(void** st) {
    cudaStream_t s;
    FDG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *st = s;
    return FDG_OK;
}
int fdg_stream_destroy(void* st) { FDG_CUDA(cudaStreamDestroy((cudaStream_t)st)); return FDG_OK; }
int fdg_stream_sync(void* st) { FDG_CUDA(cudaStreamSynchronize((cudaStream_t)st)); return FDG_OK; }
int fdg_device_sync(void) { FDG_CUDA(cudaDeviceSynchronize()); return FDG_OK; }
int fdg_event_create(void** ev) {
    cudaEvent_t e;
    FDG_CUDA(cudaEventCreate(&e));
    *ev = e;
    return FDG_OK;
}
int fdg_event_destroy(void* ev) { FDG_CUDA(cudaEventDestroy((cudaEvent_t)ev)); return FDG_OK; }
int fdg_event_record(void* ev, void* st) { FDG_CUDA(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)st)); return FDG_OK; }
int fdg_stream_wait_event(void* st, void* ev) {
    FDG_CUDA(cudaStreamWaitEvent((cudaStream_t)st, (cudaEvent_t)ev, 0));
    return FDG_OK;
}
int fdg_event_elapsed_ms(void* a, void* b, float* ms) {
    FDG_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)a, (cudaEvent_t)b));
    return FDG_OK;
}
int fdg_event_sync(void* ev) { FDG_CUDA(cudaEventSynchronize((cudaEvent_t)ev)); return FDG_OK; }
int fdg_mem_info(uint64_t* f, uint64_t* t) {
    size_t a, b;
    FDG_CUDA(cudaMemGetInfo(&a, &b));
    *f = a;
    *t = b;
    return FDG_OK;
}

// ---- context -------------------------------------------------------------------
int fdg_ctx_create(int device, fdg_ctx** out) {
    FDG_CUDA(cudaSetDevice(device));
    auto c = new fdg_ctx();
    c->device = device;
    cudaError_t e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&c->dyn_ring, 2 * kDynRing * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(c->dyn_ring, 0, 2 * kDynRing * sizeof(uint32_t));
    if (e != cudaSuccess) {
        if (c->dyn_ring) cudaFree(c->dyn_ring);
        if (c->stream) cudaStreamDestroy(c->stream);
        delete c;
        return cuda_fail(e, "fdg_ctx_create", __FILE__, __LINE__);
    }
    *out = c;
    return FDG_OK;
}

// NUMA node of the GPU's PCI device (-1 if unknown).
static int gpu_numa_node(int device) {
    char bus[32] = {};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    std::string id(bus);
    for (auto& ch : id) ch = char(std::tolower(static_cast<unsigned char>(ch)));
    FILE* f = std::fopen(("/sys/bus/pci/devices/" + id + "/numa_node").c_str(), "r");
    if (!f) return -1;
    int node = -1;
    if (std::fscanf(f, "%d", &node) != 1) node = -1;
    std::fclose(f);
    return node;
}

// The out-of-core table: either cudaHostAlloc'ed, or (option host_tier_thp) an anonymous
// mapping with transparent huge pages registered with the driver, so the GPU maps the 57 GB
// table with 2 MB pages instead of small ones (random row reads then miss the GPU TLB far
// less).
static void free_host_table(fdg_ctx* c) {
    if (!c->host_table) return;
    if (c->host_table_bytes) {
        cudaHostUnregister(c->host_table);
        munmap(c->host_table, c->host_table_bytes);
    } else {
        cudaFreeHost(c->host_table);
    }
    c->host_table = nullptr;
    c->host_table_bytes = 0;
}

int fdg_ctx_destroy(fdg_ctx* c) {
    if (!c) return FDG_OK;
    cudaSetDevice(c->device);
    if (c->indptr) cudaFree(c->indptr);
    if (c->indices) cudaFree(c->indices);
    for (void* p : c->owned_shards) cudaFree(p);
    free_host_table(c);
    if (c->shard_table) cudaFree((void*)c->shard_table);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->dyn_ring) cudaFree(c->dyn_ring);
    delete c;
    return FDG_OK;
}

int fdg_ctx_info_get(const fdg_ctx* c, fdg_ctx_info* o) {
    std::memset(o, 0, sizeof(*o));
    o->num_nodes = c->num_nodes;
    o->num_edges = c->num_edges;
    o->idx_bytes = c->idx_bytes;
    o->row_bytes = c->row_bytes;
    o->dtype = c->dtype;
    o->n_shards = c->n_shards;
    o->indptr_dev = c->indptr;
    o->indices_dev = c->indices;
    o->table_dev = c->shard_bases.empty() ? nullptr : c->shard_bases[0];
    o->rows_per_shard = c->rows_per_shard;
    o->device = c->device;
    return FDG_OK;
}

int fdg_ctx_load_topology(fdg_ctx* c, const uint64_t* indptr, uint64_t n, const uint64_t* indices, uint64_t e) {
    // Topology::load_indptr / open_indices validation (topology.hpp:84-113)
    if (!indptr) return fail(FDG_INVALID_ARG, "indptr: null array");
    for (uint64_t i = 0; i < n; ++i)
        if (indptr[i] > indptr[i + 1]) return fail(FDG_INVALID_ARG, "indptr is not non-decreasing");
    if (indptr[n] != e) return fail(FDG_INVALID_ARG, "indices size does not match indptr");
    cudaSetDevice(c->device);
    if (c->indptr) cudaFree(c->indptr);
    if (c->indices) cudaFree(c->indices);
    c->indptr = nullptr;
    c->indices = nullptr;
    c->idx_bytes = (n <= 0xFFFFFFFFull && !g_force_idx64) ? 4 : 8;
    FDG_CUDA(cudaMalloc(&c->indptr, (n + 1) * 8));
    FDG_CUDA(cudaMemcpy(c->indptr, indptr, (n + 1) * 8, cudaMemcpyHostToDevice));
    FDG_CUDA(cudaMalloc(&c->indices, std::max<uint64_t>(e, 1) * c->idx_bytes));
    if (c->idx_bytes == 8) {
        FDG_CUDA(cudaMemcpy(c->indices, indices, e * 8, cudaMemcpyHostToDevice));
    } else {
        // narrow to u32 in chunks (lossless: every id < N <= 2^32-1)
        const uint64_t chunk = 1ull << 24;
        std::vector<uint32_t> tmp(std::min<uint64_t>(chunk, std::max<uint64_t>(e, 1)));
        for (uint64_t at = 0; at < e; at += chunk) {
            uint64_t k = std::min<uint64_t>(chunk, e - at);
            for (uint64_t i = 0; i < k; ++i) {
                if (indices[at + i] >= n) return fail(FDG_INVALID_ARG, "indices entry out of range");
                tmp[i] = uint32_t(indices[at + i]);
            }
            FDG_CUDA(cudaMemcpy(static_cast<uint32_t*>(c->indices) + at, tmp.data(), k * 4, cudaMemcpyHostToDevice));
        }
    }
    c->num_nodes = n;
    c->num_edges = e;
    return FDG_OK;
}

int fdg_ctx_load_topology_files(fdg_ctx* c, const char* dir) {
    // Topology(dataset_dir): load_indptr then open_indices (topology.hpp:34-38, 76-113), with
    // the reference's checks, messages and exception categories.
    const std::string d(dir);
    const std::string ip = d + "/indptr.bin", ix = d + "/indices.bin";
    Fd fp;
    int64_t ps = 0;
    FDG_TRY(open_file(ip, "open " + ip, fp, &ps));
    if (ps < int64_t(sizeof(uint64_t)) || ps % 8 != 0) return io_fail("indptr file " + ip + " has invalid size", 0);
    std::vector<uint64_t> indptr(uint64_t(ps) / 8);
    FDG_TRY(read_at(fp, ip, 0, uint64_t(ps), indptr.data()));
    for (size_t i = 0; i + 1 < indptr.size(); ++i)
        if (indptr[i] > indptr[i + 1]) return io_fail("indptr file " + ip + " is not non-decreasing", 0);
    Fd fx;
    int64_t is = 0;
    FDG_TRY(open_file(ix, "open " + ix, fx, &is));
    if (uint64_t(is) != indptr.back() * sizeof(uint64_t))
        return io_fail("indices file " + ix + " size does not match indptr", 0);
    std::vector<uint64_t> indices(uint64_t(is) / 8);
    FDG_TRY(read_at(fx, ix, 0, uint64_t(is), indices.data()));
    return fdg_ctx_load_topology(c, indptr.data(), indptr.size() - 1, indices.data(), indices.size());
}

int fdg_ctx_generate_topology(fdg_ctx* c, uint64_t seed, uint64_t n, uint32_t avg) {
    cudaSetDevice(c->device);
    return generate_topology(*c, seed, n, avg);
}

static int install_table(fdg_ctx* c, void* dev, uint64_t n, uint32_t row_bytes, uint32_t dtype) {
    for (void* p : c->owned_shards) cudaFree(p);
    free_host_table(c);
    c->owned_shards.assign(1, dev);
    c->shard_bases.assign(1, dev);
    c->row_bytes = row_bytes;
    c->dtype = dtype;
    c->n_shards = 1;
    c->rows_per_shard = n;
    c->feat_nodes = n;
    if (c->shard_table) cudaFree((void*)c->shard_table);
    FDG_CUDA(cudaMalloc((void**)&c->shard_table, sizeof(void*)));
    FDG_CUDA(cudaMemcpy((void*)c->shard_table, &dev, sizeof(void*), cudaMemcpyHostToDevice));
    return FDG_OK;
}

int fdg_ctx_load_features(fdg_ctx* c, const void* rows, uint64_t n, uint32_t row_bytes, uint32_t dtype) {
    if (n == 0 || row_bytes == 0 || row_bytes % 4) return fail(FDG_INVALID_ARG, "feature rows: bad shape");
    cudaSetDevice(c->device);
    void* dev = nullptr;
    FDG_CUDA(cudaMalloc(&dev, n * row_bytes));
    FDG_CUDA(cudaMemcpy(dev, rows, n * row_bytes, cudaMemcpyHostToDevice));
    return install_table(c, dev, n, row_bytes, dtype);
}

int fdg_ctx_load_features_file(fdg_ctx* c, const char* path_c) {
    // storage::FeatureTable(path) (feature_file.hpp:27-51): 64-byte header decoded and
    // validated like DatasetHeader::validate (format.hpp:54-64), file length checked.
    const std::string path(path_c);
    Fd f;
    int64_t size = 0;
    FDG_TRY(open_file(path, "open feature file " + path, f, &size));
    unsigned char h[64];
    const ssize_t got = ::pread(f.fd, h, sizeof h, 0);
    if (got != ssize_t(sizeof h)) return io_fail("feature file " + path + ": truncated header", 0);
    uint32_t version, dim, dtype, row_bytes;
    uint64_t n, data_offset;
    std::memcpy(&version, h + 8, 4);
    std::memcpy(&n, h + 16, 8);
    std::memcpy(&dim, h + 24, 4);
    std::memcpy(&dtype, h + 28, 4);
    std::memcpy(&row_bytes, h + 32, 4);
    std::memcpy(&data_offset, h + 40, 8);
    if (std::memcmp(h, "FEATDRV1", 8) != 0) return io_fail("feature file: bad magic", 0);
    if (version != 1) return io_fail("feature file: unsupported version " + std::to_string(version), 0);
    if (dtype != 0) return io_fail("feature file: unsupported dtype code " + std::to_string(dtype), 0);
    if (n == 0 || dim == 0) return io_fail("feature file: empty dataset", 0);
    if (row_bytes != dim * 4) return io_fail("feature file: row_bytes != dim * 4", 0);
    if (data_offset % 512 != 0 || data_offset < 64) return io_fail("feature file: misaligned data_offset", 0);
    const uint64_t want = data_offset + n * uint64_t(row_bytes);
    if (uint64_t(size) != want)
        return io_fail("feature file " + path + ": length " + std::to_string(size) + " != header-implied " +
                           std::to_string(want),
                       0);
    // rows stream to the device in 256 MB pieces through one pinned bounce buffer
    cudaSetDevice(c->device);
    void* dev = nullptr;
    FDG_CUDA(cudaMalloc(&dev, n * row_bytes));
    const uint64_t total = n * uint64_t(row_bytes), piece = std::min<uint64_t>(total, 256ull << 20);
    void* bounce = nullptr;
    cudaError_t e = cudaMallocHost(&bounce, piece);
    if (e != cudaSuccess) {
        cudaFree(dev);
        return cuda_fail(e, "cudaMallocHost(feature bounce buffer)", __FILE__, __LINE__);
    }
    int rc = FDG_OK;
    for (uint64_t at = 0; at < total && rc == FDG_OK; at += piece) {
        const uint64_t k = std::min<uint64_t>(piece, total - at);
        rc = read_at(f, path, data_offset + at, k, bounce);
        if (rc == FDG_OK && (e = cudaMemcpy(static_cast<char*>(dev) + at, bounce, k, cudaMemcpyHostToDevice)) !=
                                cudaSuccess)
            rc = cuda_fail(e, "cudaMemcpy(feature rows)", __FILE__, __LINE__);
    }
    cudaFreeHost(bounce);
    if (rc != FDG_OK) {
        cudaFree(dev);
        return rc;
    }
    return install_table(c, dev, n, row_bytes, 0);
}

// Out-of-core tier: move the (single-shard) table to pinned host memory mapped into the
// device address space. The gather and the buffer manager's miss path then read rows
// over PCIe / C2C with the same kernels -- the paper's host-resident feature store
// with the GPU feature buffer in front of it (PAPER.md:1033-1047 future work).
int fdg_ctx_features_to_host(fdg_ctx* c) {
    if (c->row_bytes == 0 || c->shard_bases.empty()) return fail(FDG_NOT_LOADED, "features_to_host: no feature table");
    if (c->n_shards != 1 || c->owned_shards.size() != 1)
        return fail(FDG_INVALID_ARG, "features_to_host: only an owned single-shard table can move to the host tier");
    if (c->host_table) return FDG_OK;
    cudaSetDevice(c->device);
    const uint64_t bytes = c->feat_nodes * c->row_bytes;
    void* h = nullptr;
    uint64_t mapped = 0;
    cudaError_t e = cudaSuccess;
    if (g_host_tier_thp) {
        mapped = (std::max<uint64_t>(bytes, 1) + (2ull << 20) - 1) & ~((2ull << 20) - 1);
        h = mmap(nullptr, mapped, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (h == MAP_FAILED) return io_fail("features_to_host: mmap", errno);
        madvise(h, mapped, MADV_HUGEPAGE);
        // pages on the GPU's own NUMA node: a table spread over both sockets reads the far half
        // over the inter-socket link (measured: 26 vs 48 GB/s of random rows for 57 vs 4 GB)
        const int node = gpu_numa_node(c->device);
        if (node >= 0 && node < 64) {
            unsigned long mask = 1ul << node;
            syscall(SYS_mbind, h, mapped, 2 /* MPOL_BIND */, &mask, 64, 0);
        }
        e = cudaHostRegister(h, mapped, cudaHostRegisterMapped | cudaHostRegisterPortable);
        if (e != cudaSuccess) {
            munmap(h, mapped);
            return cuda_fail(e, "cudaHostRegister(feature table)", __FILE__, __LINE__);
        }
    } else {
        FDG_CUDA(cudaHostAlloc(&h, std::max<uint64_t>(bytes, 1), cudaHostAllocMapped | cudaHostAllocPortable));
    }
    e = cudaMemcpy(h, c->owned_shards[0], bytes, cudaMemcpyDeviceToHost);
    void* dptr = nullptr;
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&dptr, h, 0);
    if (e != cudaSuccess) {
        if (mapped) {
            cudaHostUnregister(h);
            munmap(h, mapped);
        } else {
            cudaFreeHost(h);
        }
        return cuda_fail(e, "fdg_ctx_features_to_host", __FILE__, __LINE__);
    }
    cudaFree(c->owned_shards[0]);
    c->owned_shards.clear();
    c->host_table = h;
    c->host_table_bytes = mapped;
    c->shard_bases.assign(1, dptr);
    FDG_CUDA(cudaMemcpy((void*)c->shard_table, &dptr, sizeof(void*), cudaMemcpyHostToDevice));
    return FDG_OK;
}

int fdg_ctx_features_on_host(const fdg_ctx* c) { return c->host_table != nullptr; }

int fdg_ctx_generate_features(fdg_ctx* c, uint64_t seed, uint64_t n, uint32_t dim, uint32_t dtype, uint32_t n_shards) {
    cudaSetDevice(c->device);
    return generate_features(*c, seed, n, dim, dtype, n_shards);
}

int fdg_ctx_set_feature_shards(fdg_ctx* c, const void* const* bases, uint32_t n_shards, uint64_t rps, uint64_t n,
                               uint32_t row_bytes, uint32_t dtype) {
    if (n_shards == 0 || rps == 0 || (n + rps - 1) / rps > n_shards)
        return fail(FDG_INVALID_ARG, "feature shards: inconsistent geometry");
    cudaSetDevice(c->device);
    // allocations owned by the context (e.g. this rank's shard) stay alive until destroy
    c->shard_bases.clear();
    for (uint32_t i = 0; i < n_shards; ++i) c->shard_bases.push_back(const_cast<void*>(bases[i]));
    c->row_bytes = row_bytes;
    c->dtype = dtype;
    c->n_shards = n_shards;
    c->rows_per_shard = rps;
    c->feat_nodes = n;
    if (c->shard_table) cudaFree((void*)c->shard_table);
    FDG_CUDA(cudaMalloc((void**)&c->shard_table, n_shards * sizeof(void*)));
    FDG_CUDA(cudaMemcpy((void*)c->shard_table, c->shard_bases.data(), n_shards * sizeof(void*), cudaMemcpyHostToDevice));
    return FDG_OK;
}

int fdg_ctx_generate_feature_shard(fdg_ctx* c, uint64_t seed, uint64_t n, uint32_t dim, uint32_t dtype, uint32_t shard,
                                   uint32_t n_shards, void** base) {
    cudaSetDevice(c->device);
    return generate_feature_shard(*c, seed, n, dim, dtype, shard, n_shards, base);
}

int fdg_ipc_get_handle(const void* base, unsigned char* handle) {
    static_assert(sizeof(cudaIpcMemHandle_t) == FDG_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    FDG_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(base)));
    std::memcpy(handle, &h, sizeof(h));
    return FDG_OK;
}

int fdg_ipc_open_handle(const unsigned char* handle, void** base) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    // lazy peer enablement: remote rows are then read over NVLink by ordinary loads
    FDG_CUDA(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
    return FDG_OK;
}

int fdg_ipc_close_handle(void* base) {
    FDG_CUDA(cudaIpcCloseMemHandle(base));
    return FDG_OK;
}

int fdg_ctx_download_topology(const fdg_ctx* c, uint64_t* indptr, void* indices) {
    if (!c->indptr) return fail(FDG_NOT_LOADED, "no topology");
    cudaSetDevice(c->device);
    if (indptr) FDG_CUDA(cudaMemcpy(indptr, c->indptr, (c->num_nodes + 1) * 8, cudaMemcpyDeviceToHost));
    if (indices) FDG_CUDA(cudaMemcpy(indices, c->indices, c->num_edges * c->idx_bytes, cudaMemcpyDeviceToHost));
    return FDG_OK;
}

int fdg_ctx_download_rows(const fdg_ctx* c, uint64_t first, uint64_t count, void* out) {
    if (c->shard_bases.empty()) return fail(FDG_NOT_LOADED, "no feature table");
    if (first + count > c->feat_nodes) return fail(FDG_OUT_OF_RANGE, "download_rows: range out of bounds");
    cudaSetDevice(c->device);
    uint64_t at = first;
    char* o = static_cast<char*>(out);
    while (at < first + count) {
        uint64_t s = at / c->rows_per_shard, local = at - s * c->rows_per_shard;
        uint64_t k = std::min<uint64_t>(c->rows_per_shard - local, first + count - at);
        FDG_CUDA(cudaMemcpy(o, static_cast<const char*>(c->shard_bases[s]) + local * c->row_bytes, k * c->row_bytes,
                            cudaMemcpyDeviceToHost));
        o += k * c->row_bytes;
        at += k;
    }
    return FDG_OK;
}

// ---- sampler -----------------------------------------------------------------------
int fdg_sampler_create(fdg_ctx* c, uint32_t max_seeds, const uint32_t* fanouts, uint32_t n_layers, fdg_sampler** out) {
    cudaSetDevice(c->device);
    Sampler* s = nullptr;
    FDG_TRY(sampler_create(c, max_seeds, fanouts, n_layers, &s));
    *out = reinterpret_cast<fdg_sampler*>(s);
    return FDG_OK;
}
int fdg_sampler_destroy(fdg_sampler* s) {
    sampler_destroy(reinterpret_cast<Sampler*>(s));
    return FDG_OK;
}
int fdg_sampler_capacity(const fdg_sampler* s, uint64_t* mn, uint64_t* me) {
    sampler_capacity(reinterpret_cast<const Sampler*>(s), mn, me);
    return FDG_OK;
}
int fdg_sample_khop(fdg_sampler* s, void* st, const uint64_t* seeds, uint32_t n_seeds, uint64_t rng_seed,
                    uint64_t* nodes, uint32_t* edges, uint64_t cap, fdg_batch_counts* cnt) {
    return sampler_sample(reinterpret_cast<Sampler*>(s), (cudaStream_t)st, seeds, n_seeds, rng_seed, nodes, edges, cap,
                          cnt);
}
int fdg_sampler_prefetch(fdg_sampler* s, void* st, const uint64_t* rng_seeds, uint32_t n) {
    return sampler_prefetch(reinterpret_cast<Sampler*>(s), (cudaStream_t)st, rng_seeds, n);
}
int fdg_sample_khop_host(fdg_sampler* s, const uint64_t* seeds, uint32_t n_seeds, uint64_t rng_seed, uint64_t* nodes,
                         uint32_t* edges, uint64_t cap, uint64_t* nn, uint64_t* ne, uint64_t* ln, uint64_t* le) {
    return sampler_sample_host(reinterpret_cast<Sampler*>(s), seeds, n_seeds, rng_seed, nullptr, 0, nodes, edges, cap,
                               nn, ne, ln, le, nullptr);
}
int fdg_sample_khop_words_host(fdg_sampler* s, const uint64_t* seeds, uint32_t n_seeds, const uint64_t* words,
                               uint64_t n_words, uint64_t* nodes, uint32_t* edges, uint64_t cap, uint64_t* nn,
                               uint64_t* ne, uint64_t* wu) {
    return sampler_sample_host(reinterpret_cast<Sampler*>(s), seeds, n_seeds, 0, words, n_words, nodes, edges, cap, nn,
                               ne, nullptr, nullptr, wu);
}
int fdg_mt_stream(void* st, uint64_t rng_seed, uint64_t n, uint64_t* out) {
    FDG_CUDA(launch_mt_streams((cudaStream_t)st, &rng_seed, 1, n, out, n));
    return FDG_OK;
}

// ---- gather -------------------------------------------------------------------------
int fdg_gather(fdg_ctx* c, void* st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host, void* out,
               uint64_t* checksum) {
    return launch_gather(*c, (cudaStream_t)st, nodes, n_dev, n_host, out, checksum);
}

int fdg_set_gather_impl(int impl) {
    if (impl != FDG_GATHER_TMA && impl != FDG_GATHER_LDG && impl != FDG_GATHER_RB_DYN)
        return fail(FDG_INVALID_ARG, "unknown gather impl");
    g_gather_impl = impl;
    return FDG_OK;
}

int fdg_set_option(const char* key, int64_t v) {
    std::string k(key);
    if (k == "gather_impl") return fdg_set_gather_impl(int(v));
    if (k == "gather_evict_first") {  // 0 off, 1 loads + stores, 2 table loads only, 3 X stores only
        if (v < 0 || v > 3) return fail(FDG_INVALID_ARG, "gather_evict_first must be in [0, 3]");
        g_gather_evict_first = int(v);
        return FDG_OK;
    }
    if (k == "l2_persist_mb") { g_l2_persist_mb = v < 0 ? 0 : v; return FDG_OK; }
    if (k == "sampler_ctas_per_sm") {
        if (v < 1 || v > 64) return fail(FDG_INVALID_ARG, "sampler_ctas_per_sm must be in [1, 64]");
        g_sampler_ctas_per_sm = v;
        return FDG_OK;
    }
    if (k == "gather_ctas_per_sm") {
        if (v < 1 || v > 4) return fail(FDG_INVALID_ARG, "gather_ctas_per_sm must be in [1, 4]");
        g_gather_ctas_per_sm = int(v);
        return FDG_OK;
    }
    if (k == "hash_clear") { g_hash_clear = v != 0; return FDG_OK; }
    if (k == "hash_keep") { g_hash_keep = v != 0; return FDG_OK; }
    if (k == "pipeline_gather_impl") {
        if (v != FDG_GATHER_TMA && v != FDG_GATHER_LDG && v != FDG_GATHER_RB_DYN)
            return fail(FDG_INVALID_ARG, "pipeline_gather_impl: unknown gather impl");
        g_pipeline_gather_impl = v;
        return FDG_OK;
    }
    if (k == "rb_chunk") {
        if (v != 128 && v != 256) return fail(FDG_INVALID_ARG, "rb_chunk must be 128 or 256");
        g_rb_chunk = v;
        return FDG_OK;
    }
    if (k == "rb_ctas_per_sm") {
        if (v < 1 || v > 4) return fail(FDG_INVALID_ARG, "rb_ctas_per_sm must be in [1, 4]");
        g_rb_ctas_per_sm = v;
        return FDG_OK;
    }
    if (k == "gather_pf64") {
        if (v < 0 || v > 2) return fail(FDG_INVALID_ARG, "gather_pf64 must be 0, 1 or 2");
        g_gather_pf64 = v;
        return FDG_OK;
    }
    if (k == "bm_overlap") {
        g_bm_overlap = v != 0;
        return FDG_OK;
    }
    if (k == "mt_adaptive") {  // samplers created from now on: 0 bound, 1 estimate, 2 test (short)
        if (v < 0 || v > 2) return fail(FDG_INVALID_ARG, "mt_adaptive must be 0, 1 or 2");
        g_mt_adaptive = v;
        return FDG_OK;
    }
    if (k == "l2_fetch_granularity") {  // cudaLimitMaxL2FetchGranularity of the current device (bytes, 0-128)
        if (v < 0 || v > 128) return fail(FDG_INVALID_ARG, "l2_fetch_granularity must be in [0, 128]");
        FDG_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(v)));
        return FDG_OK;
    }
    if (k == "bm_sorted_move") {  // host-resident tables: misses moved in node-id order (1) or batch order (0)
        g_bm_sorted_move = v != 0;
        return FDG_OK;
    }
    if (k == "host_tier_thp") {  // features_to_host: THP-backed, NUMA-local registered memory (not cudaHostAlloc)
        g_host_tier_thp = v != 0;
        return FDG_OK;
    }
    if (k == "prefetch_upfront") {  // A/B only
        g_prefetch_upfront = v != 0;
        return FDG_OK;
    }
    if (k == "replay") {  // A/B only
        g_replay = v != 0;
        return FDG_OK;
    }
    if (k == "debug_zero_word") {  // (batch << 24) | word position, -1 off (pipeline runs)
        g_debug_zero_word = v;
        return FDG_OK;
    }
    if (k == "debug_reject_batch") {
        g_debug_reject_batch = v;
        return FDG_OK;
    }
    if (k == "bm_eager_invalidate") {  // debug: buffer managers created from now on invalidate eagerly
        g_bm_eager = v != 0;
        return FDG_OK;
    }
    if (k == "sage_gemm") {
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, "sage_gemm must be 0 (CUDA cores) or 1 (tensor cores)");
        g_sage_gemm = v;
        return FDG_OK;
    }
    if (k == "force_idx64") {  // test hook: topologies loaded / generated afterwards keep u64 indices
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, "force_idx64 must be 0 or 1");
        g_force_idx64 = v;
        return FDG_OK;
    }
    if (k == "early_bloom") {
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, "early_bloom must be 0 or 1");
        g_early_bloom = v;
        return FDG_OK;
    }
    if (k == "host_tier_pf") {
        if (v < 0 || v > 2) return fail(FDG_INVALID_ARG, "host_tier_pf must be 0, 1 or 2");
        g_host_tier_pf = v;
        return FDG_OK;
    }
    if (k == "intern_lean") {
        if (v < 0 || v > 2) return fail(FDG_INVALID_ARG, "intern_lean must be 0, 1 or 2");
        g_intern_lean = v;
        return FDG_OK;
    }
    if (k == "early_fused") {
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, "early_fused must be 0 or 1");
        g_early_fused = v;
        return FDG_OK;
    }
    if (k == "hash_early_pct") {
        if (v != 0 && (v < 5 || v > 90)) return fail(FDG_INVALID_ARG, "hash_early_pct must be 0 or in [5, 90]");
        g_hash_early_pct = v;
        return FDG_OK;
    }
    if (k == "bm_move_hash") {
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, "bm_move_hash must be 0 or 1");
        g_bm_move_hash = v;
        return FDG_OK;
    }
    if (k == "bm_fuse_bind") {
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, "bm_fuse_bind must be 0 or 1");
        g_bm_fuse_bind = v;
        return FDG_OK;
    }
    if (k == "pipe_slots") {
        if (v < 0 || v > 256) return fail(FDG_INVALID_ARG, "pipe_slots must be in [0, 256]");
        g_pipe_slots = v;
        return FDG_OK;
    }
    if (k == "extract_prio") {
        if (v < 0 || v > 2) return fail(FDG_INVALID_ARG, "extract_prio must be 0, 1 or 2 (buffer manager only)");
        g_extract_prio = v;
        return FDG_OK;
    }
    if (k == "bm_split_move") {
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, "bm_split_move must be 0 or 1");
        g_bm_split_move = v;
        return FDG_OK;
    }
    if (k == "bm_move_grid" || k == "bm_meta_prio" || k == "bm_move_early" || k == "records_stream") {
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, k + " must be 0 or 1");
        (k == "bm_move_grid"    ? g_bm_move_grid
         : k == "bm_meta_prio"  ? g_bm_meta_prio
         : k == "bm_move_early" ? g_bm_move_early
                                : g_records_stream) = v;
        return FDG_OK;
    }
    if (k == "bm_move_impl") {
        if (v < 0 || v > 2) return fail(FDG_INVALID_ARG, "bm_move_impl must be 0 (LDG), 1 (TMA) or 2 (row groups)");
        g_bm_move_impl = v;
        return FDG_OK;
    }
    if (k == "hash_ctas") {
        if (v < 0 || v > 4096) return fail(FDG_INVALID_ARG, "hash_ctas must be in [0, 4096]");
        g_hash_ctas = v;
        return FDG_OK;
    }
    if (k == "hash_ctas_per_sm") {
        if (v < 0 || v > 4) return fail(FDG_INVALID_ARG, "hash_ctas_per_sm must be in [0, 4]");
        g_hash_ctas_per_sm = v;
        return FDG_OK;
    }
    if (k == "hash_dyn") {
        if (v != 0 && v != 1) return fail(FDG_INVALID_ARG, "hash_dyn must be 0 or 1");
        g_hash_dyn = v;
        return FDG_OK;
    }
    if (k == "hash_chunk") {
        if (v != 0 && v != 128 && v != 256) return fail(FDG_INVALID_ARG, "hash_chunk must be 0, 128 or 256");
        g_hash_chunk = v;
        return FDG_OK;
    }
    if (k == "checksum_impl") {
        if (v != -1 && v != FDG_GATHER_TMA && v != FDG_GATHER_LDG && v != FDG_GATHER_RB_DYN)
            return fail(FDG_INVALID_ARG, "checksum_impl must be -1 or a gather impl");
        g_checksum_impl = v;
        return FDG_OK;
    }
    if (k == "tma_cfg") {
        if (v < 0 || v > 3) return fail(FDG_INVALID_ARG, "tma_cfg must be in [0, 3]");
        g_tma_cfg = v;
        return FDG_OK;
    }
    if (k == "sampler_sms") {
        if (v < 0 || v > 1024) return fail(FDG_INVALID_ARG, "sampler_sms must be in [0, 1024]");
        g_sampler_sms = v;
        return FDG_OK;
    }
    if (k == "extract_streams") {
        if (v < 1 || v > 2) return fail(FDG_INVALID_ARG, "extract_streams must be 1 or 2");
        g_extract_streams = v;
        return FDG_OK;
    }
    if (k == "hash_load_pct") {
        if (v < 10 || v > 70) return fail(FDG_INVALID_ARG, "hash_load_pct must be in [10, 70]");
        g_hash_load_pct = v;
        return FDG_OK;
    }
    return fail(FDG_INVALID_ARG, "unknown option " + k);
}

int fdg_get_option(const char* key, int64_t* v) {
    std::string k(key);
    if (k == "gather_impl") *v = g_gather_impl;
    else if (k == "gather_evict_first") *v = g_gather_evict_first;
    else if (k == "l2_persist_mb") *v = g_l2_persist_mb;
    else if (k == "hash_load_pct") *v = g_hash_load_pct;
    else if (k == "gather_ctas_per_sm") *v = g_gather_ctas_per_sm;
    else if (k == "sampler_ctas_per_sm") *v = g_sampler_ctas_per_sm;
    else if (k == "hash_clear") *v = g_hash_clear;
    else if (k == "hash_keep") *v = g_hash_keep;
    else if (k == "hash_chunk") *v = g_hash_chunk;
    else if (k == "sage_gemm") *v = g_sage_gemm;
    else if (k == "bm_overlap") *v = g_bm_overlap;
    else if (k == "bm_eager_invalidate") *v = g_bm_eager;
    else if (k == "debug_zero_word") *v = g_debug_zero_word;
    else if (k == "mt_adaptive") *v = g_mt_adaptive;
    else if (k == "replay") *v = g_replay;
    else if (k == "prefetch_upfront") *v = g_prefetch_upfront;
    else if (k == "host_tier_thp") *v = g_host_tier_thp;
    else if (k == "bm_sorted_move") *v = g_bm_sorted_move;
    else if (k == "l2_fetch_granularity") {
        size_t g = 0;
        FDG_CUDA(cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity));
        *v = int64_t(g);
    }
    else if (k == "debug_reject_batch") *v = g_debug_reject_batch;
    else if (k == "gather_pf64") *v = g_gather_pf64;
    else if (k == "rb_ctas_per_sm") *v = g_rb_ctas_per_sm;
    else if (k == "rb_chunk") *v = g_rb_chunk;
    else if (k == "pipeline_gather_impl") *v = g_pipeline_gather_impl;
    else if (k == "checksum_impl") *v = g_checksum_impl;
    else if (k == "extract_streams") *v = g_extract_streams;
    else if (k == "sampler_sms") *v = g_sampler_sms;
    else if (k == "tma_cfg") *v = g_tma_cfg;
    else if (k == "hash_dyn") *v = g_hash_dyn;
    else if (k == "hash_ctas_per_sm") *v = g_hash_ctas_per_sm;
    else if (k == "hash_ctas") *v = g_hash_ctas;
    else if (k == "bm_move_impl") *v = g_bm_move_impl;
    else if (k == "bm_move_grid") *v = g_bm_move_grid;
    else if (k == "bm_fuse_bind") *v = g_bm_fuse_bind;
    else if (k == "bm_move_hash") *v = g_bm_move_hash;
    else if (k == "hash_early_pct") *v = g_hash_early_pct;
    else if (k == "early_fused") *v = g_early_fused;
    else if (k == "intern_lean") *v = g_intern_lean;
    else if (k == "host_tier_pf") *v = g_host_tier_pf;
    else if (k == "early_bloom") *v = g_early_bloom;
    else if (k == "force_idx64") *v = g_force_idx64;
    else if (k == "bm_meta_prio") *v = g_bm_meta_prio;
    else if (k == "bm_move_early") *v = g_bm_move_early;
    else if (k == "extract_prio") *v = g_extract_prio;
    else if (k == "records_stream") *v = g_records_stream;
    else if (k == "pipe_slots") *v = g_pipe_slots;
    else if (k == "bm_split_move") *v = g_bm_split_move;
    else if (k == "tc_write_hi") *v = tc_write_hi(nullptr);  // runs the once-per-device check
    else return fail(FDG_INVALID_ARG, "unknown option " + k);
    return FDG_OK;
}

int fdg_checksum_alias(fdg_ctx* c, void* st, const void* region, const int64_t* alias, const uint32_t* n_dev,
                       uint64_t n_host, uint64_t* checksum) {
    return launch_checksum_alias(*c, (cudaStream_t)st, region, alias, n_dev, n_host, checksum);
}

// ---- host helpers -------------------------------------------------------------------
// partition_epoch (sampling.hpp:57-70): std::shuffle with mt19937_64(splitmix64(seed)),
// the same libstdc++ as the reference build, then chunks of batch_size.
int fdg_partition_epoch(const uint64_t* ids, uint64_t n, uint64_t batch_size, uint64_t shuffle_seed, uint64_t* out) {
    if (batch_size < 1) return fail(FDG_INVALID_ARG, "partition_epoch: batch_size must be >= 1");
    std::vector<uint64_t> v(ids, ids + n);
    std::mt19937_64 rng(splitmix64(shuffle_seed));
    std::shuffle(v.begin(), v.end(), rng);
    std::memcpy(out, v.data(), n * 8);
    return FDG_OK;
}

uint64_t fdg_batch_seed(uint64_t seed, uint64_t epoch, uint64_t b) { return hash_combine(hash_combine(seed, epoch), b); }

}  // extern "C"
