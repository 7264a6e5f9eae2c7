// Communicators of the data-parallel nexel::train (dp_b200.hpp).
#include "dp_b200.hpp"

#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "nexel/error.hpp"

namespace nexel {

namespace {

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}

std::string dp_dir() {
    const char* e = std::getenv("NEXEL_DP_DIR");
    if (!e || !*e) fail("bad-config", "NEXEL_DP_WORLD > 1 needs NEXEL_DP_DIR (a fresh node-local directory)");
    return e;
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail("cuda-error", std::string("data-parallel ") + what + ": " + cudaGetErrorString(e));
}

// Waits for `path` to appear (written by another rank with an atomic rename).
void wait_for(const std::string& path, const char* what) {
    const auto t0 = std::chrono::steady_clock::now();
    struct stat sb;
    while (stat(path.c_str(), &sb) != 0) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(env_int("NEXEL_DP_TIMEOUT_S", 300)))
            fail("dp-timeout", std::string("data-parallel rendezvous: no ") + what + " at " + path);
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
}

// ---------------------------------------------------------------- NCCL
struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) fail("unsupported", std::string("NEXEL_DP_BACKEND=nccl: cannot load libnccl: ") + dlerror());
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.comm_destroy || !a.error_string)
            fail("unsupported", "libnccl lacks the entry points the data-parallel train needs");
        return a;
    }();
    return api;
}

class NcclComm final : public DpComm {
   public:
    NcclComm(int world_, int rank_) {
        world = world_;
        rank = rank_;
        const NcclApi& api = nccl();
        ncclUniqueId id;
        const std::string path = dp_dir() + "/nccl_id";
        if (rank == 0) {  // rank 0 publishes the id (written, then renamed: readers see it whole)
            check(api.get_unique_id(&id), "ncclGetUniqueId");
            const std::string tmp = path + ".tmp";
            FILE* f = std::fopen(tmp.c_str(), "wb");
            if (!f || std::fwrite(&id, sizeof id, 1, f) != 1) fail("io-error", "cannot write " + tmp);
            std::fclose(f);
            if (std::rename(tmp.c_str(), path.c_str()) != 0) fail("io-error", "cannot publish " + path);
        } else {
            wait_for(path, "NCCL id");
            FILE* f = std::fopen(path.c_str(), "rb");
            if (!f || std::fread(&id, sizeof id, 1, f) != 1) fail("io-error", "cannot read " + path);
            std::fclose(f);
        }
        check(api.comm_init_rank(&comm_, world, id, rank), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm_) nccl().comm_destroy(comm_);
    }
    void all_reduce(double* dev, size_t n, bool average, cudaStream_t stream) override {
        if (n == 0) return;
        check(nccl().all_reduce(dev, dev, n, ncclDouble, average ? ncclAvg : ncclSum, comm_, stream), "ncclAllReduce");
    }

   private:
    void check(ncclResult_t r, const char* what) {
        if (r != ncclSuccess) fail("nccl-error", std::string(what) + ": " + nccl().error_string(r));
    }
    ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------------- host (shared memory)
struct ShmHeader {
    std::atomic<int> arrived;
    std::atomic<int> generation;
    int world;
    int chunk;  // doubles per rank slot
};
static_assert(std::atomic<int>::is_always_lock_free, "process-shared atomics");
static_assert(sizeof(ShmHeader) <= 128, "slots start 128 bytes into the segment");

class HostComm final : public DpComm {
   public:
    static constexpr int kChunk = 1 << 19;  // doubles per rank slot (4 MB)

    HostComm(int world_, int rank_) {
        world = world_;
        rank = rank_;
        const std::string path = dp_dir() + "/nexel_dp_shm";
        bytes_ = 128 + static_cast<size_t>(world) * kChunk * sizeof(double);
        int fd = -1;
        if (rank == 0) {
            const std::string tmp = path + ".tmp";
            fd = ::open(tmp.c_str(), O_RDWR | O_CREAT | O_EXCL, 0600);
            if (fd < 0) fail("io-error", "cannot create " + tmp + " (NEXEL_DP_DIR must be fresh)");
            if (ftruncate(fd, static_cast<off_t>(bytes_)) != 0) fail("io-error", "cannot size " + tmp);
            map(fd);
            new (hdr_) ShmHeader{};
            hdr_->arrived.store(0);
            hdr_->generation.store(0);
            hdr_->world = world;
            hdr_->chunk = kChunk;
            if (std::rename(tmp.c_str(), path.c_str()) != 0) fail("io-error", "cannot publish " + path);
        } else {
            wait_for(path, "shared-memory segment");
            fd = ::open(path.c_str(), O_RDWR);
            if (fd < 0) fail("io-error", "cannot open " + path);
            map(fd);
            if (hdr_->world != world || hdr_->chunk != kChunk)
                fail("bad-config", "data-parallel ranks disagree on NEXEL_DP_WORLD");
        }
        ::close(fd);
        cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&pin_), kChunk * sizeof(double), cudaHostAllocDefault),
                "pinned buffer");
        barrier();  // every rank attached
    }
    ~HostComm() override {
        if (pin_) cudaFreeHost(pin_);
        if (base_) munmap(base_, bytes_);
    }
    void all_reduce(double* dev, size_t n, bool average, cudaStream_t stream) override {
        const double inv = 1.0 / world;
        for (size_t off = 0; off < n; off += kChunk) {
            const size_t m = std::min<size_t>(kChunk, n - off);
            cuda_ok(cudaMemcpyAsync(pin_, dev + off, m * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
            cuda_ok(cudaStreamSynchronize(stream), "sync");
            std::memcpy(slot(rank), pin_, m * sizeof(double));
            barrier();
            for (size_t i = 0; i < m; ++i) {  // rank order: the same sum on every rank
                double s = slot(0)[i];
                for (int r = 1; r < world; ++r) s += slot(r)[i];
                pin_[i] = average ? s * inv : s;
            }
            barrier();  // every rank has read the slots before they are reused
            cuda_ok(cudaMemcpyAsync(dev + off, pin_, m * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
            cuda_ok(cudaStreamSynchronize(stream), "sync");
        }
    }

   private:
    void map(int fd) {
        base_ = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        if (base_ == MAP_FAILED) {
            base_ = nullptr;
            fail("io-error", "cannot map the data-parallel segment");
        }
        hdr_ = static_cast<ShmHeader*>(base_);
        slots_ = reinterpret_cast<double*>(static_cast<char*>(base_) + 128);
    }
    double* slot(int r) { return slots_ + static_cast<size_t>(r) * kChunk; }
    void barrier() {  // generation barrier over the shared counters
        const int gen = hdr_->generation.load(std::memory_order_acquire);
        if (hdr_->arrived.fetch_add(1, std::memory_order_acq_rel) == world - 1) {
            hdr_->arrived.store(0, std::memory_order_relaxed);
            hdr_->generation.fetch_add(1, std::memory_order_acq_rel);
            return;
        }
        const auto t0 = std::chrono::steady_clock::now();
        for (int spin = 0; hdr_->generation.load(std::memory_order_acquire) == gen; ++spin) {
            if (spin > 1000) std::this_thread::yield();
            if ((spin & 0xffff) == 0 &&
                std::chrono::steady_clock::now() - t0 > std::chrono::seconds(env_int("NEXEL_DP_TIMEOUT_S", 300)))
                fail("dp-timeout", "data-parallel barrier: a rank did not arrive");
        }
    }
    void* base_ = nullptr;
    size_t bytes_ = 0;
    ShmHeader* hdr_ = nullptr;
    double* slots_ = nullptr;
    double* pin_ = nullptr;
};

}  // namespace

int dp_env_world() { return std::max(1, env_int("NEXEL_DP_WORLD", 1)); }
int dp_env_rank() { return dp_env_world() > 1 ? env_int("NEXEL_DP_RANK", 0) : 0; }

std::unique_ptr<DpComm> DpComm::from_env(int device) {
    const int world = dp_env_world();
    if (world <= 1) return nullptr;
    const int rank = dp_env_rank();
    if (rank < 0 || rank >= world) fail("bad-config", "NEXEL_DP_RANK must be in [0, NEXEL_DP_WORLD)");
    cuda_ok(cudaSetDevice(device), "cudaSetDevice");
    const char* b = std::getenv("NEXEL_DP_BACKEND");
    if (b && std::strcmp(b, "host") == 0) return std::make_unique<HostComm>(world, rank);
    if (b && *b && std::strcmp(b, "nccl") != 0) fail("bad-config", std::string("unknown NEXEL_DP_BACKEND ") + b);
    return std::make_unique<NcclComm>(world, rank);
}

}  // namespace nexel
