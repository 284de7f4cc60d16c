// Test-only stand-in for the five NCCL entry points psw_shard.cpp loads
// (PSW_NCCL_LIB): an all-reduce(sum, fp64) between PROCESSES that may share
// one GPU, staged through POSIX shared memory. It exists so that the
// multi-rank code path of psw_shard_solve (rank > 0 plans, communicator
// checks, the in-place sum between the two halves of the solve) can run with
// world_size 2 on a one-GPU box. No kernel waits on another process: the call
// drains its stream, copies the partial sums to the host, meets the other
// ranks at a host barrier, adds the ranks' slots in rank order and copies the
// result back. Not NCCL, not a performance path, not shipped in the library.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

extern "C" {
typedef struct { char internal[128]; } ncclUniqueId;
typedef struct FakeComm* ncclComm_t;
typedef int ncclResult_t;   // 0 = ncclSuccess
typedef int ncclDataType_t; // 8 = ncclFloat64
typedef int ncclRedOp_t;    // 0 = ncclSum
}

namespace {
constexpr size_t kSlotBytes = size_t(8) << 20;
struct Header {
    std::atomic<int> arrived;
    std::atomic<int> generation;
};
}  // namespace

struct FakeComm {
    int nranks, rank;
    char name[136];
    Header* hdr;
    char* slots;
    size_t bytes;
};

static bool barrier(FakeComm* c) {
    const int gen = c->hdr->generation.load();
    if (c->hdr->arrived.fetch_add(1) + 1 == c->nranks) {
        c->hdr->arrived.store(0);
        c->hdr->generation.fetch_add(1);
        return true;
    }
    const auto t0 = std::chrono::steady_clock::now();
    while (c->hdr->generation.load() == gen) {
        std::this_thread::sleep_for(std::chrono::microseconds(50));
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60)) return false;
    }
    return true;
}

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::memset(id, 0, sizeof(*id));
    const auto t = std::chrono::steady_clock::now().time_since_epoch().count();
    std::snprintf(id->internal, sizeof(id->internal), "/pswfake_%d_%lld", int(getpid()), (long long)t);
    return 0;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
    auto* c = new FakeComm();
    c->nranks = nranks;
    c->rank = rank;
    std::snprintf(c->name, sizeof(c->name), "%s", id.internal);
    c->bytes = 4096 + size_t(nranks) * kSlotBytes;
    const int fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, off_t(c->bytes)) != 0) return 2;
    void* m = mmap(nullptr, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return 2;
    c->hdr = static_cast<Header*>(m);  // a fresh segment is zero-filled: both counters start at 0
    c->slots = static_cast<char*>(m) + 4096;
    *out = c;
    return barrier(c) ? 0 : 6;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
    if (!c) return 0;
    barrier(c);
    munmap(c->hdr, c->bytes);
    if (c->rank == 0) shm_unlink(c->name);
    delete c;
    return 0;
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                           ncclComm_t c, cudaStream_t s) {
    if (dt != 8 || op != 0 || count * 8 > kSlotBytes) return 4;
    if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
    double* mine = reinterpret_cast<double*>(c->slots + size_t(c->rank) * kSlotBytes);
    if (cudaMemcpy(mine, send, count * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    if (!barrier(c)) return 6;
    std::vector<double> sum(count, 0.0);
    for (int r = 0; r < c->nranks; ++r) {
        const double* v = reinterpret_cast<const double*>(c->slots + size_t(r) * kSlotBytes);
        for (size_t i = 0; i < count; ++i) sum[i] += v[i];
    }
    if (!barrier(c)) return 6;  // every rank has read the slots: they may be rewritten
    if (cudaMemcpy(recv, sum.data(), count * 8, cudaMemcpyHostToDevice) != cudaSuccess) return 1;
    return 0;
}

const char* ncclGetErrorString(ncclResult_t r) {
    switch (r) {
        case 0: return "success";
        case 1: return "fake nccl: CUDA error";
        case 2: return "fake nccl: shared memory error";
        case 4: return "fake nccl: unsupported reduction";
        case 6: return "fake nccl: a rank did not arrive";
        default: return "fake nccl: error";
    }
}
}
