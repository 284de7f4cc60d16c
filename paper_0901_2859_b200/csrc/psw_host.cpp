// psw_solve_host: the end-to-end solve_batch (dichotomy/batch.hpp:57-75) on
// host buffers. RHS chunks are staged through kSlots device slots so that
// the host->device copy of chunk c+1 and the device->host copy of chunk c-1
// overlap the solve of chunk c (three streams, event-ordered; PCIe copies in
// both directions run concurrently). Streams, events and the staging buffer
// are created once per device and reused (a fresh stream-ordered allocation
// per call is returned to the OS at every synchronisation and re-mapped on
// the next call, which cost milliseconds per solve).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "psw_internal.h"

namespace {

constexpr int kSlots = 3;
constexpr size_t kChunkBytes = size_t(16) << 20;  // per chunk (>= 8 chunks when there is work)

size_t chunk_bytes() {  // PSW_HOST_CHUNK_MB: tuning override
    static const size_t b = [] {
        const char* e = std::getenv("PSW_HOST_CHUNK_MB");
        const int mb = e ? std::atoi(e) : 0;
        return mb > 0 ? size_t(mb) << 20 : kChunkBytes;
    }();
    return b;
}

struct HostPipe {
    std::mutex mu;
    bool ready = false;
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t up[kSlots] = {}, done[kSlots] = {}, freed[kSlots] = {};
    void* buf = nullptr;
    size_t buf_bytes = 0;

    int init() {
        if (ready) return PSW_OK;
        PSW_CUDA_TRY(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
        PSW_CUDA_TRY(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking));
        PSW_CUDA_TRY(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
        for (int i = 0; i < kSlots; ++i) {
            PSW_CUDA_TRY(cudaEventCreateWithFlags(&up[i], cudaEventDisableTiming));
            PSW_CUDA_TRY(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
            PSW_CUDA_TRY(cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming));
        }
        ready = true;
        return PSW_OK;
    }
    int reserve(size_t bytes) {
        if (bytes <= buf_bytes) return PSW_OK;
        if (buf) cudaFree(buf);
        buf = nullptr;
        buf_bytes = 0;
        PSW_CUDA_TRY(cudaMalloc(&buf, bytes));
        buf_bytes = bytes;
        return PSW_OK;
    }
};

HostPipe& pipe_for(int dev) {
    static std::mutex mu;
    static std::vector<HostPipe*> pipes;
    std::lock_guard<std::mutex> lk(mu);
    if (size_t(dev) >= pipes.size()) pipes.resize(size_t(dev) + 1, nullptr);
    if (!pipes[size_t(dev)]) pipes[size_t(dev)] = new HostPipe();  // lives for the process
    return *pipes[size_t(dev)];
}

}  // namespace

extern "C" int psw_solve_host(const psw_plan* plan, const void* F, int64_t ldf, void* X,
                              int64_t ldx, int64_t nrhs, int layout) {
    psw::clear_error();
    if (!plan || nrhs < 0 || (nrhs > 0 && (!F || !X)) ||
        (layout != PSW_LAYOUT_R && layout != PSW_LAYOUT_S)) {
        psw::set_error(PSW_INVALID_ARGUMENT, "invalid arguments to psw_solve_host");
        return PSW_INVALID_ARGUMENT;
    }
    const int64_t need = layout == PSW_LAYOUT_R ? nrhs : plan->n;
    if (ldf < need || ldx < need) {
        psw::set_error(PSW_INVALID_ARGUMENT, "leading dimension too small for the layout");
        return PSW_INVALID_ARGUMENT;
    }
    if (nrhs == 0) return PSW_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    PSW_CUDA_TRY(cudaSetDevice(plan->device));
    const int64_t n = plan->n;
    const size_t es = plan->dtype == PSW_F64 ? 8 : 4;
    // >= 16 MB chunks, up to 1/16 of the batch (<= 1 GB) for large batches so
    // that every chunk's solve is itself a full-GPU launch
    const size_t total = size_t(nrhs) * size_t(n) * es;
    const size_t target = std::max(chunk_bytes(), std::min(size_t(1) << 30, total / 16));
    int64_t c = std::max<int64_t>(1, int64_t(target / (size_t(n) * es)));
    c = std::min<int64_t>(c, std::max<int64_t>(1, (nrhs + 7) / 8));
    if (layout == PSW_LAYOUT_R) {
        // a layout-R chunk is a pitched copy of c * es bytes per row: keep
        // rows >= 2 KB (narrower DMA rows crawl: 16-256 B rows ran at 2-16
        // GB/s on the 2^20-row and fp32 configs), even if chunks get large
        static const int64_t min_row = [] {  // PSW_HOST_MIN_ROW: tuning override (bytes)
            const char* e = std::getenv("PSW_HOST_MIN_ROW");
            return e && std::atoll(e) > 0 ? int64_t(std::atoll(e)) : int64_t(2048);
        }();
        c = std::max<int64_t>(c, min_row / int64_t(es));
        if (c >= 32) c = c / 32 * 32;
    }
    c = std::min(c, nrhs);
    const int64_t nchunks = (nrhs + c - 1) / c;
    const size_t slot_bytes = (size_t(c) * size_t(n) * es + 255) & ~size_t(255);

    HostPipe& st = pipe_for(plan->device);
    std::lock_guard<std::mutex> lk(st.mu);
    int rc = st.init();
    if (rc == PSW_OK) rc = st.reserve(kSlots * slot_bytes);
    if (rc != PSW_OK) {
        cudaSetDevice(prev);
        return rc;
    }
    // the pipeline starts after any earlier work of this thread's device.
    // A failing call stops issuing, but every copy already queued is waited
    // for below before returning (the caller may free F and X afterwards),
    // and the caller's device is restored on every path.
    int64_t launches = 0;
#define PSW_HOST_TRY(expr)                                        \
    do {                                                          \
        if (rc == PSW_OK) {                                       \
            const cudaError_t _e = (expr);                        \
            if (_e != cudaSuccess) rc = psw::cuda_fail(_e, #expr); \
        }                                                         \
    } while (0)
    for (int64_t ci = 0; ci < nchunks && rc == PSW_OK; ++ci) {
        const int slot = int(ci % kSlots);
        const int64_t k0 = ci * c, kc = std::min(c, nrhs - k0);
        char* dbuf = static_cast<char*>(st.buf) + slot * slot_bytes;
        const int64_t dld = layout == PSW_LAYOUT_R ? kc : n;
        if (ci >= kSlots) PSW_HOST_TRY(cudaStreamWaitEvent(st.h2d, st.freed[slot], 0));
        if (layout == PSW_LAYOUT_R)
            PSW_HOST_TRY(cudaMemcpy2DAsync(dbuf, size_t(kc) * es,
                                           static_cast<const char*>(F) + size_t(k0) * es,
                                           size_t(ldf) * es, size_t(kc) * es, size_t(n),
                                           cudaMemcpyHostToDevice, st.h2d));
        else
            PSW_HOST_TRY(cudaMemcpy2DAsync(dbuf, size_t(n) * es,
                                           static_cast<const char*>(F) + size_t(k0) * size_t(ldf) * es,
                                           size_t(ldf) * es, size_t(n) * es, size_t(kc),
                                           cudaMemcpyHostToDevice, st.h2d));
        PSW_HOST_TRY(cudaEventRecord(st.up[slot], st.h2d));
        PSW_HOST_TRY(cudaStreamWaitEvent(st.comp, st.up[slot], 0));
        if (rc == PSW_OK) {
            rc = psw_solve(plan, dbuf, dld, dbuf, dld, kc, layout, st.comp);
            launches += psw_last_launch_count();
        }
        if (rc != PSW_OK) break;
        PSW_HOST_TRY(cudaEventRecord(st.done[slot], st.comp));
        PSW_HOST_TRY(cudaStreamWaitEvent(st.d2h, st.done[slot], 0));
        if (layout == PSW_LAYOUT_R)
            PSW_HOST_TRY(cudaMemcpy2DAsync(static_cast<char*>(X) + size_t(k0) * es, size_t(ldx) * es,
                                           dbuf, size_t(kc) * es, size_t(kc) * es, size_t(n),
                                           cudaMemcpyDeviceToHost, st.d2h));
        else
            PSW_HOST_TRY(cudaMemcpy2DAsync(static_cast<char*>(X) + size_t(k0) * size_t(ldx) * es,
                                           size_t(ldx) * es, dbuf, size_t(n) * es, size_t(n) * es,
                                           size_t(kc), cudaMemcpyDeviceToHost, st.d2h));
        PSW_HOST_TRY(cudaEventRecord(st.freed[slot], st.d2h));
    }
#undef PSW_HOST_TRY
    cudaError_t e1 = cudaStreamSynchronize(st.d2h);
    cudaError_t e2 = cudaStreamSynchronize(st.comp);
    cudaStreamSynchronize(st.h2d);
    cudaSetDevice(prev);
    psw::reset_launches();
    psw::note_launches(launches);
    if (rc == PSW_OK && e1 != cudaSuccess) return psw::cuda_fail(e1, "psw_solve_host d2h");
    if (rc == PSW_OK && e2 != cudaSuccess) return psw::cuda_fail(e2, "psw_solve_host solve");
    return rc;
}
