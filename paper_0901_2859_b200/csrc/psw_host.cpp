// psw_solve_host: the end-to-end solve_batch (dichotomy/batch.hpp:57-75) on
// host buffers. RHS chunks are staged through two device slots so that the
// host->device copy of chunk c+1 and the device->host copy of chunk c-1
// overlap the solve of chunk c (three streams, event-ordered).
#include <algorithm>

#include "psw_internal.h"

namespace {

struct Streams {
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t up[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr},
                freed[2] = {nullptr, nullptr};
    ~Streams() {
        for (int i = 0; i < 2; ++i) {
            if (up[i]) cudaEventDestroy(up[i]);
            if (done[i]) cudaEventDestroy(done[i]);
            if (freed[i]) cudaEventDestroy(freed[i]);
        }
        if (h2d) cudaStreamDestroy(h2d);
        if (comp) cudaStreamDestroy(comp);
        if (d2h) cudaStreamDestroy(d2h);
    }
};

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
    // ~32 MiB per chunk, at least 4 chunks when there is enough work
    int64_t c = std::max<int64_t>(1, int64_t((32u << 20) / (size_t(n) * es)));
    c = std::min<int64_t>(c, std::max<int64_t>(1, (nrhs + 3) / 4));
    if (layout == PSW_LAYOUT_R && c >= 32) c = c / 32 * 32;
    c = std::min(c, nrhs);
    const int64_t nchunks = (nrhs + c - 1) / c;
    const size_t slot_bytes = size_t(c) * size_t(n) * es;

    Streams st;
    PSW_CUDA_TRY(cudaStreamCreateWithFlags(&st.h2d, cudaStreamNonBlocking));
    PSW_CUDA_TRY(cudaStreamCreateWithFlags(&st.comp, cudaStreamNonBlocking));
    PSW_CUDA_TRY(cudaStreamCreateWithFlags(&st.d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        PSW_CUDA_TRY(cudaEventCreateWithFlags(&st.up[i], cudaEventDisableTiming));
        PSW_CUDA_TRY(cudaEventCreateWithFlags(&st.done[i], cudaEventDisableTiming));
        PSW_CUDA_TRY(cudaEventCreateWithFlags(&st.freed[i], cudaEventDisableTiming));
    }
    void* buf = nullptr;
    PSW_CUDA_TRY(cudaMallocAsync(&buf, 2 * slot_bytes, st.comp));
    PSW_CUDA_TRY(cudaStreamSynchronize(st.comp));
    int64_t launches = 0;
    int rc = PSW_OK;
    for (int64_t ci = 0; ci < nchunks && rc == PSW_OK; ++ci) {
        const int slot = int(ci & 1);
        const int64_t k0 = ci * c, kc = std::min(c, nrhs - k0);
        char* dbuf = static_cast<char*>(buf) + slot * slot_bytes;
        const int64_t dld = layout == PSW_LAYOUT_R ? kc : n;
        if (ci >= 2) PSW_CUDA_TRY(cudaStreamWaitEvent(st.h2d, st.freed[slot], 0));
        if (layout == PSW_LAYOUT_R)
            PSW_CUDA_TRY(cudaMemcpy2DAsync(dbuf, size_t(kc) * es,
                                           static_cast<const char*>(F) + size_t(k0) * es,
                                           size_t(ldf) * es, size_t(kc) * es, size_t(n),
                                           cudaMemcpyHostToDevice, st.h2d));
        else
            PSW_CUDA_TRY(cudaMemcpy2DAsync(dbuf, size_t(n) * es,
                                           static_cast<const char*>(F) + size_t(k0) * size_t(ldf) * es,
                                           size_t(ldf) * es, size_t(n) * es, size_t(kc),
                                           cudaMemcpyHostToDevice, st.h2d));
        PSW_CUDA_TRY(cudaEventRecord(st.up[slot], st.h2d));
        PSW_CUDA_TRY(cudaStreamWaitEvent(st.comp, st.up[slot], 0));
        rc = psw_solve(plan, dbuf, dld, dbuf, dld, kc, layout, st.comp);
        launches += psw_last_launch_count();
        if (rc != PSW_OK) break;
        PSW_CUDA_TRY(cudaEventRecord(st.done[slot], st.comp));
        PSW_CUDA_TRY(cudaStreamWaitEvent(st.d2h, st.done[slot], 0));
        if (layout == PSW_LAYOUT_R)
            PSW_CUDA_TRY(cudaMemcpy2DAsync(static_cast<char*>(X) + size_t(k0) * es, size_t(ldx) * es,
                                           dbuf, size_t(kc) * es, size_t(kc) * es, size_t(n),
                                           cudaMemcpyDeviceToHost, st.d2h));
        else
            PSW_CUDA_TRY(cudaMemcpy2DAsync(static_cast<char*>(X) + size_t(k0) * size_t(ldx) * es,
                                           size_t(ldx) * es, dbuf, size_t(n) * es, size_t(n) * es,
                                           size_t(kc), cudaMemcpyDeviceToHost, st.d2h));
        PSW_CUDA_TRY(cudaEventRecord(st.freed[slot], st.d2h));
    }
    cudaStreamSynchronize(st.d2h);
    cudaStreamSynchronize(st.comp);
    cudaFreeAsync(buf, st.comp);
    cudaStreamSynchronize(st.comp);
    cudaSetDevice(prev);
    psw::reset_launches();
    psw::note_launches(launches);
    return rc;
}
