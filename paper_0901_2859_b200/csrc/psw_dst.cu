// DST-I of many rows on the device: the Fourier consumer's transform
// (reference poisson/dst.hpp:85-164).
//
// out[l-1] = scale * sum_{j=1}^{N-1} in[j-1] sin(pi j l / N), l = 1..N-1,
// for `rows` rows of N-1 values (row pitch ldin / ldout, fp64).
//
// Power-of-two N (dst.hpp:96-118, 130-149): the reference's construction —
// two rows packed into the real and imaginary parts of the odd extension
// (length L = 2N), one radix-2 decimation-in-time FFT with the reference's
// bit reversal and twiddle table w_k = (cos, sin)(-2 pi k / L) (computed on
// the host with std::cos / std::sin exactly as Radix2Fft does), the two
// spectra split by conjugate symmetry. One CTA per pair of rows; the whole
// signal and the twiddles live in shared memory (L <= 8192: N <= 4096).
// Other N (dst.hpp:120-128): the direct sine sum over the reference's
// sines[m] table, one thread per output.
#include <algorithm>
#include <cmath>
#include <mutex>


#include <vector>

#include "psw_internal.h"

namespace psw {
namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;  // std::numbers::pi
constexpr int kDstThreads = 1024;
constexpr int kDstMaxL = 8192;

// Twiddle w_i lives at tw[twi(i)]: the stages read the table with power-of-two
// strides (index k * step, step up to L / 4), which in the plain layout puts
// a warp's 32 loads in one bank (16-byte entries, 8 per bank row). XOR-ing
// the low three index bits with the next three groups of three spreads every
// such stride over all eight 16-byte banks.
__device__ __forceinline__ int twi(int i) {
    return i ^ ((i >> 3) & 7) ^ ((i >> 6) & 7) ^ ((i >> 9) & 7);
}
// The signal gets the same treatment (element x at v[vsw(x)]): the bit-reversed
// scatter of the odd extension writes with strides of L / 32 entries, and the
// first passes (q < 32) read 8-element blocks 512 bytes apart.
__device__ __forceinline__ int vsw(int i) {
    return i ^ ((i >> 3) & 7) ^ ((i >> 6) & 7) ^ ((i >> 9) & 7) ^ ((i >> 12) & 7);
}

__global__ void __launch_bounds__(kDstThreads) dst_pair_kernel(
    const double* __restrict__ in, int64_t ldin, double* __restrict__ out, int64_t ldout,
    int64_t rows, int N, int logL, const double2* __restrict__ gtw, double scale) {
    extern __shared__ double2 sm[];
    const int L = 2 * N;
    double2* v = sm;        // [L]
    double2* tw = sm + L;   // [L / 2]
    const int64_t ra = 2 * int64_t(blockIdx.x), rb = ra + 1;
    const bool hasb = rb < rows;
    const double* a = in + ra * ldin;
    const double* b = in + (hasb ? rb : ra) * ldin;
    for (int k = threadIdx.x; k < L / 2; k += blockDim.x) tw[twi(k)] = gtw[k];
    // the odd extension, stored bit-reversed (Radix2Fft::transform's swap pass)
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        double re = 0.0, im = 0.0;
        if (i > 0 && i < N) {
            re = a[i - 1];
            im = hasb ? b[i - 1] : 0.0;
        } else if (i > N) {
            re = -a[L - i - 1];
            im = hasb ? -b[L - i - 1] : 0.0;
        }
        v[vsw(int(__brev(unsigned(i)) >> (32 - logL)))] = make_double2(re, im);
    }
    __syncthreads();
    // Radix2Fft::transform's stages len = 2, 4, ..., L, three at a time: the
    // eight elements k + j q (j < 8) of an 8q block in registers go through
    // the stages of half q, 2q, 4q with the same butterflies, twiddles and
    // order as the radix-2 sweep (bitwise equal to it), a third of the
    // shared-memory passes and barriers. The 1 or 2 leftover stages run first.
    int len = 2;
    const int rem = logL % 3;
    for (int t = 0; t < rem; ++t, len <<= 1) {
        const int half = len >> 1, step = L / len;
        for (int bf = threadIdx.x; bf < L / 2; bf += blockDim.x) {
            const int k = bf & (half - 1), i0 = (bf - k) * 2 + k;
            const double2 w = tw[twi(k * step)];
            const double2 x = v[vsw(i0)], y = v[vsw(i0 + half)];
            const double tr = w.x * y.x - w.y * y.y, ti = w.x * y.y + w.y * y.x;  // w * b
            v[vsw(i0 + half)] = make_double2(x.x - tr, x.y - ti);
            v[vsw(i0)] = make_double2(x.x + tr, x.y + ti);
        }
        __syncthreads();
    }
    for (; len <= L / 4; len <<= 3) {
        const int q = len >> 1;
        for (int bf = threadIdx.x; bf < L / 8; bf += blockDim.x) {
            const int k = bf & (q - 1), i0 = (bf - k) * 8 + k;
            double2 e[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) e[j] = v[vsw(i0 + j * q)];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int h = 1 << t;                  // in units of q
                const int step = L / (len << t);       // L / len_t
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (j & h) continue;
                    const double2 w = tw[twi((k + (j & (h - 1)) * q) * step)];
                    const double2 y = e[j + h];
                    const double tr = w.x * y.x - w.y * y.y, ti = w.x * y.y + w.y * y.x;
                    e[j + h] = make_double2(e[j].x - tr, e[j].y - ti);
                    e[j] = make_double2(e[j].x + tr, e[j].y + ti);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) v[vsw(i0 + j * q)] = e[j];
        }
        __syncthreads();
    }
    // split the packed spectra (dst.hpp:144-148)
    double* oa = out + ra * ldout;
    double* ob = out + rb * ldout;
    for (int l = 1 + threadIdx.x; l < N; l += blockDim.x) {
        const double2 x = v[vsw(l)], z = v[vsw(L - l)];
        const double2 y = make_double2(z.x, -z.y);  // conj(v[2N - l])
        oa[l - 1] = scale * (-0.25 * (x.y + y.y));
        if (hasb) ob[l - 1] = scale * (0.25 * (x.x - y.x));
    }
}

// dst.hpp:120-128: direct summation over sines[m] = sin(pi m / N)
__global__ void dst_direct_kernel(const double* __restrict__ in, int64_t ldin,
                                  double* __restrict__ out, int64_t ldout, int64_t rows, int N,
                                  const double* __restrict__ sines, double scale) {
    const int l = 1 + int(blockIdx.x) * blockDim.x + threadIdx.x;
    if (l >= N) return;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const double* x = in + r * ldin;
        double s = 0.0;
        for (int j = 1; j < N; ++j) {
            const int m = int((int64_t(j) * l) % (2 * N));  // sin has period 2N with sign flip
            s += x[j - 1] * (m < N ? sines[m] : -sines[m - N]);
        }
        out[r * ldout + l - 1] = scale * s;
    }
}

struct DstTables {
    std::mutex mu;
    std::vector<std::pair<std::pair<int, int>, void*>> tab;  // ((device, N), table)
};
DstTables& dst_tables() {
    static DstTables* t = new DstTables();  // lives for the process
    return *t;
}

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

// twiddles (power-of-two N, Radix2Fft(2N)) or sines (other N), cached per device
int dst_table(int device, int N, const void** out) {
    DstTables& T = dst_tables();
    std::lock_guard<std::mutex> lk(T.mu);
    for (auto& e : T.tab)
        if (e.first == std::make_pair(device, N)) {
            *out = e.second;
            return PSW_OK;
        }
    std::vector<double> h;
    if (is_pow2(N)) {
        const size_t L = 2 * size_t(N);
        h.resize(L);  // L/2 complex
        for (size_t k = 0; k < L / 2; ++k) {
            const double angle = -2.0 * kPi * static_cast<double>(k) / double(L);
            h[2 * k] = std::cos(angle);
            h[2 * k + 1] = std::sin(angle);
        }
    } else {
        h.resize(size_t(N));
        for (int j = 0; j < N; ++j) h[size_t(j)] = std::sin(kPi * static_cast<double>(j) / N);
    }
    void* d = nullptr;
    PSW_CUDA_TRY(cudaMalloc(&d, sizeof(double) * h.size()));
    PSW_CUDA_TRY(cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
    T.tab.push_back({{device, N}, d});
    *out = d;
    return PSW_OK;
}

}  // namespace
}  // namespace psw

extern "C" int psw_dst_rows(const double* in, int64_t ldin, double* out, int64_t ldout,
                            int64_t rows, int64_t N, double scale, void* stream) {
    psw::clear_error();
    if (N < 2 || rows < 0 || (rows > 0 && (!in || !out)) || ldin < N - 1 || ldout < N - 1 ||
        N > (int64_t(1) << 30)) {
        psw::set_error(PSW_INVALID_ARGUMENT, "psw_dst_rows: invalid arguments");
        return PSW_INVALID_ARGUMENT;
    }
    if (rows == 0) return PSW_OK;
    int dev = 0;
    PSW_CUDA_TRY(cudaGetDevice(&dev));
    const int n = int(N);
    const void* tab = nullptr;
    if (int rc = psw::dst_table(dev, n, &tab)) return rc;
    auto s = static_cast<cudaStream_t>(stream);
    const bool fft = psw::is_pow2(n) && 2 * n <= psw::kDstMaxL;
    if (fft) {
        const int L = 2 * n;
        int logL = 0;
        while ((1 << logL) < L) ++logL;
        const size_t smem = sizeof(double2) * (size_t(L) + size_t(L) / 2);
        static std::once_flag once;
        cudaError_t e = cudaSuccess;
        std::call_once(once, [&] {
            e = cudaFuncSetAttribute(psw::dst_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(double2) * (psw::kDstMaxL + psw::kDstMaxL / 2)));
        });
        PSW_CUDA_TRY(e);
        // one thread per 8-element block of a pass (L / 8), 64 .. kDstThreads
        const int threads = std::min(psw::kDstThreads, std::max(64, (L / 8 + 31) / 32 * 32));
        psw::dst_pair_kernel<<<unsigned((rows + 1) / 2), threads, smem, s>>>(
            in, ldin, out, ldout, rows, n, logL, static_cast<const double2*>(tab), scale);
    } else {
        const dim3 grid(unsigned((n - 1 + 127) / 128), unsigned(rows < 65535 ? rows : 65535));
        psw::dst_direct_kernel<<<grid, 128, 0, s>>>(in, ldin, out, ldout, rows, n,
                                                    static_cast<const double*>(tab), scale);
    }
    PSW_CUDA_TRY(cudaGetLastError());
    psw::note_launches(1);
    return PSW_OK;
}
