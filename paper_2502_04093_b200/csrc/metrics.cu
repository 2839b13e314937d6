// metrics.cu -- compute_metrics<T> (include/ipcomp/pipeline.hpp:354-372) on the device: the
// max pointwise error, MSE and PSNR of a reconstruction against the original, the step
// right after every retrieval in the reference's evaluation loop (tools/main.cpp:307-315).
//
// One HBM pass over both fields (2 n w bytes): 148 x 4 CTAs of 512 threads, 16-byte vector
// loads, per-thread double accumulators reduced by warp shuffles and one partial per CTA,
// then a one-CTA combine.  max_error, min and max follow std::max/std::min exactly
// (a NaN operand never replaces the running value), so they are bit-identical to the
// reference; the sum of squared differences is the same set of double products added in
// a different order (a tree instead of left to right), so MSE and PSNR agree to the sum's
// rounding (tests/test_gpu_extensions.py states the tolerance).
#include <cmath>
#include <limits>

#include "../../include/ipcomp_b200.h"
#include "util.cuh"

namespace ipcg {
namespace metrics {

struct Part {
    double maxe, sq, lo, hi;
};

__device__ __forceinline__ void acc(Part &p, double a, double b) {
    const double d = a - b;
    const double ad = fabs(d);
    p.maxe = p.maxe < ad ? ad : p.maxe;  // std::max(m, |d|)
    p.sq += d * d;
    p.lo = a < p.lo ? a : p.lo;  // std::min(lo, a)
    p.hi = p.hi < a ? a : p.hi;  // std::max(hi, a)
}

__device__ __forceinline__ void merge(Part &p, const Part &q) {
    p.maxe = p.maxe < q.maxe ? q.maxe : p.maxe;
    p.sq += q.sq;
    p.lo = q.lo < p.lo ? q.lo : p.lo;
    p.hi = p.hi < q.hi ? q.hi : p.hi;
}

__device__ __forceinline__ Part shfl_down(const Part &p, int o) {
    return Part{__shfl_down_sync(0xffffffffu, p.maxe, o), __shfl_down_sync(0xffffffffu, p.sq, o),
                __shfl_down_sync(0xffffffffu, p.lo, o), __shfl_down_sync(0xffffffffu, p.hi, o)};
}

__device__ __forceinline__ Part identity() {
    return Part{0.0, 0.0, __longlong_as_double(0x7ff0000000000000ll), -__longlong_as_double(0x7ff0000000000000ll)};
}

// block-wide reduction; the result is valid in thread 0
template <int THREADS>
__device__ Part block_reduce(Part p) {
    __shared__ Part sh[THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) merge(p, shfl_down(p, o));
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sh[w] = p;
    __syncthreads();
    if (w == 0) {
        p = (int)threadIdx.x < THREADS / 32 ? sh[threadIdx.x] : identity();
        for (int o = 16; o > 0; o >>= 1) merge(p, shfl_down(p, o));
    }
    return p;
}

constexpr int THREADS = 512;

template <class T>
__global__ void __launch_bounds__(THREADS) k_metrics(const T *__restrict__ a, const T *__restrict__ b, uint64_t n,
                                                     Part *parts) {
    Part p = identity();
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
    const bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
    const uint64_t stride = (uint64_t)gridDim.x * THREADS;
    uint64_t done = 0;
    if (aligned) {
        const uint64_t nv = n / V;
        using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
        const Vec *av = reinterpret_cast<const Vec *>(a), *bv = reinterpret_cast<const Vec *>(b);
        for (uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x; i < nv; i += stride) {
            const Vec x = __ldcs(av + i), y = __ldcs(bv + i);
            const T *xs = reinterpret_cast<const T *>(&x), *ys = reinterpret_cast<const T *>(&y);
#pragma unroll
            for (int k = 0; k < V; ++k) acc(p, (double)xs[k], (double)ys[k]);
        }
        done = nv * V;
    }
    for (uint64_t i = done + blockIdx.x * (uint64_t)THREADS + threadIdx.x; i < n; i += stride)
        acc(p, (double)a[i], (double)b[i]);
    p = block_reduce<THREADS>(p);
    if (threadIdx.x == 0) parts[blockIdx.x] = p;
}

__global__ void __launch_bounds__(THREADS) k_metrics_final(const Part *parts, int np, Part *out) {
    Part p = identity();
    for (int i = threadIdx.x; i < np; i += THREADS) merge(p, parts[i]);
    p = block_reduce<THREADS>(p);
    if (threadIdx.x == 0) *out = p;
}

}  // namespace metrics

void compute_metrics_device(int scalar, const void *a, const void *b, uint64_t n, double out[3], cudaStream_t st) {
    using namespace metrics;
    const int grid = (int)std::min<uint64_t>((uint64_t)num_sms() * 4, std::max<uint64_t>(1, (n + THREADS - 1) / THREADS));
    Part *parts = static_cast<Part *>(scratch_get((size_t)(grid + 1) * sizeof(Part), st));
    {
        ProfScope ps("metrics", st, 2 * n * (scalar == 0 ? 4 : 8));
        if (scalar == 0)
            k_metrics<float><<<grid, THREADS, 0, st>>>(static_cast<const float *>(a), static_cast<const float *>(b), n, parts);
        else
            k_metrics<double><<<grid, THREADS, 0, st>>>(static_cast<const double *>(a), static_cast<const double *>(b), n,
                                                        parts);
        CKL();
        k_metrics_final<<<1, THREADS, 0, st>>>(parts, grid, parts + grid);
        CKL();
    }
    Part r;
    readback(&r, parts + grid, sizeof(Part), st);
    scratch_put(parts, st);
    // pipeline.hpp:366-369
    out[0] = r.maxe;
    out[1] = n == 0 ? 0.0 : r.sq / (double)n;
    out[2] = out[1] == 0.0 ? std::numeric_limits<double>::infinity() : 20.0 * std::log10((r.hi - r.lo) / std::sqrt(out[1]));
}

}  // namespace ipcg
