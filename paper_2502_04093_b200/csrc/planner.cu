// planner.cu -- the retrieval planner on the GPU: plan_for_error and
// plan_for_size of the reference (proj/src/planner.cpp:125-290) over the plain ErrorModel
// (planner.hpp:13-32), as ONE single-CTA launch.  The planner is a 1024-bucket knapsack over the
// progressive levels: per level at most 33 choices (planes dropped), per bucket a max / min over
// them.  A thread owns a bucket; levels are sequential (one barrier each); the choice lists and
// the backtrack are a few hundred serial steps on thread 0.  Every floating-point expression is
// the host planner's (host.cpp), in its order, without contraction (-fmad=false), so plans are
// identical -- tests/test_gpu_parity.py compares them on random models and on every config.
// The host planner stays the default (it reads only the index and costs ~0.1 ms); this entry
// point serves callers whose model already lives on the device side of a pipeline.
#include <cmath>
#include <cstring>

#include "host.h"
#include "util.cuh"

namespace ipcg {
namespace {

constexpr int kBuckets = 1024;
constexpr int kInfCost = kBuckets + 1;
constexpr int NB = kBuckets + 1;  // DP columns e = 0 .. 1024

struct PlanIn {
    int levels, lp, mode;  // mode 0: plan_for_error, 1: plan_for_size
    double eb, max_error;
    uint64_t budget;
    double w[IPCG_MAX_LEVELS];  // amplification^(level-1), computed by the host's std::pow like the reference
    double delta[IPCG_MAX_LEVELS][33];
    uint64_t plane_bytes[IPCG_MAX_LEVELS][32];
    uint64_t outlier_bytes[IPCG_MAX_LEVELS];
    int progressive[IPCG_MAX_LEVELS];
};

struct PlanOut {
    int status;  // 0 ok; 1 below the compression bound; 2 budget below mandatory; 3 nothing fits; 4 optimum lost
    int k[IPCG_MAX_LEVELS];
};

struct Choice {
    int dropped, cost;
    uint64_t bytes;
    double err;
};

struct Value {
    double err;
    uint64_t bytes;
};

__device__ __forceinline__ uint64_t optional_bytes(const PlanIn &m, int l, int dropped) {  // level l (1-based)
    uint64_t s = 0;
    for (int p = 0; p < 32 - dropped; ++p) s += m.plane_bytes[l - 1][p];
    return s;
}

__device__ __forceinline__ bool value_lt(const Value &a, const Value &b) {
    return a.err < b.err || (a.err == b.err && a.bytes < b.bytes);
}

__device__ double bound_for_plan_dev(const PlanIn &m, const int *k) {  // planner.cpp:51-58
    double sum = 0.0;
    for (int l = 1; l <= m.levels; ++l) sum += m.w[l - 1] * m.delta[l - 1][32 - k[l - 1]];
    return sum + m.eb;
}

// best_e: (lp + 1) x NB uint64 (error mode);  best_v: (lp + 1) x NB Value (size mode)
__global__ void __launch_bounds__(1024) k_planner(const PlanIn *in, uint64_t *best_e, Value *best_v, PlanOut *out) {
    __shared__ Choice cs[IPCG_MAX_LEVELS][33];
    __shared__ int ncs[IPCG_MAX_LEVELS];
    __shared__ uint64_t base_s[IPCG_MAX_LEVELS];
    __shared__ int status_s;
    __shared__ uint64_t budget_s;
    const PlanIn &m = *in;
    const int tid = threadIdx.x;
    const int lp = m.lp;
    const double inf = INFINITY;
    if (tid == 0) {
        status_s = 0;
        for (int l = 0; l < m.levels; ++l) out->k[l] = 32;
        if (m.mode == 0) {
            // plan_for_error (planner.cpp:125-205): choice lists in increasing dropped count, equal
            // costs keep the later (more dropped) entry
            if (isnan(m.max_error) || m.max_error < m.eb) status_s = 1;
            const double slack = m.max_error - m.eb;
            for (int l = 1; l <= lp && !status_s; ++l) {
                int n = 0;
                for (int d = 0; d <= 32; ++d) {
                    const double e = m.w[l - 1] * m.delta[l - 1][d];
                    int cost;
                    if (e <= 0.0 || isinf(slack)) cost = 0;
                    else if (slack <= 0.0) cost = kInfCost;
                    else {
                        const double units = ceil(e * (double)kBuckets / slack);
                        cost = units > (double)kInfCost ? kInfCost : (int)units;
                    }
                    if (cost > kBuckets) continue;
                    const Choice c{d, cost, optional_bytes(m, l, d), e};
                    if (n && cs[l - 1][n - 1].cost == cost) cs[l - 1][n - 1] = c;
                    else cs[l - 1][n++] = c;
                }
                ncs[l - 1] = n;
                base_s[l - 1] = optional_bytes(m, l, 0);
            }
        } else {
            // plan_for_size (planner.cpp:207-290): decreasing dropped count, equal costs keep the
            // smaller error
            uint64_t mandatory = 0;
            for (int l = 1; l <= m.levels; ++l) {
                mandatory += m.outlier_bytes[l - 1];
                if (!m.progressive[l - 1]) mandatory += optional_bytes(m, l, 0);
            }
            if (m.budget < mandatory) status_s = 2;
            const uint64_t budget = m.budget - mandatory;
            budget_s = budget;
            for (int l = 1; l <= lp && !status_s; ++l) {
                int n = 0;
                for (int d = 32; d >= 0; --d) {
                    const uint64_t bytes = optional_bytes(m, l, d);
                    int cost;
                    if (bytes == 0) cost = 0;
                    else if (budget == 0) cost = kInfCost;
                    else {
                        const uint64_t units = (bytes * kBuckets + budget - 1) / budget;
                        cost = units > (uint64_t)kBuckets ? kInfCost : (int)units;
                    }
                    if (cost > kBuckets) continue;
                    const double e = m.w[l - 1] * m.delta[l - 1][d];
                    if (n && cs[l - 1][n - 1].cost == cost) {
                        if (e < cs[l - 1][n - 1].err) cs[l - 1][n - 1] = Choice{d, cost, bytes, e};
                    } else {
                        cs[l - 1][n++] = Choice{d, cost, bytes, e};
                    }
                }
                ncs[l - 1] = n;
                if (n == 0) status_s = 3;
            }
        }
    }
    __syncthreads();
    if (status_s || lp == 0) {
        if (tid == 0) out->status = status_s;
        return;
    }
    // the knapsack: row i from row i-1, a thread per bucket
    for (int e = tid; e < NB; e += blockDim.x) {
        if (m.mode == 0) best_e[e] = 0;
        else best_v[e] = Value{0.0, 0};
    }
    __syncthreads();
    for (int i = 1; i <= lp; ++i) {
        const int n = ncs[i - 1];
        for (int e = tid; e < NB; e += blockDim.x) {
            if (m.mode == 0) {
                const uint64_t base = base_s[i - 1];
                uint64_t v = 0;
                bool any = false;
                for (int q = 0; q < n; ++q) {
                    const Choice &c = cs[i - 1][q];
                    if (c.cost > e) continue;
                    const uint64_t cand = best_e[(size_t)(i - 1) * NB + e - c.cost] + (base - c.bytes);
                    if (!any || cand > v) v = cand, any = true;
                }
                best_e[(size_t)i * NB + e] = v;
            } else {
                Value v{inf, 0};
                for (int q = 0; q < n; ++q) {
                    const Choice &c = cs[i - 1][q];
                    if (c.cost > e) continue;
                    const Value prev = best_v[(size_t)(i - 1) * NB + e - c.cost];
                    if (isinf(prev.err)) continue;
                    const Value cand{prev.err + c.err, prev.bytes + c.bytes};
                    if (value_lt(cand, v)) v = cand;
                }
                best_v[(size_t)i * NB + e] = v;
            }
        }
        __syncthreads();
    }
    if (tid != 0) return;
    // backtrack (thread 0): the first choice, in the host planner's scan order, that reproduces
    // the optimum of each row
    int k[IPCG_MAX_LEVELS];
    for (int l = 0; l < m.levels; ++l) k[l] = 32;
    int st = 0;
    if (m.mode == 0) {
        int e = kBuckets;
        for (int i = lp; i >= 1 && !st; --i) {
            const uint64_t base = base_s[i - 1], want = best_e[(size_t)i * NB + e];
            bool found = false;
            for (int q = ncs[i - 1] - 1; q >= 0; --q) {
                const Choice &c = cs[i - 1][q];
                if (c.cost > e) continue;
                if (best_e[(size_t)(i - 1) * NB + e - c.cost] + (base - c.bytes) == want) {
                    k[i - 1] = 32 - c.dropped;
                    e -= c.cost;
                    found = true;
                    break;
                }
            }
            if (!found) st = 4;
        }
        // the buckets round costs up per level; the exact bound may still exceed the target by
        // rounding: give planes back to the worst level until it holds (planner.cpp:192-204)
        while (!st && bound_for_plan_dev(m, k) > m.max_error) {
            int worst = -1;
            double worst_err = 0.0;
            for (int l = 1; l <= lp; ++l) {
                const int d = 32 - k[l - 1];
                const double er = m.w[l - 1] * m.delta[l - 1][d];
                if (d > 0 && er > worst_err) worst_err = er, worst = l;
            }
            if (worst < 0) break;
            k[worst - 1] += 1;
        }
    } else {
        if (isinf(best_v[(size_t)lp * NB + kBuckets].err)) st = 3;
        int e = kBuckets;
        for (int i = lp; i >= 1 && !st; --i) {
            const Value want = best_v[(size_t)i * NB + e];
            bool found = false;
            for (int q = 0; q < ncs[i - 1]; ++q) {
                const Choice &c = cs[i - 1][q];
                if (c.cost > e) continue;
                const Value prev = best_v[(size_t)(i - 1) * NB + e - c.cost];
                if (isinf(prev.err)) continue;
                if (prev.err + c.err == want.err && prev.bytes + c.bytes == want.bytes) {
                    k[i - 1] = 32 - c.dropped;
                    e -= c.cost;
                    found = true;
                    break;
                }
            }
            if (!found) st = 4;
        }
    }
    for (int l = 0; l < m.levels; ++l) out->k[l] = k[l];
    out->status = st;
}

}  // namespace

// host side: pack the model, one launch, one readback; errors as the host planner throws them
void plan_on_device(const ipcg_error_model &m, int mode, double max_error, uint64_t budget, int *k, cudaStream_t st) {
    check_model(m);
    PlanIn in;
    std::memset(&in, 0, sizeof in);
    in.levels = m.levels, in.lp = m.progressive_levels, in.mode = mode;
    in.eb = m.eb, in.max_error = max_error, in.budget = budget;
    for (int l = 0; l < m.levels; ++l) {
        in.w[l] = std::pow(m.amplification, l);  // weight(): planner.cpp:47
        std::memcpy(in.delta[l], m.level[l].delta, sizeof in.delta[l]);
        std::memcpy(in.plane_bytes[l], m.level[l].plane_bytes, sizeof in.plane_bytes[l]);
        in.outlier_bytes[l] = m.level[l].outlier_bytes;
        in.progressive[l] = m.level[l].progressive;
    }
    const size_t rows = (size_t)(in.lp + 1) * NB;
    const size_t in_b = (sizeof(PlanIn) + 255) & ~size_t(255), out_b = 256;
    const size_t dp_b = rows * (mode == 0 ? sizeof(uint64_t) : sizeof(Value));
    uint8_t *buf = static_cast<uint8_t *>(scratch_get(in_b + out_b + dp_b, st));
    struct Put {
        void *p;
        cudaStream_t st;
        ~Put() { scratch_put(p, st); }
    } put{buf, st};
    CK(cudaMemcpyAsync(buf, &in, sizeof in, cudaMemcpyHostToDevice, st));
    PlanOut *od = reinterpret_cast<PlanOut *>(buf + in_b);
    k_planner<<<1, 1024, 0, st>>>(reinterpret_cast<const PlanIn *>(buf), reinterpret_cast<uint64_t *>(buf + in_b + out_b),
                                  reinterpret_cast<Value *>(buf + in_b + out_b), od);
    CKL();
    PlanOut ho;
    CK(cudaMemcpyAsync(&ho, od, sizeof ho, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    switch (ho.status) {
        case 0: break;
        case 1: throw Error(EINFEASIBLE, "requested error bound is below the archive's compression bound");
        case 2: throw Error(EINFEASIBLE, "byte budget is below the mandatory payload (outliers and non-progressive levels)");
        case 3: throw Error(EINFEASIBLE, "no loadable configuration fits the byte budget");
        default: throw Error(ERUNTIME, "plan reconstruction lost the optimum");
    }
    for (int l = 0; l < m.levels; ++l) k[l] = ho.k[l];
}

}  // namespace ipcg
