// util.cuh -- error plumbing and small device helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace ipcg {

// error kinds mirror the reference's exception types (ipcomp_b200.h)
enum ErrKind : int { OK = 0, EINVAL_ = 1, ERUNTIME = 2, EDOMAIN = 3, EINFEASIBLE = 4, ECUDA = 5 };

struct Error : std::runtime_error {
    int kind;
    Error(int k, const std::string &m) : std::runtime_error(m), kind(k) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char *what, const char *file, int line) {
    throw Error(ECUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " + file + ":" +
                           std::to_string(line));
}
#define CK(x)                                                          \
    do {                                                               \
        cudaError_t _e = (x);                                          \
        if (_e != cudaSuccess) ::ipcg::throw_cuda(_e, #x, __FILE__, __LINE__); \
    } while (0)
// every kernel launch goes through CKL(): checks the launch and counts it
inline unsigned long long &launch_counter() {
    static unsigned long long c = 0;
    return c;
}
#define CKL()                              \
    do {                                   \
        ++::ipcg::launch_counter();        \
        CK(cudaGetLastError());            \
    } while (0)

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
    uint64_t g = (n + block - 1) / block;
    if (g == 0) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

#if defined(__CUDACC__)
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
#endif

}  // namespace ipcg
