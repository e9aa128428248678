// fl_host.h -- host-side helpers shared by the engine and the transports:
// the error type behind the C ABI status codes and a small device array.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/flume_b200.h"

namespace fl {

struct FlumeError : std::runtime_error {
    int code;
    long pid = -1;
    int body = -1;
    long substep = -1;
    FlumeError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            throw FlumeError(FLUME_E_CUDA, std::string("cuda: ") + cudaGetErrorString(e_) + " at " \
                                               + __FILE__ + ":" + std::to_string(__LINE__));     \
    } while (0)

template <class T>
struct DevArr {
    T* p = nullptr;
    size_t n = 0;
    DevArr() = default;
    DevArr(const DevArr&) = delete;
    DevArr& operator=(const DevArr&) = delete;
    ~DevArr() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count <= n && p) return;
        release();
        if (count == 0) count = 1;
        CK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void upload(const std::vector<T>& h, cudaStream_t s) {
        alloc(h.size());
        if (!h.empty()) CK(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    }
};

// one trajectory state in HBM

}  // namespace fl
