// Internal glue of the drop-in headers: C-ABI status -> exceptions, RAII
// device buffers and host<->device copies (the legacy default stream).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <type_traits>
#include <vector>

#include "sparsek/common.hpp"
#include "sparsek_b200.h"

namespace sparsek {
namespace detail {

inline void check(int rc) {
    if (rc == SKB_OK) return;
    const std::string msg = skb_last_error();
    switch (rc) {
        case SKB_ESHAPE: throw ShapeError(msg);
        case SKB_EARG: throw ArgumentError(msg);
        case SKB_ENUMERIC: throw NumericError(msg);
        case SKB_ECONFIG: throw ConfigError(msg);
        case SKB_EIO: throw IoError(msg);
        default: throw CudaError(msg);
    }
}
inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
constexpr int dtype_of() {
    static_assert(std::is_same<T, float>::value || std::is_same<T, double>::value,
                  "sparsek: T must be float or double (as the reference instantiates)");
    return std::is_same<T, double>::value ? SKB_F64 : SKB_F32;
}

class Buf {
  public:
    Buf() = default;
    explicit Buf(size_t bytes) : n_(bytes) { cuda(cudaMalloc(&p_, bytes ? bytes : 16), "cudaMalloc"); }
    template <class T>
    explicit Buf(const std::vector<T>& v) : Buf(v.size() * sizeof(T)) {
        if (!v.empty()) cuda(cudaMemcpy(p_, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
    ~Buf() {
        if (p_) cudaFree(p_);
    }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    Buf(Buf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    Buf& operator=(Buf&& o) noexcept {
        if (this != &o) {
            if (p_) cudaFree(p_);
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
        }
        return *this;
    }
    void* get() const { return p_; }
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    template <class T>
    std::vector<T> to_host(size_t count) const {
        std::vector<T> v(count);
        if (count) cuda(cudaMemcpy(v.data(), p_, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
        return v;
    }

  private:
    void* p_ = nullptr;
    size_t n_ = 0;
};

}  // namespace detail
}  // namespace sparsek
