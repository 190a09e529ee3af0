// capi_util.hpp -- status mapping for the C ABI and small RAII device buffers.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "common.cuh"
#include "errors.hpp"

namespace fnlh {

struct ErrorState {
    std::string msg;
    int node = -1;
    int stage = -1;
};
ErrorState& last_error();

// exception -> status code (include/fnlh_b200.h enum fnlh_status)
template <class F>
int guarded(F&& f) {
    ErrorState& e = last_error();
    e.node = -1;
    e.stage = -1;
    try {
        f();
        return 0;
    } catch (const ConfigError& x) {
        e.msg = x.what();
        return 1;
    } catch (const StateError& x) {
        e.msg = x.what();
        return 2;
    } catch (const ShapeError& x) {
        e.msg = x.what();
        return 3;
    } catch (const UnsupportedCaseError& x) {
        e.msg = x.what();
        return 4;
    } catch (const FactorizationError& x) {
        e.msg = x.what();
        e.node = x.node;
        return 5;
    } catch (const DivergenceError& x) {
        e.msg = x.what();
        e.stage = x.stage;
        return 6;
    } catch (const NonConvergenceError& x) {
        e.msg = x.what();
        return 8;
    } catch (const std::exception& x) {
        e.msg = x.what();
        return 7;
    }
}

template <class T>
struct DeviceBuffer {
    T* ptr = nullptr;
    std::size_t n = 0;
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t count) { alloc(count); }
    ~DeviceBuffer() { fnlh::dfree(ptr); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : ptr(o.ptr), n(o.n) {
        o.ptr = nullptr;
        o.n = 0;
    }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            fnlh::dfree(ptr);
            ptr = o.ptr;
            n = o.n;
            o.ptr = nullptr;
            o.n = 0;
        }
        return *this;
    }
    void alloc(std::size_t count) {
        if (count == n && ptr) return;
        fnlh::dfree(ptr);
        ptr = nullptr;
        n = count;
        FNLH_CUDA_ALLOC(&ptr, std::max<std::size_t>(count, 1) * sizeof(T));
    }
    void upload(const T* h, std::size_t count) {
        alloc(count);
        if (count) {
            FNLH_CUDA(cudaMemcpy(ptr, h, count * sizeof(T), cudaMemcpyHostToDevice));
            legacy_sync();
        }
    }
    std::size_t bytes() const { return n * sizeof(T); }
};

template <class T>
void download(T* h, const T* d, std::size_t count) {
    if (count) FNLH_CUDA(cudaMemcpy(h, d, count * sizeof(T), cudaMemcpyDeviceToHost));
}

}  // namespace fnlh
