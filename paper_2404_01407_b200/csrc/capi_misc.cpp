// capi_misc.cpp -- error state and device queries of the C ABI.
#include <cuda_runtime.h>

#include "fnlh_b200.h"

#include "capi_util.hpp"

namespace fnlh {
std::atomic<long long>& launch_count() {
    static std::atomic<long long> n{0};
    return n;
}
ErrorState& last_error() {
    thread_local ErrorState e;
    return e;
}
}  // namespace fnlh

extern "C" {

const char* fnlh_last_error(void) { return fnlh::last_error().msg.c_str(); }
int fnlh_last_error_node(void) { return fnlh::last_error().node; }
int fnlh_last_error_stage(void) { return fnlh::last_error().stage; }

long long fnlh_launch_count(void) { return fnlh::launch_count().load(); }

int fnlh_set_device(int device) {
    return fnlh::guarded([&] { FNLH_CUDA(cudaSetDevice(device)); });
}

int fnlh_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

}  // extern "C"
