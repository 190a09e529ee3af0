// capi_types.hpp -- the opaque handle types behind include/fnlh_b200.h shared by the C ABI
// translation units.
#pragma once

#include <memory>

#include "la.cuh"
#include "rb.cuh"

// rb / n0 are decided once in fnlh_pattern_create and read-only afterwards, so one pattern
// handle may serve concurrent solves from several host threads (the shim's harmonic workers)
struct fnlh_pattern {
    std::unique_ptr<fnlh::DevicePattern> p;
    int rb = 0;  // 1: 2-colour colour-major ordering with one partition (rb.cuh)
    int n0 = 0;
    bool use_rb() const { return rb == 1 && fnlh::rb_enabled(); }
};
