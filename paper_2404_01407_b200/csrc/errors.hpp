// errors.hpp -- the reference's error taxonomy (core.hpp:22-56), mirrored so the C
// ABI can report the same kinds (status code + node / stage) and a C++ host shim can
// rethrow the reference's own types.
#pragma once

#include <stdexcept>
#include <string>

namespace fnlh {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct UnsupportedCaseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FactorizationError : std::runtime_error {
    int node = -1;
    FactorizationError(const std::string& msg, int node_id)
        : std::runtime_error(msg + " (node " + std::to_string(node_id) + ")"), node(node_id) {}
};
struct DivergenceError : std::runtime_error {
    int stage = -1;
    std::string field;
    DivergenceError(const std::string& msg, int stage_idx, std::string field_name = {})
        : std::runtime_error(msg + " (stage " + std::to_string(stage_idx) +
                             (field_name.empty() ? "" : ", field " + field_name) + ")"),
          stage(stage_idx),
          field(std::move(field_name)) {}
};
struct NonConvergenceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

}  // namespace fnlh
