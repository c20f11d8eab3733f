// Host-side error type shared by the CUDA and the pure-C++ translation units.
#pragma once

#include <stdexcept>
#include <string>

namespace krr {

// Exception used inside the library; converted to a krr_status at the C-ABI.
struct Error : std::runtime_error {
    int status;
    Error(int st, const std::string& msg) : std::runtime_error(msg), status(st) {}
};

[[noreturn]] inline void fail(int st, const std::string& msg) { throw Error(st, msg); }

}  // namespace krr
