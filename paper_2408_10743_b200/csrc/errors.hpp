// Exception classes used inside the library; capi.cpp maps them to sdb_status
// (the reference's symdist/errors.hpp classes plus device failures).
#pragma once

#include <stdexcept>
#include <string>

namespace sdb {

struct ParseFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ValidationFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InternalFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

}  // namespace sdb
