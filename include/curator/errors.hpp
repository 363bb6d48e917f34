#pragma once
// Error taxonomy of the curator API (mirrors proj/include/curator/errors.hpp:10-18 of the
// reference): configuration problems vs. data/runtime problems. The C ABI (mtnlg.h) maps them
// to status 1 and 2 respectively, the same split the reference CLI uses for its exit codes
// (proj/tools/curator_main.cpp:175-192).

#include <stdexcept>
#include <string>

namespace curator {

/// Invalid configuration: bad planner key/value, impossible layout. Status / exit code 1.
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
  explicit ConfigError(const char* what) : std::runtime_error(what) {}
};

/// Invalid data or a failed device/communication operation. Status / exit code 2.
class DataError : public std::runtime_error {
 public:
  explicit DataError(const std::string& what) : std::runtime_error(what) {}
  explicit DataError(const char* what) : std::runtime_error(what) {}
};

}  // namespace curator
