// Shared host-side helpers of the library's translation units.
#pragma once
#include <string>

namespace qg {

// Description of the last failed call on this thread (qg_last_error()).
inline std::string& last_message() {
  static thread_local std::string msg;
  return msg;
}
inline int fail(int status, const std::string& msg) {
  last_message() = msg;
  return status;
}

}  // namespace qg
