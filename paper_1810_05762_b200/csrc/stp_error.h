// Thread-local error channel of the C-ABI (stp_last_error).  The reference
// reports precondition failures with std::invalid_argument
// (solver.cpp:397-398, collide.cpp:271, krylov.cpp:109-114,
// scene.cpp:36-68); across a C boundary they become status codes plus this
// message.
#pragma once
#include <string>

namespace stp {

inline std::string& last_error() {
  static thread_local std::string msg;
  return msg;
}
inline const char* last_error_cstr() { return last_error().c_str(); }
inline int fail(int code, const std::string& what) {
  last_error() = what;
  return code;
}

}  // namespace stp
