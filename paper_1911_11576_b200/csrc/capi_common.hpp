// Shared state of the C ABI translation units.
#pragma once

#include <string>

namespace stitch {
// Last error message on this thread, reported by stitch_last_error().
inline std::string& capi_last_error() {
  static thread_local std::string e;
  return e;
}
}  // namespace stitch
