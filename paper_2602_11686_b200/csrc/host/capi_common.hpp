// Shared C-ABI plumbing: exception -> mp_status translation with a thread-local
// last-error string (contract of /root/reference/proj/src/capi.cpp:39-70).
#pragma once
#include <cstdlib>
#include <cstring>
#include <string>

#include "moeplan.h"
#include "moeplan/error.hpp"

namespace moeplan::capi {

std::string& last_error();

inline mp_status status_of(ErrorKind kind) {
  switch (kind) {
    case ErrorKind::invalid_argument: return MP_ERR_INVALID_ARGUMENT;
    case ErrorKind::parse: return MP_ERR_PARSE;
    case ErrorKind::io: return MP_ERR_IO;
    case ErrorKind::infeasible: return MP_ERR_INFEASIBLE;
    case ErrorKind::budget_exceeded: return MP_ERR_BUDGET_EXCEEDED;
    case ErrorKind::internal: return MP_ERR_INTERNAL;
    case ErrorKind::device: return MP_ERR_DEVICE;
  }
  return MP_ERR_INTERNAL;
}

template <typename Body>
mp_status guarded(Body&& body) noexcept {
  try {
    body();
    last_error().clear();
    return MP_OK;
  } catch (const Error& e) {
    last_error() = e.what();
    return status_of(e.kind());
  } catch (const std::exception& e) {
    last_error() = e.what();
    return MP_ERR_INTERNAL;
  } catch (...) {
    last_error() = "unknown error";
    return MP_ERR_INTERNAL;
  }
}

inline void require(bool ok, const char* what) {
  if (!ok) throw Error(ErrorKind::invalid_argument, what);
}

inline char* dup_string(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  if (!out) throw Error(ErrorKind::internal, "out of host memory");
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

}  // namespace moeplan::capi
