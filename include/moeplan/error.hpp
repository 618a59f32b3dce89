// B200 FSEP framework -- host planner error model.
// Mirrors the reference error contract (/root/reference/proj/include/moeplan/error.hpp:22-40):
// every failure is an Error carrying an ErrorKind that the C ABI maps onto mp_status.
#pragma once
#include <stdexcept>
#include <string>

namespace moeplan {

enum class ErrorKind {
  invalid_argument,
  parse,
  io,
  infeasible,
  budget_exceeded,
  internal,
  device,  // B200 extension: CUDA / NCCL failure (mp_status MP_ERR_DEVICE)
};

class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
  ErrorKind kind() const noexcept { return kind_; }

 private:
  ErrorKind kind_;
};

const char* error_kind_name(ErrorKind kind);

}  // namespace moeplan
