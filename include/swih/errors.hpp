// swih/errors.hpp — exception classes of the SWIH API.
//
// Same class names, hierarchy and payloads as the reference
// (/root/reference/proj/include/swih/errors.hpp:10-79); the GPU library
// reports each one as a status code of include/swg.h and the C++ layer
// rethrows it (detail::raise).
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

namespace swih {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : Error {
  using Error::Error;
};
struct ZeroMassError : Error {
  using Error::Error;
};
struct InvalidKernelError : Error {
  using Error::Error;
};
struct OutOfRangeError : Error {
  using Error::Error;
};
struct UnsupportedKernelError : Error {
  using Error::Error;
};
struct WindowOutOfBoundsError : Error {
  using Error::Error;
};
struct ConfigError : Error {
  using Error::Error;
};
struct ModelError : Error {
  using Error::Error;
};
struct SizeError : Error {
  using Error::Error;
};

// Table memory budget exceeded; carries the byte count that was needed.
class CapacityError : public Error {
 public:
  CapacityError(const std::string& what, std::size_t required)
      : Error(what), required_(required) {}
  std::size_t required_bytes() const noexcept { return required_; }

 private:
  std::size_t required_ = 0;
};

namespace detail {
// Throws the class matching a libswg status (no-op for SWG_OK).
void raise(int status);
}  // namespace detail

}  // namespace swih
