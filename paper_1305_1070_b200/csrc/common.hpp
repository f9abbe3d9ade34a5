// Shared host-side types for the B200 HSC path.
//
// Error taxonomy mirrors the reference's proj/include/negf/errors.hpp:15-74;
// codes are what the C ABI (include/negf_gpu.h) reports.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace negfb {

using cplx = std::complex<double>;

enum StatusCode : int {
  kOk = 0,
  kSingularBlock = 1,          // errors.hpp:36-42
  kNonSkewHermitian = 2,       // errors.hpp:61-65
  kContractViolation = 3,      // errors.hpp:27-31
  kCudaError = 4,
  kNcclError = 5,
  kOutOfMemory = 6,
  kConfigError = 7,            // errors.hpp:21-25
  kPartitionViolation = 8,     // errors.hpp:44-53
  kResidualTooLarge = 9,       // errors.hpp:67-71
  kInternal = 10,
};

struct Failure : std::runtime_error {
  int code;
  int energy_index = -1;
  int cluster = -1;
  int pivot = -1;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Kernels put the energy index of a batch in gridDim.y / gridDim.z, which
// CUDA limits to 65535: batch capacities never exceed it.
constexpr int kMaxGridYZ = 65535;

[[noreturn]] inline void fail(int code, const std::string& msg) {
  throw Failure(code, msg);
}

}  // namespace negfb
