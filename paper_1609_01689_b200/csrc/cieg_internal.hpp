// cieg_internal.hpp -- error plumbing and shared host structures of libcieg.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cieg.h"

namespace cieg {

// Error carrying a cieg_status; message already prefixed "<Type>: ".
struct Failure : std::runtime_error {
  int status;
  Failure(int s, const std::string& what) : std::runtime_error(what), status(s) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) {
  const char* type = "Error";
  switch (status) {
    case CIEG_ERR_DIMENSION: type = "DimensionMismatch"; break;
    case CIEG_ERR_CONFIG: type = "ConfigError"; break;
    case CIEG_ERR_SUBSPACE: type = "SubspaceCollapse"; break;
    case CIEG_ERR_FORMAT: type = "FormatError"; break;
    case CIEG_ERR_INDEFINITE: type = "IndefiniteGram"; break;
    case CIEG_ERR_CUDA: type = "CudaError"; break;
    case CIEG_ERR_BETA: type = "BetaTooLarge"; break;
    default: type = "Error"; break;
  }
  throw Failure(status, std::string(type) + ": " + msg);
}

void set_last_error(const std::string& msg);
void clear_last_error();

// Run f, translating exceptions into a status + cieg_last_error().
template <typename F>
int guarded(F&& f) {
  try {
    clear_last_error();
    f();
    return CIEG_OK;
  } catch (const Failure& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("Error: host allocation failed");
    return CIEG_ERR_ARGUMENT;
  } catch (const std::exception& e) {
    set_last_error(std::string("Error: ") + e.what());
    return CIEG_ERR_ARGUMENT;
  }
}

// Host copy of a generated CSB matrix (flattened ci::CsbMatrix).
struct HostCsb {
  std::uint32_t dim = 0;
  std::uint32_t nb = 0;
  int precision = 0;
  std::vector<std::uint32_t> block_boundaries;
  std::vector<std::uint64_t> entry_offsets;
  std::vector<std::uint16_t> rows, cols;
  std::vector<float> values32;
  std::vector<double> values64;
  std::vector<std::uint32_t> group_bounds;
};

}  // namespace cieg

struct cieg_host_csb {
  cieg::HostCsb h;
};
