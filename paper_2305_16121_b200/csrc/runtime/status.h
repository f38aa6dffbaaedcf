// Error plumbing behind the C-ABI: C++ exceptions of the tmpsim error types
// (reference errors.hpp:11-26) and CUDA/NCCL failures map to oases_status codes
// (the reference CLI's exit codes, main.cpp:281-293).
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../../include/oases.h"
#include "../../../include/oases/tmpsim.hpp"

namespace oases {

struct CudaError : tmpsim::DeviceError {
  explicit CudaError(const std::string& w) : tmpsim::DeviceError(w) {}
};
struct NcclError : tmpsim::DeviceError {
  explicit NcclError(const std::string& w) : tmpsim::DeviceError(w) {}
};

void set_last_error(const std::string& msg);

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Runs f, converting exceptions into a status + thread-local message.
template <typename F>
oases_status guarded(F&& f) {
  try {
    f();
    return OASES_OK;
  } catch (const tmpsim::ConfigError& e) {
    set_last_error(e.what());
    return OASES_ERR_CONFIG;
  } catch (const tmpsim::InfeasibleError& e) {
    set_last_error(e.what());
    return OASES_ERR_INFEASIBLE;
  } catch (const tmpsim::IoError& e) {
    set_last_error(e.what());
    return OASES_ERR_IO;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return OASES_ERR_CUDA;
  } catch (const NcclError& e) {
    set_last_error(e.what());
    return OASES_ERR_NCCL;
  } catch (const tmpsim::DeviceError& e) {
    set_last_error(e.what());
    return OASES_ERR_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return OASES_ERR_CONFIG;
  }
}

}  // namespace oases
