// covap_capi_common.hpp — helpers shared by the C-ABI translation units
// (covap_capi.cpp, covap_feedback_capi.cpp): the communicator handle, error
// mapping onto covap_status + covap_last_error(), device guard.  Internal.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "covap/errors.hpp"
#include "covap_c.h"

namespace covapb {
struct NcclPeerMem;
}

struct covap_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 1;
  int rank = 0;
  int device = 0;
  // NCCL windows registered on this communicator (symmetric send buffers,
  // covap_state_use_symmetric): deregistered at the latest when it is destroyed
  std::vector<ncclWindow_t> windows;
  // peer-collective memory on this communicator (covap_peer_create_nccl):
  // its window / device communicator released at the latest then
  std::vector<covapb::NcclPeerMem*> peer_mems;
};

namespace covapb {

extern thread_local std::string g_last_error;


inline covap_status fail(covap_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

inline covap_status from_exception() {
  try {
    throw;
  } catch (const covap::InvalidInput& e) {
    return fail(COVAP_ERR_INVALID_INPUT, e.what());
  } catch (const covap::InvalidState& e) {
    return fail(COVAP_ERR_INVALID_STATE, e.what());
  } catch (const covap::UndefinedRatio& e) {
    return fail(COVAP_ERR_UNDEFINED_RATIO, e.what());
  } catch (const covap::IncompleteProfile& e) {
    return fail(COVAP_ERR_INCOMPLETE_PROFILE, e.what());
  } catch (const covap::ConfigError& e) {
    return fail(COVAP_ERR_CONFIG, e.what());
  } catch (const covap::Error& e) {
    return fail(COVAP_ERR_GENERIC, e.what());
  } catch (const std::bad_alloc&) {
    return fail(COVAP_ERR_GENERIC, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(COVAP_ERR_GENERIC, e.what());
  } catch (...) {
    return fail(COVAP_ERR_GENERIC, "unknown error");
  }
}

struct CudaError {
  cudaError_t e;
  const char* where;
};
struct NcclError {
  ncclResult_t r;
  const char* where;
};

#define CK(x)                                            \
  do {                                                   \
    cudaError_t _e = (x);                                \
    if (_e != cudaSuccess) throw CudaError{_e, #x};      \
  } while (0)
#define NK(x)                                            \
  do {                                                   \
    ncclResult_t _r = (x);                               \
    if (_r != ncclSuccess) throw NcclError{_r, #x};      \
  } while (0)

// Runs body; maps every failure onto a status code + message.
template <typename F>
inline covap_status guarded(F&& body) {
  try {
    body();
    return COVAP_OK;
  } catch (const CudaError& ce) {
    return fail(ce.e == cudaErrorNoDevice || ce.e == cudaErrorInsufficientDriver
                    ? COVAP_ERR_NO_DEVICE
                    : COVAP_ERR_CUDA,
                std::string(ce.where) + ": " + cudaGetErrorString(ce.e));
  } catch (const NcclError& ne) {
    return fail(COVAP_ERR_NCCL, std::string(ne.where) + ": " + ncclGetErrorString(ne.r));
  } catch (...) {
    return from_exception();
  }
}

// Restores the caller's current device on scope exit (no device switch, and
// so no extra runtime calls, when the caller is already on dev).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev == dev) {
      prev = -1;
      return;
    }
    CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

inline void need(bool cond, const char* msg) {
  if (!cond) throw covap::InvalidInput(msg);
}

inline void need_aligned(const void* p, const char* what) {
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
    throw covap::InvalidInput(std::string(what) + " must be 16-byte aligned");
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

inline ncclDataType_t nccl_type(int dtype) { return dtype == COVAP_F64 ? ncclFloat64 : ncclFloat32; }

inline int world(const covap_comm* c) { return c ? c->nranks : 1; }

}  // namespace covapb

using namespace covapb;  // NOLINT: the C-ABI units use these unqualified
