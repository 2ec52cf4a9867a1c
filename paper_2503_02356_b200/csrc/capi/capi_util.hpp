// Exception -> status-code translation for the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../../include/chunkflow_b200.h"
#include "../host/plan.hpp"

namespace cfb {

extern thread_local std::string g_last_error;

// Relative cost of one attention (query, key) pair vs one token of GEMM work
// for the DP partition.  FLOP ratio 12*L*H*dh / (6*N) = 4.4e-5 for
// Llama-7B-GQA8; the attention kernels run at about half the
// GEMM rate, and the per-op times of a measured C2 step fit 8.4e-5
// (profiles/round1_step_breakdown.json).
constexpr double kPairWeight = 8.4e-5;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return CF_OK;
  } catch (const ValidationError& e) {
    g_last_error = e.what();
    return CF_EVALIDATION;
  } catch (const ParseError& e) {
    g_last_error = e.what();
    return CF_EPARSE;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return CF_ECUDA;
  } catch (const NcclError& e) {
    g_last_error = e.what();
    return CF_ENCCL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CF_EINTERNAL;
  }
}

}  // namespace cfb

struct cf_plan {
  cfb::Plan p;
};
