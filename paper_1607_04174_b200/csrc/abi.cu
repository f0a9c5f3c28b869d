// ABI plumbing: version, status strings, CUDA error capture, SM count.
#include <atomic>
#include "swb_common.cuh"

namespace {
thread_local cudaError_t g_last = cudaSuccess;
std::atomic<int> g_sms{0};
std::atomic<unsigned long long> g_launches{0};
}  // namespace

void swb_set_last_cuda(cudaError_t e) { g_last = e; }
void swb_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" unsigned long long swb_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int swb_sm_count() {
  int v = g_sms.load(std::memory_order_relaxed);
  if (v > 0) return v;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  g_sms.store(sms, std::memory_order_relaxed);
  return sms;
}

extern "C" int swb_abi_version(void) { return 1; }

extern "C" const char* swb_status_string(int status) {
  switch (status) {
    case SWB_OK: return "ok";
    case SWB_INVALID_PARAM: return "InvalidParam";
    case SWB_INSUFFICIENT_BASIS: return "InsufficientBasis";
    case SWB_SINGULAR_SMALL_SYSTEM: return "SingularSmallSystem";
    case SWB_DEGENERATE_GRAPH: return "DegenerateGraph";
    case SWB_CUDA_ERROR: return "CudaError";
    case SWB_WORKSPACE_TOO_SMALL: return "WorkspaceTooSmall";
    case SWB_COMM_ERROR: return "CommError";
    default: return "unknown";
  }
}

extern "C" const char* swb_last_cuda_error(void) { return cudaGetErrorString(g_last); }
