// gg_common.cuh -- shared definitions of the B200 GGArray library: error
// plumbing, CUDA driver VMM entry points, constants, element types.  Part of
// the single translation unit built from ggarray.cu.
#ifndef GG_COMMON_CUH
#define GG_COMMON_CUH

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>
#include <type_traits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ggarray.h"
#include "../../include/ggarray_device.cuh"

#define GG_VERSION 1


namespace gg {


typedef gg_device_view Tables;

thread_local std::string g_err;
std::atomic<unsigned long long> g_launches{0};   // kernels launched by this library

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

// Driver VMM entry points resolved through cudaGetDriverEntryPoint, so the
// library has no link-time libcuda dependency (it loads on GPU-less hosts).
struct Drv {
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuGetErrorString) err_string = nullptr;
  bool ok = false;
};

Drv &drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char *name, void **fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn != nullptr;
    };
    d.ok = get("cuMemGetAllocationGranularity", (void **)&d.granularity) &&
           get("cuMemAddressReserve", (void **)&d.reserve) &&
           get("cuMemAddressFree", (void **)&d.addr_free) &&
           get("cuMemCreate", (void **)&d.create) && get("cuMemRelease", (void **)&d.release) &&
           get("cuMemMap", (void **)&d.map) && get("cuMemUnmap", (void **)&d.unmap) &&
           get("cuMemSetAccess", (void **)&d.set_access) &&
           get("cuGetErrorString", (void **)&d.err_string);
  });
  return d;
}

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(GG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define CU_TRY(expr)                                                                   \
  do {                                                                                 \
    CUresult r_ = (expr);                                                              \
    if (r_ != CUDA_SUCCESS) {                                                          \
      const char *s_ = nullptr;                                                        \
      if (drv().err_string) drv().err_string(r_, &s_);                                 \
      return fail(r_ == CUDA_ERROR_OUT_OF_MEMORY ? GG_ENOMEM : GG_ECUDA,               \
                  std::string(#expr) + ": " + (s_ ? s_ : "?"));                        \
    }                                                                                  \
  } while (0)

constexpr int kMaxBuckets = 64;
constexpr uint64_t kDefaultVaBudget = uint64_t(16) << 40;   // slab VA per array (16 TiB)
constexpr int kThreads = 256;          // CTA size of the streaming kernels
constexpr uint64_t kFlatChunk = 16 * 1024;  // bytes per CTA of the contiguous +c kernel

// ctl word per shard (only uploaded when an op plans a failure)
constexpr uint32_t kCtlLimitMask = 0xffu;   // allocate buckets < limit
constexpr uint32_t kCtlWrite = 1u << 8;     // write the values
constexpr uint32_t kCtlZero = 1u << 9;      // write zeros instead (failed shard)

inline uint32_t elem_bytes_of(uint32_t dt) {
  switch (dt) {
    case GG_I8: case GG_U8: return 1;
    case GG_I16: case GG_U16: case GG_F16: return 2;
    case GG_I32: case GG_U32: case GG_F32: return 4;
    case GG_I64: case GG_U64: case GG_F64: return 8;
    default: return 0;
  }
}

inline uint64_t round16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

inline int ilog2(uint64_t x) { return 63 - __builtin_clzll(x); }

}  // namespace gg

#endif  // GG_COMMON_CUH
