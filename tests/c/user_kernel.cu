// A THIRD-PARTY kernel growing a GGArray from inside a running kernel with the
// public device header (include/ggarray_device.cuh) -- the paper's use case --
// compiled separately from the library.  Thread i of block b emits i-th value
// if it is odd; the warp appends its odd values to shard (b % S) with
// gg::warp_push_back, the block variant with gg::block_push_back (modes 2-5:
// the mask variants, 4 = block_push_back_staged, 5 = warp_push_back_staged,
// vector stores).
// Built and driven by tests/test_gpu_user_kernel.py.
#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>

#include "ggarray_device.cuh"

template <int BLOCK>
__global__ void user_emit(gg::gg_device_view v, const int32_t *in, uint64_t n, int block_mode) {
  __shared__ unsigned long long scratch[34];
  __shared__ __align__(16) int32_t stage[BLOCK * 4 + (BLOCK / 32) * 8];
  const uint32_t s = blockIdx.x % v.S;
  if (block_mode >= 2) {            // mask variants: 4 rounds of candidates per thread
    constexpr int K = 4;
    const uint64_t round = (uint64_t)gridDim.x * BLOCK;
    for (uint64_t r0 = 0; (uint64_t)blockIdx.x * BLOCK + r0 * round < n; r0 += K) {
      int32_t cand[K];
      uint32_t mask = 0;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const uint64_t i = (uint64_t)blockIdx.x * BLOCK + (r0 + j) * round + threadIdx.x;
        cand[j] = i < n ? in[i] : 0;
        mask |= (uint32_t)(i < n && (cand[j] & 1)) << j;
      }
      if (block_mode == 5)
        gg::warp_push_back_staged<int32_t, K>(v, s, mask, cand, stage + (threadIdx.x >> 5) * (32 * K + 8));
      else if (block_mode == 4) gg::block_push_back_staged<BLOCK, int32_t, K>(v, s, mask, cand, scratch, stage);
      else if (block_mode == 3) gg::block_push_back_mask<BLOCK, int32_t, K>(v, s, mask, cand, scratch);
      else gg::warp_push_back_mask<int32_t, K>(v, s, mask, cand);
    }
    return;
  }
  for (uint64_t base = (uint64_t)blockIdx.x * BLOCK; base < n; base += (uint64_t)gridDim.x * BLOCK) {
    const uint64_t i = base + threadIdx.x;
    const int32_t x = i < n ? in[i] : 0;
    const bool odd = i < n && (x & 1);
    if (block_mode) gg::block_push_back<BLOCK, int32_t>(v, s, odd ? 1u : 0u, &x, scratch);
    else gg::warp_push_back<int32_t>(v, s, odd, x);
  }
}

extern "C" int user_emit_launch(const void *view_bytes, uint64_t view_size, const int32_t *d_in,
                                uint64_t n, uint32_t grid, int block_mode, void *stream) {
  if (view_size != sizeof(gg::gg_device_view)) return 1;
  gg::gg_device_view v;
  memcpy(&v, view_bytes, sizeof v);
  user_emit<256><<<grid, 256, 0, (cudaStream_t)stream>>>(v, d_in, n, block_mode);
  return (int)cudaGetLastError();
}
