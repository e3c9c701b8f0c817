// Streaming-copy variants on B200 (probe, not product): which loop shape
// reaches the measured torch-copy bandwidth?
#include <cuda_runtime.h>
#include <cstdint>

template <int U, int LS>
__device__ __forceinline__ uint4 ld(const uint4 *p) {
  if (LS == 0) return __ldcg(p);
  if (LS == 1) return __ldg(p);
  if (LS == 3) return __ldcs(p);
  return *p;
}
template <int LS>
__device__ __forceinline__ void st(uint4 *p, uint4 v) {
  if (LS == 0) __stcg(p, v);
  else if (LS == 3) __stcs(p, v);
  else *p = v;
}

// non-persistent: each CTA copies one contiguous chunk of U*blockDim vectors
template <int U, int LS>
__global__ void k_chunk(uint4 *d, const uint4 *s, uint64_t nv) {
  uint64_t base = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  uint4 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { uint64_t i = base + u * blockDim.x; if (i < nv) r[u] = ld<U, LS>(s + i); }
#pragma unroll
  for (int u = 0; u < U; ++u) { uint64_t i = base + u * blockDim.x; if (i < nv) st<LS>(d + i, r[u]); }
}

// persistent grid-stride over tiles of T vectors per CTA
template <int U, int LS>
__global__ void k_tiles(uint4 *d, const uint4 *s, uint64_t nv, uint32_t tilev) {
  const uint64_t ntiles = (nv + tilev - 1) / tilev;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t lo = t * tilev, hi = min(nv, lo + tilev);
    for (uint64_t v0 = lo + threadIdx.x; v0 < hi; v0 += U * blockDim.x) {
      uint4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = ld<U, LS>(s + min(v0 + u * blockDim.x, hi - 1));
#pragma unroll
      for (int u = 0; u < U; ++u) if (v0 + u * blockDim.x < hi) st<LS>(d + v0 + u * blockDim.x, r[u]);
    }
  }
}

// TMA bulk: CTA streams its chunks through a smem ring with cp.async.bulk
// (global -> smem, mbarrier completion) and cp.async.bulk (smem -> global).
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32) k_tma(char *d, const char *s, uint64_t nbytes) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const uint64_t nchunks = nbytes / CHUNK;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t phase[STAGES] = {0};
  uint64_t c = blockIdx.x;
  // prologue: fill stages
  int issued = 0;
  for (int i = 0; i < STAGES && c + (uint64_t)i * gridDim.x < nchunks; ++i) {
    const uint64_t ch = c + (uint64_t)i * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(buf + i * CHUNK)), "l"(s + ch * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[i])) : "memory");
    ++issued;
  }
  int k = 0;
  for (uint64_t ch = c; ch < nchunks; ch += gridDim.x, k = (k + 1) % STAGES) {
    // wait for stage k
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}"
                 ::"r"(smem_u32(&bar[k])), "r"(phase[k]) : "memory");
    phase[k] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(d + ch * CHUNK), "r"(smem_u32(buf + k * CHUNK)), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill stage k with chunk ch + STAGES*grid once its store has read smem
    const uint64_t nxt = ch + (uint64_t)STAGES * gridDim.x;
    if (nxt < nchunks) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[k])), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf + k * CHUNK)), "l"(s + nxt * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[k])) : "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

extern "C" int probe_copy(void *d, const void *s, uint64_t nbytes, int variant, int threads, int grid_or_tile) {
  const uint64_t nv = nbytes / 16;
  uint4 *dv = (uint4 *)d; const uint4 *sv = (const uint4 *)s;
  switch (variant) {
#define CH(U, LS) { int g = (int)((nv + (uint64_t)threads * U - 1) / ((uint64_t)threads * U)); k_chunk<U, LS><<<g, threads>>>(dv, sv, nv); break; }
    case 0: CH(4, 2)
    case 1: CH(4, 0)
    case 2: CH(4, 3)
    case 3: CH(8, 2)
    case 4: CH(2, 2)
    case 5: CH(1, 2)
    case 6: CH(8, 3)
#undef CH
    case 10: { k_tiles<4, 0><<<148 * 8, threads>>>(dv, sv, nv, grid_or_tile / 16); break; }
    case 11: { k_tiles<4, 2><<<148 * 8, threads>>>(dv, sv, nv, grid_or_tile / 16); break; }
    case 12: { k_tiles<8, 2><<<148 * 4, threads>>>(dv, sv, nv, grid_or_tile / 16); break; }
    case 20: {
      constexpr int ST = 4, CHK = 32768;
      cudaFuncSetAttribute(k_tma<ST, CHK>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CHK);
      k_tma<ST, CHK><<<148 * grid_or_tile, 32, ST * CHK>>>((char *)d, (const char *)s, nbytes); break; }
    case 21: {
      constexpr int ST = 6, CHK = 16384;
      cudaFuncSetAttribute(k_tma<ST, CHK>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CHK);
      k_tma<ST, CHK><<<148 * grid_or_tile, 32, ST * CHK>>>((char *)d, (const char *)s, nbytes); break; }
    case 22: {
      constexpr int ST = 2, CHK = 65536;
      cudaFuncSetAttribute(k_tma<ST, CHK>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CHK);
      k_tma<ST, CHK><<<148 * grid_or_tile, 32, ST * CHK>>>((char *)d, (const char *)s, nbytes); break; }
    default: return -1;
  }
  return (int)cudaGetLastError();
}
