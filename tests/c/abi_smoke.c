/* End-to-end use of the C ABI (include/ggarray.h) from plain C, as a caller in
 * another language would bind it: create, CSR insert, commit, grow,
 * duplicate insert, +1 pass, flatten, state read-back, error codes.
 * Built and run by tests/test_gpu_c_abi.py; prints "OK" on success. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "ggarray.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_) {                                                                \
      fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_,   \
              gg_last_error());                                               \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(void) {
  enum { S = 64, PER = 1000 };
  const uint64_t n = (uint64_t)S * PER;
  int32_t *h_vals = malloc(n * sizeof(int32_t));
  for (uint64_t i = 0; i < n; ++i) h_vals[i] = (int32_t)i;
  void *d_vals = NULL, *d_out = NULL;
  CHECK(gg_buf_alloc(n * 4, NULL, &d_vals));
  if (cudaMemcpy(d_vals, h_vals, n * 4, cudaMemcpyHostToDevice) != cudaSuccess) return 1;

  gg_array *bad = NULL;
  if (gg_create(0, S, 3, GG_I32, 58, 0, &bad) != GG_EVALUE || bad) {
    fprintf(stderr, "fb=3 must be GG_EVALUE\n");
    return 1;
  }
  gg_array *a = NULL;
  CHECK(gg_create(0, S, 32, GG_I32, 58, 0, &a));
  uint64_t off[S + 1];
  for (int s = 0; s <= S; ++s) off[s] = (uint64_t)s * PER;
  int32_t status[S];
  CHECK(gg_insert(a, d_vals, off, NULL, status, NULL));          /* one atomicAdd per LFVector */
  CHECK(gg_commit(a, NULL));
  uint64_t target[S];
  for (int s = 0; s < S; ++s) target[s] = 2 * PER;
  int64_t failed = -1;
  CHECK(gg_reserve(a, target, &failed, NULL));                    /* grow(2n) */
  CHECK(gg_insert_duplicate_ex(a, GG_F_COMMIT, status, NULL));    /* every shard appends itself */
  int32_t one = 1;
  CHECK(gg_rw_add(a, &one, 1, GG_RW_PER_SHARD, NULL));
  CHECK(gg_buf_alloc(2 * n * 4, NULL, &d_out));
  CHECK(gg_flatten(a, d_out, NULL));
  int32_t *h_out = malloc(2 * n * 4);
  if (cudaMemcpy(h_out, d_out, 2 * n * 4, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  for (uint64_t g = 0; g < 2 * n; ++g) {
    const uint64_t s = g / (2 * PER), i = g % (2 * PER);
    const int32_t want = (int32_t)(s * PER + i % PER + 1);
    if (h_out[g] != want) {
      fprintf(stderr, "flat[%llu] = %d, want %d\n", (unsigned long long)g, h_out[g], want);
      return 1;
    }
  }
  uint64_t sizes[S], caps[S], flags[S], prefix[S + 1], ops[S];
  CHECK(gg_device_state(a, sizes, caps, flags, prefix, ops, NULL));
  for (int s = 0; s < S; ++s)
    if (sizes[s] != 2 * PER || caps[s] != 32u * 63u || flags[s] != 63u || ops[s] != 2) {
      fprintf(stderr, "shard %d state %llu %llu %llu %llu\n", s, (unsigned long long)sizes[s],
              (unsigned long long)caps[s], (unsigned long long)flags[s], (unsigned long long)ops[s]);
      return 1;
    }
  if (prefix[S] != 2 * n) return 1;
  int32_t x = 0;
  CHECK(gg_get(a, 3, 5, &x, NULL));
  if (x != 3 * PER + 5 + 1) return 1;
  if (gg_get(a, 3, 2 * PER, &x, NULL) != GG_EINDEX) return 1;    /* IndexError past size */
  uint64_t mem[6];
  CHECK(gg_mem_stats(a, mem, NULL));
  if (mem[0] != (uint64_t)S * 32 * 63 * 4 || mem[3] != 2 * n * 4) return 1;
  CHECK(gg_destroy(a));
  CHECK(gg_buf_free(d_vals, NULL));
  CHECK(gg_buf_free(d_out, NULL));
  cudaDeviceSynchronize();
  free(h_vals);
  free(h_out);
  printf("OK\n");
  return 0;
}
