/* Plain-C GPU client of include/hpz.h, no Python or PyTorch anywhere: two ranks emulated
 * on device 0 (P=2, P'=1 — the arenas are allocated by the library and bound to each
 * other with hpz_bind), three flat layers (one smaller than P*A), three training steps of
 * Algorithm 1 through the C ABI on one CUDA stream:
 *   fwd gathers (fused secondary store) -> bwd gathers from the secondaries -> seeded
 *   gradients -> fused reduce-scatter + Adam,
 * with EXACT verification (every backward-gathered element compared with its owner's
 * primary on the device).  Checks on the host: each rank's backward gather equals its
 * forward gather byte for byte, both ranks gathered the same bytes, the counters report
 * 0 mismatches / NaN reads / timeouts, and the step counter advanced.
 * Prints C_STEP_OK and exits 0 on success. */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hpz.h"

#define P 2
#define L 3
#define CHECK(x)                                                                   \
  do {                                                                             \
    int rc_ = (x);                                                                 \
    if (rc_ != HPZ_OK) {                                                           \
      fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #x, rc_);            \
      return 1;                                                                    \
    }                                                                              \
  } while (0)
#define CUCHECK(x)                                                                 \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main(void) {
  const int64_t numel[L] = {300007, 65536, 77};
  hpz_ctx* ctx[P];
  void* arena[P];
  for (int r = 0; r < P; ++r) {
    CHECK(hpz_init(P, 1, r, 0, &ctx[r]));
    uint64_t bytes = 0;
    CHECK(hpz_register_flat_params(ctx[r], L, numel, HPZ_BF16, 256, L, &bytes));
    CHECK(hpz_arena_alloc(ctx[r], NULL));
    CHECK(hpz_arena_ptr(ctx[r], r, &arena[r]));
  }
  for (int r = 0; r < P; ++r) {
    CHECK(hpz_bind(ctx[r], arena));
    CHECK(hpz_set_verify(ctx[r], HPZ_VERIFY_EXACT));
  }
  cudaStream_t s;
  CUCHECK(cudaStreamCreate(&s));
  hpz_layer_info_t info[L];
  size_t maxb = 0;
  for (int i = 0; i < L; ++i) {
    CHECK(hpz_layer_info(ctx[0], i, &info[i]));
    if ((size_t)info[i].numel_pad * 2 > maxb) maxb = (size_t)info[i].numel_pad * 2;
  }
  void *fwd[P][L], *bwd[P][L];
  for (int r = 0; r < P; ++r)
    for (int i = 0; i < L; ++i) {
      CUCHECK(cudaMalloc(&fwd[r][i], (size_t)info[i].numel_pad * 2));
      CUCHECK(cudaMalloc(&bwd[r][i], (size_t)info[i].numel_pad * 2));
    }
  for (int i = 0; i < L; ++i)
    for (int r = 0; r < P; ++r) CHECK(hpz_synth_master(ctx[r], i, 0x5EED0001ull + (uint64_t)i, 1.0f / 32, s));
  hpz_adam adam = {1e-3, 0.9, 0.999, 1e-8, 0.0, 0};
  unsigned char* ha = (unsigned char*)malloc(maxb);
  unsigned char* hb = (unsigned char*)malloc(maxb);
  for (int t = 0; t < 3; ++t) {
    for (int i = 0; i < L; ++i)
      for (int r = 0; r < P; ++r) CHECK(hpz_fwd_gather(ctx[r], i, fwd[r][i], s));
    for (int i = L - 1; i >= 0; --i) {
      for (int r = 0; r < P; ++r) CHECK(hpz_bwd_gather(ctx[r], i, bwd[r][i], s));
      for (int r = 0; r < P; ++r)
        CHECK(hpz_synth_grads(ctx[r], i, 0x5EED0002ull ^ ((uint64_t)t << 32) ^ ((uint64_t)i << 16) ^ (uint64_t)r,
                              1.0f / 4096, 0, s));
      for (int r = 0; r < P; ++r) CHECK(hpz_grads_ready(ctx[r], i, s));   /* one stream: publish first */
      for (int r = 0; r < P; ++r) CHECK(hpz_reduce_scatter_adam(ctx[r], i, &adam, s));
    }
    CUCHECK(cudaStreamSynchronize(s));
    for (int i = 0; i < L; ++i) {
      const size_t nb = (size_t)info[i].numel_pad * 2;
      for (int r = 0; r < P; ++r) {
        CUCHECK(cudaMemcpy(ha, fwd[r][i], nb, cudaMemcpyDeviceToHost));
        CUCHECK(cudaMemcpy(hb, bwd[r][i], nb, cudaMemcpyDeviceToHost));
        if (memcmp(ha, hb, nb) != 0) {
          fprintf(stderr, "step %d layer %d rank %d: backward gather != forward gather\n", t, i, r);
          return 1;
        }
      }
      CUCHECK(cudaMemcpy(hb, fwd[1][i], nb, cudaMemcpyDeviceToHost));
      CUCHECK(cudaMemcpy(ha, fwd[0][i], nb, cudaMemcpyDeviceToHost));
      if (memcmp(ha, hb, nb) != 0) {
        fprintf(stderr, "step %d layer %d: ranks gathered different parameters\n", t, i);
        return 1;
      }
    }
  }
  unsigned long long bad = 0, checked = 0;
  for (int r = 0; r < P; ++r) {
    hpz_counters_t c;
    CHECK(hpz_counters(ctx[r], &c, 0));
    bad += c.mismatches + c.nan_reads + c.timeouts;
    checked += c.launches;
    int64_t step = -1;
    CHECK(hpz_current_step(ctx[r], &step));
    if (step != 3) {
      fprintf(stderr, "rank %d: step counter %lld, expected 3\n", r, (long long)step);
      return 1;
    }
  }
  printf("mismatches+nan+timeouts=%llu launches=%llu\n", bad, checked);
  for (int r = 0; r < P; ++r) {
    for (int i = 0; i < L; ++i) {
      cudaFree(fwd[r][i]);
      cudaFree(bwd[r][i]);
    }
    hpz_finalize(ctx[r]);
  }
  free(ha);
  free(hb);
  if (bad != 0) return 1;
  printf("C_STEP_OK\n");
  return 0;
}
