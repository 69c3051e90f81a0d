// NVLink P2P bandwidth probe (design experiment, not part of the product path).
//
// All N GPUs run at once (the hpZ collectives are all-to-all).  Each GPU moves
// `mb` MiB per peer with one of four strategies and reports its NVLink ingress:
//   pull_ldg : LDG.128 from every peer's buffer, STG to local       (current gather/RS)
//   push_stg : LDG.128 local, STG.128 into every peer's buffer
//   pull_tma : cp.async.bulk peer->smem (mbarrier), cp.async.bulk smem->local
//   push_tma : cp.async.bulk local->smem, cp.async.bulk smem->peer
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe p2p_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int kMaxG = 8;
struct Ptrs {
  const char* src[kMaxG];
  char* dst[kMaxG];
  int n;
  int64_t bytes;   // per peer
};

__device__ __forceinline__ int4 ldg(const int4* p) {
  int4 r;
  asm volatile("ld.global.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int U>
__global__ void __launch_bounds__(256) copy_ldg(const Ptrs p) {
  const int64_t vec = p.bytes >> 4;
  const int64_t tile = 256 * U;
  const int64_t tiles = (vec + tile - 1) / tile;
  for (int64_t w = blockIdx.x; w < tiles * p.n; w += gridDim.x) {
    const int j = w % p.n;
    const int64_t t = w / p.n;
    const int4* s = (const int4*)p.src[j];
    int4* d = (int4*)p.dst[j];
    int4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t v = t * tile + threadIdx.x + u * 256;
      if (v < vec) r[u] = ldg(s + v);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t v = t * tile + threadIdx.x + u * 256;
      if (v < vec) d[v] = r[u];
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// TMA 1D bulk copy pipeline: one elected thread per CTA.
template <int STAGES>
__global__ void __launch_bounds__(32) copy_tma(const Ptrs p, int chunk) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t per = (p.bytes + chunk - 1) / chunk;
  const int64_t total = per * p.n;
  // chunks of this CTA: k-th is w = blockIdx.x + k*gridDim.x
  int64_t nk = 0;
  if (blockIdx.x < total) nk = (total - blockIdx.x + gridDim.x - 1) / gridDim.x;
  uint32_t phase[STAGES];
  for (int s = 0; s < STAGES; ++s) phase[s] = 0;
  auto issue_load = [&](int64_t k) {
    const int64_t w = blockIdx.x + k * gridDim.x;
    const int j = w % p.n;
    const int64_t c = w / p.n;
    const int64_t off = c * chunk;
    const int64_t n = (p.bytes - off) < chunk ? (p.bytes - off) : chunk;
    const int s = k % STAGES;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"((uint32_t)n) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(smem + (size_t)s * chunk)), "l"(p.src[j] + off), "r"((uint32_t)n), "r"(smem_u32(&bar[s]))
                 : "memory");
  };
  for (int64_t k = 0; k < nk && k < STAGES - 1; ++k) issue_load(k);
  for (int64_t k = 0; k < nk; ++k) {
    const int s = k % STAGES;
    // wait for load k
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                   : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(phase[s]) : "memory");
    }
    phase[s] ^= 1;
    const int64_t w = blockIdx.x + k * gridDim.x;
    const int j = w % p.n;
    const int64_t c = w / p.n;
    const int64_t off = c * chunk;
    const int64_t n = (p.bytes - off) < chunk ? (p.bytes - off) : chunk;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(p.dst[j] + off), "r"(smem_u32(smem + (size_t)s * chunk)), "r"((uint32_t)n) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // stage (k+STAGES-1)%STAGES == (k-1)%STAGES: its store (k-1) must have read smem
    if (k + STAGES - 1 < nk) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue_load(k + STAGES - 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int G = argc > 1 ? atoi(argv[1]) : 2;
  const char* mode = argc > 2 ? argv[2] : "pull_ldg";
  int64_t mb = argc > 3 ? atoll(argv[3]) : 256;
  int ctas_per_sm = argc > 4 ? atoi(argv[4]) : 4;
  int chunk = argc > 5 ? atoi(argv[5]) : 32768;
  const bool with_self = argc > 6 && atoi(argv[6]) != 0;   // also copy the local buffer (like a gather)
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (G > ndev) G = ndev;
  const int64_t bytes = mb << 20;
  char* buf_src[kMaxG];
  char* buf_dst[kMaxG];   // each GPU: G regions of `bytes` (one per source peer)
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h)
      if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    cudaGetLastError();
    CK(cudaMalloc(&buf_src[g], bytes));
    CK(cudaMalloc(&buf_dst[g], bytes * G));
    CK(cudaMemset(buf_src[g], g + 1, bytes));
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const bool pull = strstr(mode, "pull") != nullptr;
  const bool tma = strstr(mode, "tma") != nullptr;
  // pull_mix / push_mix: a TMA kernel (1 CTA/SM) moves the first `mix_pct`% of every peer
  // buffer while an LDG/STG kernel (ctas_per_sm CTAs/SM) moves the rest, concurrently on two
  // streams: does mixing the two request paths exceed either alone?
  const bool mix = strstr(mode, "mix") != nullptr;
  const int mix_pct = argc > 7 ? atoi(argv[7]) : 50;
  // TMA stage ring depth (argv[8], default 4): the ceiling is the best over depths
  const int stages = argc > 8 ? atoi(argv[8]) : 4;
  void (*tma_k)(const Ptrs, int) = stages == 2 ? copy_tma<2> : stages == 3 ? copy_tma<3> : stages == 6 ? copy_tma<6> : copy_tma<4>;
  const int n_stages = (stages == 2 || stages == 3 || stages == 6) ? stages : 4;
  cudaStream_t st[kMaxG], st2[kMaxG];
  cudaEvent_t e0[kMaxG], e1[kMaxG], e2[kMaxG];
  Ptrs P[kMaxG], PA[kMaxG], PB[kMaxG];
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&st2[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
    CK(cudaEventCreate(&e2[g]));
    Ptrs& p = P[g];
    p.n = 0;
    p.bytes = bytes;
    for (int h = 0; h < G; ++h) {
      if (h == g && !with_self) continue;
      if (pull) {   // g reads peer h's src into its own dst region h
        p.src[p.n] = buf_src[h];
        p.dst[p.n] = buf_dst[g] + (int64_t)h * bytes;
      } else {      // g writes its src into peer h's dst region g
        p.src[p.n] = buf_src[g];
        p.dst[p.n] = buf_dst[h] + (int64_t)g * bytes;
      }
      p.n++;
    }
    if (tma || mix) {
      int smem = n_stages * chunk;
      CK(cudaFuncSetAttribute(tma_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    if (mix) {   // split every peer buffer: [0, a) by TMA, [a, bytes) by LDG/STG
      const int64_t a = (bytes * mix_pct / 100) / 4096 * 4096;
      PA[g] = p;
      PB[g] = p;
      PA[g].bytes = a;
      PB[g].bytes = bytes - a;
      for (int k = 0; k < p.n; ++k) {
        PB[g].src[k] = p.src[k] + a;
        PB[g].dst[k] = p.dst[k] + a;
      }
    }
  }
  for (int it = 0; it < 4; ++it) {
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventRecord(e0[g], st[g]));
      if (mix) {
        CK(cudaStreamWaitEvent(st2[g], e0[g], 0));
        tma_k<<<sms, 32, n_stages * chunk, st[g]>>>(PA[g], chunk);
        copy_ldg<8><<<sms * ctas_per_sm, 256, 0, st2[g]>>>(PB[g]);
        CK(cudaEventRecord(e2[g], st2[g]));
        CK(cudaStreamWaitEvent(st[g], e2[g], 0));
      } else if (tma)
        tma_k<<<sms * ctas_per_sm, 32, n_stages * chunk, st[g]>>>(P[g], chunk);
      else
        copy_ldg<8><<<sms * ctas_per_sm, 256, 0, st[g]>>>(P[g]);
      CK(cudaGetLastError());
      CK(cudaEventRecord(e1[g], st[g]));
    }
    double worst = 1e30, sum = 0;
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventSynchronize(e1[g]));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
      double gbs = (double)bytes * (G - 1) / (ms * 1e-3) / 1e9;   // peer (NVLink) bytes only
      if (gbs < worst) worst = gbs;
      sum += gbs;
    }
    if (it == 3)
      printf("mode=%s G=%d MB/peer=%lld ctas/sm=%d chunk=%d stages=%d  per-GPU GB/s: min %.1f avg %.1f\n", mode, G,
             (long long)mb, ctas_per_sm, chunk, n_stages, worst, sum / G);
  }
  // verify one region
  CK(cudaSetDevice(0));
  unsigned char v = 0;
  const int h = G > 1 ? 1 : 0;
  CK(cudaMemcpy(&v, buf_dst[0] + (int64_t)h * bytes + bytes / 2, 1, cudaMemcpyDeviceToHost));
  printf("  check dst[0] region %d byte = %d (expect %d)\n", h, v, h + 1);
  return 0;
}
