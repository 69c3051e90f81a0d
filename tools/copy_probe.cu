// Device-local copy structures at the N = 1 gather's size (one Falcon-7B block, 414 MB of
// bf16 read + 414 MB written per copy), 34 back-to-back copies timed with CUDA events:
//   tma_persist  : 1 CTA/SM grid-stride, one thread issues cp.async.bulk loads into an
//                  S-stage smem ring and bulk-stores each stage (the library's gather)
//   ldg_persist  : grid-stride LDG.128/STG.128, CTAS CTAs/SM, U loads in flight per thread
//   ldg_wide     : one short-lived CTA per TILE bytes (a huge grid, like an elementwise
//                  kernel), U loads in flight per thread
//   tma_wide     : one short-lived CTA per TILE bytes, bulk load + bulk store through smem
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/copy_probe tools/copy_probe.cu
//   tools/copy_probe [MB]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));   \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* s, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(s)),
               "l"(g), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_store(void* g, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int S>
__global__ void __launch_bounds__(32, 1) tma_persist(const char* src, char* dst, int64_t bytes, int chunk) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t total = (bytes + chunk - 1) / chunk;
  const int64_t nk = blockIdx.x < total ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](int64_t k) {
    const int64_t off = (blockIdx.x + k * gridDim.x) * (int64_t)chunk;
    const uint32_t b = (uint32_t)(bytes - off < chunk ? bytes - off : chunk);
    const int s = (int)(k % S);
    mbar_expect_tx(&full[s], b);
    tma_load(smem + (size_t)s * chunk, src + off, b, &full[s]);
  };
  for (int64_t k = 0; k < nk && k < S - 1; ++k) issue(k);
  for (int64_t k = 0; k < nk; ++k) {
    const int s = (int)(k % S);
    mbar_wait(&full[s], (uint32_t)((k / S) & 1));
    const int64_t off = (blockIdx.x + k * gridDim.x) * (int64_t)chunk;
    const uint32_t b = (uint32_t)(bytes - off < chunk ? bytes - off : chunk);
    tma_store(dst + off, smem + (size_t)s * chunk, b);
    bulk_commit();
    if (k + S - 1 < nk) {
      bulk_wait_read<1>();
      issue(k + S - 1);
    }
  }
  bulk_wait_all();
}

// persistent, but chunks handed out in order by a global counter (the hardware block
// scheduler's order, without relaunching CTAs): the producer grabs the next chunk index when
// it refills a stage and leaves it in smem for the stage's store
template <int S>
__global__ void __launch_bounds__(32, 1) tma_dyn(const char* src, char* dst, int64_t bytes, int chunk,
                                                 unsigned long long* ctr) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ int64_t wk[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t total = (bytes + chunk - 1) / chunk;
  int64_t issued = 0;
  auto issue = [&]() -> bool {
    const int64_t w = (int64_t)atomicAdd(ctr, 1ull);
    if (w >= total) return false;
    const int64_t off = w * chunk;
    const uint32_t b = (uint32_t)(bytes - off < chunk ? bytes - off : chunk);
    const int s = (int)(issued % S);
    wk[s] = w;
    mbar_expect_tx(&full[s], b);
    tma_load(smem + (size_t)s * chunk, src + off, b, &full[s]);
    ++issued;
    return true;
  };
  bool more = true;
  for (int k = 0; k < S - 1 && more; ++k) more = issue();
  for (int64_t k = 0; k < issued; ++k) {
    const int s = (int)(k % S);
    mbar_wait(&full[s], (uint32_t)((k / S) & 1));
    const int64_t off = wk[s] * chunk;
    const uint32_t b = (uint32_t)(bytes - off < chunk ? bytes - off : chunk);
    tma_store(dst + off, smem + (size_t)s * chunk, b);
    bulk_commit();
    if (more) {
      bulk_wait_read<1>();
      more = issue();
    }
  }
  bulk_wait_all();
}

// the library's gather shape: producer thread + 4 "fingerprint" warps that read every
// landed stage from smem and free it through an empty barrier before it is refilled;
// DYN 0 = static grid-stride chunks, 1 = counter per grab, 2 = counter read one grab ahead
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
template <int S, int DYN, int LAG = 1, int GATE = 1, int READ = 1>
__global__ void __launch_bounds__(160, 1) tma_fp(const char* src, char* dst, int64_t bytes, int chunk,
                                                 unsigned* ctr, unsigned long long* out_fp) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t empty[S];
  __shared__ int64_t wk[S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t total = (bytes + chunk - 1) / chunk;
  if (warp == 0) {
    if (lane != 0) return;
    int64_t issued = 0;
    unsigned ahead = DYN == 2 ? atomicAdd(ctr, 1u) : 0u;
    auto grab = [&]() -> int64_t {
      int64_t w;
      if (DYN == 2) {
        w = ahead;
        if (w < total) ahead = atomicAdd(ctr, 1u);
      } else if (DYN == 1) {
        w = atomicAdd(ctr, 1u);
      } else {
        w = blockIdx.x + issued * (int64_t)gridDim.x;
      }
      return w < total ? w : -1;
    };
    auto issue = [&](int64_t w) {
      const int64_t off = w * chunk;
      const uint32_t b = (uint32_t)(bytes - off < chunk ? bytes - off : chunk);
      const int s = (int)(issued % S);
      wk[s] = w;
      mbar_expect_tx(&full[s], b);
      tma_load(smem + (size_t)s * chunk, src + off, b, &full[s]);
      ++issued;
    };
    bool more = true;
    for (int k = 0; k < S - LAG && more; ++k) {
      const int64_t w = grab();
      if (w < 0) more = false;
      else issue(w);
    }
    for (int64_t k = 0; k < issued; ++k) {
      const int s = (int)(k % S);
      mbar_wait(&full[s], (uint32_t)((k / S) & 1));
      const int64_t off = wk[s] * chunk;
      const uint32_t b = (uint32_t)(bytes - off < chunk ? bytes - off : chunk);
      tma_store(dst + off, smem + (size_t)s * chunk, b);
      bulk_commit();
      if (more) {
        const int64_t w = grab();
        if (w < 0) {
          more = false;
        } else {
          bulk_wait_read<LAG>();
          if (GATE && k >= LAG) mbar_wait(&empty[(k - LAG) % S], (uint32_t)(((k - LAG) / S) & 1));
          issue(w);
        }
      }
    }
    const int s = (int)(issued % S);
    if (issued >= S) mbar_wait(&empty[s], (uint32_t)(((issued - S) / S) & 1));
    wk[s] = -1;
    mbar_arrive(&full[s]);
    bulk_wait_all();
  } else {
    unsigned long long acc = 0;
    const int ct = threadIdx.x - 32;
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      mbar_wait(&full[s], (uint32_t)((k / S) & 1));
      const int64_t w = *reinterpret_cast<volatile int64_t*>(&wk[s]);
      if (w < 0) break;
      const int4* st = reinterpret_cast<const int4*>(smem + (size_t)s * chunk);
      const uint32_t g0 = (uint32_t)(w * chunk / 16);
      for (int v = ct; READ && v < chunk / 16; v += 128) {
        const int4 x = st[v];
        const uint32_t q = (g0 + v) * 4u * 0x9E3779B1u;
        acc += (unsigned long long)(uint32_t)x.x * (q | 1u) + (unsigned long long)(uint32_t)x.y * ((q + 0x9E3779B1u) | 1u) +
               (unsigned long long)(uint32_t)x.z * ((q + 2u * 0x9E3779B1u) | 1u) +
               (unsigned long long)(uint32_t)x.w * ((q + 3u * 0x9E3779B1u) | 1u);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc) atomicAdd(out_fp, acc);
  }
}

template <int U>
__global__ void __launch_bounds__(256) ldg_persist(const int4* src, int4* dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < n; base += stride) {
    int4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * blockDim.x < n) r[u] = __ldcs(src + base + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * blockDim.x < n) dst[base + u * blockDim.x] = r[u];
  }
}

template <int U>
__global__ void __launch_bounds__(128) ldg_wide(const int4* src, int4* dst, int64_t n) {
  const int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  int4 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (base + u * blockDim.x < n) r[u] = src[base + u * blockDim.x];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (base + u * blockDim.x < n) dst[base + u * blockDim.x] = r[u];
}

// the wide LDG copy with the library's per-launch obligations: a fingerprint of every 16-byte
// word computed from registers (block-reduced, one RED per CTA) and a completion counter
// (one returning atomic per CTA, the last CTA resets it)
template <int U, int T>
__global__ void __launch_bounds__(T) ldg_wide_fp(const int4* src, int4* dst, int64_t n, unsigned long long* fp_out,
                                                 unsigned* done) {
  __shared__ unsigned long long red[T / 32];
  const int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x;
  int4 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (base + u * T < n) r[u] = src[base + u * T];
  unsigned long long acc = 0;
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (base + u * T < n) {
      dst[base + u * T] = r[u];
      const uint32_t q = (uint32_t)(base + u * T) * 4u * 0x9E3779B1u;
      acc += (unsigned long long)(uint32_t)r[u].x * (q | 1u) + (unsigned long long)(uint32_t)r[u].y * ((q + 0x9E3779B1u) | 1u) +
             (unsigned long long)(uint32_t)r[u].z * ((q + 2u * 0x9E3779B1u) | 1u) +
             (unsigned long long)(uint32_t)r[u].w * ((q + 3u * 0x9E3779B1u) | 1u);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < T / 32; ++w) t += red[w];
    atomicAdd(fp_out, t);
    __threadfence_system();
    if (atomicAdd(done, 1u) == gridDim.x - 1) *done = 0;
  }
}

// persistent warps, each taking runs of R warp-tiles (32 lanes x U int4) from a counter with
// the next run's counter read issued ahead; copy through registers + register fingerprint
template <int U, int R>
__global__ void __launch_bounds__(256) ldg_dyn_fp(const int4* src, int4* dst, int64_t n, unsigned* ctr,
                                                  unsigned long long* fp_out) {
  const int lane = threadIdx.x & 31;
  const int64_t tiles = (n + 32 * U - 1) / (32 * U);
  unsigned nxt = 0;
  if (lane == 0) nxt = atomicAdd(ctr, (unsigned)R);
  unsigned long long acc = 0;
  for (;;) {
    const int64_t run = (int64_t)__shfl_sync(0xffffffffu, nxt, 0);
    if (run >= tiles) break;
    if (lane == 0) nxt = atomicAdd(ctr, (unsigned)R);
    for (int t = 0; t < R && run + t < tiles; ++t) {
      const int64_t base = (run + t) * 32 * U + lane;
      int4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (base + u * 32 < n) r[u] = src[base + u * 32];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (base + u * 32 < n) {
          dst[base + u * 32] = r[u];
          const uint32_t q = (uint32_t)(base + u * 32) * 4u * 0x9E3779B1u;
          acc += (unsigned long long)(uint32_t)r[u].x * (q | 1u) + (unsigned long long)(uint32_t)r[u].y * ((q + 0x9E3779B1u) | 1u) +
                 (unsigned long long)(uint32_t)r[u].z * ((q + 2u * 0x9E3779B1u) | 1u) +
                 (unsigned long long)(uint32_t)r[u].w * ((q + 3u * 0x9E3779B1u) | 1u);
        }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc) atomicAdd(fp_out, acc);
}

__global__ void __launch_bounds__(32) tma_wide(const char* src, char* dst, int64_t bytes, int tile) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full;
  if (threadIdx.x != 0) return;
  mbar_init(&full, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t off = (int64_t)blockIdx.x * tile;
  const uint32_t b = (uint32_t)(bytes - off < tile ? bytes - off : tile);
  mbar_expect_tx(&full, b);
  tma_load(smem, src + off, b, &full);
  mbar_wait(&full, 0);
  tma_store(dst + off, smem, b);
  bulk_commit();
  bulk_wait_all();
}

template <typename F>
double timeit(F f, int64_t bytes) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a));
    for (int i = 0; i < 34; ++i) f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double gbs = 2.0 * bytes * 34 / (ms * 1e-3) / 1e9;
    if (gbs > best) best = gbs;
  }
  return best;
}

int main(int argc, char** argv) {
  const int64_t bytes = (argc > 1 ? atoll(argv[1]) : 414142464LL / (1 << 20)) << 20;
  char *src, *dst;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&dst, bytes));
  CK(cudaMemset(src, 1, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t n16 = bytes / 16;
  printf("bytes per copy %lld (read) + same written, %d SMs\n", (long long)bytes, sms);
  printf("memcpy_d2d           %.1f GB/s\n", timeit([&] { CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice)); }, bytes));
#define TMA_P(S, CH)                                                                              \
  {                                                                                               \
    CK(cudaFuncSetAttribute(tma_persist<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH)); \
    printf("tma_persist %2dx%3dK  %.1f GB/s\n", S, CH / 1024,                                      \
           timeit([&] { tma_persist<S><<<sms, 32, S * CH>>>(src, dst, bytes, CH); }, bytes));     \
  }
  TMA_P(8, 16384)
  TMA_P(4, 32768)
  TMA_P(12, 16384)
  unsigned long long* ctr;
  CK(cudaMalloc(&ctr, 8 * 64));
  CK(cudaMemset(ctr, 0, 8 * 64));
  int rep = 0;
#define TMA_D(S, CH)                                                                              \
  {                                                                                               \
    CK(cudaFuncSetAttribute(tma_dyn<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH));     \
    printf("tma_dyn     %2dx%3dK  %.1f GB/s\n", S, CH / 1024, timeit([&] {                        \
             CK(cudaMemsetAsync(ctr, 0, 8));                                                      \
             tma_dyn<S><<<sms, 32, S * CH>>>(src, dst, bytes, CH, ctr);                            \
           }, bytes));                                                                            \
  }
  TMA_D(8, 16384)
  TMA_D(4, 32768)
  TMA_D(6, 32768)
  (void)rep;
  unsigned long long* fpo;
  CK(cudaMalloc(&fpo, 8));
#define TMA_F(S, CH, D)                                                                           \
  {                                                                                               \
    CK(cudaFuncSetAttribute(tma_fp<S, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH));   \
    printf("tma_fp dyn%d %2dx%3dK  %.1f GB/s\n", D, S, CH / 1024, timeit([&] {                     \
             CK(cudaMemsetAsync(ctr, 0, 8));                                                      \
             tma_fp<S, D><<<sms, 160, S * CH>>>(src, dst, bytes, CH, (unsigned*)ctr, fpo);         \
           }, bytes));                                                                            \
  }
  TMA_F(8, 16384, 0)
  TMA_F(8, 16384, 1)
  TMA_F(8, 16384, 2)
#define TMA_FL(S, CH, D, LAG, GATE)                                                                       \
  {                                                                                                       \
    CK(cudaFuncSetAttribute(tma_fp<S, D, LAG, GATE>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH)); \
    printf("tma_fp dyn%d lag%d gate%d %2dx%3dK  %.1f GB/s\n", D, LAG, GATE, S, CH / 1024, timeit([&] {     \
             CK(cudaMemsetAsync(ctr, 0, 8));                                                              \
             tma_fp<S, D, LAG, GATE><<<sms, 160, S * CH>>>(src, dst, bytes, CH, (unsigned*)ctr, fpo);      \
           }, bytes));                                                                                    \
  }
  {
    CK(cudaFuncSetAttribute(tma_fp<8, 1, 1, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384));
    printf("tma_fp dyn1 noread     8x 16K  %.1f GB/s\n", timeit([&] {
             CK(cudaMemsetAsync(ctr, 0, 8));
             tma_fp<8, 1, 1, 1, 0><<<sms, 160, 8 * 16384>>>(src, dst, bytes, 16384, (unsigned*)ctr, fpo);
           }, bytes));
  }
  TMA_FL(8, 16384, 1, 1, 0)
  TMA_FL(8, 16384, 1, 2, 1)
  TMA_FL(8, 16384, 1, 3, 1)
  TMA_FL(8, 16384, 0, 2, 1)
  TMA_FL(12, 16384, 1, 2, 1)
#define LDG_P(U, C)                                                                                 \
  printf("ldg_persist U=%d %2d CTA/SM  %.1f GB/s\n", U, C,                                          \
         timeit([&] { ldg_persist<U><<<sms * C, 256>>>((const int4*)src, (int4*)dst, n16); }, bytes));
  LDG_P(4, 4)
  LDG_P(4, 8)
  LDG_P(8, 4)
#define LDG_W(U)                                                                                               \
  printf("ldg_wide U=%d        %.1f GB/s\n", U,                                                                 \
         timeit([&] { ldg_wide<U><<<(unsigned)((n16 + 128 * U - 1) / (128 * U)), 128>>>((const int4*)src, (int4*)dst, n16); }, \
                bytes));
  LDG_W(4)
  LDG_W(8)
#define TMA_W(T)                                                                                       \
  {                                                                                                    \
    CK(cudaFuncSetAttribute(tma_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, T));               \
    printf("tma_wide %3dK        %.1f GB/s\n", T / 1024,                                              \
           timeit([&] { tma_wide<<<(unsigned)((bytes + T - 1) / T), 32, T>>>(src, dst, bytes, T); }, bytes)); \
  }
  unsigned* dn;
  CK(cudaMalloc(&dn, 64));
  CK(cudaMemset(dn, 0, 64));
#define LDG_WF(U, T)                                                                                            \
  printf("ldg_wide_fp U=%d T=%d  %.1f GB/s\n", U, T,                                                            \
         timeit([&] { ldg_wide_fp<U, T><<<(unsigned)((n16 + (int64_t)T * U - 1) / ((int64_t)T * U)), T>>>((const int4*)src, (int4*)dst, n16, fpo, dn); }, \
                bytes));
  LDG_WF(8, 128)
  LDG_WF(8, 256)
  LDG_WF(8, 512)
  LDG_WF(4, 512)
  LDG_WF(16, 256)
#define LDG_DF(U, R, C)                                                                                   \
  printf("ldg_dyn_fp U=%d R=%d %d CTA/SM  %.1f GB/s\n", U, R, C, timeit([&] {                               \
           CK(cudaMemsetAsync(ctr, 0, 8));                                                                  \
           ldg_dyn_fp<U, R><<<sms * C, 256>>>((const int4*)src, (int4*)dst, n16, (unsigned*)ctr, fpo);      \
         }, bytes));
  LDG_DF(8, 4, 8)
  LDG_DF(8, 8, 8)
  LDG_DF(8, 4, 4)
  LDG_DF(4, 8, 8)
  LDG_DF(16, 4, 4)
  TMA_W(16384)
  TMA_W(32768)
  TMA_W(65536)
  return 0;
}
