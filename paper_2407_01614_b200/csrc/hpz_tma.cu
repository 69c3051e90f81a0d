// TMA (cp.async.bulk) pipelines of the hpZ hot path for sm_100a.
//
// One persistent CTA per SM.  A single elected producer thread streams chunks of the
// sources (peer arenas over NVLink, or local HBM) into a ring of shared-memory stages
// with 1-D bulk copies completing on mbarriers; the data never passes through
// registers unless it must be computed on:
//   * gather_tma_kernel: producer bulk-loads a 32 KiB chunk of source j, then bulk-stores
//     the same smem stage to the full buffer and (fused secondary store, a2) to the
//     secondary; optional fingerprint consumer warps read the stage (a7).
//   * rs_tma_kernel<P, ADAM, MODE>: producer bulk-loads the P peers' gradient slices of a
//     chunk (fp32 / bf16 / qgZ codes; + the master/m/v chunk when ADAM); up to 512
//     consumer threads sum in the fixed pairwise-by-rank order (R7) and apply Adam (R8)
//     from smem, storing with STG.128.
//   * qgz_quantize_kernel / qwz_quantize_kernel / gather_qwz_kernel: the ZeRO++ qgZ / qwZ
//     blockwise quantizers and the dequantizing forward gather (f1, f2).
// Flags are acquired by the producer before the first bulk read of a source; a
// fence.proxy.async orders the generic-proxy acquire before the async-proxy reads, and
// the bulk stores are drained (wait_group 0) and proxy-fenced before the grid-wide
// release.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "hpz_device.cuh"
#include "hpz_internal.h"

namespace hpz {

namespace {

#ifndef HPZ_GATHER_STAGES
#define HPZ_GATHER_STAGES 3
#endif
#ifndef HPZ_GATHER_CHUNK
#define HPZ_GATHER_CHUNK 32768
#endif
// Gather stage geometry, two instantiations: sources over NVLink pull 32 KiB chunks through
// 3 stages (96 KiB in flight per SM: at N = 4 the gathers reach 0.81 of 770 GB/s vs 0.79
// with 4 stages and 0.74 with 2; N = 2 equal; r02_ab_remote_gather.jsonl); a single local
// source (P = 1, or P' = 1 backward) is a device-local copy and streams 16 KiB chunks
// through 8 stages (measured at N = 1: fwd / bwd gathers at 0.91 of the HBM copy peak vs
// 0.85-0.87 with 32 KiB; at N = 4 the 16 KiB geometry loses 2-5% on NVLink pulls, 8 KiB
// loses 10-20% everywhere).
constexpr int kGatherChunk = HPZ_GATHER_CHUNK;   // bytes per gather stage (remote sources)
constexpr int kGatherStages = HPZ_GATHER_STAGES;
#ifndef HPZ_GATHER_LOCAL_CHUNK
#define HPZ_GATHER_LOCAL_CHUNK 16384
#endif
#ifndef HPZ_GATHER_LOCAL_STAGES
#define HPZ_GATHER_LOCAL_STAGES 8
#endif
constexpr int kGatherChunkLocal = HPZ_GATHER_LOCAL_CHUNK;
constexpr int kGatherStagesLocal = HPZ_GATHER_LOCAL_STAGES;
constexpr int kFpWarps = 4;             // fingerprint consumer warps
constexpr int kRsChunk = 1024;          // base shard elements per RS stage
#ifndef HPZ_RS_P1_MUL
#define HPZ_RS_P1_MUL 1                 // P = 1 (local, HBM-bound) chunk multiplier (A/B builds)
#endif
#ifndef HPZ_RS_PN_MUL
#define HPZ_RS_PN_MUL 2                 // 2 <= P <= 8 chunk multiplier (A/B builds)
#endif
#ifndef HPZ_RS_BUDGET_KB
#define HPZ_RS_BUDGET_KB 224            // shared-memory stage budget per CTA (4 stages at P = 4 under the budget alone; fp32 RS is capped, HPZ_RS_STAGES_P4PLUS)
                                        // (0.820 vs 0.814 of 770 GB/s with 200 KiB, N=4 A/B)
#endif
#ifndef HPZ_RS_MAX_STAGES
#define HPZ_RS_MAX_STAGES 6
#endif
#ifndef HPZ_RS_STAGES_P4PLUS
#define HPZ_RS_STAGES_P4PLUS 2          // stage cap for P >= 4 (0 = none): less peer data in flight per
                                        // SM measured faster in the all-to-all (P=4: 2 stages 1.2%
                                        // faster than 4; r02_ab_rs_stages.jsonl); P = 8 fits 2 anyway
#endif
#ifndef HPZ_GATHER_ROTATE
#define HPZ_GATHER_ROTATE 0             // 1: rotate each gather CTA through the sources (chunk_of);
                                        // measured slower (local copies -23%, N=4 bwd -1%), kept off
#endif
#ifndef HPZ_RS_ROTATE
#define HPZ_RS_ROTATE 1                 // rotate the order of the P slice loads per CTA and chunk
                                        // (N=4 RS+Adam 0.817 vs 0.799-0.811 of 770 GB/s; N=2 equal)
#endif
#ifndef HPZ_RS_WMV_LDG
#define HPZ_RS_WMV_LDG 0                // P >= 2: consumers load master/m/v with LDG (prefetched
#endif                                  // one chunk ahead) so the smem ring holds only peer data
constexpr int kRsMaxConsumers = 512;    // up to 16 consumer warps (one float4 each per chunk)

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done;
}
// Consumer-side wait: a bare try_wait loop.  Measured (A/B on one B200, N=1 fused RS+Adam):
// adding an iteration bound or a clock check to this loop costs 12-14% of the kernel.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
// Cold path, out of line.
__device__ __noinline__ void mbar_timeout(const SyncCommon& sc) {
  atomicAdd(sc.timeouts, 1ull);
  atomicExch(sc.abort_flag, 1u);
  *sc.host_err = 1u;
  __threadfence_system();
}
// Producer-side wait (one thread per CTA): bounded, so a pipeline that stops draining
// records a timeout (HPZ_ETIMEOUT on the next call) after ~2^26 tries instead of spinning
// forever.  Consumers only ever wait for stages the producer has issued, and every issued
// bulk copy completes (or faults the kernel), so the producer is the one place a lost
// dependency can stall.
__device__ __forceinline__ bool mbar_wait_bounded(uint64_t* bar, uint32_t parity, const SyncCommon& sc) {
  uint32_t spins = 0;
  while (!mbar_try(bar, parity)) {
    if (++spins == (1u << 26)) {
      mbar_timeout(sc);
      return false;
    }
  }
  return true;
}
__device__ __forceinline__ void tma_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// Programmatic dependent launch (sm_90+), OFF unless built with -DHPZ_PDL: a kernel
// launched with programmatic stream serialization may start while the previous kernel of
// the stream drains, and must `griddep_wait` before touching memory that kernel produced
// (everything else our kernels read from a previous kernel is ordered by flags).  Measured
// on B200 without per-call events: N=1 step 50.0 ms with PDL vs 44.6 ms without, N=2 37.6 vs
// 37.3 ms — the early-launched CTAs cost more than the drained tails save.
__device__ __forceinline__ void griddep_wait() {
#ifdef HPZ_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void griddep_launch_dependents() {
#ifdef HPZ_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ------------------------------------------------------------------ gather (a2, a4)
// Block = 1 producer warp (+ kFpWarps fingerprint warps when FP).  Dynamic smem =
// kGatherStages * kGatherChunk bytes.
template <bool FP, int kGatherChunk, int kGatherStages>
__global__ void __launch_bounds__(32 * (1 + kFpWarps), 1)
    gather_tma_kernel(const __grid_constant__ GatherParams p) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full_bar[kGatherStages];
  __shared__ __align__(8) uint64_t empty_bar[kGatherStages];
  __shared__ unsigned long long fp_red[kFpWarps];

  const int n_src = p.n_src;
  const int64_t chunks_per_src = (p.src_bytes + kGatherChunk - 1) / kGatherChunk;
  const int64_t total = chunks_per_src * n_src;
  // HPZ_GATHER_ROTATE: round k hands CTA b item k*G + (b + k) % G (a permutation inside each
  // round of G items), so every CTA rotates through the sources instead of pinning one
  // (G % n_src == 0 would give CTA b source b % n_src for good: the CTAs of the local source
  // finish early and the NVLink pulls run on the rest of the SMs).
  const int64_t G = gridDim.x;
  const int64_t nk = HPZ_GATHER_ROTATE
      ? total / G + (((int64_t)blockIdx.x + total / G) % G < total % G ? 1 : 0)
      : (blockIdx.x < total ? (total - blockIdx.x + G - 1) / G : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGatherStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kFpWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  auto chunk_of = [&](int64_t k, int& j, int64_t& off, uint32_t& bytes) {
    const int64_t w = HPZ_GATHER_ROTATE ? k * G + ((int64_t)blockIdx.x + k) % G : blockIdx.x + k * G;
    j = (int)(w % n_src);
    off = (w / n_src) * kGatherChunk;
    const int64_t rem = p.src_bytes - off;
    bytes = (uint32_t)(rem < kGatherChunk ? rem : kGatherChunk);
  };

  if (warp == 0) {
    if (lane == 0) {
      uint32_t waited = 0;
      bool war_done = false;
      const uint32_t src_target = layer_epoch(p.src_target, p.sync);
      auto issue_load = [&](int64_t k) {
        int j;
        int64_t off;
        uint32_t bytes;
        chunk_of(k, j, off, bytes);
        if (!((waited >> j) & 1u)) {
          if (p.src_flag[j] != nullptr) wait_geq(p.src_flag[j], src_target, p.sync);   // E1 / E3
          fence_proxy_async();
          waited |= 1u << j;
        }
        const int s = (int)(k % kGatherStages);
        mbar_expect_tx(&full_bar[s], bytes);
        tma_load(smem + (size_t)s * kGatherChunk, p.src[j] + off, bytes, &full_bar[s]);
      };
      const int64_t pre = nk < kGatherStages - 1 ? nk : kGatherStages - 1;
      for (int64_t k = 0; k < pre; ++k) issue_load(k);
      griddep_wait();   // the previous kernel of the stream may still write `out` / the secondary
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % kGatherStages);
        mbar_wait(&full_bar[s], (uint32_t)((k / kGatherStages) & 1));   // issued bulk loads always land
        int j;
        int64_t off;
        uint32_t bytes;
        chunk_of(k, j, off, bytes);
        const char* stage = smem + (size_t)s * kGatherChunk;
        tma_store(p.out + (int64_t)j * p.src_bytes + off, stage, bytes);
        if (p.sec != nullptr && j >= p.sec_lo && j < p.sec_hi) {
          if (!war_done) {
            wait_all(p.war, p.sync);   // E4: node peers' backward reads of step t-1 are done
            fence_proxy_async();
            war_done = true;
          }
          tma_store(p.sec + (int64_t)(j - p.sec_lo) * p.src_bytes + off, stage, bytes);
        }
        bulk_commit();
        if (k + kGatherStages - 1 < nk) {
          // the stage of chunk k-1 is refilled: its stores must have read it ...
          bulk_wait_read<1>();
          // ... and the fingerprint warps must be done with it
          if (FP && k >= 1) mbar_wait_bounded(&empty_bar[(k - 1) % kGatherStages], (uint32_t)(((k - 1) / kGatherStages) & 1), p.sync);
          issue_load(k + kGatherStages - 1);
        }
      }
      griddep_launch_dependents();   // every load and store of this CTA is issued
      bulk_wait_all();       // all bulk stores performed
      fence_proxy_async();   // ... and ordered before the generic-proxy release below
    }
  } else if (FP) {
    // fingerprint consumers: order-independent checksum of every 16-byte word
    uint64_t fp = 0;
    const int ct = threadIdx.x - 32;
    for (int64_t k = 0; k < nk; ++k) {
      const int s = (int)(k % kGatherStages);
      mbar_wait(&full_bar[s], (uint32_t)((k / kGatherStages) & 1));
      int j;
      int64_t off;
      uint32_t bytes;
      chunk_of(k, j, off, bytes);
      const int4* st = reinterpret_cast<const int4*>(smem + (size_t)s * kGatherChunk);
      const int64_t gv0 = ((int64_t)j * p.src_bytes + off) >> 4;
      for (uint32_t v = ct; v < bytes / 16; v += 32 * kFpWarps) fp += fp_word((uint32_t)(gv0 + v), st[v]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fp += __shfl_xor_sync(0xffffffffu, fp, o);
    if (lane == 0) fp_red[warp - 1] = fp;
  }
  __syncthreads();
  if (FP && threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < kFpWarps; ++w) s += fp_red[w];
    if (s) atomicAdd(p.fp_acc + 2 * ((p.fp_par + epoch_base(p.sync)) & 1u), s);
  }
  if (last_cta(p.done_ctr)) gather_finish(p);
}

// ------------------------------------------------------------------ RS (+ Adam) (a5, a6)
enum RsMode { RS_F32 = 0, RS_BF16 = 1, RS_QGZ = 2 };

template <int P, bool ADAM, int MODE, bool FP = false>
struct RsCfg {
  static constexpr bool QGZ = MODE == RS_QGZ;
  // per stage: P gradient slices (fp32, or qgZ int4 codes + (min, scale) per 64) (+ w, m, v);
  // qgZ chunks are longer so its small code/param copies stay >= 1 KiB / 256 B
  // P=1 (local, HBM-bound): 1024-element chunks keep 6 stages in flight; 2 <= P <= 8: 2048
  static constexpr int kChunk = (P >= 2 && P <= 8 ? HPZ_RS_PN_MUL : (P == 1 ? HPZ_RS_P1_MUL : 1)) * (QGZ ? 2 * kRsChunk : kRsChunk);
  static constexpr int kGradBytes = MODE == RS_BF16 ? 2 : 4;
  static constexpr int kCodeBytes = kChunk / 2;
  static constexpr int kParamBytes = kChunk / kQgzBlock * 8;
  static constexpr int kSrcBytes = QGZ ? kCodeBytes + kParamBytes : kChunk * kGradBytes;
  static constexpr int kWmvOff = P * kSrcBytes;
  static constexpr bool kWmvLdg = ADAM && HPZ_RS_WMV_LDG && P >= 2 && kChunk / 4 <= kRsMaxConsumers;
  static constexpr int kPrimOff = kWmvOff + (ADAM && !kWmvLdg ? 3 * kChunk * 4 : 0);
  static constexpr int kStageBytes = kPrimOff;
  static constexpr int kBudget = HPZ_RS_BUDGET_KB * 1024;
  static constexpr int kFit = kBudget / kStageBytes;
  // the P >= 4 cap was measured on the fp32 RS only: qgZ / bf16 gradients keep the budget rule
  static constexpr int kMax = (P >= 4 && MODE == RS_F32 && HPZ_RS_STAGES_P4PLUS > 0) ? HPZ_RS_STAGES_P4PLUS
                                                                                 : HPZ_RS_MAX_STAGES;
  static constexpr int kStages = kFit >= kMax ? kMax : (kFit < 2 ? 2 : kFit);
  // consumer threads: one float4 per thread per chunk, at most 16 warps (idle polling
  // warps would steal issue slots from the working ones)
  static constexpr int kConsumers = kChunk / 4 < kRsMaxConsumers ? kChunk / 4 : kRsMaxConsumers;
  static constexpr int kLead = 32;   // producer warp
  static constexpr int kThreads = kLead + kConsumers;
};

// Block = 1 producer warp + consumer warps.  Dynamic smem = kStages * kStageBytes.
// FP (with ADAM): the consumers also fingerprint the primary words they write (a7, E1/E2;
// a few integer ops per thread, prim_word_fp).  A separate instantiation, so the plain
// kernel keeps its code.  (Measured: a dedicated fingerprint warp fed through smem was
// slower — this kernel's time tracks the consumers' instruction stream, and a polling warp
// steals their issue slots.)
template <int P, bool ADAM, int MODE, bool FP>
__global__ void __launch_bounds__(RsCfg<P, ADAM, MODE, FP>::kThreads, 1)
    rs_tma_kernel(const __grid_constant__ RSParams r, const __grid_constant__ AdamParams a) {
  using C = RsCfg<P, ADAM, MODE, FP>;
  static_assert(ADAM || !FP, "fingerprints are emitted by the optimizer");
  constexpr bool QGZ = C::QGZ;
  constexpr bool BF16 = MODE == RS_BF16;
  static_assert(C::kStages >= 2, "stage ring too small");
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full_bar[C::kStages];
  __shared__ __align__(8) uint64_t empty_bar[C::kStages];
  uint64_t fp = 0;                 // FP consumers: fingerprint of the primary words written
  const int64_t n = r.n_vec * 4;   // shard elements (multiple of 256)
  const int64_t total = (n + C::kChunk - 1) / C::kChunk;
  const int64_t nk = blockIdx.x < total ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    griddep_wait();                      // the caller's gradient writes (previous kernel) are done
    if (r.ready.n) {
      __threadfence_system();
      release_all(r.ready, r.sync);      // E5
    }
    wait_all(r.ready_wait, r.sync);      // E5: every rank's gradient slot is written
    if (ADAM) wait_all(a.wait, a.sync);  // E2 (+E7): nobody still reads my primary
    fence_proxy_async();
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], C::kConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % C::kStages);
        if (k >= C::kStages) mbar_wait_bounded(&empty_bar[s], (uint32_t)(((k / C::kStages) - 1) & 1), r.sync);
        const int64_t e0 = (blockIdx.x + k * gridDim.x) * (int64_t)C::kChunk;
        const int64_t rem = n - e0;
        const uint32_t cnt = (uint32_t)(rem < C::kChunk ? rem : C::kChunk);
        const uint32_t bytes = cnt * 4;
        char* st = smem + (size_t)s * C::kStageBytes;
        const uint32_t src_bytes = QGZ ? cnt / 2 + cnt / kQgzBlock * 8 : (BF16 ? cnt * 2 : bytes);
        mbar_expect_tx(&full_bar[s], src_bytes * P + (ADAM && !C::kWmvLdg ? 3 * bytes : 0));
#pragma unroll
        for (int jj = 0; jj < P; ++jj) {
          // HPZ_RS_ROTATE: each CTA starts its chunk's loads at a different source rank
          const int j = HPZ_RS_ROTATE ? (int)((jj + blockIdx.x + k) % P) : jj;
          char* dst = st + j * C::kSrcBytes;
          if (QGZ) {
            tma_load(dst, r.qcodes[j] + e0 / 2, cnt / 2, &full_bar[s]);
            tma_load(dst + C::kCodeBytes, r.qparams[j] + e0 / kQgzBlock, cnt / kQgzBlock * 8, &full_bar[s]);
          } else if (BF16) {
            tma_load(dst, reinterpret_cast<const __nv_bfloat16*>(r.src[j]) + e0, cnt * 2, &full_bar[s]);
          } else {
            tma_load(dst, r.src[j] + e0, bytes, &full_bar[s]);
          }
        }
        if (ADAM && !C::kWmvLdg) {
          float* wmv = reinterpret_cast<float*>(st + C::kWmvOff);
          tma_load(wmv + 0 * C::kChunk, a.w + e0, bytes, &full_bar[s]);
          tma_load(wmv + 1 * C::kChunk, a.m + e0, bytes, &full_bar[s]);
          tma_load(wmv + 2 * C::kChunk, a.v + e0, bytes, &full_bar[s]);
        }
      }
      griddep_launch_dependents();
    }
  } else {
    const float4 sc = ADAM ? adam_scalars(a) : make_float4(0.f, 0.f, 0.f, 0.f);
    // kWmvLdg: this thread's master/m/v float4s of the next chunk, loaded one chunk ahead
    float4 nw = make_float4(0.f, 0.f, 0.f, 0.f), nm = nw, nv = nw;
    auto load_wmv = [&](int64_t kk) {
      const int64_t e0k = (blockIdx.x + kk * gridDim.x) * (int64_t)C::kChunk;
      const int ct0 = threadIdx.x - C::kLead;
      if (e0k + ct0 * 4 < n) {
        const int64_t ii = e0k / 4 + ct0;
        nw = __ldcs(reinterpret_cast<const float4*>(a.w) + ii);
        nm = __ldcs(reinterpret_cast<const float4*>(a.m) + ii);
        nv = __ldcs(reinterpret_cast<const float4*>(a.v) + ii);
      }
    };
    static_assert(!C::kWmvLdg || C::kConsumers * 4 == C::kChunk, "LDG master/m/v: one float4 per consumer");
    if constexpr (C::kWmvLdg) if (nk > 0) load_wmv(0);
    for (int64_t k = 0; k < nk; ++k) {
      const int s = (int)(k % C::kStages);
      mbar_wait(&full_bar[s], (uint32_t)((k / C::kStages) & 1));
      const int64_t e0 = (blockIdx.x + k * gridDim.x) * (int64_t)C::kChunk;
      const int64_t rem = n - e0;
      const int cnt = (int)(rem < C::kChunk ? rem : C::kChunk);
      const char* stc = smem + (size_t)s * C::kStageBytes;
      const float4* wmv = reinterpret_cast<const float4*>(stc + C::kWmvOff);
      float4 cw = nw, cm = nm, cv = nv;   // kWmvLdg: this chunk's master/m/v
      if constexpr (C::kWmvLdg) if (k + 1 < nk) load_wmv(k + 1);
      // one float4 `ct` of the chunk: fixed-order sum (R7) of the P slices, then Adam (R8);
      // w / pk: the new master and bf16 primary (for the fingerprint)
      auto process = [&](const int ct, float4& w, uint2& pk) {
        const int64_t i = e0 / 4 + ct;   // float4 index in the shard
        float4 x[P];
#pragma unroll
        for (int j = 0; j < P; ++j) {
          const char* sj = stc + j * C::kSrcBytes;
          if (QGZ) {
            // dequantize 4 elements: v = min_b + code * scale_b (multiply, then add)
            const uint32_t c2 = reinterpret_cast<const uint16_t*>(sj)[ct];
            const float2 ms = reinterpret_cast<const float2*>(sj + C::kCodeBytes)[ct * 4 / kQgzBlock];
            x[j].x = __fadd_rn(ms.x, __fmul_rn((float)(c2 & 15u), ms.y));
            x[j].y = __fadd_rn(ms.x, __fmul_rn((float)((c2 >> 4) & 15u), ms.y));
            x[j].z = __fadd_rn(ms.x, __fmul_rn((float)((c2 >> 8) & 15u), ms.y));
            x[j].w = __fadd_rn(ms.x, __fmul_rn((float)((c2 >> 12) & 15u), ms.y));
          } else if (BF16) {
            // bf16 -> fp32 is exact; the reduction itself stays fp32
            const uint2 b = reinterpret_cast<const uint2*>(sj)[ct];
            x[j] = make_float4(__uint_as_float(b.x << 16), __uint_as_float(b.x & 0xFFFF0000u),
                               __uint_as_float(b.y << 16), __uint_as_float(b.y & 0xFFFF0000u));
          } else {
            x[j] = reinterpret_cast<const float4*>(sj)[ct];
          }
        }
        float4 g = pairwise_sum<P>(x);
        g.x = __fmul_rn(g.x, r.inv_p);
        g.y = __fmul_rn(g.y, r.inv_p);
        g.z = __fmul_rn(g.z, r.inv_p);
        g.w = __fmul_rn(g.w, r.inv_p);
        if (r.out) reinterpret_cast<float4*>(r.out)[i] = g;
        if (ADAM) {
          float4 m, v;
          if constexpr (C::kWmvLdg) {
            w = cw;
            m = cm;
            v = cv;
          } else {
            w = wmv[0 * (C::kChunk / 4) + ct];
            m = wmv[1 * (C::kChunk / 4) + ct];
            v = wmv[2 * (C::kChunk / 4) + ct];
          }
          adam1(w.x, m.x, v.x, g.x, a, sc);
          adam1(w.y, m.y, v.y, g.y, a, sc);
          adam1(w.z, m.z, v.z, g.z, a, sc);
          adam1(w.w, m.w, v.w, g.w, a, sc);
          reinterpret_cast<float4*>(a.w)[i] = w;
          reinterpret_cast<float4*>(a.m)[i] = m;
          reinterpret_cast<float4*>(a.v)[i] = v;
          if (a.prim_bf16) {
            pk = pack_bf16x4(w);
            reinterpret_cast<uint2*>(a.prim)[i] = pk;
          } else {
            reinterpret_cast<float4*>(a.prim)[i] = w;
          }
          if constexpr (FP) prim_word_fp(fp, a.prim_bf16, i, w, pk, a.fpe.word_base);
        }
      };
      // consumer thread ct handles float4 ct of the chunk (and ct + kConsumers, ... when the
      // chunk holds more float4s than there are consumers).  The single-pass form is a
      // separate branch: compiled as a loop it measured ~13% slower.
      float4 w;
      uint2 pk;
      if constexpr (C::kConsumers * 4 == C::kChunk) {
        const int ct = threadIdx.x - C::kLead;
        if (ct * 4 < cnt) process(ct, w, pk);
      } else {
        for (int ct = threadIdx.x - C::kLead; ct * 4 < cnt; ct += C::kConsumers) process(ct, w, pk);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
  }
  if constexpr (FP) emit_fp(fp, a.fpe, a.sync);
  if (last_cta(r.done_ctr)) {
    release_all(r.rel, r.sync);             // E6
    if (ADAM) release_all(a.rel, a.sync);   // E1 (t+1)
  }
}

// Launch with programmatic stream serialization (PDL): the kernel may begin while the
// previous kernel in the stream finishes its tail.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, int smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
#ifdef HPZ_PDL
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#else
  (void)attr;
  cfg.numAttrs = 0;
#endif
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Opt a kernel into `smem` bytes of dynamic shared memory on the CURRENT device (the
// attribute is per device: a process that drives several GPUs sets it once on each).
template <auto Kernel>
cudaError_t set_smem_attr(int smem) {
  constexpr int kMaxDev = 64;
  static bool done[kMaxDev] = {};   // one flag array per kernel (template argument)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < kMaxDev && done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess && dev >= 0 && dev < kMaxDev) done[dev] = true;
  return e;
}

template <int P, bool ADAM, int MODE, bool FP = false>
cudaError_t launch_rs_tma_t(const RSParams& r, const AdamParams& a, int grid, cudaStream_t s) {
  using C = RsCfg<P, ADAM, MODE, FP>;
  const int smem = C::kStages * C::kStageBytes;
  cudaError_t e = set_smem_attr<rs_tma_kernel<P, ADAM, MODE, FP>>(smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(rs_tma_kernel<P, ADAM, MODE, FP>, grid, C::kThreads, smem, s, r, a);
}

template <int P, int MODE>
cudaError_t launch_rs_adam_tma(const RSParams& r, const AdamParams& a, int grid, cudaStream_t s) {
  return a.fpe.n_dst > 0 ? launch_rs_tma_t<P, true, MODE, true>(r, a, grid, s)
                         : launch_rs_tma_t<P, true, MODE, false>(r, a, grid, s);
}

// qgZ quantizer: 4 threads per 64-element block, each holding 4 float4s (elements
// 4*(q + 4u) .. +3 of the block, q = lane % 4, u = 0..3) so a warp-wide 16-byte load
// touches 64 contiguous bytes of 8 blocks; block min/max take 2 shuffle levels.  NaN
// anywhere in a block makes its (min, scale) NaN so it surfaces after dequantization.
// fp32, one IEEE op per operator, round-half-even codes — the oracle's
// quantize_blockwise decisions, bit for bit.
__global__ void __launch_bounds__(256, 4) qgz_quantize_kernel(const __grid_constant__ QuantParams q) {
  if (threadIdx.x == 0 && q.war.n) wait_all(q.war, q.sync);   // E6: peers done with the old codes
  __syncthreads();
  const int64_t n_blocks = q.n / kQgzBlock;
  const int sub = threadIdx.x & 3;
  const int64_t grp = (int64_t)blockIdx.x * (blockDim.x / 4) + (threadIdx.x >> 2);   // 4-thread group id
  const int64_t n_grp = (int64_t)gridDim.x * (blockDim.x / 4);
  const float4* g4 = reinterpret_cast<const float4*>(q.g);
  uint16_t* c16 = reinterpret_cast<uint16_t*>(q.codes);
  for (int64_t b = grp; b < n_blocks; b += n_grp) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = g4[b * 16 + sub + 4 * u];
    int nan = 0;
    float mn = v[0].x, mx = v[0].x;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      nan |= isnan(v[u].x) | isnan(v[u].y) | isnan(v[u].z) | isnan(v[u].w);
      mn = fminf(mn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
      mx = fmaxf(mx, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
    }
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      nan |= __shfl_xor_sync(0xffffffffu, nan, o);
    }
    float scale = __fdiv_rn(__fsub_rn(mx, mn), 15.0f);
    if (nan) {
      mn = __int_as_float(0x7fc00000);
      scale = mn;
    }
    const bool pos = scale > 0.0f;
    const float rcp = pos ? __frcp_rn(scale) : 0.0f;
    const float e[16] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w,
                         v[2].x, v[2].y, v[2].z, v[2].w, v[3].x, v[3].y, v[3].z, v[3].w};
    int c[16];
    if (pos) {
      quant_codes<16>(e, mn, scale, rcp, 15, 0x1p-17f, c);
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) c[k] = 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      c16[b * 16 + sub + 4 * u] =
          (uint16_t)(c[4 * u] | (c[4 * u + 1] << 4) | (c[4 * u + 2] << 8) | (c[4 * u + 3] << 12));
    if (sub == 0) q.params[b] = make_float2(mn, scale);
  }
}

// ------------------------------------------------------------------ qwZ (f2)
// One warp per 256-element block of the owner's primary shard: each lane converts 8
// elements to fp32, the warp reduces min/max/NaN, and the block's codes are
// round-half-even((v - min) / scale) with scale = (max - min) / 255 — the oracle's
// quantize_blockwise(bits=8, block=256), bit for bit.  The last CTA releases E1.
__global__ void __launch_bounds__(256, 4) qwz_quantize_kernel(const __grid_constant__ QwzQuantParams q) {
  constexpr int U = 4;   // blocks per warp step: their loads are all in flight before any is used
  const int lane = threadIdx.x & 31;
  const int64_t n_blocks = q.n / kQwzBlock;
  const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x / 32);
  const bool emit = q.fpe.n_dst > 0;
  uint64_t fp = 0;
  for (int64_t b0 = warp_id * U; b0 < n_blocks; b0 += n_warps * U) {
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t b = b0 + u;
      if (b >= n_blocks) break;
      if (q.prim_bf16) {
        const uint4 w = reinterpret_cast<const uint4*>(q.prim)[b * 32 + lane];
        const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[u][2 * k] = __uint_as_float(x[k] << 16);
          v[u][2 * k + 1] = __uint_as_float(x[k] & 0xFFFF0000u);
        }
      } else {
        const float4 a = reinterpret_cast<const float4*>(q.prim)[(b * 32 + lane) * 2];
        const float4 c = reinterpret_cast<const float4*>(q.prim)[(b * 32 + lane) * 2 + 1];
        v[u][0] = a.x; v[u][1] = a.y; v[u][2] = a.z; v[u][3] = a.w;
        v[u][4] = c.x; v[u][5] = c.y; v[u][6] = c.z; v[u][7] = c.w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t b = b0 + u;
      if (b >= n_blocks) break;
      int nan = 0;
      float mn = v[u][0], mx = v[u][0];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        nan |= isnan(v[u][k]);
        mn = fminf(mn, v[u][k]);
        mx = fmaxf(mx, v[u][k]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        nan |= __shfl_xor_sync(0xffffffffu, nan, o);
      }
      float scale = __fdiv_rn(__fsub_rn(mx, mn), 255.0f);
      if (nan) {
        mn = __int_as_float(0x7fc00000);
        scale = mn;
      }
      uint32_t lo = 0, hi = 0;
      const bool pos = scale > 0.0f;
      const float rcp = pos ? __frcp_rn(scale) : 0.0f;
      if (pos) {
        int c[8];
        quant_codes<8>(v[u], mn, scale, rcp, 255, 0x1p-13f, c);
        lo = (uint32_t)c[0] | ((uint32_t)c[1] << 8) | ((uint32_t)c[2] << 16) | ((uint32_t)c[3] << 24);
        hi = (uint32_t)c[4] | ((uint32_t)c[5] << 8) | ((uint32_t)c[6] << 16) | ((uint32_t)c[7] << 24);
      }
      reinterpret_cast<uint2*>(q.codes)[b * 32 + lane] = make_uint2(lo, hi);
      if (lane == 0) q.params[b] = make_float2(mn, scale);
      if (emit) {
        // the words the forward gather will produce from these codes: min + code * scale in
        // fp32, rounded to the parameter dtype (gather_qwz_kernel's arithmetic)
        float d[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t code = ((k < 4 ? lo : hi) >> (8 * (k & 3))) & 0xFFu;
          d[k] = __fadd_rn(mn, __fmul_rn((float)code, scale));
        }
        const int64_t e = b * kQwzBlock + lane * 8;   // shard element of d[0]
        if (q.prim_bf16) {
          const uint2 a = pack_bf16x4(make_float4(d[0], d[1], d[2], d[3]));
          const uint2 c = pack_bf16x4(make_float4(d[4], d[5], d[6], d[7]));
          fp += fp_word((uint32_t)(q.fpe.word_base + e / 8), make_int4((int)a.x, (int)a.y, (int)c.x, (int)c.y));
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            fp += fp_word((uint32_t)(q.fpe.word_base + e / 4 + h),
                          make_int4(__float_as_int(d[4 * h]), __float_as_int(d[4 * h + 1]),
                                    __float_as_int(d[4 * h + 2]), __float_as_int(d[4 * h + 3])));
        }
      }
    }
  }
  if (emit) emit_fp(fp, q.fpe, q.sync);
  if (last_cta(q.done_ctr)) release_all(q.rel, q.sync);   // E1: codes of step t+1 are ready
}

// qwZ forward gather: producer TMA-pulls 8192-element chunks of source j's codes (8 KiB)
// and (min, scale) pairs (256 B); 8 consumer warps dequantize 8 elements per thread-step
// (fp32 min + code*scale, then the parameter dtype), store 16-byte words to the full
// buffer and — fused secondary store — to the secondary, and fingerprint them.
#ifndef HPZ_QW_CHUNK
#define HPZ_QW_CHUNK 16384   // 16 KiB of codes x 4 stages, 16 consumer warps: fwd qwZ gather
#endif                       // 7.2 vs 7.6 ms/step (N=2) for 8 KiB / 8 warps
#ifndef HPZ_QW_STAGES
#define HPZ_QW_STAGES 4
#endif
#ifndef HPZ_QW_CONSUMERS
#define HPZ_QW_CONSUMERS 512
#endif
constexpr int kQwChunk = HPZ_QW_CHUNK;
constexpr int kQwStages = HPZ_QW_STAGES;
constexpr int kQwConsumers = HPZ_QW_CONSUMERS;
__global__ void __launch_bounds__(32 + kQwConsumers, 1) gather_qwz_kernel(const __grid_constant__ GatherParams p) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full_bar[kQwStages];
  __shared__ __align__(8) uint64_t empty_bar[kQwStages];
  __shared__ unsigned long long fp_red[kQwConsumers / 32];
  constexpr int kStage = kQwChunk + kQwChunk / kQwzBlock * 8;
  const int n_src = p.n_src;
  const int64_t n_el = p.src_bytes;                     // codes: 1 byte per element
  const int64_t chunks_per_src = (n_el + kQwChunk - 1) / kQwChunk;
  const int64_t total = chunks_per_src * n_src;
  const int64_t G = gridDim.x;   // HPZ_GATHER_ROTATE schedule: see gather_tma_kernel
  const int64_t nk = HPZ_GATHER_ROTATE
      ? total / G + (((int64_t)blockIdx.x + total / G) % G < total % G ? 1 : 0)
      : (blockIdx.x < total ? (total - blockIdx.x + G - 1) / G : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int eb = p.elem_bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQwStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kQwConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto chunk_of = [&](int64_t k, int& j, int64_t& off, uint32_t& cnt) {
    const int64_t w = HPZ_GATHER_ROTATE ? k * G + ((int64_t)blockIdx.x + k) % G : blockIdx.x + k * G;
    j = (int)(w % n_src);
    off = (w / n_src) * kQwChunk;
    const int64_t rem = n_el - off;
    cnt = (uint32_t)(rem < kQwChunk ? rem : kQwChunk);
  };
  if (warp == 0) {
    if (lane == 0) {
      uint32_t waited = 0;
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % kQwStages);
        if (k >= kQwStages) mbar_wait_bounded(&empty_bar[s], (uint32_t)(((k / kQwStages) - 1) & 1), p.sync);
        int j;
        int64_t off;
        uint32_t cnt;
        chunk_of(k, j, off, cnt);
        if (!((waited >> j) & 1u)) {
          if (p.src_flag[j] != nullptr) wait_geq(p.src_flag[j], layer_epoch(p.src_target, p.sync), p.sync);   // E1
          fence_proxy_async();
          waited |= 1u << j;
        }
        char* st = smem + (size_t)s * kStage;
        // bulk copies move multiples of 16 bytes: a one-block tail carries 8 bytes of
        // (min, scale) plus 8 padding bytes (inside the 4 KiB-aligned params buffer)
        const uint32_t pbytes = (cnt / kQwzBlock * 8 + 15) & ~15u;
        mbar_expect_tx(&full_bar[s], cnt + pbytes);
        tma_load(st, p.src[j] + off, cnt, &full_bar[s]);
        tma_load(st + kQwChunk, p.qw_params[j] + off / kQwzBlock, pbytes, &full_bar[s]);
      }
    }
  } else {
    uint64_t fp = 0;
    bool war_done = false;
    for (int64_t k = 0; k < nk; ++k) {
      const int s = (int)(k % kQwStages);
      mbar_wait(&full_bar[s], (uint32_t)((k / kQwStages) & 1));
      int j;
      int64_t off;
      uint32_t cnt;
      chunk_of(k, j, off, cnt);
      const bool to_sec = p.sec != nullptr && j >= p.sec_lo && j < p.sec_hi;
      if (to_sec && !war_done) {
        // E4 once per thread before its first secondary store (cheap local flag reads)
        wait_all(p.war, p.sync);
        war_done = true;
      }
      const char* st = smem + (size_t)s * kStage;
      const float2* prm = reinterpret_cast<const float2*>(st + kQwChunk);
      for (uint32_t e = (threadIdx.x - 32) * 8; e < cnt; e += kQwConsumers * 8) {
        const uint2 c = *reinterpret_cast<const uint2*>(st + e);
        const float2 ms = prm[e / kQwzBlock];
        float v[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
          const uint32_t code = ((k2 < 4 ? c.x : c.y) >> (8 * (k2 & 3))) & 0xFFu;
          v[k2] = __fadd_rn(ms.x, __fmul_rn((float)code, ms.y));
        }
        const int64_t ge = (int64_t)j * n_el + off + e;      // element index in the full buffer
        if (eb == 2) {
          uint4 w;
          uint32_t* wp = &w.x;
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * k2], v[2 * k2 + 1]);
            wp[k2] = *reinterpret_cast<uint32_t*>(&b2);
          }
          reinterpret_cast<uint4*>(p.out)[ge / 8] = w;
          if (to_sec) reinterpret_cast<uint4*>(p.sec)[((int64_t)(j - p.sec_lo) * n_el + off + e) / 8] = w;
          if (p.fp_acc) fp += fp_word((uint32_t)(ge / 8), *reinterpret_cast<int4*>(&w));
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 w = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
            reinterpret_cast<float4*>(p.out)[ge / 4 + h] = w;
            if (to_sec) reinterpret_cast<float4*>(p.sec)[((int64_t)(j - p.sec_lo) * n_el + off + e) / 4 + h] = w;
            if (p.fp_acc) fp += fp_word((uint32_t)(ge / 4 + h), *reinterpret_cast<const int4*>(&w));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fp += __shfl_xor_sync(0xffffffffu, fp, o);
    if (lane == 0) fp_red[warp - 1] = fp;
  }
  __syncthreads();
  if (p.fp_acc && threadIdx.x == 0) {
    unsigned long long sum = 0;
    for (int w = 0; w < kQwConsumers / 32; ++w) sum += fp_red[w];
    if (sum) atomicAdd(p.fp_acc + 2 * ((p.fp_par + epoch_base(p.sync)) & 1u), sum);
  }
  if (last_cta(p.done_ctr)) gather_finish(p);
}

}  // namespace

template <int CHUNK, int STAGES>
cudaError_t launch_gather_tma_t(const GatherParams& p, int grid, cudaStream_t s) {
  const int smem = STAGES * CHUNK;
  const bool fp = p.fp_acc != nullptr;
  cudaError_t e = fp ? set_smem_attr<gather_tma_kernel<true, CHUNK, STAGES>>(smem)
                     : set_smem_attr<gather_tma_kernel<false, CHUNK, STAGES>>(smem);
  if (e != cudaSuccess) return e;
  return fp ? launch_pdl(gather_tma_kernel<true, CHUNK, STAGES>, grid, 32 * (1 + kFpWarps), smem, s, p)
            : launch_pdl(gather_tma_kernel<false, CHUNK, STAGES>, grid, 32, smem, s, p);
}

cudaError_t launch_gather_tma(const GatherParams& p, int grid, cudaStream_t s) {
  // one source = this rank's own arena (P = 1, or the P' = 1 backward): a local copy
  return p.n_src == 1 ? launch_gather_tma_t<kGatherChunkLocal, kGatherStagesLocal>(p, grid, s)
                      : launch_gather_tma_t<kGatherChunk, kGatherStages>(p, grid, s);
}

cudaError_t launch_qwz_quantize(const QwzQuantParams& q, int grid, cudaStream_t s) {
  qwz_quantize_kernel<<<grid, 256, 0, s>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_gather_qwz(const GatherParams& p, int grid, cudaStream_t s) {
  constexpr int smem = kQwStages * (kQwChunk + kQwChunk / kQwzBlock * 8);
  cudaError_t e = set_smem_attr<gather_qwz_kernel>(smem);
  if (e != cudaSuccess) return e;
  gather_qwz_kernel<<<grid, 32 + kQwConsumers, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_qgz_quantize(const QuantParams& q, int grid, cudaStream_t s) {
  qgz_quantize_kernel<<<grid, 256, 0, s>>>(q);
  return cudaGetLastError();
}

template <int P>
cudaError_t launch_rs_tma_p(const RSParams& r, const AdamParams* a, int grid, cudaStream_t s, int mode) {
  AdamParams none{};
  switch (mode) {
    case RS_F32: return a ? launch_rs_adam_tma<P, RS_F32>(r, *a, grid, s) : launch_rs_tma_t<P, false, RS_F32>(r, none, grid, s);
    case RS_BF16: return a ? launch_rs_adam_tma<P, RS_BF16>(r, *a, grid, s) : launch_rs_tma_t<P, false, RS_BF16>(r, none, grid, s);
    case RS_QGZ: return a ? launch_rs_adam_tma<P, RS_QGZ>(r, *a, grid, s) : launch_rs_tma_t<P, false, RS_QGZ>(r, none, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rs_tma(const RSParams& r, const AdamParams* a, int world, int grid, cudaStream_t s, int mode) {
  switch (world) {
#define HPZ_RST_CASE(P) \
  case P: return launch_rs_tma_p<P>(r, a, grid, s, mode);
    HPZ_RST_CASE(1) HPZ_RST_CASE(2) HPZ_RST_CASE(3) HPZ_RST_CASE(4) HPZ_RST_CASE(5) HPZ_RST_CASE(6)
    HPZ_RST_CASE(7) HPZ_RST_CASE(8) HPZ_RST_CASE(9) HPZ_RST_CASE(10) HPZ_RST_CASE(11) HPZ_RST_CASE(12)
    HPZ_RST_CASE(13) HPZ_RST_CASE(14) HPZ_RST_CASE(15) HPZ_RST_CASE(16)
#undef HPZ_RST_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hpz
