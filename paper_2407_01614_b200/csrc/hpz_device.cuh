// Device helpers shared by the sm_100a kernels (hpz_kernels.cu, hpz_tma.cu): the
// memory-model primitives of the cross-GPU flag protocol, bounded waits,
// grid completion, the fingerprint, and the R7 reduction / R8 Adam arithmetic that both
// copy engines must evaluate identically.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hpz_internal.h"

namespace hpz {
namespace {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Acquire one flag (>= target) with a timeout; returns false on timeout (and records it:
// device abort flag so later waits are skipped, host-mapped error word for the runtime).
__device__ __forceinline__ bool wait_geq(const uint32_t* flag, uint32_t target, const SyncCommon& s) {
  if (ld_acquire_sys(flag) >= target) return true;
  if (*(volatile uint32_t*)s.abort_flag) return false;
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while (ld_acquire_sys(flag) < target) {
    if ((++spins & 63u) == 0) {
      if (*(volatile uint32_t*)s.abort_flag) return false;
      if (globaltimer() - t0 > s.timeout_ns) {
        atomicAdd(s.timeouts, 1ull);
        atomicExch(s.abort_flag, 1u);
        *s.host_err = 1u;
        __threadfence_system();
        return false;
      }
    }
    __nanosleep(32);
  }
  return true;
}

__device__ __forceinline__ void wait_all(const WaitList& w, const SyncCommon& s) {
  for (int k = 0; k < w.n; ++k) wait_geq(w.ptr[k], w.target, s);
}

__device__ __forceinline__ void release_all(const ReleaseList& r) {
  for (int k = 0; k < r.n; ++k) st_release_sys(r.ptr[k], r.value);
}

// Last-CTA detection: returns true in thread 0 of the CTA that finishes last.  Every
// CTA's global stores are made visible at system scope before it is counted, so the
// last CTA may release flags that cover the whole grid's output.
__device__ __forceinline__ bool last_cta(uint32_t* ctr) {
  __syncthreads();
  bool last = false;
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t prev = atomicAdd(ctr, 1u);
    if (prev == gridDim.x - 1) {
      *ctr = 0u;   // reset for the next launch (ordered by the stream)
      __threadfence_system();
      last = true;
    }
  }
  return last;
}

// Order-independent 64-bit checksum contribution of one 16-byte word at global word
// index gi (a7).  Not cryptographic: it detects stale/garbage words; EXACT mode counts
// elements.
__device__ __forceinline__ uint64_t fp_word(uint32_t gi, const int4& w) {
  uint32_t h = (uint32_t)w.x * 0x85EBCA6Bu ^ (uint32_t)w.y * 0xC2B2AE35u ^ (uint32_t)w.z * 0x27D4EB2Fu ^
               (uint32_t)w.w * 0x165667B1u ^ gi * 0x9E3779B1u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  uint32_t h2 = h * 0x297A2D39u;
  h2 ^= h2 >> 16;
  return ((uint64_t)h2 << 32) | h;
}

__device__ __forceinline__ float4 add4(const float4& a, const float4& b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// Fixed association (reading R7): adjacent rank pairs summed level by level, an odd
// last operand carried up — for P=8: ((G0+G1)+(G2+G3))+((G4+G5)+(G6+G7)).
template <int P>
__device__ __forceinline__ float4 pairwise_sum(float4 (&x)[P]) {
#pragma unroll
  for (int n = P; n > 1; n = (n + 1) / 2) {
#pragma unroll
    for (int k = 0; k < n / 2; ++k) x[k] = add4(x[2 * k], x[2 * k + 1]);
    if (n & 1) x[n / 2] = x[n - 1];
  }
  return x[0];
}

// One Adam element (reading R8), exactly the oracle's operation sequence: every
// operation is an explicit round-to-nearest intrinsic, so nothing is contracted to fma.
__device__ __forceinline__ void adam1(float& w, float& m, float& v, float g, const AdamParams& p) {
  m = __fadd_rn(__fmul_rn(p.beta1, m), __fmul_rn(p.omb1, g));
  v = __fadd_rn(__fmul_rn(p.beta2, v), __fmul_rn(__fmul_rn(p.omb2, g), g));
  const float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), p.bc2_sqrt), p.eps);
  if (p.lr_wd != 0.0f) w = __fsub_rn(w, __fmul_rn(p.lr_wd, w));
  w = __fsub_rn(w, __fmul_rn(p.step_size, __fdiv_rn(m, d)));
}

// Blockwise quantization code round-half-even((v - mn) / scale) clamped to [0, maxc] —
// bit-identical to the IEEE quotient the oracle rounds (R26, R28) but without a division
// per element: q1 = (v - mn) * RN(1/scale) differs from RN((v - mn)/scale) by less than
// 1.5 * 2^-23 * q <= 2^-14.4 for q <= 255, so unless q1 lies within `tie_eps` (2^-17 for
// 4-bit, 2^-13 for 8-bit codes) of a half-integer both round to the same integer; near a
// tie (or for NaN / inf) the exact quotient is computed.  Caller guarantees scale > 0.
__device__ __forceinline__ int quant_code(float v, float mn, float scale, float rcp, int maxc, float tie_eps) {
  const float a = __fsub_rn(v, mn);
  float q = __fmul_rn(a, rcp);
  const float fr = __fsub_rn(q, floorf(q));
  if (!(fabsf(__fsub_rn(fr, 0.5f)) >= tie_eps)) q = __fdiv_rn(a, scale);
  int c = __float2int_rn(q);
  return c < 0 ? 0 : (c > maxc ? maxc : c);
}

// quant_code for N elements of one block at once, same results element by element: the
// fast quotient for all N, one (rarely taken) branch that recomputes the elements near a
// tie with the IEEE division — instead of a divergent branch per element, which measured
// ~38 issued instructions per element in the qgZ quantizer (ncu: issue-bound at 77%).
template <int N>
__device__ __forceinline__ void quant_codes(const float (&e)[N], float mn, float scale, float rcp, int maxc,
                                            float tie_eps, int (&c)[N]) {
  float q[N];
  bool near = false;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    q[k] = __fmul_rn(__fsub_rn(e[k], mn), rcp);
    const float fr = __fsub_rn(q[k], floorf(q[k]));
    near |= !(fabsf(__fsub_rn(fr, 0.5f)) >= tie_eps);
  }
  if (near) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const float fr = __fsub_rn(q[k], floorf(q[k]));
      if (!(fabsf(__fsub_rn(fr, 0.5f)) >= tie_eps)) q[k] = __fdiv_rn(__fsub_rn(e[k], mn), scale);
    }
  }
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const int ci = __float2int_rn(q[k]);
    c[k] = ci < 0 ? 0 : (ci > maxc ? maxc : ci);
  }
}

}  // namespace
}  // namespace hpz
