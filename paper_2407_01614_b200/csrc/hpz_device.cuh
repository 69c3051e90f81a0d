// Device helpers shared by the sm_100a kernels (hpz_kernels.cu, hpz_tma.cu): the
// memory-model primitives of the cross-GPU flag protocol, bounded waits,
// grid completion, the fingerprint, and the R7 reduction / R8 Adam arithmetic that both
// copy engines must evaluate identically.
#pragma once
#include <cuda_bf16.h>
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
        if (s.timeout_info != nullptr &&
            atomicCAS(s.timeout_info, 0ull, (unsigned long long)(uintptr_t)flag) == 0ull)   // first timeout: which edge
          s.timeout_info[1] = ((unsigned long long)target << 32) | ld_acquire_sys(flag);
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

// The rank's device step counter (device-epoch mode) or 0 (host epochs are absolute).
// Written only by the epoch-advance kernel of the previous step's last call, so a plain
// load after kernel start sees it.
__device__ __forceinline__ uint32_t epoch_base(const SyncCommon& s) {
  return s.epoch ? *(const volatile uint32_t*)s.epoch : 0u;
}
// A layer-flag value (one use per step): relative value + epoch.
__device__ __forceinline__ uint32_t layer_epoch(uint32_t v, const SyncCommon& s) { return v + epoch_base(s); }

// mul 0 means 1 (a layer flag: one use per step).
__device__ __forceinline__ void wait_all(const WaitList& w, const SyncCommon& s) {
  const uint32_t target = w.target + (w.mul ? w.mul : 1u) * epoch_base(s);
  for (int k = 0; k < w.n; ++k) wait_geq(w.ptr[k], target, s);
}

__device__ __forceinline__ void release_all(const ReleaseList& r, const SyncCommon& s) {
  const uint32_t v = r.value + (r.mul ? r.mul : 1u) * epoch_base(s);
  for (int k = 0; k < r.n; ++k) st_release_sys(r.ptr[k], v);
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

// Fingerprint (a7): F(buffer) = sum over its 32-bit words x_q of x_q * M(q) mod 2^64, with
// q the word's index in the full parameter buffer and M(q) = (q * 0x9E3779B1) | 1, an odd
// position-dependent multiplier.  Additive, so CTAs, owners and gathers combine partial sums
// in any order; one IMAD + one wide IMAD per word, so the optimizer can emit it in registers
// almost for free.  It detects any single changed word exactly (an odd M(q) times a nonzero
// 32-bit difference is never 0 mod 2^64); a multi-word change escapes only if the weighted
// differences cancel mod 2^64 — a stale or garbage read does not do that by accident.  EXACT
// mode counts elements.
constexpr uint32_t kFpMul = 0x9E3779B1u;
// acc += x * (qm | 1) with qm = q * kFpMul, as ONE 32x32->64 multiply-add (mad.wide.u32)
__device__ __forceinline__ void fp_mad(uint64_t& acc, uint32_t qm, uint32_t x) {
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(x), "r"(qm | 1u));
}
__device__ __forceinline__ uint64_t fp_u32(uint32_t q, uint32_t x) {
  uint64_t acc = 0;
  fp_mad(acc, q * kFpMul, x);
  return acc;
}
// ... of one 16-byte word at 16-byte-word index gi (32-bit words 4gi .. 4gi+3)
__device__ __forceinline__ uint64_t fp_word(uint32_t gi, const int4& w) {
  const uint32_t qm = gi * (4u * kFpMul);
  uint64_t acc = 0;
  fp_mad(acc, qm, (uint32_t)w.x);
  fp_mad(acc, qm + kFpMul, (uint32_t)w.y);
  fp_mad(acc, qm + 2u * kFpMul, (uint32_t)w.z);
  fp_mad(acc, qm + 3u * kFpMul, (uint32_t)w.w);
  return acc;
}

// Fingerprint contribution of the primary elements a thread of an Adam kernel just wrote:
// float4 index i of the shard (bf16: the 8 bytes pk, 32-bit words 2i, 2i+1 of the shard;
// fp32: the 16 bytes w, words 4i .. 4i+3).  word_base = the shard's first 16-byte word in
// the full buffer.  Per thread, no cross-lane work.
__device__ __forceinline__ void prim_word_fp(uint64_t& acc, bool bf16, int64_t i, const float4& w, const uint2& pk,
                                             int64_t word_base) {
  if (bf16) {
    const uint32_t qm = (uint32_t)(word_base * 4 + 2 * i) * kFpMul;
    fp_mad(acc, qm, pk.x);
    fp_mad(acc, qm + kFpMul, pk.y);
  } else {
    const uint32_t qm = (uint32_t)(word_base * 4 + 4 * i) * kFpMul;
    fp_mad(acc, qm, __float_as_uint(w.x));
    fp_mad(acc, qm + kFpMul, __float_as_uint(w.y));
    fp_mad(acc, qm + 2u * kFpMul, __float_as_uint(w.z));
    fp_mad(acc, qm + 3u * kFpMul, __float_as_uint(w.w));
  }
}

// Block-wide sum of per-thread fingerprints, added (thread 0) into every reader's slot of
// the step parity.  Every thread of the block must call it.
__device__ __forceinline__ void emit_fp(uint64_t fp, const FpEmit& e, const SyncCommon& s) {
  __shared__ unsigned long long red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fp += __shfl_xor_sync(0xffffffffu, fp, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = fp;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < (int)((blockDim.x + 31) / 32); ++k) t += red[k];
    const int par = (int)((e.par + epoch_base(s)) & 1u);
    if (t)
      for (int q = 0; q < e.n_dst; ++q) atomicAdd(e.dst[q] + par, t);
  }
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

// The step's bias-corrected scalars (step_size = lr / (1 - beta1^t), bc2_sqrt =
// sqrt(1 - beta2^t)): host-computed for the call (host epochs), or looked up for the device
// step (device epochs) in the host-filled table.
// .x step_size, .y bc2_sqrt, .z RN(1 / bc2_sqrt) (IEEE reciprocal, for div_by_const)
__device__ __forceinline__ float4 adam_scalars(const AdamParams& p) {
  float2 t = make_float2(p.step_size, p.bc2_sqrt);
  if (p.tab != nullptr) {
    int64_t k = p.tab_k0 + (int64_t)epoch_base(p.sync);
    if (k >= p.tab_len) k = p.tab_len - 1;
    t = p.tab[k];
  }
  return make_float4(t.x, t.y, __frcp_rn(t.y), 0.0f);
}

#ifndef HPZ_ADAM_RCP_DIV
#define HPZ_ADAM_RCP_DIV 0
#endif
// RN(a / b) for a constant divisor b > 0 with rb = RN(1/b): Markstein's correction
// (q0 = RN(a*rb) is faithful, r = a - b*q0 is exact with an FMA, RN(q0 + r*rb) = RN(a/b)
// for normal operands and results); 3 instructions instead of the IEEE division's
// ~10.  a = sqrt(v) is 0, normal, inf or NaN here; the non-finite cases take the division.
// A/B only (off): bit-identical in every GPU parity test (273 incl. the 128-case fuzz and
// special values) but the fused RS+Adam measured 5% SLOWER (35.4 vs 33.6 ms/step at N=1).
__device__ __forceinline__ float div_by_const(float a, float b, float rb) {
#if HPZ_ADAM_RCP_DIV
  const float q0 = __fmul_rn(a, rb);
  const float r = __fmaf_rn(-q0, b, a);
  const float q1 = __fmaf_rn(r, rb, q0);
  return a < 3.0e38f ? q1 : __fdiv_rn(a, b);
#else
  (void)rb;
  return __fdiv_rn(a, b);
#endif
}

// One Adam element (reading R8), exactly the oracle's operation sequence: every
// operation is an explicit round-to-nearest intrinsic, so nothing is contracted to fma.
// sc = adam_scalars(p).
__device__ __forceinline__ void adam1(float& w, float& m, float& v, float g, const AdamParams& p, const float4 sc) {
  m = __fadd_rn(__fmul_rn(p.beta1, m), __fmul_rn(p.omb1, g));
  v = __fadd_rn(__fmul_rn(p.beta2, v), __fmul_rn(__fmul_rn(p.omb2, g), g));
  const float d = __fadd_rn(div_by_const(__fsqrt_rn(v), sc.y, sc.z), p.eps);
  if (p.lr_wd != 0.0f) w = __fsub_rn(w, __fmul_rn(p.lr_wd, w));
  w = __fsub_rn(w, __fmul_rn(sc.x, __fdiv_rn(m, d)));
}

// bf16 RNE of 4 fp32 values packed as 8 bytes (cvt.rn.bf16x2.f32).
__device__ __forceinline__ uint2 pack_bf16x4(const float4& w) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(w.x, w.y);
  __nv_bfloat162 hi = __floats2bfloat162_rn(w.z, w.w);
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  return pk;
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

// The last CTA of a gather: (forward) compare the gathered fingerprint with the one the
// owners emitted when they wrote their primaries (catches a forward read of stale or
// half-updated primaries: E1 / E2); (backward) compare it with the forward one (E3 / E4);
// then release the kernel's flags.  Slots are zeroed for their next use two steps later.
__device__ __forceinline__ void gather_finish(const GatherParams& p) {
  const int par = (int)((p.fp_par + epoch_base(p.sync)) & 1u);
  if (p.fp_exp != nullptr) {
    wait_all(p.exp_wait, p.sync);      // every owner's emission for this step is complete
    const unsigned long long got = *(volatile unsigned long long*)(p.fp_acc + 2 * par);
    const unsigned long long want = atomicExch(p.fp_exp + par, 0ull);
    atomicAdd(p.fpx_checked, 1ull);
    if (got != want) atomicAdd(p.fpx_mism, 1ull);
    __threadfence_system();            // the zeroed slot before the release that lets owners refill it
  }
  if (p.fp_a != nullptr) {
    wait_all(p.cmp_wait, p.sync);      // the forward checksum of this step is complete
    const unsigned long long a = atomicExch(p.fp_a + 2 * par, 0ull);
    const unsigned long long b = atomicExch(p.fp_b + 2 * par, 0ull);
    atomicAdd(p.fp_checked, 1ull);
    if (a != b) atomicAdd(p.fp_mism, 1ull);
  }
  release_all(p.rel, p.sync);
}

}  // namespace
}  // namespace hpz
