// Internal interface between the host runtime (hpz_runtime.cpp) and the sm_100a
// kernels (hpz_kernels.cu).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hpz.h"

namespace hpz {

constexpr int kMaxWorld = HPZ_MAX_WORLD;

// Device-side error/timeout plumbing shared by every waiting kernel, and the epoch base.
//
// Flag values are epochs.  Host-epoch mode (default): every value / target
// in a kernel's parameters is absolute, computed on the host from its step counter, and
// `epoch` is nullptr.  Device-epoch mode (HPZ_OPT_DEVICE_EPOCH, for CUDA-graph capture):
// parameters hold values RELATIVE to the step the call was issued in, and the kernel adds
// mul * (*epoch), the rank's step counter in device memory, which the call that completes
// a step advances on the device.  A captured step therefore replays with fresh epochs.
struct SyncCommon {
  uint64_t timeout_ns;                 // per-wait timeout
  uint32_t* abort_flag;                // local arena: set after the first timeout -> later waits skip
  unsigned long long* timeouts;        // local arena counter
  volatile uint32_t* host_err;         // host-mapped pinned word polled by the runtime
  const uint32_t* epoch;               // device step counter (device-epoch mode) or nullptr
  unsigned long long* timeout_info;    // [0] address of the first flag that timed out, [1] target<<32 | seen
};

// A list of flags to release (st.release.sys of value + mul * epoch), possibly in peer arenas.
struct ReleaseList {
  uint32_t* ptr[2 * kMaxWorld];
  int n;
  uint32_t value;
  uint32_t mul;                        // per-step increment of the value (device-epoch mode)
};

// A list of local flags to acquire (ld.acquire.sys until >= target + mul * epoch).
struct WaitList {
  const uint32_t* ptr[2 * kMaxWorld];
  int n;
  uint32_t target;
  uint32_t mul;
};

// Owner-emitted primary fingerprints (a7, E1/E2 coverage): the kernel that writes a primary
// shard (Adam, the qwZ quantizer, the init / resume refresh) adds the fingerprint of every
// 16-byte word it wrote (the word as the forward gather will read it) into every reader's
// "expected forward fingerprint" accumulator of the step that will gather it.
struct FpEmit {
  unsigned long long* dst[kMaxWorld];  // reader q's accumulator (parity-0 slot), nullptr: off
  int n_dst;
  int par;                             // parity of the gathering step (+ epoch in device mode)
  int64_t word_base;                   // my shard's first 16-byte word in the full buffer
};

// Forward / backward gather (a2 / a4): out[j*src_bytes ...] = src[j][...] for j < n_src.
struct GatherParams {
  const char* src[kMaxWorld];          // source shards (peer-mapped), in output order
  const uint32_t* src_flag[kMaxWorld]; // local flag acquired before reading src[j] (nullptr: none)
  uint32_t src_target;
  int n_src;
  int64_t src_bytes;                   // multiple of 16
  char* out;
  // fused secondary store (a2): sources [sec_lo, sec_hi) also go to sec + (j-sec_lo)*src_bytes
  char* sec;
  int sec_lo, sec_hi;
  WaitList war;                        // acquired before the first secondary store (E4)
  // verification (a7).  Accumulators are parity-0 slots; the step's slot is +2*par with
  // par = (fp_par + epoch) & 1
  int fp_par;
  unsigned long long* fp_acc;          // fingerprint accumulator (nullptr: off)
  const char* prim[kMaxWorld];         // EXACT: primaries of all ranks
  int64_t prim_bytes;                  // EXACT: bytes per primary shard
  int64_t valid_bytes;                 // numel * elem_bytes: elements past it are padding
  int elem_bytes;                      // 2 (bf16) or 4 (f32)
  unsigned long long* mism;            // EXACT counters
  unsigned long long* nans;
  // completion
  uint32_t* done_ctr;
  ReleaseList rel;
  // post-completion fingerprint compare (backward): waits cmp_wait, compares a vs b, zeroes both
  unsigned long long* fp_a;
  unsigned long long* fp_b;
  WaitList cmp_wait;
  unsigned long long* fp_mism;
  unsigned long long* fp_checked;
  // forward: compare my gathered fingerprint (fp_acc) with the owners' emitted one (fp_exp,
  // parity-0 slot, +par) once every owner released E1 (exp_wait); zero fp_exp
  unsigned long long* fp_exp;
  WaitList exp_wait;
  unsigned long long* fpx_mism;
  unsigned long long* fpx_checked;
  // qwZ (f2): src[j] are INT8 codes (1 byte per element, src_bytes = shard elements) and
  // qw_params[j] their (min, scale) per 256 elements; the kernel dequantizes to elem_bytes
  const float2* qw_params[kMaxWorld];
  SyncCommon sync;
};

// qgZ (f1): blockwise INT4 quantization of one rank's gradient slot.
constexpr int kQgzBlock = 64;          // elements per (min, scale) block
struct QuantParams {
  const float* g;                      // local gradient slot (n elements, n % 64 == 0)
  uint8_t* codes;                      // n/2 bytes: element 2i in the low nibble, 2i+1 high
  float2* params;                      // n/64 (min, scale) pairs
  int64_t n;
  WaitList war;                        // E6 of the previous use: peers done reading codes
  SyncCommon sync;
};

// qwZ (f2): blockwise INT8 quantization of one owner's primary shard (after Adam / load);
// its last CTA releases E1 (PRIMARY_READY) because peers gather the codes, not the primary.
constexpr int kQwzBlock = 256;
struct QwzQuantParams {
  const void* prim;                    // primary shard (bf16 or fp32), n elements, n % 256 == 0
  int prim_bf16;
  uint8_t* codes;                      // n bytes
  float2* params;                      // n/256 (min, scale) pairs
  int64_t n;
  uint32_t* done_ctr;
  ReleaseList rel;                     // E1
  FpEmit fpe;                          // expected fingerprint of the DEQUANTIZED words
  SyncCommon sync;
};

// Reduce-scatter (a5).
struct RSParams {
  const uint8_t* qcodes[kMaxWorld];    // qgZ: rank j's codes of my shard (peer-mapped), or unused
  const float2* qparams[kMaxWorld];    // qgZ: rank j's (min, scale) of my shard's blocks
  const float* src[kMaxWorld];         // src[j] = rank j's gradient slot + r*shard (peer-mapped);
                                       // with bf16 gradients the pointer addresses __nv_bfloat16 data
  float* out;                          // local gradient shard
  int64_t n_vec;                       // shard / 4
  float inv_p;
  ReleaseList ready;                   // E5 release (may be empty if already released)
  WaitList ready_wait;                 // E5 acquire of every rank
  uint32_t* done_ctr;
  ReleaseList rel;                     // E6 release
  SyncCommon sync;
};

// Fused Adam + primary refresh (a6).
struct AdamParams {
  float* w;
  float* m;
  float* v;
  const float* g;
  void* prim;
  int prim_bf16;
  int64_t n_vec;                       // shard / 4
  float beta1, beta2, omb1, omb2, step_size, bc2_sqrt, eps, lr_wd;
  // device-epoch mode: (step_size, bc2_sqrt) of 1-based Adam step k at tab[k - 1] (host
  // computed in double, rounded once), k = tab_k0 + epoch + 1, clamped to the last entry
  // (the scalars are constant from there on)
  const float2* tab;
  int64_t tab_k0, tab_len;
  WaitList wait;                       // E2 (+ backward-primary readers)
  uint32_t* done_ctr;
  ReleaseList rel;                     // E1 for t+1
  FpEmit fpe;                          // expected fingerprint of the new primary (nullptr dst: off)
  SyncCommon sync;
};

// Kernel launchers (hpz_kernels.cu).  Each returns the cudaError_t of the launch.
cudaError_t launch_gather(const GatherParams& p, int grid, cudaStream_t s);
cudaError_t launch_reduce_scatter(const RSParams& p, int world, int grid, cudaStream_t s);
cudaError_t launch_adam(const AdamParams& p, int grid, cudaStream_t s);
// Fused reduce-scatter + Adam (r.out may be nullptr: the reduced gradient is not stored).
cudaError_t launch_rs_adam(const RSParams& r, const AdamParams& a, int world, int grid, cudaStream_t s);
// TMA (cp.async.bulk) variants, one persistent CTA per SM (hpz_tma.cu).  The gather
// variant does not implement EXACT verification (p.mism must be nullptr).
cudaError_t launch_gather_tma(const GatherParams& p, int grid, cudaStream_t s);
// mode: 0 fp32 gradients, 1 bf16 gradients (fp32 accumulation), 2 qgZ INT4 codes
cudaError_t launch_rs_tma(const RSParams& r, const AdamParams* a, int world, int grid, cudaStream_t s,
                          int mode = 0);
cudaError_t launch_qgz_quantize(const QuantParams& q, int grid, cudaStream_t s);
cudaError_t launch_qwz_quantize(const QwzQuantParams& q, int grid, cudaStream_t s);
// qwZ forward gather: TMA-pulls codes + params, dequantizes, STG to out (+ secondary).
cudaError_t launch_gather_qwz(const GatherParams& p, int grid, cudaStream_t s);
cudaError_t launch_wait(const WaitList& w, const SyncCommon& sync, cudaStream_t s);
cudaError_t launch_release(const ReleaseList& r, const SyncCommon& sync, cudaStream_t s);
// *epoch += 1 (device-epoch mode: the call that completes a step)
cudaError_t launch_epoch_advance(uint32_t* epoch, cudaStream_t s);
// fingerprint of a freshly written primary shard (init / resume) into the readers' slots
cudaError_t launch_prim_fp(const void* prim, int64_t n_words, const FpEmit& fpe, const SyncCommon& sync, int grid,
                           cudaStream_t s);
cudaError_t launch_copy(void* dst, const void* src, int64_t bytes, int grid, cudaStream_t s);
cudaError_t launch_refresh_primary(const float* master, void* prim, int prim_bf16, int64_t n, int grid, cudaStream_t s);
cudaError_t launch_fill_u32(void* dst, uint32_t value, int64_t bytes, int grid, cudaStream_t s);
cudaError_t launch_delay(int us, cudaStream_t s);
// Seeded generator; e0 = global element index of dst[0]; values for
// e >= numel are 0.  kind 0: uniform*scale, 1: dyadic.
cudaError_t launch_synth_f32(float* dst, int64_t n, int64_t e0, int64_t numel, uint64_t key,
                             float scale, int kind, int grid, cudaStream_t s);
// Same generator, each value rounded to bf16 (RNE).
cudaError_t launch_synth_bf16(void* dst, int64_t n, int64_t e0, int64_t numel, uint64_t key,
                              float scale, int kind, int grid, cudaStream_t s);
// Master init from a generator or an fp32 source (src == nullptr: generator), m = v = 0,
// primary = rne(master).  n = shard elements, e0 = rank*shard.
cudaError_t launch_init_shard(float* master, float* m, float* v, void* prim, int prim_bf16,
                              const float* src_full, int64_t n, int64_t e0, int64_t numel,
                              uint64_t key, float scale, int grid, cudaStream_t s);

}  // namespace hpz
