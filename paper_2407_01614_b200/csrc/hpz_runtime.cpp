// Host runtime of libhpz: layout (a1), context/epoch bookkeeping, peer mappings and
// the C ABI declared in include/hpz.h.  Every hot-path call validates on the host,
// builds one parameter block and enqueues kernels on the caller's stream.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hpz_internal.h"

using namespace hpz;

namespace {

constexpr uint64_t kBufAlign = 4096;      // every per-layer buffer starts 4 KiB-aligned
constexpr uint64_t kCtrlAlign = 65536;

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

enum FlagKind { F_PRIM_READY = 0, F_FWD_DONE, F_SEC_READY, F_BWD_DONE, F_BWDP_DONE, F_NUM_LAYER_KINDS };
enum SlotFlagKind { S_GRAD_READY = 0, S_RS_DONE, S_NUM };
enum CtrKind { C_FWD = 0, C_BWD, C_RS, C_ADAM, C_QWZ, C_NUM };

struct Layer {
  int64_t numel, numel_pad, shard, sec_shard;
  uint64_t off_primary, off_master, off_m, off_v, off_gshard, off_secondary;
  uint64_t off_qw_codes = 0, off_qw_params = 0;   // qwZ (f2)
  int slot;
  // host bookkeeping of the step t the layer's ops were issued for (-1: never)
  int64_t fwd_t = -1, bwd_t = -1, rs_t = -1, step_t = -1;
  int64_t fpx_t = -1;    // step whose forward gather the owner's last fingerprint emission targets
  char* fwd_out = nullptr;          // full buffer of the last forward gather
  int64_t copy_t = -1;              // stock / paper: step of the last secondary copy issued
  const char* copy_src = nullptr;   // ... its source range while it may still be pending
  int64_t copy_bytes = 0;
};

}  // namespace

struct hpz_ctx {
  int world = 0, node_size = 0, rank = 0, device = 0, k = 0, sm_count = 0;
  int dtype = HPZ_BF16, elem = 2;
  int64_t align = 256;
  int n_layers = 0, n_slots = 0;
  std::vector<Layer> layers;
  std::vector<int64_t> slot_numel;        // numel_pad capacity of each grad slot
  std::vector<uint64_t> off_slot;
  std::vector<uint64_t> slot_use;         // completed-or-issued reduce-scatters per slot
  std::vector<uint8_t> slot_ready_sent;   // E5 already released for the current use
  uint64_t off_flags = 0, off_ctr = 0, off_fp = 0, off_stats = 0, ctrl_bytes = 0, arena_bytes = 0;
  bool registered = false, bound = false, owns_arena = false;
  // P' == P (one node): the secondary slice of rank r is its own primary shard
  // (Eq. (1) with P' = P), so the layout aliases it instead of storing a second copy; the
  // forward gather writes no secondary and the backward gather reads the node's primaries
  // (E1 acquire, E7 release).  Not with qwZ, whose secondary holds dequantized weights.
  bool alias_sec = false;
  bool alias_opt = true;                  // HPZ_OPT_ALIAS_SECONDARY
  bool copy_by_caller = false;            // HPZ_OPT_COPY_BY_CALLER
  char* arena[kMaxWorld] = {};            // mapped arena base of every rank
  bool opened[kMaxWorld] = {};            // arena[j] was opened via IPC here
  int64_t t = 0;                          // current step (flag epochs)
  int64_t adam_base = 0;                  // Adam steps done before this context (resume)
  int order = HPZ_ORDER_FIXED, stock_delay_us = 0, stock_poison = 0;
  int verify = HPZ_VERIFY_NONE;
  double timeout_s = 20.0;
  uint32_t* host_err = nullptr;           // pinned, mapped
  uint32_t* host_err_dev = nullptr;
  cudaStream_t side = nullptr;            // stock-mode copy stream
  cudaEvent_t side_ev = nullptr;
  std::vector<cudaEvent_t> copy_ev;       // ORDER_PAPER: per-layer "MemcpyD2D finished" host events
  uint64_t launches = 0;
  bool store_grad_shard = true;           // fused RS+Adam also stores the reduced gradient
  int ctas_per_sm = 4;                    // LDG/STG kernels
  int copy_engine = HPZ_COPY_TMA;
  int qgz_bits = 0;                       // f1: 4 = INT4 quantized gradient all-to-all
  int grad_bytes = 4;                     // f4: 2 = bf16 gradients (fp32 accumulation)
  int qwz_bits = 0;                       // f2: 8 = INT8 blockwise weights in the forward gather
  int max_ctas = 0;                       // cap on every grid (0 = all SMs)
  int bwd_ctas = 0, rs_ctas = 0;          // caps of the backward gathers / reduce-scatters (overlap)
  std::vector<uint64_t> off_qcodes, off_qparams;   // per grad slot (qgZ)
  std::vector<uint32_t> slot_uses;        // layers sharing each gradient slot (uses per step)
  uint64_t off_fpx = 0, off_epoch = 0;    // expected-forward-fingerprint slots; device step counter
  std::vector<int64_t> fpx_for;           // per layer: the step whose forward the last emission targets
  bool dev_epoch = false;                 // HPZ_OPT_DEVICE_EPOCH
  int fault = 0;                          // HPZ_OPT_FAULT (test-only ordering faults)
  float2* adam_tab = nullptr;             // device-epoch Adam scalars (cudaMalloc'd)
  int64_t adam_tab_len = 0;
  double adam_tab_key[4] = {-1, -1, -1, -1};
  std::string err;

  // ---- arena addressing (identical on every rank) ----
  uint32_t* flag(int rank_arena, int kind, int layer, int src) const {
    const uint64_t idx = ((uint64_t)kind * n_layers + layer) * world + src;
    return reinterpret_cast<uint32_t*>(arena[rank_arena] + off_flags) + idx;
  }
  uint32_t* slot_flag(int rank_arena, int kind, int slot, int src) const {
    const uint64_t base = (uint64_t)F_NUM_LAYER_KINDS * n_layers * world;
    const uint64_t idx = base + ((uint64_t)kind * n_slots + slot) * world + src;
    return reinterpret_cast<uint32_t*>(arena[rank_arena] + off_flags) + idx;
  }
  uint32_t* ctr(int kind, int idx) const {
    return reinterpret_cast<uint32_t*>(arena[rank] + off_ctr) + (uint64_t)kind * (n_layers + n_slots) + idx;
  }
  unsigned long long* fp(int layer, int parity, int which) const {
    return reinterpret_cast<unsigned long long*>(arena[rank] + off_fp) + ((uint64_t)layer * 2 + parity) * 2 + which;
  }
  // stats: 0 mismatches, 1 nans, 2 fp_mism, 3 fp_checked, 4 timeouts, 5 abort flag (u32),
  // 6 fwd-vs-owner fingerprint mismatches, 7 ... checked
  unsigned long long* stat(int i) const {
    return reinterpret_cast<unsigned long long*>(arena[rank] + off_stats) + i;
  }
  // rank `r`'s expected-forward-fingerprint slot pair of `layer` (parity 0; +1 = parity 1)
  unsigned long long* fpx(int r, int layer) const {
    return reinterpret_cast<unsigned long long*>(arena[r] + off_fpx) + (uint64_t)layer * 2;
  }
  uint32_t* epoch_word() const { return reinterpret_cast<uint32_t*>(arena[rank] + off_epoch); }
  SyncCommon sync() const {
    SyncCommon s;
    s.timeout_ns = (uint64_t)(timeout_s * 1e9);
    s.abort_flag = reinterpret_cast<uint32_t*>(stat(5));
    s.timeouts = stat(4);
    s.host_err = host_err_dev;
    s.epoch = dev_epoch ? epoch_word() : nullptr;
    s.timeout_info = stat(8);
    return s;
  }
  // Flag value for the absolute epoch x of a layer flag: absolute (host epochs) or relative
  // to the current step t, the kernel adding its device step counter (device epochs).
  uint32_t lv(int64_t x) const { return (uint32_t)(dev_epoch ? x - t : x); }
  // ... of a gradient-slot flag (slot_uses[slot] uses per step); the list's mul is set by sl()
  uint32_t sv(int slot, int64_t x) const { return (uint32_t)(dev_epoch ? x - t * (int64_t)slot_uses[slot] : x); }
  uint32_t sl(int slot) const { return slot_uses[slot]; }
  int node_first() const { return (rank / node_size) * node_size; }
  int local() const { return rank % node_size; }
};

namespace {

int fail(hpz_ctx* c, int code, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return code;
}

#define HPZ_CUDA(c, call)                                                              \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) return fail(c, HPZ_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

// Which ordering edge a flag address belongs to (for the timeout message).
std::string describe_flag(const hpz_ctx* c, uint64_t addr) {
  static const char* kLayerKinds[] = {"PRIM_READY (E1)", "FWD_DONE (E2)", "SEC_READY (E3)", "BWD_DONE (E4)",
                                      "BWDP_DONE (E7)"};
  static const char* kSlotKinds[] = {"GRAD_READY (E5)", "RS_DONE (E6)"};
  char buf[160];
  for (int r = 0; r < c->world; ++r) {
    const uint64_t base = reinterpret_cast<uint64_t>(c->arena[r] + c->off_flags);
    const uint64_t n_layer = (uint64_t)F_NUM_LAYER_KINDS * c->n_layers * c->world;
    const uint64_t n_all = n_layer + (uint64_t)S_NUM * c->n_slots * c->world;
    if (addr < base || addr >= base + n_all * 4) continue;
    uint64_t idx = (addr - base) / 4;
    if (idx < n_layer) {
      const uint64_t src = idx % c->world, layer = (idx / c->world) % c->n_layers, kind = idx / c->world / c->n_layers;
      snprintf(buf, sizeof buf, "%s of layer %llu from rank %llu (flag in rank %d's arena)", kLayerKinds[kind],
               (unsigned long long)layer, (unsigned long long)src, r);
    } else {
      idx -= n_layer;
      const uint64_t src = idx % c->world, slot = (idx / c->world) % c->n_slots, kind = idx / c->world / c->n_slots;
      snprintf(buf, sizeof buf, "%s of gradient slot %llu from rank %llu (flag in rank %d's arena)", kSlotKinds[kind],
               (unsigned long long)slot, (unsigned long long)src, r);
    }
    return buf;
  }
  snprintf(buf, sizeof buf, "flag at %#llx", (unsigned long long)addr);
  return buf;
}

int check_ready(hpz_ctx* c) {
  if (!c) return HPZ_EINVAL;
  if (!c->registered || !c->bound) return fail(c, HPZ_ESTATE, "context not registered/bound");
  if (c->host_err && *(volatile uint32_t*)c->host_err) {
    unsigned long long info[2] = {0, 0};
    cudaMemcpy(info, c->stat(8), sizeof info, cudaMemcpyDeviceToHost);   // the waits have returned
    cudaGetLastError();
    if (info[0])
      return fail(c, HPZ_ETIMEOUT, "a device-side flag wait timed out: %s stayed at %u, needed >= %u",
                  describe_flag(c, info[0]).c_str(), (unsigned)(info[1] & 0xffffffffu), (unsigned)(info[1] >> 32));
    return fail(c, HPZ_ETIMEOUT, "a device-side flag wait timed out (a peer never released)");
  }
  return HPZ_OK;
}

int check_layer(hpz_ctx* c, int layer) {
  if (layer < 0 || layer >= c->n_layers) return fail(c, HPZ_EINVAL, "layer %d out of range", layer);
  return HPZ_OK;
}

int grid_for(const hpz_ctx* c, int64_t work_items, int per_sm, int cap = 0) {
  int64_t g = (int64_t)c->sm_count * per_sm;
  if (c->max_ctas > 0 && g > c->max_ctas) g = c->max_ctas;   // leave SMs to overlapped compute
  if (cap > 0 && g > cap) g = cap;                            // per-collective cap (overlap)
  if (work_items < g) g = work_items;
  return g < 1 ? 1 : (int)g;
}


// Pick the gather kernel: TMA bulk pipeline (one CTA/SM) or the LDG/STG kernel (EXACT
// verification, or when selected with HPZ_OPT_COPY_ENGINE).
cudaError_t gather_launch(const hpz_ctx* c, const GatherParams& p, cudaStream_t s, int cap = 0) {
  if (c->copy_engine == HPZ_COPY_TMA && p.mism == nullptr) {
    const int64_t cb = p.n_src == 1 ? 16384 : 32768;   // launch_gather_tma's chunk for this case (grid sizing only)
    const int64_t chunks = (p.src_bytes + cb - 1) / cb * p.n_src;
    return launch_gather_tma(p, grid_for(c, chunks, 1, cap), s);
  }
  const int64_t tiles = (p.src_bytes / 16 + 2047) / 2048 * p.n_src;
  return launch_gather(p, grid_for(c, tiles, c->ctas_per_sm, cap > 0 ? cap * c->ctas_per_sm : 0), s);
}

#ifndef HPZ_RS_CTAS_PER_SM
#define HPZ_RS_CTAS_PER_SM 1   // TMA reduce-scatter CTAs per SM (A/B builds; needs a smaller stage budget)
#endif
cudaError_t rs_launch(const hpz_ctx* c, const RSParams& r, const AdamParams* a, cudaStream_t s) {
  const int per_sm = HPZ_RS_CTAS_PER_SM;
  if (c->qgz_bits || c->grad_bytes == 2)   // qgZ codes / bf16 gradients: TMA engine only
    return launch_rs_tma(r, a, c->world, grid_for(c, (r.n_vec * 4 + 1023) / 1024, per_sm, c->rs_ctas), s, c->qgz_bits ? 2 : 1);
  if (c->copy_engine == HPZ_COPY_TMA)
    return launch_rs_tma(r, a, c->world, grid_for(c, (r.n_vec * 4 + 1023) / 1024, per_sm, c->rs_ctas), s);
  const int grid = grid_for(c, (r.n_vec + 511) / 512, c->ctas_per_sm, c->rs_ctas > 0 ? c->rs_ctas * c->ctas_per_sm : 0);
  return a ? launch_rs_adam(r, *a, c->world, grid, s) : launch_reduce_scatter(r, c->world, grid, s);
}

// Owner-side fingerprint emission (a7): into every reader's expected-forward slot of the
// step `for_t` whose forward gather will read what the emitting kernel writes.
FpEmit fp_emit(hpz_ctx* c, int layer, int64_t for_t) {
  FpEmit e{};
  const Layer& L = c->layers[layer];
  for (int q = 0; q < c->world; ++q) e.dst[e.n_dst++] = c->fpx(q, layer);
  e.par = (int)(c->lv(for_t) & 1u);
  e.word_base = (int64_t)c->rank * L.shard * c->elem / 16;
  c->layers[layer].fpx_t = for_t;
  return e;
}

// qwZ: quantize my primary shard of `layer` (just written by Adam or the init) and release
// E1 (value) from the quantizer's last CTA: peers gather the codes, not the primary.
// `emit`: also emit the expected forward fingerprint (of the dequantized words) for step for_t.
int qwz_quantize(hpz_ctx* c, int layer, uint32_t value, cudaStream_t s, bool emit, int64_t for_t) {
  const Layer& L = c->layers[layer];
  char* a = c->arena[c->rank];
  QwzQuantParams q{};
  q.prim = a + L.off_primary;
  q.prim_bf16 = c->dtype == HPZ_BF16;
  q.codes = reinterpret_cast<uint8_t*>(a + L.off_qw_codes);
  q.params = reinterpret_cast<float2*>(a + L.off_qw_params);
  q.n = L.shard;
  q.done_ctr = c->ctr(C_QWZ, layer);
  for (int j = 0; j < c->world; ++j) q.rel.ptr[q.rel.n++] = c->flag(j, F_PRIM_READY, layer, c->rank);
  q.rel.value = value;
  if (emit) q.fpe = fp_emit(c, layer, for_t);
  q.sync = c->sync();
  cudaError_t e = launch_qwz_quantize(q, grid_for(c, (L.shard / kQwzBlock + 31) / 32, 4), s);   // one wave of 4 CTAs/SM, 8 warps x 4 blocks per CTA step
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "qwZ quantize launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  return HPZ_OK;
}

int publish_primary(hpz_ctx* c, int layer, cudaStream_t s);

int do_init_shard(hpz_ctx* c, int layer, const float* src, uint64_t key, float scale, cudaStream_t s) {
  Layer& L = c->layers[layer];
  char* a = c->arena[c->rank];
  if (L.fwd_t >= 0) return fail(c, HPZ_ESTATE, "layer %d already in use; load before the first gather", layer);
  cudaError_t e = launch_init_shard(reinterpret_cast<float*>(a + L.off_master), reinterpret_cast<float*>(a + L.off_m),
                                    reinterpret_cast<float*>(a + L.off_v), a + L.off_primary, c->dtype == HPZ_BF16,
                                    src, L.shard, (int64_t)c->rank * L.shard, L.numel, key, scale,
                                    grid_for(c, (L.shard + 255) / 256, 8), s);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "init_shard launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  return publish_primary(c, layer, s);
}

// A freshly loaded primary (init / resume): its expected forward fingerprint for the current
// step (always: one pass over the shard, once), then E1 (the qwZ quantizer's, with qwZ).
int publish_primary(hpz_ctx* c, int layer, cudaStream_t s) {
  const Layer& L = c->layers[layer];
  if (c->qwz_bits) return qwz_quantize(c, layer, c->lv(c->t + 1), s, true, c->t);   // E1 from the quantizer
  const int64_t words = L.shard * c->elem / 16;
  cudaError_t e = launch_prim_fp(c->arena[c->rank] + L.off_primary, words, fp_emit(c, layer, c->t), c->sync(),
                                 grid_for(c, (words + 255) / 256, 4), s);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "fingerprint launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  // E1 for the current step: PRIMARY_READY_j[layer][me] = t+1 in every rank's arena
  ReleaseList r{};
  for (int j = 0; j < c->world; ++j) r.ptr[r.n++] = c->flag(j, F_PRIM_READY, layer, c->rank);
  r.value = c->lv(c->t + 1);
  e = launch_release(r, c->sync(), s);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "release launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  return HPZ_OK;
}

// E6: wait until every rank finished reading the previous use of the layer's slot.
int slot_acquire(hpz_ctx* c, int layer, cudaStream_t s) {
  const int slot = c->layers[layer].slot;
  const uint64_t use = c->slot_use[slot];
  if (use == 0) return HPZ_OK;
  WaitList w{};
  for (int j = 0; j < c->world; ++j) w.ptr[w.n++] = c->slot_flag(c->rank, S_RS_DONE, slot, j);
  w.target = c->sv(slot, use);
  w.mul = c->sl(slot);
  cudaError_t e = launch_wait(w, c->sync(), s);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "wait launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  return HPZ_OK;
}

ReleaseList grad_ready_list(hpz_ctx* c, int slot) {
  ReleaseList r{};
  for (int j = 0; j < c->world; ++j) r.ptr[r.n++] = c->slot_flag(j, S_GRAD_READY, slot, c->rank);
  r.value = c->sv(slot, c->slot_use[slot] + 1);
  r.mul = c->sl(slot);
  return r;
}

}  // namespace

extern "C" {

int hpz_version(void) { return HPZ_VERSION; }

int hpz_init(int world, int node_size, int rank, int device, hpz_ctx** out) {
  if (!out) return HPZ_EINVAL;
  *out = nullptr;
  if (world < 1 || world > kMaxWorld || node_size < 1 || world % node_size != 0 || rank < 0 || rank >= world)
    return HPZ_EINVAL;
  if (device == -1) {   // host-only context: layout queries only (no CUDA calls)
    hpz_ctx* c = new hpz_ctx();
    c->world = world;
    c->node_size = node_size;
    c->k = world / node_size;
    c->rank = rank;
    c->device = -1;
    *out = c;
    return HPZ_OK;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return HPZ_EINVAL;
  }
  if (cudaSetDevice(device) != cudaSuccess) return HPZ_ECUDA;
  hpz_ctx* c = new hpz_ctx();
  c->world = world;
  c->node_size = node_size;
  c->k = world / node_size;
  c->rank = rank;
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaHostAlloc(reinterpret_cast<void**>(&c->host_err), sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess) {
    delete c;
    return HPZ_ECUDA;
  }
  *c->host_err = 0;
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->host_err_dev), c->host_err, 0);
  *out = c;
  return HPZ_OK;
}

int hpz_register_flat_params(hpz_ctx* c, int n_layers, const int64_t* numel, int param_dtype,
                             int64_t align_elems, int n_grad_slots, uint64_t* arena_bytes) {
  if (!c) return HPZ_EINVAL;
  if (c->registered) return fail(c, HPZ_ESTATE, "register_flat_params called twice");
  if (n_layers < 1 || !numel) return fail(c, HPZ_EINVAL, "n_layers must be >= 1");
  if (param_dtype != HPZ_BF16 && param_dtype != HPZ_F32) return fail(c, HPZ_EINVAL, "bad param dtype");
  const int elem = param_dtype == HPZ_BF16 ? 2 : 4;
  if (align_elems < 8 || (align_elems & (align_elems - 1)) || (align_elems * elem) % 16)
    return fail(c, HPZ_EINVAL, "align_elems must be a power of two >= 8 covering 16 bytes");
  if (n_grad_slots < 1 || n_grad_slots > n_layers) return fail(c, HPZ_EINVAL, "n_grad_slots must be in [1, n_layers]");
  if (c->qwz_bits && align_elems % kQwzBlock)
    return fail(c, HPZ_EINVAL, "qwZ needs align_elems to be a multiple of 256 (whole quantization blocks per shard)");
  if (c->qgz_bits && align_elems % 256)   // whole 64-blocks per shard, 16-byte bulk copies of their params
    return fail(c, HPZ_EINVAL, "qgZ needs align_elems to be a multiple of 256");
  c->dtype = param_dtype;
  c->elem = elem;
  c->alias_sec = c->alias_opt && c->node_size == c->world && !c->qwz_bits;
  c->align = align_elems;
  c->n_layers = n_layers;
  c->n_slots = n_grad_slots;
  c->layers.assign(n_layers, Layer{});
  c->slot_numel.assign(n_grad_slots, 0);
  c->slot_use.assign(n_grad_slots, 0);
  c->slot_ready_sent.assign(n_grad_slots, 0);
  c->slot_uses.assign(n_grad_slots, 0);
  const int64_t q = (int64_t)c->world * align_elems;
  for (int i = 0; i < n_layers; ++i) {
    if (numel[i] < 1) return fail(c, HPZ_EINVAL, "layer %d: numel must be >= 1", i);
    Layer& L = c->layers[i];
    L.numel = numel[i];
    L.numel_pad = (numel[i] + q - 1) / q * q;        // Eq. (1) with padding reading R2
    L.shard = L.numel_pad / c->world;
    L.sec_shard = L.numel_pad / c->node_size;
    L.slot = i % n_grad_slots;
    c->slot_uses[L.slot] += 1;
    if (L.numel_pad > c->slot_numel[L.slot]) c->slot_numel[L.slot] = L.numel_pad;
  }
  // control region: flags | completion counters | fingerprints | stats
  const uint64_t n_flags = (uint64_t)F_NUM_LAYER_KINDS * n_layers * c->world + (uint64_t)S_NUM * n_grad_slots * c->world;
  uint64_t off = 0;
  c->off_flags = off;
  off = align_up(off + n_flags * 4, 256);
  c->off_ctr = off;
  off = align_up(off + (uint64_t)C_NUM * (n_layers + n_grad_slots) * 4, 256);
  c->off_fp = off;
  off = align_up(off + (uint64_t)n_layers * 4 * 8, 256);
  c->off_stats = off;
  off = align_up(off + 16 * 8, 256);
  c->off_fpx = off;
  off = align_up(off + (uint64_t)n_layers * 2 * 8, 256);
  c->off_epoch = off;
  off = align_up(off + 4, 256);
  c->ctrl_bytes = align_up(off, kCtrlAlign);
  off = c->ctrl_bytes;
  for (int i = 0; i < n_layers; ++i) {
    Layer& L = c->layers[i];
    L.off_primary = off;   off = align_up(off + (uint64_t)L.shard * elem, kBufAlign);
    L.off_master = off;    off = align_up(off + (uint64_t)L.shard * 4, kBufAlign);
    L.off_m = off;         off = align_up(off + (uint64_t)L.shard * 4, kBufAlign);
    L.off_v = off;         off = align_up(off + (uint64_t)L.shard * 4, kBufAlign);
    L.off_gshard = off;    off = align_up(off + (uint64_t)L.shard * 4, kBufAlign);
    if (c->alias_sec) {
      L.off_secondary = L.off_primary;   // secondary == primary (P' == P)
    } else {
      L.off_secondary = off;
      off = align_up(off + (uint64_t)L.sec_shard * elem, kBufAlign);
    }
    if (c->qwz_bits) {   // int8 codes + (min, scale) per 256 elements of the primary shard
      L.off_qw_codes = off;
      off = align_up(off + (uint64_t)L.shard, kBufAlign);
      L.off_qw_params = off;
      off = align_up(off + (uint64_t)L.shard / kQwzBlock * 8, kBufAlign);
    }
  }
  c->off_slot.assign(n_grad_slots, 0);
  c->off_qcodes.assign(n_grad_slots, 0);
  c->off_qparams.assign(n_grad_slots, 0);
  for (int s = 0; s < n_grad_slots; ++s) {
    c->off_slot[s] = off;
    off = align_up(off + (uint64_t)c->slot_numel[s] * c->grad_bytes, kBufAlign);
    if (c->qgz_bits) {   // int4 codes + (min, scale) per 64-element block
      c->off_qcodes[s] = off;
      off = align_up(off + (uint64_t)c->slot_numel[s] / 2, kBufAlign);
      c->off_qparams[s] = off;
      off = align_up(off + (uint64_t)c->slot_numel[s] / kQgzBlock * 8, kBufAlign);
    }
  }
  c->arena_bytes = off;
  c->registered = true;
  if (arena_bytes) *arena_bytes = off;
  return HPZ_OK;
}

int hpz_arena_alloc(hpz_ctx* c, void* ipc_handle_out) {
  if (!c) return HPZ_EINVAL;
  if (!c->registered) return fail(c, HPZ_ESTATE, "arena_alloc before register");
  if (c->device < 0) return fail(c, HPZ_ESTATE, "host-only context (device -1) has no arena");
  if (c->arena[c->rank]) return fail(c, HPZ_ESTATE, "arena already allocated/bound");
  HPZ_CUDA(c, cudaSetDevice(c->device));
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, c->arena_bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, HPZ_ENOMEM, "cudaMalloc(%llu bytes): %s", (unsigned long long)c->arena_bytes, cudaGetErrorString(e));
  }
  c->arena[c->rank] = static_cast<char*>(p);
  c->owns_arena = true;
  HPZ_CUDA(c, cudaMemset(p, 0, c->ctrl_bytes));
  HPZ_CUDA(c, cudaDeviceSynchronize());
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    HPZ_CUDA(c, cudaIpcGetMemHandle(&h, p));
    static_assert(sizeof(h) == HPZ_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(ipc_handle_out, &h, sizeof h);
  }
  return HPZ_OK;
}

static int finish_bind(hpz_ctx* c) {
  HPZ_CUDA(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  HPZ_CUDA(c, cudaEventCreateWithFlags(&c->side_ev, cudaEventDisableTiming));
  c->copy_ev.assign(c->n_layers, nullptr);
  for (auto& ev : c->copy_ev) HPZ_CUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  c->bound = true;
  return HPZ_OK;
}

int hpz_arena_open(hpz_ctx* c, const void* all_handles) {
  if (!c || !all_handles) return HPZ_EINVAL;
  if (!c->registered || !c->arena[c->rank] || !c->owns_arena) return fail(c, HPZ_ESTATE, "arena_open needs arena_alloc first");
  if (c->bound) return fail(c, HPZ_ESTATE, "already bound");
  HPZ_CUDA(c, cudaSetDevice(c->device));
  const char* hs = static_cast<const char*>(all_handles);
  for (int j = 0; j < c->world; ++j) {
    if (j == c->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hs + (size_t)j * HPZ_IPC_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, HPZ_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", j, cudaGetErrorString(e));
    }
    c->arena[j] = static_cast<char*>(p);
    c->opened[j] = true;
  }
  return finish_bind(c);
}

int hpz_bind(hpz_ctx* c, void* const* ptrs) {
  if (!c || !ptrs) return HPZ_EINVAL;
  if (!c->registered) return fail(c, HPZ_ESTATE, "bind before register");
  if (c->device < 0) return fail(c, HPZ_ESTATE, "host-only context (device -1) cannot bind");
  if (c->bound) return fail(c, HPZ_ESTATE, "already bound");
  for (int j = 0; j < c->world; ++j) {
    if (!ptrs[j] || (reinterpret_cast<uintptr_t>(ptrs[j]) & 255)) return fail(c, HPZ_EINVAL, "arena_ptrs[%d] null or not 256-byte aligned", j);
  }
  if (c->arena[c->rank] && c->arena[c->rank] != ptrs[c->rank]) return fail(c, HPZ_EINVAL, "arena_ptrs[rank] differs from the allocated arena");
  HPZ_CUDA(c, cudaSetDevice(c->device));
  const bool zero = c->arena[c->rank] == nullptr;
  for (int j = 0; j < c->world; ++j) c->arena[j] = static_cast<char*>(ptrs[j]);
  if (zero) {
    HPZ_CUDA(c, cudaMemset(c->arena[c->rank], 0, c->ctrl_bytes));
    HPZ_CUDA(c, cudaDeviceSynchronize());
  }
  return finish_bind(c);
}

int hpz_finalize(hpz_ctx* c) {
  if (!c) return HPZ_EINVAL;
  if (c->device < 0) {
    delete c;
    return HPZ_OK;
  }
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int j = 0; j < c->world; ++j)
    if (c->opened[j]) cudaIpcCloseMemHandle(c->arena[j]);
  if (c->owns_arena && c->arena[c->rank]) cudaFree(c->arena[c->rank]);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->side_ev) cudaEventDestroy(c->side_ev);
  for (auto ev : c->copy_ev)
    if (ev) cudaEventDestroy(ev);
  if (c->host_err) cudaFreeHost(c->host_err);
  if (c->adam_tab) cudaFree(c->adam_tab);
  delete c;
  return HPZ_OK;
}

int hpz_layer_info(const hpz_ctx* cc, int layer, hpz_layer_info_t* out) {
  hpz_ctx* c = const_cast<hpz_ctx*>(cc);
  if (!c || !out) return HPZ_EINVAL;
  if (!c->registered) return fail(c, HPZ_ESTATE, "not registered");
  if (int rc = check_layer(c, layer)) return rc;
  const Layer& L = c->layers[layer];
  out->numel = L.numel;
  out->numel_pad = L.numel_pad;
  out->shard = L.shard;
  out->sec_shard = L.sec_shard;
  out->off_primary = L.off_primary;
  out->off_master = L.off_master;
  out->off_m = L.off_m;
  out->off_v = L.off_v;
  out->off_grad_shard = L.off_gshard;
  out->off_secondary = L.off_secondary;
  out->off_grad_slot = c->off_slot[L.slot];
  out->grad_slot = L.slot;
  out->_pad = 0;
  return HPZ_OK;
}

int hpz_arena_ptr(const hpz_ctx* cc, int rank, void** out) {
  hpz_ctx* c = const_cast<hpz_ctx*>(cc);
  if (!c || !out || rank < 0 || rank >= c->world) return HPZ_EINVAL;
  if (!c->arena[rank]) return fail(c, HPZ_ESTATE, "arena of rank %d not mapped", rank);
  *out = c->arena[rank];
  return HPZ_OK;
}

int hpz_buffer(const hpz_ctx* cc, int layer, int kind, void** ptr, int64_t* n) {
  hpz_ctx* c = const_cast<hpz_ctx*>(cc);
  if (!c || !ptr) return HPZ_EINVAL;
  if (!c->registered || !c->arena[c->rank]) return fail(c, HPZ_ESTATE, "arena not allocated/bound");
  if (int rc = check_layer(c, layer)) return rc;
  const Layer& L = c->layers[layer];
  char* a = c->arena[c->rank];
  int64_t cnt = L.shard;
  switch (kind) {
    case HPZ_BUF_PRIMARY: *ptr = a + L.off_primary; break;
    case HPZ_BUF_MASTER: *ptr = a + L.off_master; break;
    case HPZ_BUF_ADAM_M: *ptr = a + L.off_m; break;
    case HPZ_BUF_ADAM_V: *ptr = a + L.off_v; break;
    case HPZ_BUF_GRAD_SHARD: *ptr = a + L.off_gshard; break;
    case HPZ_BUF_SECONDARY: *ptr = a + L.off_secondary; cnt = L.sec_shard; break;
    case HPZ_BUF_GRAD_SLOT: *ptr = a + c->off_slot[L.slot]; cnt = L.numel_pad; break;
    default: return fail(c, HPZ_EINVAL, "bad buffer kind %d", kind);
  }
  if (n) *n = cnt;
  return HPZ_OK;
}

int hpz_current_step(const hpz_ctx* c, int64_t* t) {
  if (!c || !t) return HPZ_EINVAL;
  *t = c->t;
  return HPZ_OK;
}

int hpz_resync_step(hpz_ctx* c) {
  if (int rc = check_ready(c)) return rc;
  if (!c->dev_epoch) return fail(c, HPZ_ESTATE, "hpz_resync_step needs device epochs");
  HPZ_CUDA(c, cudaSetDevice(c->device));
  HPZ_CUDA(c, cudaDeviceSynchronize());
  uint32_t d = 0;
  HPZ_CUDA(c, cudaMemcpy(&d, c->epoch_word(), 4, cudaMemcpyDeviceToHost));
  for (const Layer& L : c->layers)
    if (L.step_t != c->t - 1) return fail(c, HPZ_ESTATE, "hpz_resync_step between complete steps only");
  const int64_t t = (int64_t)d;
  for (Layer& L : c->layers) {
    L.fwd_t = L.bwd_t = L.rs_t = L.step_t = t - 1;
    if (L.fpx_t == c->t) L.fpx_t = t;   // the last step's emission targets step t's forward
  }
  for (size_t k = 0; k < c->slot_use.size(); ++k) {
    c->slot_use[k] = (uint64_t)t * c->slot_uses[k];
    c->slot_ready_sent[k] = 0;
  }
  c->t = t;
  return HPZ_OK;
}

int hpz_counters(hpz_ctx* c, hpz_counters_t* out, int reset) {
  if (!c || !out) return HPZ_EINVAL;
  if (c->device < 0) return fail(c, HPZ_ESTATE, "host-only context has no counters");
  if (!c->registered || !c->arena[c->rank]) return fail(c, HPZ_ESTATE, "arena not allocated/bound");
  HPZ_CUDA(c, cudaSetDevice(c->device));
  HPZ_CUDA(c, cudaDeviceSynchronize());
  unsigned long long s[8];
  HPZ_CUDA(c, cudaMemcpy(s, c->stat(0), sizeof s, cudaMemcpyDeviceToHost));
  out->mismatches = s[0];
  out->nan_reads = s[1];
  out->fp_mismatches = s[2];
  out->fp_checked = s[3];
  out->timeouts = s[4];
  out->launches = c->launches;
  out->fp_fwd_mismatches = s[6];
  out->fp_fwd_checked = s[7];
  if (reset) {
    HPZ_CUDA(c, cudaMemset(c->stat(0), 0, 4 * sizeof(unsigned long long)));
    HPZ_CUDA(c, cudaMemset(c->stat(6), 0, 2 * sizeof(unsigned long long)));
  }
  return HPZ_OK;
}

const char* hpz_last_error(const hpz_ctx* c) { return c ? c->err.c_str() : "null context"; }

int hpz_set_order(hpz_ctx* c, int order, int stock_delay_us, int stock_poison) {
  if (!c) return HPZ_EINVAL;
  if (order < HPZ_ORDER_FIXED || order > HPZ_ORDER_PAPER || stock_delay_us < 0) return fail(c, HPZ_EINVAL, "bad order");
  c->order = order;
  c->stock_delay_us = stock_delay_us;
  c->stock_poison = stock_poison;
  return HPZ_OK;
}

int hpz_set_verify(hpz_ctx* c, int mode) {
  if (!c) return HPZ_EINVAL;
  if (mode < HPZ_VERIFY_NONE || mode > HPZ_VERIFY_EXACT) return fail(c, HPZ_EINVAL, "bad verify mode");
  c->verify = mode;
  return HPZ_OK;
}

int hpz_set_timeout(hpz_ctx* c, double seconds) {
  if (!c || !(seconds > 0)) return HPZ_EINVAL;
  c->timeout_s = seconds;
  return HPZ_OK;
}

int hpz_load_master(hpz_ctx* c, int layer, const float* full, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  if (!full) return fail(c, HPZ_EINVAL, "null source");
  return do_init_shard(c, layer, full, 0, 0.f, static_cast<cudaStream_t>(stream));
}

int hpz_load_state(hpz_ctx* c, int layer, const float* master, const float* m, const float* v,
                   int64_t adam_steps_done, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  if (!master || !m || !v || adam_steps_done < 0) return fail(c, HPZ_EINVAL, "bad checkpoint arguments");
  Layer& L = c->layers[layer];
  if (L.fwd_t >= 0) return fail(c, HPZ_ESTATE, "layer %d already in use; load state before the first gather", layer);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* a = c->arena[c->rank];
  const size_t bytes = (size_t)L.shard * 4;
  HPZ_CUDA(c, cudaMemcpyAsync(a + L.off_master, master, bytes, cudaMemcpyDefault, s));
  HPZ_CUDA(c, cudaMemcpyAsync(a + L.off_m, m, bytes, cudaMemcpyDefault, s));
  HPZ_CUDA(c, cudaMemcpyAsync(a + L.off_v, v, bytes, cudaMemcpyDefault, s));
  cudaError_t e = launch_refresh_primary(reinterpret_cast<const float*>(a + L.off_master), a + L.off_primary,
                                         c->dtype == HPZ_BF16, L.shard, grid_for(c, (L.shard + 255) / 256, 8), s);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "refresh launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  c->adam_base = adam_steps_done;
  return publish_primary(c, layer, s);
}

int hpz_synth_master(hpz_ctx* c, int layer, uint64_t key, float scale, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  return do_init_shard(c, layer, nullptr, key, scale, static_cast<cudaStream_t>(stream));
}

// Stock / paper secondary write (Alg. 1: "L_i,second <- empty(|L_i|/P');
// Copy to L_i,second (Async MemcpyD2D)"): a copy from the layer's forward-gathered full
// buffer on the context's side stream, after the work already on `s`.  STOCK: no edge to the
// backward AllGather (the race).  PAPER: SEC_READY + a host-visible
// "MemcpyD2D finished" event the backward gather waits for on the HOST (Alg. 1 blue lines).
// The copy reads the caller's full buffer after this call returns: the next hpz gather into
// the same buffer waits for it (the stream-side equivalent of record_stream on L_i).
static int secondary_copy(hpz_ctx* c, int layer, cudaStream_t s) {
  Layer& L = c->layers[layer];
  const int nf = c->node_first();
  char* sec = c->arena[c->rank] + L.off_secondary;
  const int64_t sec_bytes = L.sec_shard * c->elem;
  cudaError_t e;
  HPZ_CUDA(c, cudaEventRecord(c->side_ev, s));
  HPZ_CUDA(c, cudaStreamWaitEvent(c->side, c->side_ev, 0));
  if (c->order == HPZ_ORDER_PAPER && c->t > 0) {
    // E4 (P2P needs it; NCCL's rendezvous would cover it): node peers' step t-1 reads done
    WaitList w{};
    for (int q = 0; q < c->node_size; ++q) w.ptr[w.n++] = c->flag(c->rank, F_BWD_DONE, layer, nf + q);
    w.target = c->lv(c->t);
    e = launch_wait(w, c->sync(), c->side);
    if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "wait launch: %s", cudaGetErrorString(e));
    c->launches += 1;
  }
  if (c->stock_poison) {
    e = launch_fill_u32(sec, c->elem == 2 ? 0x7FC07FC0u : 0x7FC00000u, sec_bytes, grid_for(c, sec_bytes / 4096 + 1, 4), c->side);
    if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "poison launch: %s", cudaGetErrorString(e));
    c->launches += 1;
  }
  if (c->stock_delay_us > 0) {
    e = launch_delay(c->stock_delay_us, c->side);
    if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "delay launch: %s", cudaGetErrorString(e));
    c->launches += 1;
  }
  e = launch_copy(sec, L.fwd_out + (int64_t)c->local() * sec_bytes, sec_bytes, grid_for(c, sec_bytes / 4096 + 1, 4), c->side);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "stock copy launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  if (c->order == HPZ_ORDER_PAPER) {
    // publish SEC_READY to the node (what the collective's rendezvous does for NCCL)
    ReleaseList r{};
    for (int q = 0; q < c->node_size; ++q) r.ptr[r.n++] = c->flag(nf + q, F_SEC_READY, layer, c->rank);
    r.value = c->lv(c->t + 1);
    e = launch_release(r, c->sync(), c->side);
    if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "release launch: %s", cudaGetErrorString(e));
    c->launches += 1;
  }
  HPZ_CUDA(c, cudaEventRecord(c->copy_ev[layer], c->side));
  L.copy_t = c->t;
  L.copy_src = L.fwd_out;
  L.copy_bytes = L.numel_pad * c->elem;
  return HPZ_OK;
}

// A gather about to write [out, out + bytes) waits for every pending stock / paper copy that
// reads from that range (issued earlier on the side stream), then forgets it.
static int wait_pending_copies(hpz_ctx* c, const char* out, int64_t bytes, cudaStream_t s) {
  for (int i = 0; i < c->n_layers; ++i) {
    Layer& L = c->layers[i];
    if (!L.copy_src || L.copy_src >= out + bytes || L.copy_src + L.copy_bytes <= out) continue;
    HPZ_CUDA(c, cudaStreamWaitEvent(s, c->copy_ev[i], 0));
    L.copy_src = nullptr;
  }
  return HPZ_OK;
}

int hpz_fwd_gather(hpz_ctx* c, int layer, void* full_out, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  if (!full_out || (reinterpret_cast<uintptr_t>(full_out) & 15)) return fail(c, HPZ_EINVAL, "full_out null or not 16-byte aligned");
  Layer& L = c->layers[layer];
  if (L.fwd_t == c->t) return fail(c, HPZ_ESTATE, "layer %d already forward-gathered at step %lld", layer, (long long)c->t);
  if (c->qwz_bits && (c->verify == HPZ_VERIFY_EXACT || c->order == HPZ_ORDER_OFF))
    return fail(c, HPZ_ESTATE, "qwZ gathers dequantized weights: EXACT verification and ORDER_OFF compare/read raw primaries");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->dev_epoch && (c->order == HPZ_ORDER_STOCK || c->order == HPZ_ORDER_PAPER))
    return fail(c, HPZ_ESTATE, "device epochs (graph capture) support ORDER_FIXED and ORDER_OFF only");
  const uint32_t t1 = c->lv(c->t + 1);
  GatherParams p{};
  p.n_src = c->world;
  p.src_bytes = L.shard * c->elem;
  for (int j = 0; j < c->world; ++j) {
    p.src[j] = c->arena[j] + L.off_primary;
    // E1 (HPZ_FAULT_SKIP_E1: test-only, the data reads skip it; the fingerprint check keeps it)
    p.src_flag[j] = (c->fault & HPZ_FAULT_SKIP_E1) ? nullptr : c->flag(c->rank, F_PRIM_READY, layer, j);
  }
  p.src_target = t1;
  p.out = static_cast<char*>(full_out);
  p.elem_bytes = c->elem;
  p.valid_bytes = L.numel * c->elem;
  const int l = c->local();
  const int nf = c->node_first();
  const bool write_sec = c->order == HPZ_ORDER_FIXED && !c->alias_sec;
  if (write_sec) {
    // fused secondary store: my secondary slice l holds primaries l*k .. l*k+k-1 (R2 nesting)
    p.sec = c->arena[c->rank] + L.off_secondary;
    p.sec_lo = l * c->k;
    p.sec_hi = (l + 1) * c->k;
    for (int q = 0; q < c->node_size; ++q) p.war.ptr[p.war.n++] = c->flag(c->rank, F_BWD_DONE, layer, nf + q);   // E4
    p.war.target = c->lv(c->t);
  }
  p.fp_par = (int)(c->lv(c->t) & 1u);
  if (c->verify != HPZ_VERIFY_NONE) {
    p.fp_acc = c->fp(layer, 0, 0);
    if (L.fpx_t == c->t) {
      // the owners emitted this step's expected fingerprint (a7, E1/E2): compare once all E1s
      p.fp_exp = c->fpx(c->rank, layer);
      for (int j = 0; j < c->world; ++j) p.exp_wait.ptr[p.exp_wait.n++] = c->flag(c->rank, F_PRIM_READY, layer, j);
      p.exp_wait.target = t1;
      p.fpx_mism = c->stat(6);
      p.fpx_checked = c->stat(7);
    }
  }
  p.done_ctr = c->ctr(C_FWD, layer);
  if (write_sec)
    for (int q = 0; q < c->node_size; ++q) p.rel.ptr[p.rel.n++] = c->flag(nf + q, F_SEC_READY, layer, c->rank);   // E3
  for (int j = 0; j < c->world; ++j) p.rel.ptr[p.rel.n++] = c->flag(j, F_FWD_DONE, layer, c->rank);            // E2
  p.rel.value = t1;
  p.sync = c->sync();
  if (int rc = wait_pending_copies(c, p.out, L.numel_pad * c->elem, s)) return rc;
  cudaError_t e;
  if (c->qwz_bits) {
    // qwZ: pull every owner's INT8 codes + (min, scale) and dequantize (f2, R28)
    p.src_bytes = L.shard;   // one code byte per element
    for (int j = 0; j < c->world; ++j) {
      p.src[j] = c->arena[j] + L.off_qw_codes;
      p.qw_params[j] = reinterpret_cast<const float2*>(c->arena[j] + L.off_qw_params);
    }
    e = launch_gather_qwz(p, grid_for(c, (L.shard + 8191) / 8192 * c->world, 1), s);
  } else {
    e = gather_launch(c, p, s);
  }
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "fwd gather launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  L.fwd_t = c->t;
  L.fwd_out = p.out;
  if ((c->order == HPZ_ORDER_STOCK || c->order == HPZ_ORDER_PAPER) && !c->alias_sec && !c->copy_by_caller)
    return secondary_copy(c, layer, s);
  return HPZ_OK;
}

int hpz_secondary_copy(hpz_ctx* c, int layer, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  const Layer& L = c->layers[layer];
  if (!c->copy_by_caller || (c->order != HPZ_ORDER_STOCK && c->order != HPZ_ORDER_PAPER))
    return fail(c, HPZ_ESTATE, "hpz_secondary_copy: only with HPZ_OPT_COPY_BY_CALLER in ORDER_STOCK / ORDER_PAPER");
  if (L.fwd_t != c->t) return fail(c, HPZ_ESTATE, "layer %d: secondary copy before its forward gather", layer);
  if (L.copy_t == c->t) return fail(c, HPZ_ESTATE, "layer %d: secondary copy already issued at step %lld", layer, (long long)c->t);
  if (c->alias_sec) return HPZ_OK;   // P' == P: the secondary is the primary, nothing to copy
  return secondary_copy(c, layer, static_cast<cudaStream_t>(stream));
}

int hpz_bwd_gather(hpz_ctx* c, int layer, void* full_out, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  if (!full_out || (reinterpret_cast<uintptr_t>(full_out) & 15)) return fail(c, HPZ_EINVAL, "full_out null or not 16-byte aligned");
  Layer& L = c->layers[layer];
  if (L.fwd_t != c->t) return fail(c, HPZ_ESTATE, "layer %d: backward gather without its forward gather at step %lld", layer, (long long)c->t);
  if (L.bwd_t == c->t) return fail(c, HPZ_ESTATE, "layer %d already backward-gathered at step %lld", layer, (long long)c->t);
  if (c->order == HPZ_ORDER_PAPER && !c->alias_sec) {
    // Alg. 1: "Repeat wait Until MemcpyD2D on L_k,second finishes" (host)
    if (L.copy_t != c->t) return fail(c, HPZ_ESTATE, "layer %d: backward gather before its secondary copy (hpz_secondary_copy)", layer);
    HPZ_CUDA(c, cudaEventSynchronize(c->copy_ev[layer]));
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t t1 = c->lv(c->t + 1);
  const int nf = c->node_first();
  const bool from_prim = c->order == HPZ_ORDER_OFF || c->alias_sec;
  const bool reads_prim = from_prim || c->verify == HPZ_VERIFY_EXACT;
  GatherParams p{};
  if (from_prim) {
    // no hpZ: AllGather(L_i, P) from the primaries again (ZeRO-3 backward);
    // P' == P: the node's secondaries ARE the primaries, same gather
    p.n_src = c->world;
    p.src_bytes = L.shard * c->elem;
    for (int j = 0; j < c->world; ++j) {
      p.src[j] = c->arena[j] + L.off_primary;
      p.src_flag[j] = c->flag(c->rank, F_PRIM_READY, layer, j);
    }
  } else {
    // hpZ: AllGather(L_i, P') over the node's secondaries
    p.n_src = c->node_size;
    p.src_bytes = L.sec_shard * c->elem;
    for (int q = 0; q < c->node_size; ++q) {
      p.src[q] = c->arena[nf + q] + L.off_secondary;
      // THE FIX: acquire SEC_READY of the owner for step t.
      // STOCK reproduces the bug: no wait.
      p.src_flag[q] = c->order != HPZ_ORDER_STOCK ? c->flag(c->rank, F_SEC_READY, layer, nf + q) : nullptr;
    }
  }
  p.src_target = t1;
  p.out = static_cast<char*>(full_out);
  p.elem_bytes = c->elem;
  p.valid_bytes = L.numel * c->elem;
  if (c->verify == HPZ_VERIFY_EXACT) {
    for (int j = 0; j < c->world; ++j) p.prim[j] = c->arena[j] + L.off_primary;
    p.prim_bytes = L.shard * c->elem;
    p.mism = c->stat(0);
    p.nans = c->stat(1);
  }
  p.fp_par = (int)(c->lv(c->t) & 1u);
  if (c->verify != HPZ_VERIFY_NONE) {
    p.fp_acc = c->fp(layer, 0, 1);
    p.fp_a = c->fp(layer, 0, 0);
    p.fp_b = c->fp(layer, 0, 1);
    p.cmp_wait.ptr[p.cmp_wait.n++] = c->flag(c->rank, F_FWD_DONE, layer, c->rank);   // my forward finished
    p.cmp_wait.target = t1;
    p.fp_mism = c->stat(2);
    p.fp_checked = c->stat(3);
  }
  p.done_ctr = c->ctr(C_BWD, layer);
  // E4 (released in every order, so the order may change between steps: the next step's
  // secondary writes wait for it even after an OFF step that read no secondary)
  for (int q = 0; q < c->node_size; ++q) p.rel.ptr[p.rel.n++] = c->flag(nf + q, F_BWD_DONE, layer, c->rank);
  if (reads_prim)
    for (int j = 0; j < c->world; ++j) p.rel.ptr[p.rel.n++] = c->flag(j, F_BWDP_DONE, layer, c->rank);
  p.rel.value = t1;
  p.sync = c->sync();
  if (reads_prim) {
    // the primaries read here must still be W_t: they are, because Adam(t) waits for BWDP_DONE
    // and the sources' PRIMARY_READY >= t+1 is acquired per source (OFF) or below (EXACT)
    if (!from_prim) {
      WaitList w{};
      for (int j = 0; j < c->world; ++j) w.ptr[w.n++] = c->flag(c->rank, F_PRIM_READY, layer, j);
      w.target = t1;
      cudaError_t e = launch_wait(w, c->sync(), s);
      if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "wait launch: %s", cudaGetErrorString(e));
      c->launches += 1;
    }
  }
  if (int rc = wait_pending_copies(c, p.out, L.numel_pad * c->elem, s)) return rc;
  cudaError_t e = gather_launch(c, p, s, c->bwd_ctas);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "bwd gather launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  L.bwd_t = c->t;
  return HPZ_OK;
}

int hpz_grad_buffer(hpz_ctx* c, int layer, void** slot_ptr, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = slot_acquire(c, layer, static_cast<cudaStream_t>(stream))) return rc;
  if (slot_ptr) *slot_ptr = c->arena[c->rank] + c->off_slot[c->layers[layer].slot];
  return HPZ_OK;
}

int hpz_grad_upload(hpz_ctx* c, int layer, const void* src, int64_t n, void* stream) {
  void* slot = nullptr;
  if (int rc = hpz_grad_buffer(c, layer, &slot, stream)) return rc;
  const Layer& L = c->layers[layer];
  if (!src || n < 0 || n > L.numel) return fail(c, HPZ_EINVAL, "bad gradient source or length");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t gb = (size_t)c->grad_bytes;
  HPZ_CUDA(c, cudaMemcpyAsync(slot, src, (size_t)n * gb, cudaMemcpyDefault, s));
  if (n < L.numel_pad)
    HPZ_CUDA(c, cudaMemsetAsync(static_cast<char*>(slot) + n * gb, 0, (size_t)(L.numel_pad - n) * gb, s));
  return HPZ_OK;
}

int hpz_synth_grads(hpz_ctx* c, int layer, uint64_t key, float scale, int kind, void* stream) {
  void* slot = nullptr;
  if (int rc = hpz_grad_buffer(c, layer, &slot, stream)) return rc;
  if (kind != 0 && kind != 1) return fail(c, HPZ_EINVAL, "bad generator kind");
  const Layer& L = c->layers[layer];
  const int grid = grid_for(c, (L.numel_pad + 255) / 256, 8);
  cudaError_t e = c->grad_bytes == 2
                      ? launch_synth_bf16(slot, L.numel_pad, 0, L.numel, key, scale, kind, grid, static_cast<cudaStream_t>(stream))
                      : launch_synth_f32(static_cast<float*>(slot), L.numel_pad, 0, L.numel, key, scale, kind, grid,
                                         static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "synth launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  return HPZ_OK;
}

// qgZ: quantize this rank's gradient slot of `layer` (whole numel_pad) before the RS kernel
// publishes E5; waits E6 of the slot's previous use (peers done reading the old codes).
static int qgz_quantize(hpz_ctx* c, int layer, cudaStream_t s) {
  const Layer& L = c->layers[layer];
  const int slot = L.slot;
  QuantParams q{};
  q.g = reinterpret_cast<const float*>(c->arena[c->rank] + c->off_slot[slot]);
  q.codes = reinterpret_cast<uint8_t*>(c->arena[c->rank] + c->off_qcodes[slot]);
  q.params = reinterpret_cast<float2*>(c->arena[c->rank] + c->off_qparams[slot]);
  q.n = L.numel_pad;
  if (c->slot_use[slot] > 0) {
    for (int j = 0; j < c->world; ++j) q.war.ptr[q.war.n++] = c->slot_flag(c->rank, S_RS_DONE, slot, j);
    q.war.target = c->sv(slot, c->slot_use[slot]);
    q.war.mul = c->sl(slot);
  }
  q.sync = c->sync();
  cudaError_t e = launch_qgz_quantize(q, grid_for(c, (L.numel_pad / kQgzBlock + 63) / 64, 4), s);   // 4 resident CTAs/SM: one wave
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "qgZ quantize launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  return HPZ_OK;
}

int hpz_grads_ready(hpz_ctx* c, int layer, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  const int slot = c->layers[layer].slot;
  if (c->slot_ready_sent[slot]) return fail(c, HPZ_ESTATE, "grads_ready already published for this use of the slot");
  if (c->qgz_bits)
    if (int rc = qgz_quantize(c, layer, static_cast<cudaStream_t>(stream))) return rc;
  cudaError_t e = launch_release(grad_ready_list(c, slot), c->sync(), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "release launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  c->slot_ready_sent[slot] = 1;
  return HPZ_OK;
}

static void build_rs(hpz_ctx* c, int layer, RSParams& p) {
  Layer& L = c->layers[layer];
  const int slot = L.slot;
  const uint32_t u1 = c->sv(slot, c->slot_use[slot] + 1);
  p = RSParams{};
  for (int j = 0; j < c->world; ++j)
    p.src[j] = reinterpret_cast<const float*>(c->arena[j] + c->off_slot[slot] + (uint64_t)c->rank * L.shard * c->grad_bytes);
  p.out = reinterpret_cast<float*>(c->arena[c->rank] + L.off_gshard);
  p.n_vec = L.shard / 4;
  p.inv_p = (float)(1.0 / c->world);
  if (!c->slot_ready_sent[slot]) p.ready = grad_ready_list(c, slot);   // E5 release
  for (int j = 0; j < c->world; ++j) p.ready_wait.ptr[p.ready_wait.n++] = c->slot_flag(c->rank, S_GRAD_READY, slot, j);
  p.ready_wait.target = u1;
  p.ready_wait.mul = c->sl(slot);
  p.done_ctr = c->ctr(C_RS, c->n_layers + slot);
  for (int j = 0; j < c->world; ++j) p.rel.ptr[p.rel.n++] = c->slot_flag(j, S_RS_DONE, slot, c->rank);   // E6
  p.rel.value = u1;
  p.rel.mul = c->sl(slot);
  p.sync = c->sync();
  if (c->qgz_bits) {
    for (int j = 0; j < c->world; ++j) {
      p.qcodes[j] = reinterpret_cast<const uint8_t*>(c->arena[j] + c->off_qcodes[slot]) + (int64_t)c->rank * L.shard / 2;
      p.qparams[j] = reinterpret_cast<const float2*>(c->arena[j] + c->off_qparams[slot]) + (int64_t)c->rank * L.shard / kQgzBlock;
    }
  }
}

static void rs_issued(hpz_ctx* c, int layer) {
  Layer& L = c->layers[layer];
  c->slot_use[L.slot] += 1;
  c->slot_ready_sent[L.slot] = 0;
  L.rs_t = c->t;
}

int hpz_reduce_scatter(hpz_ctx* c, int layer, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  Layer& L = c->layers[layer];
  if (L.rs_t == c->t) return fail(c, HPZ_ESTATE, "layer %d already reduce-scattered at step %lld", layer, (long long)c->t);
  RSParams p;
  build_rs(c, layer, p);
  if (c->qgz_bits && !c->slot_ready_sent[L.slot])
    if (int rc = qgz_quantize(c, layer, static_cast<cudaStream_t>(stream))) return rc;
  cudaError_t e = rs_launch(c, p, nullptr, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "reduce-scatter launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  rs_issued(c, layer);
  return HPZ_OK;
}

static int check_adam(hpz_ctx* c, const hpz_adam* a) {
  if (!a) return fail(c, HPZ_EINVAL, "null adam");
  if (!(a->lr >= 0) || !(a->beta1 >= 0 && a->beta1 < 1) || !(a->beta2 >= 0 && a->beta2 < 1) || !(a->eps > 0) ||
      !(a->weight_decay >= 0))
    return fail(c, HPZ_EINVAL, "bad Adam hyper-parameters");
  return HPZ_OK;
}

// Device epochs: the per-step Adam scalars as a device table (Adam step k at [k - 1]),
// computed exactly like build_adam's host path, up to the step from which they no longer
// change in fp32.  Rebuilt (synchronously) when the hyper-parameters change; not while a
// stream is being captured.
static int adam_table(hpz_ctx* c, const hpz_adam* a, cudaStream_t s) {
  const double key[4] = {a->lr, a->beta1, a->beta2, (double)c->adam_base};
  if (c->adam_tab && !std::memcmp(key, c->adam_tab_key, sizeof key)) return HPZ_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  HPZ_CUDA(c, cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    return fail(c, HPZ_ESTATE, "device epochs: run one step with these Adam hyper-parameters before capturing");
  std::vector<float2> tab;
  constexpr int64_t kMax = 1 << 22;
  const float lr_f = (float)a->lr;
  for (int64_t k = 1;; ++k) {
    const double bc1 = 1.0 - std::pow(a->beta1, (double)k);
    const double bc2 = 1.0 - std::pow(a->beta2, (double)k);
    const float2 v = make_float2((float)(a->lr / bc1), (float)std::sqrt(bc2));
    tab.push_back(v);
    if (v.x == lr_f && v.y == 1.0f) break;   // constant from here on (monotone, rounded)
    if (k == kMax) return fail(c, HPZ_EINVAL, "device epochs: beta1/beta2 too close to 1 for the scalar table");
  }
  if (c->adam_tab) cudaFree(c->adam_tab);
  c->adam_tab = nullptr;
  HPZ_CUDA(c, cudaMalloc(&c->adam_tab, tab.size() * sizeof(float2)));
  HPZ_CUDA(c, cudaMemcpy(c->adam_tab, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  c->adam_tab_len = (int64_t)tab.size();
  std::memcpy(c->adam_tab_key, key, sizeof key);
  return HPZ_OK;
}

static int build_adam(hpz_ctx* c, int layer, const hpz_adam* a, AdamParams& p, cudaStream_t s) {
  Layer& L = c->layers[layer];
  const int64_t tad = a->step > 0 ? a->step : c->adam_base + c->t + 1;    // 1-based Adam count (R24)
  const double bc1 = 1.0 - std::pow(a->beta1, (double)tad);
  const double bc2 = 1.0 - std::pow(a->beta2, (double)tad);
  char* ar = c->arena[c->rank];
  p = AdamParams{};
  p.w = reinterpret_cast<float*>(ar + L.off_master);
  p.m = reinterpret_cast<float*>(ar + L.off_m);
  p.v = reinterpret_cast<float*>(ar + L.off_v);
  p.g = reinterpret_cast<const float*>(ar + L.off_gshard);
  p.prim = ar + L.off_primary;
  p.prim_bf16 = c->dtype == HPZ_BF16;
  p.n_vec = L.shard / 4;
  p.beta1 = (float)a->beta1;
  p.beta2 = (float)a->beta2;
  p.omb1 = (float)(1.0 - a->beta1);
  p.omb2 = (float)(1.0 - a->beta2);
  p.step_size = (float)(a->lr / bc1);
  p.bc2_sqrt = (float)std::sqrt(bc2);
  p.eps = (float)a->eps;
  p.lr_wd = (float)(a->lr * a->weight_decay);
  if (c->dev_epoch && a->step <= 0) {   // scalars of the device step, from the table
    if (int rc = adam_table(c, a, s)) return rc;
    p.tab = c->adam_tab;
    p.tab_k0 = c->adam_base;
    p.tab_len = c->adam_tab_len;
  }
  const uint32_t t1 = c->lv(c->t + 1);
  if (!(c->fault & HPZ_FAULT_SKIP_E2))   // test-only fault: overwrite the primary under its readers
    for (int j = 0; j < c->world; ++j) p.wait.ptr[p.wait.n++] = c->flag(c->rank, F_FWD_DONE, layer, j);   // E2
  if (c->order == HPZ_ORDER_OFF || c->verify == HPZ_VERIFY_EXACT || c->alias_sec)
    for (int j = 0; j < c->world; ++j) p.wait.ptr[p.wait.n++] = c->flag(c->rank, F_BWDP_DONE, layer, j);   // E7
  p.wait.target = t1;
  p.done_ctr = c->ctr(C_ADAM, layer);
  if (!c->qwz_bits) {   // with qwZ the quantizer launched after Adam releases E1 (and emits)
    for (int j = 0; j < c->world; ++j) p.rel.ptr[p.rel.n++] = c->flag(j, F_PRIM_READY, layer, c->rank);   // E1
    if (c->verify != HPZ_VERIFY_NONE) p.fpe = fp_emit(c, layer, c->t + 1);
  }
  p.rel.value = c->lv(c->t + 2);
  p.sync = c->sync();
  return HPZ_OK;
}

// The call that completes step t: host t advances; with device epochs the device step
// counter advances too, after every kernel this call enqueued on `s`.
static int advance_step(hpz_ctx* c, cudaStream_t s) {
  c->t += 1;
  if (!c->dev_epoch) return HPZ_OK;
  cudaError_t e = launch_epoch_advance(c->epoch_word(), s);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "epoch advance launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  return HPZ_OK;
}

static int stepped(hpz_ctx* c, int layer, cudaStream_t s) {
  c->layers[layer].step_t = c->t;
  bool all = true;
  for (int i = 0; i < c->n_layers; ++i) all = all && c->layers[i].step_t == c->t;
  return all ? advance_step(c, s) : HPZ_OK;
}

static int step_one(hpz_ctx* c, int layer, const hpz_adam* a, cudaStream_t s) {
  Layer& L = c->layers[layer];
  if (L.rs_t != c->t) return fail(c, HPZ_ESTATE, "layer %d: step without its reduce-scatter at step %lld", layer, (long long)c->t);
  if (L.step_t == c->t) return fail(c, HPZ_ESTATE, "layer %d already stepped at step %lld", layer, (long long)c->t);
  AdamParams p;
  if (int rc = build_adam(c, layer, a, p, s)) return rc;
  cudaError_t e = launch_adam(p, grid_for(c, (p.n_vec + 511) / 512, c->ctas_per_sm), s);
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "adam launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  if (c->qwz_bits) return qwz_quantize(c, layer, c->lv(c->t + 2), s, c->verify != HPZ_VERIFY_NONE, c->t + 1);
  return HPZ_OK;
}

int hpz_step(hpz_ctx* c, int layer, const hpz_adam* a, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_adam(c, a)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (layer == -1) {
    for (int i = 0; i < c->n_layers; ++i)
      if (c->layers[i].rs_t != c->t || c->layers[i].step_t == c->t)
        return fail(c, HPZ_ESTATE, "layer %d not reduce-scattered (or already stepped) at step %lld", i, (long long)c->t);
    const int64_t t = c->t;
    for (int i = 0; i < c->n_layers; ++i) {
      if (int rc = step_one(c, i, a, s)) return rc;
      c->layers[i].step_t = t;
    }
    return advance_step(c, s);
  }
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = step_one(c, layer, a, s)) return rc;
  return stepped(c, layer, s);
}

int hpz_reduce_scatter_adam(hpz_ctx* c, int layer, const hpz_adam* a, void* stream) {
  if (int rc = check_ready(c)) return rc;
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = check_adam(c, a)) return rc;
  Layer& L = c->layers[layer];
  if (L.rs_t == c->t) return fail(c, HPZ_ESTATE, "layer %d already reduce-scattered at step %lld", layer, (long long)c->t);
  if (L.step_t == c->t) return fail(c, HPZ_ESTATE, "layer %d already stepped at step %lld", layer, (long long)c->t);
  RSParams r;
  AdamParams p;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  build_rs(c, layer, r);
  if (int rc = build_adam(c, layer, a, p, s)) return rc;
  if (!c->store_grad_shard) r.out = nullptr;
  if (c->qgz_bits && !c->slot_ready_sent[L.slot])
    if (int rc = qgz_quantize(c, layer, static_cast<cudaStream_t>(stream))) return rc;
  cudaError_t e = rs_launch(c, r, &p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(c, HPZ_ECUDA, "rs+adam launch: %s", cudaGetErrorString(e));
  c->launches += 1;
  if (c->qwz_bits)
    if (int rc = qwz_quantize(c, layer, c->lv(c->t + 2), s, c->verify != HPZ_VERIFY_NONE, c->t + 1)) return rc;
  rs_issued(c, layer);
  return stepped(c, layer, s);
}

int hpz_set_option(hpz_ctx* c, int option, int64_t value) {
  if (!c) return HPZ_EINVAL;
  switch (option) {
    case HPZ_OPT_STORE_GRAD_SHARD: c->store_grad_shard = value != 0; return HPZ_OK;
    case HPZ_OPT_CTAS_PER_SM:
      if (value < 1 || value > 32) return fail(c, HPZ_EINVAL, "ctas_per_sm must be in [1, 32]");
      c->ctas_per_sm = (int)value;
      return HPZ_OK;
    case HPZ_OPT_QGZ:
      if (c->registered) return fail(c, HPZ_ESTATE, "qgZ must be chosen before hpz_register_flat_params");
      if (value != 0 && value != 4) return fail(c, HPZ_EINVAL, "qgZ bits must be 0 (off) or 4");
      if (value && c->grad_bytes != 4) return fail(c, HPZ_EINVAL, "qgZ quantizes fp32 gradients");
      c->qgz_bits = (int)value;
      return HPZ_OK;
    case HPZ_OPT_MAX_CTAS:
      if (value < 0 || value > 1 << 20) return fail(c, HPZ_EINVAL, "max_ctas must be >= 0");
      c->max_ctas = (int)value;
      return HPZ_OK;
    case HPZ_OPT_QWZ:
      if (c->registered) return fail(c, HPZ_ESTATE, "qwZ must be chosen before hpz_register_flat_params");
      if (value != 0 && value != 8) return fail(c, HPZ_EINVAL, "qwZ bits must be 0 (off) or 8");
      c->qwz_bits = (int)value;
      return HPZ_OK;
    case HPZ_OPT_GRAD_DTYPE:
      if (c->registered) return fail(c, HPZ_ESTATE, "the gradient dtype must be chosen before hpz_register_flat_params");
      if (value != HPZ_F32 && value != HPZ_BF16) return fail(c, HPZ_EINVAL, "gradient dtype must be HPZ_F32 or HPZ_BF16");
      if (value == HPZ_BF16 && c->qgz_bits) return fail(c, HPZ_EINVAL, "qgZ quantizes fp32 gradients");
      c->grad_bytes = value == HPZ_BF16 ? 2 : 4;
      return HPZ_OK;
    case HPZ_OPT_BWD_CTAS:
    case HPZ_OPT_RS_CTAS:
      if (value < 0 || value > 1 << 20) return fail(c, HPZ_EINVAL, "CTA caps must be >= 0");
      (option == HPZ_OPT_BWD_CTAS ? c->bwd_ctas : c->rs_ctas) = (int)value;
      return HPZ_OK;
    case HPZ_OPT_DEVICE_EPOCH: {
      if (value != 0 && value != 1) return fail(c, HPZ_EINVAL, "device_epoch must be 0 or 1");
      if (!c->bound) return fail(c, HPZ_ESTATE, "device epochs need a bound arena");
      if (c->dev_epoch && value == 0)   // back to host epochs: take over the device's step count first
        if (int rc = hpz_resync_step(c)) return rc;
      // between steps, device idle: the device counter starts at the host's step
      HPZ_CUDA(c, cudaSetDevice(c->device));
      HPZ_CUDA(c, cudaDeviceSynchronize());
      const uint32_t t32 = (uint32_t)c->t;
      HPZ_CUDA(c, cudaMemcpy(c->epoch_word(), &t32, 4, cudaMemcpyHostToDevice));
      c->dev_epoch = value != 0;
      return HPZ_OK;
    }
    case HPZ_OPT_ALIAS_SECONDARY:
      if (c->registered) return fail(c, HPZ_ESTATE, "the secondary layout must be chosen before hpz_register_flat_params");
      if (value != 0 && value != 1) return fail(c, HPZ_EINVAL, "alias_secondary must be 0 or 1");
      c->alias_opt = value != 0;
      return HPZ_OK;
    case HPZ_OPT_COPY_BY_CALLER:
      if (value != 0 && value != 1) return fail(c, HPZ_EINVAL, "copy_by_caller must be 0 or 1");
      c->copy_by_caller = value != 0;
      return HPZ_OK;
    case HPZ_OPT_FAULT:
      if (value < 0 || value > (HPZ_FAULT_SKIP_E1 | HPZ_FAULT_SKIP_E2)) return fail(c, HPZ_EINVAL, "bad fault mask");
      c->fault = (int)value;
      return HPZ_OK;
    case HPZ_OPT_COPY_ENGINE:
      if (value != HPZ_COPY_LDG && value != HPZ_COPY_TMA) return fail(c, HPZ_EINVAL, "copy engine must be 0 (LDG) or 1 (TMA)");
      c->copy_engine = (int)value;
      return HPZ_OK;
    default: return fail(c, HPZ_EINVAL, "unknown option %d", option);
  }
}

}  // extern "C"
