/*
 * hpz.h — C ABI of libhpz: the ZeRO++ hpZ data-parallel hot path of
 * arXiv 2407.01614 ("Enhancing Stability for Large Language Models Training in
 * Constrained Bandwidth Networks"), written natively for B200 (sm_100a).
 *
 * Citations are PAPER.md:<line> (the paper's LaTeX source) with the algorithm /
 * equation they fall in.  DESIGN.md lists every reading (R1..R25) taken where
 * the paper is silent.
 *
 * What the library does (Algorithm 1):
 *   forward  : AllGather(L_i, P) of the primary 1/P shards
 *              + the rank's secondary 1/P' copy, Eq. (1)
 *              (one fused kernel: the same in-flight tile is stored twice)
 *   backward : AllGather(L_i, P') over the secondary shards of the rank's (virtual)
 *              node, ordered after the secondary write — the paper's fix
 *              ("Repeat wait Until MemcpyD2D on L_k,second finishes")
 *   gradients: ReduceScatter(∇L_i, P), fp32, fixed pairwise-by-rank order
 *   step     : partitioned Adam on the fp32 master shard + bf16 primary refresh PAPER.md:117
 * Cross-GPU data moves by P2P loads over NVLink peer mappings of every rank's
 * arena; ordering between ranks is carried by release/acquire epoch flags that
 * the writer pushes into the waiter's arena (edges E1..E6).
 *
 * Conventions (all functions):
 *   - Return HPZ_OK (0) or a negative hpz_status.  On error the context keeps a
 *     message readable with hpz_last_error(); the call has no other effect.
 *   - Hot-path calls are host-asynchronous: they validate, enqueue kernels on the
 *     caller's stream and return.  They never block on the device.  A device-side
 *     wait that exceeds the timeout (hpz_set_timeout) records an error word; the
 *     next call on the context returns HPZ_ETIMEOUT and all later waits are
 *     skipped so a broken run cannot hang the GPU.
 *   - Streams are cudaStream_t values passed as void* (NULL = legacy default).
 *   - Device pointers are CUDA device (or managed) addresses on the context's
 *     device; "host" pointers may be pageable or pinned.
 *   - All ranks of a world must make the same sequence of hot-path calls
 *     (SPMD).  Calls of one rank may be spread over several streams: the
 *     library's flags order every cross-GPU hazard, and the caller's streams order
 *     the library against its own compute.
 *   - Ownership: the library allocates exactly one device arena per context
 *     (hpz_arena_alloc) or borrows a caller-provided one (hpz_bind), plus — with
 *     HPZ_OPT_DEVICE_EPOCH only — a small table of Adam scalars; full_out buffers
 *     always belong to the caller.
 */
#ifndef HPZ_H
#define HPZ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define HPZ_API __attribute__((visibility("default")))
#else
#define HPZ_API
#endif

#define HPZ_VERSION 1
#define HPZ_MAX_WORLD 16          /* P <= 16 ranks */
#define HPZ_IPC_HANDLE_BYTES 64   /* sizeof(cudaIpcMemHandle_t) */

typedef struct hpz_ctx hpz_ctx;   /* opaque; one per (process, GPU, rank) */

typedef enum {
  HPZ_OK = 0,
  HPZ_EINVAL = -1,    /* bad argument (SPEC invalid-argument)                       */
  HPZ_ESTATE = -2,    /* call out of lifecycle order (SPEC lifecycle/invalid-program) */
  HPZ_ECUDA = -3,     /* a CUDA runtime call failed; message names it              */
  HPZ_ETIMEOUT = -4,  /* a device-side flag wait timed out (peer missing / deadlock); the
                         message names the first flag that timed out (edge, layer or
                         gradient slot, source rank, value seen vs needed) */
  HPZ_ENOMEM = -5     /* arena allocation failed                                    */
} hpz_status;

typedef enum { HPZ_F32 = 0, HPZ_BF16 = 1 } hpz_dtype;

/* Ordering scheme (Table 1 columns):
 *  FIXED : modified hpZ, the paper's fix — backward gathers wait for the secondary write.
 *  STOCK : stock ZeRO++ hpZ, the bug reproduced on purpose — the secondary is written by
 *          a separate copy on a side stream after the forward gather, optionally preceded
 *          by a poison fill (torch.empty analog) and a delay, and backward
 *          gathers do not wait for it.
 *  OFF   : no hpZ (plain ZeRO-3) — no secondary; backward gathers over all P primaries.
 *  PAPER : the paper's own fix, literally (Alg. 1 blue lines): the stock side-stream copy,
 *          then hpz_bwd_gather blocks the HOST until that layer's copy finished before it
 *          enqueues the gather (plus the device-side acquire of the node peers' copies that
 *          P2P pulls need).  Correct like FIXED; kept to measure the host stall FIXED avoids. */
typedef enum { HPZ_ORDER_FIXED = 0, HPZ_ORDER_STOCK = 1, HPZ_ORDER_OFF = 2, HPZ_ORDER_PAPER = 3 } hpz_order;

/* Stale-parameter detection (a7):
 *  NONE        : off.
 *  FINGERPRINT : an order-independent 64-bit checksum of every gathered 16-byte word is
 *                accumulated by the forward and the backward gather of each layer; a
 *                layer whose two checksums differ counts one fp_mismatch (E3/E4: the
 *                backward read stale / half-written secondaries).  The kernel that writes
 *                a primary shard (Adam, the qwZ quantizer, load) also emits the checksum
 *                of the words it wrote into every reader's slot for the step that will
 *                gather them; a forward gather whose checksum differs from the owners'
 *                counts one fp_fwd_mismatch (E1/E2: the forward read pre-step or
 *                half-updated primaries).  Cheap; on in the bench.
 *  EXACT       : the backward gather additionally reads every element's owner primary
 *                and counts elements whose bits differ (mismatches) and NaN elements
 *                read (nan_reads).  Test/stress mode; doubles backward traffic. */
typedef enum { HPZ_VERIFY_NONE = 0, HPZ_VERIFY_FINGERPRINT = 1, HPZ_VERIFY_EXACT = 2 } hpz_verify;

/* Which per-layer arena buffer hpz_buffer() returns. */
typedef enum {
  HPZ_BUF_PRIMARY = 0,    /* param dtype, shard elements          */
  HPZ_BUF_MASTER = 1,     /* fp32, shard                          */
  HPZ_BUF_ADAM_M = 2,     /* fp32, shard                          */
  HPZ_BUF_ADAM_V = 3,     /* fp32, shard                          */
  HPZ_BUF_GRAD_SHARD = 4, /* fp32, shard: reduce-scatter output   */
  HPZ_BUF_SECONDARY = 5,  /* param dtype, sec_shard elements      */
  HPZ_BUF_GRAD_SLOT = 6   /* fp32, numel_pad: full local gradient */
} hpz_buffer_kind;

/* Adam hyper-parameters (the paper names no optimizer; reading R8).  Bias corrections
 * are evaluated in double on the host from the 1-based step count and rounded once
 * to fp32.  step == 0 means "use the context's step counter + 1". */
typedef struct {
  double lr, beta1, beta2, eps, weight_decay;
  int64_t step;
} hpz_adam;

/* Layout of one flat layer buffer (a1).  Eq. (1), with the padding
 * reading R2: numel_pad = ceil(numel / (P*A)) * P*A, shard = numel_pad/P,
 * sec_shard = numel_pad/P'.  Offsets are byte offsets into every rank's arena (all
 * ranks share one layout). */
typedef struct {
  int64_t numel, numel_pad, shard, sec_shard;
  uint64_t off_primary, off_master, off_m, off_v, off_grad_shard, off_secondary, off_grad_slot;
  int32_t grad_slot;
  int32_t _pad;
} hpz_layer_info_t;

typedef struct {
  uint64_t mismatches;      /* EXACT: elements e < numel whose backward-gathered bits != W_t */
  uint64_t nan_reads;       /* EXACT: NaN elements returned by backward gathers             */
  uint64_t fp_mismatches;   /* FINGERPRINT: layers whose fwd/bwd checksums differed         */
  uint64_t fp_checked;      /* FINGERPRINT: layer-gathers compared                          */
  uint64_t timeouts;        /* device flag waits that timed out                              */
  uint64_t launches;        /* kernels this context launched (host count)                   */
  uint64_t fp_fwd_mismatches; /* FINGERPRINT: forward gathers whose checksum != the owners'   */
  uint64_t fp_fwd_checked;    /* FINGERPRINT: forward gathers compared with the owners'       */
} hpz_counters_t;

/* ---- lifecycle ------------------------------------------------------------------ */

/* Create a context for global rank `rank` of a world of `world` ranks split into
 * consecutive virtual nodes of `node_size` = P' ranks (readings R3, R4: node
 * n(r) = r / P', local slice l(r) = r mod P').  Calls cudaSetDevice(device).
 * EINVAL: world not in [1,16], node_size does not divide world, rank not in
 * [0,world), device invalid.  device == -1 creates a host-only context that supports
 * only register/layer_info/finalize (layout queries without a GPU; no CUDA calls).
 * *out is owned by the caller; free with hpz_finalize. */
HPZ_API int hpz_init(int world, int node_size, int rank, int device, hpz_ctx** out);

/* Register the model as n_layers flat buffers (one per ZeRO-3 module)
 * of numel[i] elements each, parameters stored as param_dtype (HPZ_BF16 or HPZ_F32),
 * padded to a multiple of world*align_elems (align_elems: power of two, >= 8 and a
 * multiple of 16/elem_size; 256 recommended).  n_grad_slots full-length fp32 gradient
 * slots are laid out (layer i uses slot i % n_grad_slots; n_grad_slots == n_layers
 * gives every layer its own).  Writes the arena size every rank must provide.
 * Once per context (ESTATE if repeated); EINVAL on bad sizes. */
HPZ_API int hpz_register_flat_params(hpz_ctx* ctx, int n_layers, const int64_t* numel, int param_dtype,
                             int64_t align_elems, int n_grad_slots, uint64_t* arena_bytes);

/* Allocate this rank's arena (cudaMalloc, arena_bytes), zero its flag/counter region
 * and export a CUDA IPC handle (HPZ_IPC_HANDLE_BYTES bytes written to ipc_handle_out)
 * for peers in other processes.  ESTATE before register; ENOMEM on failure. */
HPZ_API int hpz_arena_alloc(hpz_ctx* ctx, void* ipc_handle_out);

/* Open the IPC handles of all ranks (world * HPZ_IPC_HANDLE_BYTES bytes, rank order;
 * the own entry is ignored) as NVLink peer mappings and bind them.  Synchronous.
 * The caller must barrier all ranks after every rank returned, before any hot-path
 * call.  ECUDA if a peer mapping fails (no P2P between the GPUs). */
HPZ_API int hpz_arena_open(hpz_ctx* ctx, const void* all_ipc_handles);

/* Alternative to hpz_arena_open: bind caller-provided arena base pointers of all ranks
 * (arena_ptrs[world], each >= arena_bytes, mapped in this process, 256-byte aligned).
 * arena_ptrs[rank] is this rank's own arena; if the library did not allocate it, its
 * flag region is zeroed here (synchronously).  Borrowed for the context lifetime.
 * Used e.g. for single-process emulation of several ranks on one GPU. */
HPZ_API int hpz_bind(hpz_ctx* ctx, void* const* arena_ptrs);

/* Release the arena (if allocated here), peer mappings, streams and the context. */
HPZ_API int hpz_finalize(hpz_ctx* ctx);

/* ---- inspection ------------------------------------------------------------------- */

HPZ_API int hpz_layer_info(const hpz_ctx* ctx, int layer, hpz_layer_info_t* out);
/* Device pointer of rank `rank`'s arena as mapped in this process. */
HPZ_API int hpz_arena_ptr(const hpz_ctx* ctx, int rank, void** out);
/* Device pointer + element count of one per-layer buffer of this rank's arena. */
HPZ_API int hpz_buffer(const hpz_ctx* ctx, int layer, int kind, void** dev_ptr, int64_t* numel);
/* The step t the next forward gather belongs to (0-based). */
HPZ_API int hpz_current_step(const hpz_ctx* ctx, int64_t* t);
/* Device epochs only (HPZ_OPT_DEVICE_EPOCH): after replaying a captured step graph, set the
 * host's step bookkeeping to the device step counter (synchronizes the device).  Call
 * between complete steps, before issuing hot-path calls eagerly again or capturing anew. */
HPZ_API int hpz_resync_step(hpz_ctx* ctx);
/* Read (synchronising the device) and optionally reset the detection counters. */
HPZ_API int hpz_counters(hpz_ctx* ctx, hpz_counters_t* out, int reset);
HPZ_API const char* hpz_last_error(const hpz_ctx* ctx);
HPZ_API int hpz_version(void);

/* ---- configuration ------------------------------------------------------------------ */

/* Ordering scheme (see hpz_order); stock_delay_us delays the stock / paper secondary
 * copy on its side stream, stock_poison != 0 fills the secondary with quiet NaNs first
 * (bf16 0x7FC0 / f32 0x7FC00000, reading R16).  Must be identical on all ranks and
 * changed only between steps (FIXED, PAPER and OFF may follow each other directly; after
 * STOCK, whose side-stream copy is ordered with nothing by design, synchronize the device
 * before the next step). */
HPZ_API int hpz_set_order(hpz_ctx* ctx, int order, int stock_delay_us, int stock_poison);
HPZ_API int hpz_set_verify(hpz_ctx* ctx, int mode);
/* Device-side flag wait timeout in seconds (default 20). */
HPZ_API int hpz_set_timeout(hpz_ctx* ctx, double seconds);

/* ---- initial state ------------------------------------------------------------------ */

/* Load layer `layer`'s initial parameters from a full fp32 DEVICE buffer of numel elements: master shard = the rank's slice (zero padding), m = v = 0,
 * primary = bf16_rne(master) (or an fp32 copy).  Releases E1 for step 0.  Must precede
 * the layer's first forward gather. */
HPZ_API int hpz_load_master(hpz_ctx* ctx, int layer, const float* full_fp32, void* stream);

/* Same, with the parameters produced on the device by the seeded counter-based generator
 * of DESIGN.md §6 (value(e) = (int(mix(key + (e+1)*golden) >> 40) - 2^23) * 2^-23 * scale
 * for e < numel, 0 in padding); key is the 64-bit stream key computed by the caller. */
HPZ_API int hpz_synth_master(hpz_ctx* ctx, int layer, uint64_t key, float scale, void* stream);

/* Resume from a checkpoint: this rank's master / Adam m / Adam v shards of
 * `layer` (fp32, `shard` elements each, host or device pointers, as read through
 * hpz_buffer) and the number of Adam steps already taken (bias corrections continue from
 * adam_steps_done + 1).  Refreshes the primary (RNE) and releases E1 like hpz_load_master;
 * must precede the layer's first gather on this context. */
HPZ_API int hpz_load_state(hpz_ctx* ctx, int layer, const float* master, const float* m, const float* v,
                           int64_t adam_steps_done, void* stream);

/* ---- hot path ------------------------------------------------------------------------ */

/* Forward gather of layer `layer` at the current step t (Alg. 1 PAPER.md:101,
 * AllGather(L_i, P)): full_out[numel_pad] (param dtype, device, caller-owned,
 * 16-byte aligned) = concatenation of the P primary shards, each pulled over NVLink.
 * FIXED: the same tiles are also stored into this rank's secondary slice
 * l(r) (Eq. (1)) after the node peers' backward reads of step t-1 are done
 * (E4); releases SEC_READY (E3) to the node and FWD_DONE (E2) to every owner.
 * STOCK: the secondary is written by a side-stream copy instead (no ordering edge).
 * OFF: no secondary. */
HPZ_API int hpz_fwd_gather(hpz_ctx* ctx, int layer, void* full_out, void* stream);

/* ORDER_STOCK / ORDER_PAPER with HPZ_OPT_COPY_BY_CALLER: enqueue Alg. 1's "L_i,second <-
 * empty(|L_i|/P'); Copy to L_i,second (Async MemcpyD2D)" for this step's
 * forward-gathered full buffer of `layer`, on the context's side stream after the work
 * already enqueued on `stream` (optional poison fill and delay first, hpz_set_order).  The
 * copy reads that full buffer after the call returns; later hpz gathers into the same buffer
 * wait for it, other writes by the caller must be ordered after it by the caller.  ESTATE
 * outside those orders / without the option, before the layer's forward gather of the step,
 * or twice in a step.  No-op when the secondary is aliased (P' = P). */
HPZ_API int hpz_secondary_copy(hpz_ctx* ctx, int layer, void* stream);

/* Backward gather of layer `layer` at step t (Alg. 1, AllGather(L_i, P')):
 * full_out[numel_pad] = concatenation of the P' secondaries of this rank's node.
 * FIXED: each source is read only after its owner released SEC_READY for step t — the
 * paper's fix as a device-side acquire.  OFF: gathers the P
 * primaries.  ESTATE if the layer's forward gather of step t was not issued. */
HPZ_API int hpz_bwd_gather(hpz_ctx* ctx, int layer, void* full_out, void* stream);

/* The gradient slot (fp32 — or bf16 with HPZ_OPT_GRAD_DTYPE — numel_pad elements, device)
 * the caller fills with this rank's
 * local gradient of `layer` (zero in padding).  Enqueues on `stream` the wait for every
 * rank's reduce-scatter of the slot's previous use (E6) before returning the pointer. */
HPZ_API int hpz_grad_buffer(hpz_ctx* ctx, int layer, void** grad_slot, void* stream);

/* hpz_grad_buffer + copy of n <= numel gradient values (fp32 or bf16) from `src` (host or device) into the
 * slot, zero-filling [n, numel_pad).  The end-to-end entry point for host gradients. */
HPZ_API int hpz_grad_upload(hpz_ctx* ctx, int layer, const void* src, int64_t n, void* stream);

/* hpz_grad_buffer + fill the slot on the device with the seeded generator (kind 0:
 * uniform*scale, 1: dyadic grid), zero in padding. */
HPZ_API int hpz_synth_grads(hpz_ctx* ctx, int layer, uint64_t key, float scale, int kind, void* stream);

/* Optional: publish "my gradient slot of `layer` is written" (E5) early (with qgZ: after
 * quantizing it).  Done implicitly by hpz_reduce_scatter if not called for this use. */
HPZ_API int hpz_grads_ready(hpz_ctx* ctx, int layer, void* stream);

/* Reduce-scatter of layer `layer` (Alg. 1, ReduceScatter(∇L_i, P)): the
 * grad shard (arena, fp32, shard elements) = (Σ_j G_j[r*s + e]) * (1/P), summed in the
 * fixed pairwise-by-rank association (R7) over the P ranks' slots pulled over NVLink.
 * Waits for every rank's E5, releases E6. */
HPZ_API int hpz_reduce_scatter(hpz_ctx* ctx, int layer, void* stream);

/* Partitioned Adam (Alg. 1, optimizer.step(); R8) on layer `layer`'s shard
 * (layer = -1: all layers), then primary = bf16_rne(master); waits until every rank
 * finished reading this primary for step t (E2) and releases PRIMARY_READY for t+1
 * (E1).  The step counter t advances once every layer has been stepped.  ESTATE if the
 * layer's reduce-scatter of step t was not issued. */
HPZ_API int hpz_step(hpz_ctx* ctx, int layer, const hpz_adam* adam, void* stream);

/* Fused reduce-scatter + partitioned Adam of one layer (a5 + a6 in one kernel): the
 * fixed-order reduced gradient feeds the Adam update of the same shard elements in
 * registers (the per-layer optimizer step of ZeRO-3 overlapped with the backward pass;
 * mathematically identical to hpz_reduce_scatter + hpz_step, bit for bit).  Waits E5,
 * E2 (+E7); releases E6 and E1(t+1).  The grad shard is stored only if
 * HPZ_OPT_STORE_GRAD_SHARD is on (default on).  Counts as both calls for the layer. */
HPZ_API int hpz_reduce_scatter_adam(hpz_ctx* ctx, int layer, const hpz_adam* adam, void* stream);

/* Tuning / behaviour options (identical on all ranks). */
typedef enum {
  HPZ_OPT_STORE_GRAD_SHARD = 0,  /* 0/1: fused RS+Adam writes the reduced gradient shard */
  HPZ_OPT_CTAS_PER_SM = 1,       /* 1..32: persistent-grid CTAs per SM of the LDG/STG kernels */
  HPZ_OPT_COPY_ENGINE = 2,       /* HPZ_COPY_TMA (default) or HPZ_COPY_LDG */
  HPZ_OPT_QGZ = 3,               /* 0 (default) or 4: ZeRO++ qgZ (Alg. 1 comment
                                    PAPER.md:114 "Replaced with INT4 AllToAll if with qgZ").
                                    The reduce-scatter quantizes this rank's gradient slot
                                    blockwise to INT4 (64-element blocks, fp32 min + scale,
                                    round-half-even codes; reading R26) and the owner pulls
                                    every rank's codes of its shard (0.625 B/elem instead of
                                    4), dequantizes (min + code*scale) and reduces in the R7
                                    order.  Set BEFORE hpz_register_flat_params (it sizes the
                                    arena); needs align_elems % 256 == 0.  With qgZ,
                                    hpz_grads_ready also quantizes. */
  HPZ_OPT_GRAD_DTYPE = 4,        /* HPZ_F32 (default) or HPZ_BF16: gradient slots hold
                                    bf16; the reduce-scatter converts (exactly) to fp32 and
                                    reduces in fp32 in the R7 order — half the NVLink bytes.
                                    Set before hpz_register_flat_params; not with qgZ. */
  HPZ_OPT_QWZ = 5,               /* 0 (default) or 8: ZeRO++ qwZ ("quantizes weights
                                    before AllGather"; reading R28): after every
                                    optimizer step (and at load) the owner quantizes its primary
                                    shard blockwise to INT8 (256-element blocks, fp32 min +
                                    scale, round-half-even codes) and the forward gather pulls
                                    codes (1 + 8/256 B/elem instead of 2), dequantizes
                                    (min + code*scale, then RNE to the param dtype) and writes
                                    the full buffer and the secondary; the backward gather is
                                    unchanged and returns the same values.  Needs align_elems
                                    % 256 == 0; not with EXACT verification or ORDER_OFF.  Set
                                    before hpz_register_flat_params. */
  HPZ_OPT_MAX_CTAS = 6,          /* cap on the CTAs of every launch (0 = whole GPU): bounds the SMs
                                    the collectives occupy while compute overlaps them (f3) */
  HPZ_OPT_BWD_CTAS = 10,         /* CTA cap of the backward gathers (0 = none) and ... */
  HPZ_OPT_RS_CTAS = 11,          /* ... of the reduce-scatters: with caps summing to at most the
                                    SM count, a backward gather on one stream and a
                                    reduce-scatter on another run side by side (no kernel of
                                    either waits on the other, so they may share the GPU) */
  HPZ_OPT_DEVICE_EPOCH = 13,     /* 0 (default) / 1: the rank's step counter lives in device
                                    memory and every kernel derives its flag epochs (and the
                                    Adam bias-correction scalars, from a host-filled table) from
                                    it, so a whole step can be captured in a CUDA graph and
                                    replayed (SURVEY §8(b) conventions).  The call that
                                    completes a step (last hpz_step / hpz_reduce_scatter_adam)
                                    advances the counter on its stream, so every other call of
                                    the step must be stream-ordered before it and the next
                                    step's calls after it (one graph replay after another on
                                    one stream does this).  ORDER_FIXED / ORDER_OFF only (the
                                    stock / paper side-stream copies cannot be captured).  Set
                                    between steps with the device idle; bound arenas only. */
  HPZ_OPT_FAULT = 14,            /* TEST ONLY, 0 = off: HPZ_FAULT_* bits remove an ordering
                                    edge on purpose to prove the detector sees the violation */
  HPZ_OPT_ALIAS_SECONDARY = 15,  /* 1 (default) / 0, before hpz_register_flat_params.  With
                                    P' = P (one node) the secondary slice of a rank IS its primary
                                    shard (Eq. (1) with P' = P): the arena stores no
                                    second copy, the forward gather writes no secondary and the
                                    backward gather reads the node's primaries (E1 acquire, E7
                                    release; every order behaves so, the stock race included).
                                    0 keeps a separate secondary at P' = P — needed only to
                                    reproduce the stock / paper copy on a one-node world.  No
                                    effect with qwZ (its secondary holds dequantized weights). */
  HPZ_OPT_COPY_BY_CALLER = 16    /* 0 (default) / 1, ORDER_STOCK / ORDER_PAPER: hpz_fwd_gather
                                    does not enqueue the secondary copy; the caller issues it with
                                    hpz_secondary_copy where Alg. 1 does (after L_i.forward(),
                                    PAPER.md:103-105) — e.g. to reproduce which backward gathers a
                                    prefetching schedule races. */
} hpz_option;
#define HPZ_FAULT_SKIP_E1 1   /* forward gathers read primaries without acquiring PRIMARY_READY */
#define HPZ_FAULT_SKIP_E2 2   /* Adam overwrites the primary without waiting for its readers   */
/* Copy engine of the gathers and the reduce-scatter: TMA 1-D bulk copies through a
 * shared-memory stage ring (cp.async.bulk, one persistent CTA per SM), or 16-byte
 * LDG/STG streams (several CTAs per SM).  EXACT verification always uses LDG/STG. */
typedef enum { HPZ_COPY_LDG = 0, HPZ_COPY_TMA = 1 } hpz_copy_engine;
HPZ_API int hpz_set_option(hpz_ctx* ctx, int option, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* HPZ_H */
