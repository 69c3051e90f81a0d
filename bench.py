#!/usr/bin/env python
"""Benchmark of the hpZ hot path (arXiv 2407.01614, Algorithm 1) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model falcon7b] [--impl hpz|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = one pass of the whole hot path over the model's flat layer buffers:
forward gather (+ fused secondary write) of every layer, backward gather +
reduce-scatter of every layer in reverse order, partitioned Adam of every layer
(DESIGN.md §7).  Inputs (parameters, optimizer state, gradients) are resident in HBM
before the timed region; gradients are synthetic (the model's backward compute is out
of scope).  The N GPUs form a world of P = N ranks split into 2 virtual nodes of
P' = N/2 (P' = 1 at N = 1).

Rank 0 prints ONE JSON line.  `value` = whole-job gather+reduce-scatter throughput:
Σ over ranks of the collectives' algorithmic bytes per step (AllGather output bytes of
the forward and backward gathers + ReduceScatter input bytes, the nccl-tests "algbw"
convention) ÷ the max over ranks of the device time of the whole step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "hpZ gather+reduce-scatter NVLink GB/s per step; stale-param mismatches (must be 0)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--model", default="falcon7b")
    ap.add_argument("--node-size", type=int, default=None)
    ap.add_argument("--impl", default="hpz", choices=["hpz", "reference"])
    ap.add_argument("--order", default="fixed", choices=["fixed", "stock", "off"])
    ap.add_argument("--verify", default="fingerprint", choices=["none", "fingerprint", "exact"])
    ap.add_argument("--unfused", action="store_true",
                    help="separate reduce-scatter and Adam kernels (default: fused per-layer RS+Adam)")
    ap.add_argument("--ctas-per-sm", type=int, default=None)
    ap.add_argument("--copy-engine", default="tma", choices=["tma", "ldg"])
    ap.add_argument("--qgz", action="store_true", help="ZeRO++ qgZ: INT4 gradient all-to-all (SURVEY f1)")
    ap.add_argument("--qwz", action="store_true", help="ZeRO++ qwZ: INT8 weights in the forward gather (SURVEY f2)")
    ap.add_argument("--overlap-bwd", type=int, default=0,
                    help="run each layer's backward gather on a second stream, capped at this many CTAs, "
                         "beside the previous layer's reduce-scatter (capped at the remaining SMs); 0 = one stream")
    ap.add_argument("--grad-dtype", default="f32", choices=["f32", "bf16"],
                    help="gradient slot dtype (bf16: SURVEY f4, fp32 accumulation)")
    ap.add_argument("--grad-slots", type=int, default=0,
                    help="gradient slots (0 = one per layer, resident).  Fewer slots (large models) "
                         "regenerate each layer's gradient on the device inside the step (timed, "
                         "reported as grad_synth)")
    ap.add_argument("--trace", default=None, help="write a JSONL op trace (one line per hpz_* call) of the "
                    "instrumented breakdown steps to this file (per rank: FILE.rankR)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--graph", type=int, default=1,
                    help="1: device-side epochs, one whole step captured in a CUDA graph and replayed each timed "
                         "step (fixed/off orders); 0: every call issued eagerly")
    ap.add_argument("--graph-events", type=int, default=1,
                    help="graph mode: 1 = per-call timing events inside the captured (timed) graph; 0 = a plain "
                         "graph, per-call times from eager steps after the timed region")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-p2p-ceiling", action="store_true")
    ap.add_argument("--share-gpus", action="store_true",
                    help="FUNCTIONAL CHECK ONLY, not a measurement: rank r runs on GPU r %% device_count "
                         "(several time-sliced processes per GPU, gloo control plane, no NCCL baseline / "
                         "p2p ceiling), so the N-rank path runs on a box with fewer than N GPUs")
    ap.add_argument("--oracle-numel", type=int, default=0,
                    help="elements of the oracle's sample (0: 2^25/P; tests use small samples)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", ",".join(str(g) for g in self.gpus)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
            out, _ = self.p.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic():
    """Per-element DRAM traffic of each kernel from a committed `ncu --set full` capture
    (profiles/ncu_traffic.json), or {}."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return {}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def host_mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 8 << 30


class ExtEvent:
    """A timing event recorded as an EXTERNAL event-record node when the stream is being
    captured (cuEventRecordWithFlags(..., CU_EVENT_RECORD_EXTERNAL)): its timestamp is taken
    every time the graph replays, so per-call device times can be read from inside a
    CUDA-graph replay.  Same elapsed_time() interface as torch.cuda.Event."""
    _lib = None

    def __init__(self):
        import ctypes
        if ExtEvent._lib is None:
            ExtEvent._lib = ctypes.CDLL("libcuda.so.1")
        self._ct = ctypes
        self.h = ctypes.c_void_p()
        self._check(ExtEvent._lib.cuEventCreate(ctypes.byref(self.h), 0), "cuEventCreate")

    def _check(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"{what} failed: CUresult {rc}")

    def record(self, stream):
        self._check(ExtEvent._lib.cuEventRecordWithFlags(self.h, self._ct.c_void_p(stream.cuda_stream), 1),
                    "cuEventRecordWithFlags")

    def __del__(self):
        try:
            if ExtEvent._lib is not None and self.h:
                ExtEvent._lib.cuEventDestroy_v2(self.h)
        except Exception:          # noqa: BLE001  (interpreter shutdown)
            pass

    def elapsed_time(self, other):
        ms = self._ct.c_float()
        self._check(ExtEvent._lib.cuEventElapsedTime(self._ct.byref(ms), self.h, other.h), "cuEventElapsedTime")
        return ms.value


# ----------------------------------------------------------------------------- oracle legs
def oracle_sample_numel(world, override=0):
    """The bounded sample of the workload the oracle is timed on: the first S elements of
    one flat layer, S = 2^25 / P (rounded to whole P*256 blocks) — the oracle simulates all P
    ranks, so its work per sample is ~constant in P.  Deterministic: both arms time exactly
    this sample."""
    q = world * 256
    return max(q, ((override or (1 << 25) // world)) // q * q)


def _oracle_worker(world, node_size, dtype, S, rounds, barrier, out_q):
    """One oracle process: build a one-layer HpzOracle of S elements (all P ranks), then
    `rounds` times: wait for every process, time one full step (fwd gather + secondary,
    bwd gather, RS, Adam)."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import hpz_oracle as O
    o = O.HpzOracle([S], world, node_size, align=256, param_dtype=dtype)
    for k in range(rounds):
        barrier.wait()
        t0 = time.time()
        o.step()
        out_q.put((k, t0, time.time()))


def oracle_bytes(world, S, dtype):
    """Algorithmic bytes of one sample step (same algbw accounting as the GPU arm)."""
    e = 2 if dtype == "bf16" else 4
    return world * (2 * S * e + 4 * S)


def oracle_time(world, node_size, dtype, S, procs, rounds=1):
    """Wall time of each of `rounds` rounds of `procs` concurrent one-step samples
    (processes, one per core)."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(procs)
    q = ctx.Queue()
    ps = [ctx.Process(target=_oracle_worker, args=(world, node_size, dtype, S, rounds, barrier, q))
          for _ in range(procs)]
    for p in ps:
        p.start()
    spans = [q.get() for _ in range(procs * rounds)]
    for p in ps:
        p.join()
    walls = []
    for k in range(rounds):
        sk = [(a, b) for kk, a, b in spans if kk == k]
        walls.append(max(b for _, b in sk) - min(a for a, _ in sk))
    return walls if rounds > 1 else walls[0]


def oracle_procs(world, S):
    """Processes for the all-cores leg: every core, bounded so the samples' memory (about
    80 B per element per simulated rank, measured) stays under half of MemAvailable."""
    per = 80 * S * world + (300 << 20)
    return max(1, min(host_cores(), int(host_mem_available() * 0.5 // per)))


def cpu_baseline(world, node_size, dtype, model_elems, override=0):
    """The oracle as it stands, timed on this box's host cores: one thread, then one
    process per core; plus the per-step time extrapolated to the whole model."""
    S = oracle_sample_numel(world, override)
    bytes1 = oracle_bytes(world, S, dtype)
    dt1 = oracle_time(world, node_size, dtype, S, 1)
    C = oracle_procs(world, S)
    dtc = oracle_time(world, node_size, dtype, S, C) if C > 1 else dt1
    v1 = bytes1 / dt1 / 1e9
    vc = C * bytes1 / dtc / 1e9
    step1 = model_elems / S * dt1
    return {"value": round(vc, 4), "unit": "GB/s", "cores": C, "kind": "oracle",
            "sample": f"oracle/hpz_oracle.py HpzOracle, one full step (fwd gather + secondary, bwd gather, RS, Adam) "
                      f"of the first {S} elements of one flat layer, all {world} rank(s) simulated (P={world}, "
                      f"P'={node_size}); {C} such samples in {C} concurrent processes ({dtc:.2f} s wall); "
                      f"numpy; same algbw byte accounting as the GPU arm; host has {host_cores()} cores",
            "single_thread": {"value": round(v1, 4), "unit": "GB/s", "cores": 1, "seconds": round(dt1, 3)},
            "extrapolated_step_s": {"single_thread": round(step1, 1), "all_cores": round(step1 * v1 / vc, 1),
                                    "note": "EXTRAPOLATED: (model elements / sample elements) x sample time"}}


# ----------------------------------------------------------------------------- main arm
def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n):
    """`python bench.py --gpus N` outside torchrun: start N ranks (one process per GPU)
    through torch.distributed.run on 127.0.0.1 and relay rank 0's JSON line; everything
    else the ranks print goes to stderr.  Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, text=True, cwd=ROOT)
    for line in p.stdout:
        s = line.strip()
        if s.startswith("{") and s.endswith("}"):
            print(s, flush=True)
        else:
            sys.stderr.write(line)
    return p.wait()


def step_bytes(numel_pad, shard, P, Pp, e, grad_dtype="f32", qgz=False, qwz=False, fused=True):
    """Algorithmic bytes per rank per step (SURVEY §8(d) per padded model
    element: forward gather 2(P-1)/P, backward 2(P'-1)/P', RS 4(P-1)/P of NVLink ingress,
    fused Adam 30/P of HBM).  numel_pad / shard: per layer.  Returns
      ag      AllGather output bytes (N̂·e), coll = 2·ag + fp32 RS input (the `value` bytes),
      rs_in   RS input bytes in the slot dtype, adam = the optimizer's HBM bytes,
      nvlink  per kernel: NVLink ingress (busbw convention; qgZ / qwZ: wire bytes),
      hbm     per kernel: every byte it reads or writes in this GPU's memory, incl. what it
              serves to peers,
      hbm_p1  per kernel at P = 1: the local copy / update bytes (the N = 1 roofline)."""
    N, S = sum(numel_pad), sum(shard)
    ag = N * e
    coll = 2 * ag + N * 4
    rs_in = N * (2 if grad_dtype == "bf16" else 4)
    rs_wire = rs_in * (0.625 / 4 if qgz else 1.0)          # qgZ: int4 codes + (min, scale) per 64
    fwd_wire = ag * ((1 + 8 / 256) / e if qwz else 1.0)     # qwZ: int8 codes + (min, scale) per 256
    adam = S * (30 if e == 2 else 32)
    sec = 0 if (Pp == P and not qwz) else ag / Pp           # P' == P: secondary is the primary
    rs_name = "reduce_scatter+adam" if fused else "reduce_scatter"
    nvlink = {"fwd_gather": fwd_wire * (P - 1) / P, "bwd_gather": ag * (Pp - 1) / Pp,
              "reduce_scatter": rs_wire * (P - 1) / P, "reduce_scatter+adam": rs_wire * (P - 1) / P, "adam": adam}
    hbm = {"fwd_gather": 2 * ag + sec,                      # serve primary; write out (+ secondary)
           "bwd_gather": 2 * ag,                            # serve secondary; write out
           # RS: my slot is read once in total (by its owners); fused Adam: w, m, v read +
           # written (24 B) and the primary refreshed (e); unfused: the fp32 shard written
           rs_name: rs_in + (S * (24 + e) if fused else S * 4)}
    hbm_p1 = {"fwd_gather": 2 * ag + sec, "bwd_gather": 2 * ag, "reduce_scatter": 2 * rs_in, "adam": adam,
              # fused at P=1: read grad slot 4 + w,m,v 12; write w,m,v 12 + primary e
              "reduce_scatter+adam": S * (28 + e)}
    ingress = nvlink["fwd_gather"] + nvlink["bwd_gather"] + nvlink["reduce_scatter"]
    return {"ag": ag, "coll": coll, "rs_in": rs_in, "adam": adam, "sec": sec, "nvlink": nvlink, "hbm": hbm,
            "hbm_p1": hbm_p1, "ingress": ingress}


def make_config(args, world, node_size, n_layers, n_params, n_slots):
    """The workload this line measures (identical for both arms)."""
    extra = {"share_gpus": "FUNCTIONAL CHECK: ranks time-slice shared GPUs; the timings are not "
                           "measurements"} if getattr(args, "share_gpus", False) else {}
    return {**extra, "workload": f"{args.model}-shaped flat parameter buffers ({n_layers} layers, "
                        f"{n_params} params), bf16 params + fp32 master/Adam",
            "world": world, "node_size": node_size, "virtual_nodes": world // node_size,
            "parallelism": f"hpZ dp{world} (P={world}, P'={node_size})", "order": args.order,
            "verify": args.verify, "copy_engine": args.copy_engine,
            "launch": ("one step captured in a CUDA graph (device-side epochs), replayed per timed step"
                       if args.graph and args.order in ("fixed", "off") else "eager calls"),
            "reduce_scatter": "pull" if world > 1 else "local",
            "overlap_bwd": (f"backward gathers on a second stream ({args.overlap_bwd} CTAs) beside "
                            f"the reduce-scatters") if args.overlap_bwd else None,
            "qgz": "int4 blockwise (64) gradient all-to-all; RS bytes counted as the fp32 "
                   "gradient bytes reduced, wire bytes 0.625 B/elem" if args.qgz else None,
            "grad_dtype": args.grad_dtype, "grad_slots": n_slots,
            "qwz": "int8 blockwise (256) weights in the forward gather; AG bytes counted as the "
                   "bf16 parameter bytes delivered" if args.qwz else None,
            "l2": "no flush: per-step working set >> 126 MB L2 (every layer buffer is "
                  "touched once per phase)",
            "value_def": "sum over ranks of AllGather output bytes (fwd+bwd) + ReduceScatter "
                         "input bytes per step (nccl-tests algbw bytes) / max-over-ranks device time "
                         "of the whole step (gathers, reduce-scatter and Adam)"}


def main():
    args = parse()
    under_launcher = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n_gpus = args.gpus if args.gpus is not None else world
    if args.impl == "reference":
        # the oracle arm needs no GPU ranks: rank 0 (or this lone process) simulates all N
        return reference_arm(args, n_gpus if not under_launcher else world, rank,
                             args.node_size or (n_gpus // 2 if n_gpus >= 2 else 1))
    if not under_launcher and n_gpus > 1:
        sys.exit(relaunch(n_gpus))
    if n_gpus != world:
        sys.exit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    node_size = args.node_size or (world // 2 if world >= 2 else 1)

    import torch
    import torch.distributed as dist
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200 import shapes
    from paper_2407_01614_b200.world import DistWorld, EmulatedWorld, max_over_ranks, sum_over_ranks
    from synth import inputs as S

    if args.share_gpus:
        local_rank %= torch.cuda.device_count()
        args.no_nccl = args.no_p2p_ceiling = True
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if args.share_gpus:
            dist.init_process_group("gloo")      # NCCL refuses two ranks on one device
        else:
            dist.init_process_group("nccl", device_id=dev)
    numels = shapes.numels(args.model)
    dtype = shapes.PARAM_DTYPE.get(args.model, "bf16")
    e = 2 if dtype == "bf16" else 4
    L = len(numels)

    n_slots = args.grad_slots if 0 < args.grad_slots < L else L
    if world > 1:
        W = DistWorld(numels, node_size, dtype=dtype, n_grad_slots=n_slots, device=local_rank, timeout_s=60.0,
                      qgz=args.qgz, grad_dtype=args.grad_dtype, qwz=args.qwz)
    else:
        W = EmulatedWorld(numels, 1, 1, dtype=dtype, n_grad_slots=n_slots, device=local_rank, timeout_s=60.0,
                          qgz=args.qgz, grad_dtype=args.grad_dtype, qwz=args.qwz)
    rc = W.ranks[0]
    ctx = rc.ctx
    H.hpz_set_order(ctx, args.order)
    H.hpz_set_verify(ctx, args.verify)
    fused = not args.unfused
    H.hpz_set_option(ctx, "store_grad_shard", 0 if fused else 1)
    if args.ctas_per_sm:
        H.hpz_set_option(ctx, "ctas_per_sm", args.ctas_per_sm)
    H.hpz_set_option(ctx, "copy_engine", H.COPY[args.copy_engine])
    stream = torch.cuda.Stream(device=dev)      # a non-default stream: CUDA graphs capture on it
    torch.cuda.set_stream(stream)
    use_graph = bool(args.graph) and args.order in ("fixed", "off")
    if use_graph:
        H.hpz_set_option(ctx, "device_epoch", 1)     # epochs from the device: a step can be replayed
    gstream = torch.cuda.Stream(device=dev) if args.overlap_bwd else stream   # backward gathers
    if args.overlap_bwd:
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        H.hpz_set_option(ctx, "bwd_ctas", args.overlap_bwd)
        H.hpz_set_option(ctx, "rs_ctas", n_sm - args.overlap_bwd)
    infos = rc.infos
    # resident inputs: initial params (device generator) and this rank's gradients
    for i in range(L):
        H.hpz_synth_master(ctx, i, S.stream_key(S.SEED_PARAMS, i, 0, 0), S.PARAM_SCALE, stream)
        if n_slots == L:
            H.hpz_synth_grads(ctx, i, S.stream_key(S.SEED_GRADS, i, 0, rank), S.GRAD_SCALE, 0, stream)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    nmax = max(x.numel_pad for x in infos)
    fwd_buf = torch.empty(nmax, dtype=tdt, device=dev)     # caller-owned full buffers, reused
    # per layer (repartition); with --overlap-bwd the gathers run ahead of the
    # reduce-scatters, so a small ring of buffers stands in for the backward compute's reads
    bwd_bufs = [torch.empty(nmax, dtype=tdt, device=dev) for _ in range(2 if args.overlap_bwd else 1)]
    adam = H.make_adam()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    copy_stream = torch.cuda.Stream(device=dev)

    def one_step(ev=None, grads_from=None):
        """ev: dict of per-call event lists (or None).  grads_from: pinned host buffer
        uploaded into every layer's gradient slot (end-to-end arm): the uploads run on a
        copy stream from the start of the step, in backward order, each reduce-scatter
        waiting only for its own layer's upload."""
        def rec(k, st=None, layer=None):
            if ev is not None:
                x = ExtEvent() if torch.cuda.is_current_stream_capturing() else torch.cuda.Event(enable_timing=True)
                x.record(stream if st is None else st)
                ev[k].append(x)
                if k.endswith("0"):
                    ev["_layer_" + k[:-1]].append(layer)
        up = {}
        if grads_from is not None:
            copy_stream.wait_stream(stream)
            for i in reversed(range(L)):
                H.hpz_grad_upload(ctx, i, grads_from.data_ptr(), infos[i].numel, copy_stream)
                up[i] = torch.cuda.Event()
                up[i].record(copy_stream)
        for i in range(L):
            rec("fwd0", layer=i)
            H.hpz_fwd_gather(ctx, i, fwd_buf.data_ptr(), stream)
            rec("fwd1")
        if gstream is not stream:
            gstream.wait_stream(stream)
        rs_done = {}
        for i in reversed(range(L)):
            if gstream is not stream and i + len(bwd_bufs) in rs_done:
                # buffer reuse: layer i+2's backward (here: its reduce-scatter) is done with it
                gstream.wait_event(rs_done[i + len(bwd_bufs)])
            rec("bwd0", gstream, layer=i)
            H.hpz_bwd_gather(ctx, i, bwd_bufs[i % len(bwd_bufs)].data_ptr(), gstream)
            rec("bwd1", gstream)
            if gstream is not stream:      # the layer's gradient exists only after its bwd gather
                done = torch.cuda.Event()
                done.record(gstream)
                stream.wait_event(done)
            if grads_from is not None:
                stream.wait_event(up[i])
            elif n_slots < L:    # shared slots: this layer's gradient is produced in the step
                rec("g0", layer=i)
                H.hpz_synth_grads(ctx, i, S.stream_key(S.SEED_GRADS, i, 0, rank), S.GRAD_SCALE, 0, stream)
                rec("g1")
            if args.qgz:
                rec("q0", layer=i)
                H.hpz_grads_ready(ctx, i, stream)      # qgZ: INT4-quantize my slot, publish E5
                rec("q1")
            rec("rs0", layer=i)
            if fused:
                H.hpz_reduce_scatter_adam(ctx, i, adam, stream)   # RS + this layer's Adam
            else:
                H.hpz_reduce_scatter(ctx, i, stream)
            rec("rs1")
            if gstream is not stream:
                rs_done[i] = torch.cuda.Event()
                rs_done[i].record(stream)
        if gstream is not stream:
            stream.wait_stream(gstream)
        if not fused:
            for i in range(L):
                rec("adam0", layer=i)
                H.hpz_step(ctx, i, adam, stream)
                rec("adam1")

    for _ in range(args.warmup):
        one_step()
    K = args.steps
    graph = None
    evs = {k: [] for k in ("fwd0", "fwd1", "bwd0", "bwd1", "rs0", "rs1", "adam0", "adam1", "q0", "q1", "g0", "g1")}
    evs.update({"_layer_" + k: [] for k in ("fwd", "bwd", "rs", "adam", "q", "g")})
    if use_graph:
        # capture the K timed steps (every layer's gathers and fused RS+Adam, K times) as ONE
        # CUDA graph with an external timing event around every call: each step reads its
        # flag epochs and Adam scalars from the device step counter, and the per-call device
        # times come from inside the timed replay itself
        torch.cuda.synchronize()
        l0 = H.hpz_counters(ctx)["launches"]
        graph = torch.cuda.CUDAGraph()
        t_ref = ExtEvent()
        with torch.cuda.graph(graph, stream=stream):
            t_ref.record(stream)
            for _ in range(K):
                one_step(evs if args.graph_events else None)
        graph_launches = H.hpz_counters(ctx)["launches"] - l0
        torch.cuda.synchronize()
    H.hpz_counters(ctx, reset=True)
    launches0 = H.hpz_counters(ctx)["launches"]
    clocks = ClockSampler(list(range(world)) if rank == 0 else [])
    barrier()
    if rank == 0:
        clocks.start()
    # timed region: K whole steps bracketed by two events (graph mode: one replay of the K-step
    # graph; eager mode: K steps without per-call events)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for _ in range(args.steps):
            one_step()
    t_end.record(stream)
    barrier()
    clk = clocks.stop() if rank == 0 else None
    barrier()        # rank 0 spent ~0.25 s stopping the sampler: realign before the breakdown steps
    cnt = H.hpz_counters(ctx)
    launches = graph_launches if graph is not None else cnt["launches"] - launches0
    if graph is not None:
        H.hpz_resync_step(ctx)    # host bookkeeping = the device step counter, for the eager steps below
    step_ms = t_start.elapsed_time(t_end) / K
    if graph is not None and args.graph_events:
        KB = K                    # per-call times of the timed steps themselves
    else:
        # eager mode: extra instrumented steps (events around every call) after the timed region
        KB = max(1, min(K, 5))
        t_ref = torch.cuda.Event(enable_timing=True)
        t_ref.record(stream)
        for _ in range(KB):
            one_step(evs)
        barrier()
    if args.trace:
        # JSONL op trace of the instrumented steps (one line per call; SURVEY §5 tracing)
        names = {"fwd": "hpz_fwd_gather", "bwd": "hpz_bwd_gather", "rs": "hpz_reduce_scatter" + ("_adam" if fused else ""),
                 "adam": "hpz_step", "q": "hpz_grads_ready(qgZ quantize)", "g": "hpz_synth_grads"}
        recs = []
        for k, nm in names.items():
            per_step = len(evs[k + "0"]) // KB if evs[k + "0"] else 0
            for idx, (a, b) in enumerate(zip(evs[k + "0"], evs[k + "1"])):
                recs.append({"rank": rank, "step": idx // max(per_step, 1), "op": nm, "layer": evs["_layer_" + k][idx],
                             "start_ms": round(t_ref.elapsed_time(a), 4), "dur_ms": round(a.elapsed_time(b), 4)})
        recs.sort(key=lambda r: r["start_ms"])
        with open(args.trace if world == 1 else f"{args.trace}.rank{rank}", "w") as f:
            for r in recs:
                f.write(json.dumps(r) + "\n")
    tot = {k: sum(a.elapsed_time(b) for a, b in zip(evs[k + "0"], evs[k + "1"])) / KB
           for k in ("fwd", "bwd", "rs", "adam", "q", "g")}
    P, Pp = world, node_size
    B = step_bytes([x.numel_pad for x in infos], [x.shard for x in infos], P, Pp, e, args.grad_dtype,
                   args.qgz, args.qwz, fused)
    ag_bytes, coll_bytes, rs_bytes, adam_bytes = B["ag"], B["coll"], B["rs_in"], B["adam"]

    vals = max_over_ranks([step_ms, tot["fwd"], tot["bwd"], tot["rs"], tot["adam"],
                           tot["fwd"] + tot["bwd"] + tot["rs"] + tot["q"], tot["q"], tot["g"]], device=dev)
    stats = sum_over_ranks([cnt["fp_mismatches"], cnt["mismatches"], cnt["nan_reads"], cnt["timeouts"],
                            cnt["fp_checked"], launches, cnt["fp_fwd_mismatches"], cnt["fp_fwd_checked"]], device=dev)
    step_ms, fwd_ms, bwd_ms, rs_ms, adam_ms, coll_ms, q_ms, g_ms = vals
    # whole-job throughput of the step: the collectives' algorithmic bytes of all ranks per
    # step / the max-over-ranks time of the whole step (incl. the optimizer)
    value = world * coll_bytes / (step_ms * 1e-3) / 1e9

    # ------------------------------------------------ roofline of the dominant kernel
    pk = peaks()
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    rs_name = "reduce_scatter+adam" if fused else "reduce_scatter"
    share = {"fwd_gather": fwd_ms, "bwd_gather": bwd_ms, rs_name: rs_ms}
    if not fused:
        share["adam"] = adam_ms
    dom = max(share, key=share.get)
    if world == 1:
        alg = B["hbm_p1"][dom]
        bound, peak, unit = "hbm", hbm_peak, "GB/s"
    else:
        alg = B["nvlink"][dom]
        if dom == "adam":
            bound, peak, unit = "hbm", hbm_peak, "GB/s"
        else:
            bound, peak, unit = "nvlink", 770.0, "GB/s"
    achieved = alg / (share[dom] * 1e-3) / 1e9          # per-launch bytes / per-launch time, summed over L launches
    traffic = traffic_alg = None
    traffic_src = None if world == 1 else (
        f"not captured for world {world} (P'={node_size}): the capture drives all P GPUs from one process under "
        f"ncu (tools/nvlink_bytes.py; ncu must not wrap the multi-rank bench) and exists for N = 2, 4 "
        f"(profiles/ncu_traffic.json)")
    tr = ncu_traffic().get(f"P{world}_{dom}")
    if tr and tr.get("node_size", node_size) != node_size:
        tr = None                                       # captured on another (P, P')
    nvl_rx = None
    if tr and not (args.qgz or args.qwz or args.grad_dtype != "f32"):
        # DRAM bytes of ONE captured launch (ncu) next to that launch's algorithmic bytes
        traffic, traffic_alg, traffic_src = tr["dram_bytes_per_launch"], tr["launch_alg_bytes"], tr["source"]
        if "nvlink_rx_bytes_per_launch" in tr:          # N > 1: the same capture's NVLink ingress
            nvl_rx = {"nvlink_rx_bytes_per_launch": tr["nvlink_rx_bytes_per_launch"],
                      "nvlink_alg_ingress_bytes": tr["nvlink_alg_ingress_bytes"],
                      "rx_over_alg": round(tr["nvlink_rx_bytes_per_launch"] / tr["nvlink_alg_ingress_bytes"], 4),
                      "traffic_is": tr["alg_bytes_are"]}
    roofline = {"bound": bound, "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_launch_alg_bytes": traffic_alg, "traffic_source": traffic_src,
                **({"traffic_nvlink": nvl_rx} if nvl_rx else {}),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if bound == "hbm" else
                "B200_PROFILING.md measured peer copy 770 GB/s per direction (900 nominal)",
                "alg_bytes_per_step": alg, "launches_per_step": L, "ms_per_step": round(share[dom], 4),
                "timing": (f"external CUDA events around every call inside the captured graph, read from the timed "
                           f"replay itself ({KB} steps), on the stream the kernels run on"
                           if graph is not None and args.graph_events else
                           f"CUDA events around every call of {KB} instrumented steps run right after the timed "
                           f"region (same config, eager issue), on the stream the kernels run on"),
                "share_of_step": round(share[dom] / max(fwd_ms + bwd_ms + rs_ms + adam_ms + q_ms + g_ms, 1e-9), 4)}

    # per-kernel table (north_star: per-step gather / reduce-scatter time, NVLink GB/s
    # against 900 per direction, HBM GB/s against the measured copy peak); algorithmic bytes
    # per rank and step: NVLink ingress as above; HBM = every byte each kernel must read or
    # write in this GPU's memory (incl. the shards it serves to peers)
    hbm_k, nv_k = B["hbm"], B["nvlink"]
    kernels = {}
    for k, ms in (("fwd_gather", fwd_ms), ("bwd_gather", bwd_ms), (rs_name, rs_ms)):
        if ms <= 0:
            continue
        nv = nv_k[k] / (ms * 1e-3) / 1e9
        hb = hbm_k[k] / (ms * 1e-3) / 1e9
        kernels[k] = {"ms_per_step": round(ms, 3), "nvlink_GB": round(nv_k[k] / 1e9, 3), "nvlink_GBps": round(nv, 1),
                      "nvlink_frac_of_770": round(nv / 770.0, 4), "nvlink_frac_of_900": round(nv / 900.0, 4),
                      "hbm_GB": round(hbm_k[k] / 1e9, 3), "hbm_GBps": round(hb, 1),
                      "hbm_frac_of_measured": round(hb / hbm_peak, 4)}

    # ------------------------------------------------ end-to-end arm (host buffers)
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        host = torch.empty(max(x.numel for x in infos), pin_memory=True,
                           dtype=torch.bfloat16 if args.grad_dtype == "bf16" else torch.float32)
        H.hpz_synth_grads(ctx, 0, S.stream_key(S.SEED_GRADS, 0, 0, rank), S.GRAD_SCALE, 0, stream)
        # fill the pinned buffer with this rank's synthetic gradient values (device generator)
        from paper_2407_01614_b200.world import buffer_view
        src = buffer_view(rc, 0, "grad_slot", "f32")
        if args.grad_dtype == "bf16":
            from paper_2407_01614_b200.world import device_view
            src = device_view(H.hpz_buffer(ctx, 0, "grad_slot")[0], infos[0].numel_pad, "bf16")
        host[: infos[0].numel].copy_(src[: infos[0].numel])
        one_step(grads_from=host)          # warm-up of the e2e path
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            one_step(grads_from=host)
            res = torch.empty(6, dtype=torch.int64)   # the step's result: detection counters, D2H
            c = H.hpz_counters(ctx)
            res[:] = torch.tensor([c["fp_mismatches"], c["mismatches"], c["nan_reads"], c["timeouts"],
                                   c["fp_checked"], c["launches"]])
        b.record(stream)
        barrier()
        e2e_ms = max_over_ranks([a.elapsed_time(b) / args.e2e_steps], device=dev)[0]
        e2e = {"value": round(world * coll_bytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": sum(x.numel for x in infos) * (2 if args.grad_dtype == "bf16" else 4),
               "d2h_bytes_per_step": 5 * 8,
               "ms_per_step": round(e2e_ms, 3),
               "note": "through the C ABI: every layer's gradient uploaded from pinned host memory "
                       "(hpz_grad_upload, on a copy stream overlapping the gathers) inside the timed "
                       "step; counters read back (hpz_counters); PCIe-bound"}

    # ------------------------------------------------ NCCL baseline (same collectives, same sizes)
    nccl = None
    if world > 1 and not args.no_nccl:
        nccl = nccl_baseline(infos, e, node_size, dev, tdt, args)
    ceiling = None
    if world > 1 and not args.no_p2p_ceiling:
        torch.cuda.synchronize()
        dist.barrier()
        ceiling = p2p_ceiling(world, rank)
        if ceiling:
            for k in kernels.values():
                k["nvlink_frac_of_measured_ceiling"] = round(k["nvlink_GBps"] / ceiling["pull_tma_GBps_per_gpu_avg"], 4)

    W.close()
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(world, node_size, dtype, sum(x.numel_pad for x in infos), args.oracle_numel)
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16 gathers / f32 reduce-scatter+Adam", "data": "synthetic",
            "config": make_config(args, world, node_size, L, sum(x.numel for x in infos), n_slots),
            "stale_param_mismatches": {"fingerprint_layers": int(stats[0]), "exact_elements": int(stats[1]),
                                       "nan_reads": int(stats[2]), "timeouts": int(stats[3]),
                                       "layers_checked": int(stats[4]),
                                       "fwd_vs_owner_fingerprint_layers": int(stats[6]),
                                       "fwd_layers_checked": int(stats[7]),
                                       "what": "timed steps; FINGERPRINT: backward vs forward gather of every "
                                               "layer (E3/E4) and forward gather vs the checksum the owners "
                                               "emitted when writing their primaries (E1/E2); EXACT: elements"},
            "breakdown_steps": KB,
            "breakdown_ms_per_step": {"fwd_gather": round(fwd_ms, 3), "bwd_gather": round(bwd_ms, 3),
                                      rs_name: round(rs_ms, 3), "adam": round(adam_ms, 3),
                                      "qgz_quantize": round(q_ms, 3), "grad_synth": round(g_ms, 3),
                                      "collectives": round(coll_ms, 3)},
            "fused_rs_adam": fused,
            "nvlink_ingress_GBps_per_gpu": round(B["ingress"] / (step_ms * 1e-3) / 1e9, 2) if world > 1 else None,
            "nvlink_frac_of_900": round(B["ingress"] / (step_ms * 1e-3) / 1e9 / 900, 4) if world > 1 else None,
            "collectives_only_GBps": round(world * coll_bytes / (coll_ms * 1e-3) / 1e9, 2),
            "roofline": roofline, "kernels": kernels,
            "cpu_baseline": cpu,
            "nccl_baseline": nccl,
            "p2p_ceiling": ceiling,
            "e2e": e2e,
            "gpu_launches": int(stats[5]),
            "clocks": clk,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def p2p_ceiling(world, rank):
    """The fabric's measured all-to-all pull ceiling: after the timed work,
    rank 0 runs tools/p2p_probe (every GPU TMA-pulls 512 MiB from every peer at once, the
    traffic pattern of these collectives) while the other ranks wait on the host (TCP store,
    no GPU work).  Returns {per-GPU ingress GB/s} or None."""
    import re
    import torch.distributed as dist
    store = dist.distributed_c10d._get_default_store()
    res = None
    if rank == 0:
        exe = os.path.join(ROOT, "tools", "p2p_probe")
        try:
            by_depth = {}
            for depth in (2, 3, 4):           # the ceiling: the best stage-ring depth
                out = subprocess.run([exe, str(world), "pull_tma", "512", "1", "32768", "0", "50", str(depth)],
                                     capture_output=True, text=True, timeout=120).stdout
                m = re.search(r"per-GPU GB/s: min ([0-9.]+) avg ([0-9.]+)", out)
                if m:
                    by_depth[depth] = (float(m.group(1)), float(m.group(2)))
            if by_depth:
                best = max(by_depth, key=lambda d: by_depth[d][1])
                res = {"pull_tma_GBps_per_gpu_min": by_depth[best][0], "pull_tma_GBps_per_gpu_avg": by_depth[best][1],
                       "avg_by_stage_depth": {str(d): v[1] for d, v in by_depth.items()},
                       "how": f"tools/p2p_probe {world} pull_tma 512 1 32768 0 50 DEPTH: all {world} GPUs TMA-pull "
                              f"512 MiB from every peer concurrently (bulk copies through a DEPTH x 32 KiB smem ring, "
                              f"1 CTA/SM), per-GPU ingress; best depth of 2, 3, 4 ({best})"}
        except Exception:          # noqa: BLE001  (a missing or failing probe only drops this field)
            res = None
        finally:
            store.set("hpz_p2p_probe_done", "1")   # never leave the other ranks waiting
    else:
        store.wait(["hpz_p2p_probe_done"])
    return res


def nccl_baseline(infos, e, node_size, dev, tdt, args):
    """NCCL (torch.distributed, NCCL 2.28) on the same message sizes: AllGather over P into
    a full buffer + copy of the secondary slice; AllGather over the virtual-node group;
    fp32 ReduceScatter(AVG).  Timed with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    P = dist.get_world_size()
    r = dist.get_rank()
    from paper_2407_01614_b200.world import virtual_nodes
    groups = [dist.new_group(g) for g in virtual_nodes(P, node_size)]
    my_group = groups[r // node_size]
    nmax = max(x.numel_pad for x in infos)
    smax = max(x.shard for x in infos)
    full = torch.empty(nmax, dtype=tdt, device=dev)
    prim = torch.ones(smax, dtype=tdt, device=dev)
    sec = torch.empty(nmax // node_size, dtype=tdt, device=dev)
    grad = torch.ones(nmax, dtype=torch.float32, device=dev)
    gsh = torch.empty(smax, dtype=torch.float32, device=dev)
    l = r % node_size

    def step(ev=None):
        t = {"fwd": 0.0, "bwd": 0.0, "rs": 0.0}
        marks = []
        for x in infos:
            a = torch.cuda.Event(enable_timing=True); a.record()
            dist.all_gather_into_tensor(full[: x.numel_pad], prim[: x.shard])
            sec[: x.sec_shard].copy_(full[l * x.sec_shard:(l + 1) * x.sec_shard])
            b = torch.cuda.Event(enable_timing=True); b.record()
            marks.append(("fwd", a, b))
        for x in reversed(infos):
            a = torch.cuda.Event(enable_timing=True); a.record()
            dist.all_gather_into_tensor(full[: x.numel_pad], sec[: x.sec_shard], group=my_group)
            b = torch.cuda.Event(enable_timing=True); b.record()
            dist.reduce_scatter_tensor(gsh[: x.shard], grad[: x.numel_pad], op=dist.ReduceOp.AVG)
            c = torch.cuda.Event(enable_timing=True); c.record()
            marks.append(("bwd", a, b))
            marks.append(("rs", b, c))
        return marks

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    K = max(1, min(args.steps, 5))
    allm = []
    for _ in range(K):
        allm += step()
    torch.cuda.synchronize()
    t = {"fwd": 0.0, "bwd": 0.0, "rs": 0.0}
    for k, a, b in allm:
        t[k] += a.elapsed_time(b) / K
    v = torch.tensor([t["fwd"], t["bwd"], t["rs"]], dtype=torch.float64, device=dev)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    fwd, bwd, rs = v.tolist()
    ag = sum(x.numel_pad for x in infos) * e
    rsb = sum(x.numel_pad for x in infos) * 4
    coll = fwd + bwd + rs
    return {"value": round(P * (2 * ag + rsb) / (coll * 1e-3) / 1e9, 2), "unit": "GB/s",
            "ms_per_step": {"fwd_gather+copy": round(fwd, 3), "bwd_gather": round(bwd, 3),
                            "reduce_scatter": round(rs, 3)},
            "steps": K, "impl": f"torch.distributed NCCL {'.'.join(map(str, torch.cuda.nccl.version()))}"}


def reference_arm(args, world, rank, node_size):
    """--impl reference: the CPU oracle as it stands, on this arm's config/metric/unit, each
    step the bounded sample of the workload that `cpu_baseline` times (one process per host
    core, each simulating one step of all P ranks on the first S elements of a layer).
    Under torchrun only rank 0 runs; the other ranks exit without work."""
    if rank != 0:
        return
    from paper_2407_01614_b200 import shapes
    dtype = shapes.PARAM_DTYPE.get(args.model, "bf16")
    numels = shapes.numels(args.model)
    L = len(numels)
    n_slots = args.grad_slots if 0 < args.grad_slots < L else L
    S = oracle_sample_numel(world, args.oracle_numel)
    C = oracle_procs(world, S)
    walls = oracle_time(world, node_size, dtype, S, C, rounds=args.warmup + args.steps)
    walls = walls if isinstance(walls, list) else [walls]
    timed = walls[args.warmup:]
    bytes_round = C * oracle_bytes(world, S, dtype)
    value = statistics.median(bytes_round / w / 1e9 for w in timed)
    ms = statistics.median(timed) * 1e3
    q = world * 256
    model_elems = sum(-(-n // q) * q for n in numels)
    sample = (f"oracle/hpz_oracle.py HpzOracle, one full step of the first {S} elements of one flat layer, all "
              f"{world} rank(s) simulated (P={world}, P'={node_size}); {C} such samples in {C} concurrent "
              f"processes per step; numpy; host has {host_cores()} cores")
    out = {"metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 1), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "bf16 gathers / f32 reduce-scatter+Adam", "data": "synthetic",
           "impl": "reference",
           "config": make_config(args, world, node_size, L, sum(numels), n_slots),
           "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "kind": "oracle", "cores": C, "sample": sample,
                            "extrapolated_step_s": round(model_elems / (C * S) * statistics.median(timed), 1)},
           "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
