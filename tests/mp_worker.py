"""Worker for the multi-process GPU parity test (one process per GPU, torchrun).

Every rank builds the real DistWorld (arena in libhpz, CUDA IPC peer mappings over
NVLink), runs T steps of Algorithm 1 with seeded inputs, and compares its own outputs
element by element with the CPU oracle (simulated locally at test sizes).  Exit code
0 = parity; any mismatch raises.

    torchrun --nproc-per-node N tests/mp_worker.py --node-size P' [--order fixed|off|stock]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import hpz_oracle as O  # noqa: E402
from synth import inputs as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--node-size", type=int, required=True)
    ap.add_argument("--order", default="fixed")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--numels", default="300007,65536,4099,77")
    ap.add_argument("--stock-delay-us", type=int, default=0)
    ap.add_argument("--engine", default="tma")
    ap.add_argument("--verify", default="fingerprint")
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--qgz", type=int, default=0)
    ap.add_argument("--grad-dtype", default="f32")
    ap.add_argument("--qwz", type=int, default=0)
    ap.add_argument("--grad-slots", type=int, default=0)
    ap.add_argument("--share-gpus", type=int, default=0,
                    help="1: rank r runs on GPU r %% device_count (several processes per GPU, time-sliced; "
                         "gloo control plane, since NCCL refuses two ranks on one device)")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    if args.share_gpus:
        local %= torch.cuda.device_count()
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if args.share_gpus else "cuda"
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.world import DistWorld, buffer_view, run_step

    numels = [int(x) for x in args.numels.split(",")]
    P, r = dist.get_world_size(), dist.get_rank()
    W = DistWorld(numels, args.node_size, timeout_s=20.0, qgz=bool(args.qgz), grad_dtype=args.grad_dtype,
                  qwz=bool(args.qwz), n_grad_slots=args.grad_slots or None,
                  alias_secondary=args.order != "stock")     # the stock race needs a real secondary
    rc = W.ranks[0]
    s = torch.cuda.current_stream()
    H.hpz_set_order(rc.ctx, args.order, stock_delay_us=args.stock_delay_us, stock_poison=args.order == "stock")
    H.hpz_set_verify(rc.ctx, "exact" if args.order == "stock" else args.verify)
    H.hpz_set_option(rc.ctx, "copy_engine", H.COPY[args.engine])
    for i, n in enumerate(numels):
        w0 = torch.from_numpy(S.layer_params(i, n)).cuda()
        H.hpz_load_master(rc.ctx, i, w0.data_ptr(), s)
    torch.cuda.synchronize()
    fwd = [torch.zeros(x.numel_pad, dtype=torch.bfloat16, device="cuda") for x in rc.infos]
    bwd = [torch.zeros(x.numel_pad, dtype=torch.bfloat16, device="cuda") for x in rc.infos]
    o = O.HpzOracle(numels, P, args.node_size, order="off" if args.order == "off" else "fixed",
                    qgz=bool(args.qgz), grad_dtype=args.grad_dtype, qwz=bool(args.qwz))
    adam = H.make_adam()
    keep = []
    t_box = [0]

    def grad_fn(rcx, i):
        g = torch.from_numpy(S.layer_grads(i, t_box[0], r, numels[i])).cuda()
        if args.grad_dtype == "bf16":
            g = g.to(torch.bfloat16)
        keep.append(g)
        H.hpz_grad_upload(rcx.ctx, i, g.data_ptr(), numels[i], s)

    for t in range(args.steps):
        t_box[0] = t
        run_step([rc], {r: (lambda i: fwd[i].data_ptr())}, {r: (lambda i: bwd[i].data_ptr())}, adam,
                 stream=s, grad_fn=grad_fn, fused=bool(args.fused))
        torch.cuda.synchronize()
        rec = o.step()
        if args.order == "stock":
            continue
        for i, lay in enumerate(o.layouts):
            W_t = O.param_bits(rec.W[i], "bf16")
            got_f = fwd[i].cpu().view(torch.int16).numpy().view(np.uint16)
            got_b = bwd[i].cpu().view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(got_f, W_t), f"rank {r} step {t} layer {i}: fwd gather"
            assert np.array_equal(got_b, W_t), f"rank {r} step {t} layer {i}: bwd gather"
            st = o.state[i][r]
            if args.order == "fixed":
                # P' == P: the secondary is aliased to the primary, which holds W_{t+1}
                want = st.prim if (args.node_size == P and not args.qwz) else st.sec
                sec = buffer_view(rc, i, "secondary", "bf16").cpu().numpy().view(np.uint16)
                assert np.array_equal(sec, O.param_bits(want, "bf16")), f"rank {r} layer {i}: secondary"
            g = buffer_view(rc, i, "grad_shard", "f32").cpu().numpy()
            rs = O.qgz_reduce_scatter if args.qgz else O.reduce_scatter
            Gs = [S.layer_grads(i, t, j, lay.numel, lay.numel_pad) for j in range(P)]
            if args.grad_dtype == "bf16":
                Gs = [O.bf16_to_f32(O.bf16_rne(x)) for x in Gs]
            ref = rs(Gs, lay, r)
            assert np.array_equal(g.view(np.uint32), ref.view(np.uint32)), f"rank {r} layer {i}: RS"
            for kind, refv in (("master", st.master), ("m", st.m), ("v", st.v)):
                got = buffer_view(rc, i, kind, "f32").cpu().numpy()
                assert np.array_equal(got.view(np.uint32), refv.view(np.uint32)), f"rank {r} layer {i}: {kind}"
            prim = buffer_view(rc, i, "primary", "bf16").cpu().numpy().view(np.uint16)
            assert np.array_equal(prim, O.param_bits(st.prim, "bf16")), f"rank {r} layer {i}: primary"
        keep.clear()
    c = H.hpz_counters(rc.ctx)
    tot = torch.tensor([c["mismatches"], c["nan_reads"], c["timeouts"], c["fp_mismatches"]],
                       dtype=torch.int64, device=red_dev)
    dist.all_reduce(tot)
    tot = tot.tolist()
    if r == 0:
        print(f"counters mismatches={tot[0]} nan_reads={tot[1]} timeouts={tot[2]} fp_mismatches={tot[3]}", flush=True)
    assert tot[2] == 0, "device flag wait timed out"
    if args.order == "stock":
        assert tot[0] > 0, "stock ordering should show stale reads"
    else:
        assert tot[0] == 0 and tot[1] == 0 and tot[3] == 0
    W.close()
    dist.barrier()
    dist.destroy_process_group()
    if r == 0:
        print("MP_PARITY_OK", flush=True)


if __name__ == "__main__":
    main()
