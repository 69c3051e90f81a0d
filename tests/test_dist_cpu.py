"""Multi-process host logic on CPU: world_size-2 gloo (no GPU).  Covers the control plane
of the N>1 path: IPC-handle exchange, virtual-node groups, max-over-ranks timing, and the
bench's reference arm under torchrun (rank 0 prints one JSON line, rank 1 exits 0)."""
import json
import os
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2407_01614_b200.world import exchange_handles, max_over_ranks, sum_over_ranks, virtual_nodes
    h = bytes([rank]) * 64
    got = exchange_handles(h)
    mx = max_over_ranks([float(rank), 10.0 - rank])
    sm = sum_over_ranks([1.0, float(rank)])
    # gloo (the --share-gpus control plane): a CUDA device argument reduces on the host
    assert max_over_ranks([float(rank)], device="cuda") == [1.0]
    assert sum_over_ranks([1.0], device=torch.device("cuda", 0)) == [2.0]
    groups = virtual_nodes(world, 1)
    subg = [dist.new_group(g) for g in groups]
    mine = subg[rank]
    t = torch.tensor([rank + 1.0])
    dist.all_reduce(t, group=mine)          # a node group of size 1 only sees itself
    q.put((rank, [x[0] for x in got], mx, sm, t.item()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_control_plane():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, 29731, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, handles, mx, sm, node_sum in res:
        assert handles == [0, 1]
        assert mx == [1.0, 10.0]
        assert sm == [2.0, 1.0]
        assert node_sum == rank + 1.0


def test_virtual_nodes():
    from paper_2407_01614_b200.world import virtual_nodes
    assert virtual_nodes(8, 4) == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert virtual_nodes(8, 2) == [[0, 1], [2, 3], [4, 5], [6, 7]]
    assert virtual_nodes(1, 1) == [[0]]
    with pytest.raises(ValueError):
        virtual_nodes(8, 3)


def test_bench_reference_arm_torchrun_gloo():
    """--impl reference under torchrun (2 ranks): rank 0 alone prints one JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port=29741", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--oracle-numel", "200000"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["cores"] >= 1 and "extrapolated_step_s" in d["cpu_baseline"]
    assert d["config"]["world"] == 2 and d["config"]["node_size"] == 1


def test_bench_reference_arm_without_launcher():
    """The driver starts `python bench.py --impl reference --gpus N` without torchrun: the
    oracle arm simulates all N ranks in this one process and prints one line (exit 0), with
    the same `config` the GPU arm prints for that N (2 x 4 virtual nodes at N = 8)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "8", "--steps", "2",
           "--warmup", "1", "--oracle-numel", "65536"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 8 and d["config"]["node_size"] == 4 and d["config"]["virtual_nodes"] == 2
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    import bench
    import argparse
    args = argparse.Namespace(model="falcon7b", order="fixed", verify="fingerprint", copy_engine="tma", overlap_bwd=0,
                              qgz=False, grad_dtype="f32", qwz=False, graph=1)
    from paper_2407_01614_b200 import shapes
    n = shapes.numels("falcon7b")
    assert d["config"] == bench.make_config(args, 8, 4, len(n), sum(n), len(n))


def test_share_gpus_config_is_labelled():
    """`bench.py --share-gpus` lines say they are functional checks, not measurements."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    args = argparse.Namespace(model="falcon7b_block", order="fixed", verify="fingerprint", copy_engine="tma",
                              overlap_bwd=0, qgz=False, grad_dtype="f32", qwz=False, graph=1, share_gpus=True)
    cfg = bench.make_config(args, 8, 4, 1, 207070080, 1)
    assert "FUNCTIONAL CHECK" in cfg["share_gpus"] and cfg["parallelism"] == "hpZ dp8 (P=8, P'=4)"
    args.share_gpus = False
    assert "share_gpus" not in bench.make_config(args, 8, 4, 1, 207070080, 1)
