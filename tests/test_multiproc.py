"""The bench's multi-rank plumbing (barrier + max-over-ranks) on CPU with gloo,
world_size 2 — the same code path torchrun drives with NCCL on GPUs."""
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, json
sys.path.insert(0, %r)
import torch.distributed as dist
import bench
world, rank, local = bench.dist_setup("replicas")
t = bench.max_over_ranks(0.5 + rank, world)
bench.barrier(world)
# each rank plans its own replica of a small memgraph: identical plans
from paper_2405_16283_b200 import workloads as W
g = W.llama_prefill(W.LlamaConfig(dim=256, layers=1, heads=2, ffn=512, vocab=300), 128)
mg, st = W.plan(g, 64 << 20)
import hashlib
h = hashlib.sha256(mg.encode()).hexdigest()
import torch
obj = [None] * world
dist.all_gather_object(obj, h)
print(json.dumps({"rank": rank, "max": t, "same_plan": len(set(obj)) == 1}))
dist.destroy_process_group()
"""


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo():
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(r), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER % ROOT], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    import json
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    assert all(r["max"] == 1.5 and r["same_plan"] for r in res)


def test_reference_arm_two_ranks_rank0_only():
    """`bench.py --impl reference` under a 2-rank launch: rank 0 alone times the
    CPU arm and prints the JSON line, rank 1 exits 0 without work (gloo here,
    NCCL on the GPU box)."""
    import json
    ref_so = os.path.join(ROOT, "oracle", "_ref")
    if not (os.path.isdir(ref_so) and any(f.startswith("_memplan") for f in os.listdir(ref_so))):
        import pytest
        pytest.skip("oracle/_ref (the reference planner) is not built")
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(r), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                                       "--gpus", "2", "--steps", "1", "--warmup", "0", "--seq", "256",
                                       "--layers", "1"], env=env, cwd=ROOT, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    lines0 = [l for l in outs[0][0].splitlines() if l.startswith("{")]
    assert len(lines0) == 1 and not [l for l in outs[1][0].splitlines() if l.startswith("{")]
    d = json.loads(lines0[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    # the arm's config is the one our arm prints (same workload: the TP graph over 2 GPUs)
    assert d["config"]["workload"] == "llama7b_prefill_seq4096_cap16GiB_tp2" and d["scaling"] == "strong"
    assert abs(d["ms_per_step"] - d["cpu_baseline"]["layer_s"][0] * 1e3) < 6  # the actually-timed sample
    assert d["reference_planner"]["vertices"] > 0


TP_WORKER = r"""
import os, sys, json, time
sys.path.insert(0, %r)
import bench
calls = []
def fake(args, world, rank, local, n, tp):  # stands in for the GPU work of rank 0
    time.sleep(1.0)
    calls.append((world, rank, n, tp))
bench.run_ours_on = fake
args = bench.argparse.Namespace(mode="tp", gpus=2)
world, rank, local = bench.dist_setup("tp")
import torch.distributed as dist
assert dist.get_backend() == "gloo"  # no NCCL: the idle rank never touches a GPU
t0 = time.time()
bench.run_ours(args, world, rank, local)
print(json.dumps({"rank": rank, "calls": calls, "waited": time.time() - t0}))
dist.destroy_process_group()
"""


def test_tp_mode_rank0_drives_all_gpus():
    """tp mode under a 2-rank launch: rank 0 alone runs the partitioned memgraph
    over both GPUs (one host process), rank 1 waits for it at one barrier."""
    import json
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(r), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", TP_WORKER % ROOT], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    res = {d["rank"]: d for d in (json.loads(o.strip().splitlines()[-1]) for o, _ in outs)}
    assert res[0]["calls"] == [[1, 0, 2, True]] and res[1]["calls"] == []
    assert res[1]["waited"] >= 0.9  # rank 1 left only after rank 0 finished
