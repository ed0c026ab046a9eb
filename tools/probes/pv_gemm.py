"""Config-5 P·V GEMM shape (M 4096 x N 128 x K 4096, bf16 in, fp32 out +
fp32 residual) with and without split-K, one launch each (for ncu)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor

for ks in (0, 2, 4, 8):
    g = W.GraphBuilder()
    a = g.input("P", (4096, 4096), "bf16")
    b = g.input("vt", (128, 4096), "bf16")
    r = g.input("R", (4096, 128), "f32")
    g.gemm("O", a, b, 4096, 128, 4096, r=r, out_dtype="f32", out_shape=(4096, 128), ksplit=ks or None)
    mg, _ = W.plan(g, 1 << 30)
    with Executor(mg, g.to_json(), {"input_residency": "device"}) as ex:
        ex.set_input(a, torch.randn(4096, 4096, device="cuda").to(torch.bfloat16))
        ex.set_input(b, torch.randn(128, 4096, device="cuda").to(torch.bfloat16))
        ex.set_input(r, torch.randn(4096, 128, device="cuda"))
        for _ in range(2):
            ex.run(trace=False)
