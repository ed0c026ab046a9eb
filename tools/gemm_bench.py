"""GEMM microbenchmark through the executor: TFLOP/s per shape from CUDA
events (trace) and error vs a torch fp32 matmul of the same bf16 inputs."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor

SHAPES = [(4096, 4096, 4096), (4096, 12288, 4096), (4096, 22016, 4096), (4096, 4096, 11008), (8192, 8192, 8192),
          (4096, 32000, 4096), (300, 4096, 4096), (4096, 200, 4096)]
TILE = os.environ.get("TN_GEMM_TILE", "auto")  # auto | narrow | wide
RESID = "--residual" in sys.argv  # fused residual epilogue (C = A·Bᵀ + R), as in attn_out / ffn_out
# --sustain: also time back-to-back runs for ~3 s (power-capped steady state, like inside a step)
SUSTAIN = "--sustain" in sys.argv
args = [x for x in sys.argv[1:] if not x.startswith("--")]
if args:
    SHAPES = [tuple(int(x) for x in s.split("x")) for s in args]
for M, N, K in SHAPES:
    g = W.GraphBuilder()
    a = g.input("A", (M, K), "bf16")
    b = g.input("B", (N, K), "bf16")
    r = g.input("R", (M, N), "bf16") if RESID else None
    c = g.gemm("C", a, b, M, N, K, r=r, out_shape=(M, N), tile=TILE)
    mg, _ = W.plan(g, 1 << 36)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    with Executor(mg, g.to_json(), {"input_residency": "device"}) as ex:
        ex.set_input(a, A)
        ex.set_input(b, B)
        if RESID:
            Rt = torch.randn(M, N, device="cuda").to(torch.bfloat16)
            ex.set_input(r, Rt)
        best = 1e9
        for _ in range(5):
            t = json.loads(ex.run())
            row = [r for r in t["rows"] if r["vertex"] == c][0]
            best = min(best, row["end"] - row["start"])
        sus = None
        if SUSTAIN:
            import time
            n, t_end = 0, time.time() + 3.0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            while time.time() < t_end:
                ex.run(trace=False)
                n += 1
            e1.record()
            e1.synchronize()
            sus = e0.elapsed_time(e1) * 1e-3 / n
        out = torch.frombuffer(bytearray(ex.get_output(c, M * N * 2)), dtype=torch.bfloat16).view(M, N).cuda()
    ref = A.float() @ B.float().T
    if RESID:
        ref = ref + Rt.float()
    Bt = B.t()
    for _ in range(3):
        torch.matmul(A, Bt)
    cb = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(A, Bt)
        e1.record()
        e1.synchronize()
        cb = min(cb, e0.elapsed_time(e1) * 1e-3)
    err = ((out.float() - ref).norm() / ref.norm()).item()
    print(json.dumps({"M": M, "N": N, "K": K, "us": round(best * 1e6, 1), "tflops": round(2 * M * N * K / best / 1e12, 1),
                      "rel_err": err, "cublas_us": round(cb * 1e6, 1),
                      "cublas_tflops": round(2 * M * N * K / cb / 1e12, 1), "tile": TILE, "sk": os.environ.get("TN_GEMM_SK", "0"),
                      "sustained_us_per_run": round(sus * 1e6, 1) if sus else None,
                      "sustained_tflops": round(2 * M * N * K / sus / 1e12, 1) if sus else None,
                      "residual": RESID}), flush=True)
