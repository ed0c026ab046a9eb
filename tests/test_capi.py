"""The C-ABI library loads without a GPU and exports every declared symbol."""
import ctypes
import os
import re

from paper_2405_16283_b200 import _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "turnip.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(tn_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported():
    L = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert _lib.lib().tn_version().decode().startswith("turnip-b200")


def test_errors_are_codes_not_aborts():
    err = _lib.Out()
    out = _lib.Out()
    rc = _lib.lib().tn_simulate(b"not json", None, None, None, 0, None, out.ref, err.ref)
    assert rc == 2 and "invalid JSON" in err.take()


def test_executor_without_gpu_fails_loudly():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_16283_b200 import memplan, workloads as W
    from paper_2405_16283_b200.executor import Executor
    g = W.llama_prefill(W.LlamaConfig(dim=256, layers=1, heads=2, ffn=512, vocab=300), 128)
    mg, _ = W.plan(g, 64 << 20)
    with pytest.raises(memplan.MemplanError) as e:
        Executor(mg, g.to_json())
    assert e.value.code == 3


def test_executor_config_keys_are_validated_before_any_cuda_call():
    """Bad executor configuration is a usage error (code 2) with the key named,
    raised before the CUDA runtime is touched (so it reproduces on CPU)."""
    import pytest
    from paper_2405_16283_b200 import memplan, workloads as W
    from paper_2405_16283_b200.executor import Executor
    g = W.GraphBuilder()
    a = g.input("A", (128, 128), "bf16")
    b = g.input("B", (128, 128), "bf16")
    g.gemm("C", a, b, 128, 128, 128, out_shape=(128, 128))
    mg, _ = W.plan(g, 1 << 24)
    for cfg, key in (({"timestamps": "bogus"}, "timestamps"), ({"input_residency": "gpu"}, "input_residency"),
                     ({"completion": "spin"}, "completion"), ({"device_inputs": "move"}, "device_inputs")):
        with pytest.raises(memplan.MemplanError) as e:
            Executor(mg, g.to_json(), cfg)
        assert e.value.code == 2 and key in str(e.value)
