"""Microbenchmark: MoE router logits + top-k (opx_moe_route) at the C2 per-rank shape."""
import sys

import torch

sys.path.insert(0, ".")
from tests.gpu_util import P, S, call  # noqa: E402

T, H, E, k = 8192, 2048, 128, 8
h = torch.randn(T, H, device="cuda").to(torch.bfloat16)
w = (torch.randn(E, H, device="cuda") * 0.02).to(torch.bfloat16)
logits = torch.empty(T, E, device="cuda")
idx = torch.empty(T, k, device="cuda", dtype=torch.int32)
wts = torch.empty(T, k, device="cuda")
for _ in range(3):
    call("opx_moe_route", P(h), P(w), T, H, E, k, P(logits), P(idx), P(wts), S())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    call("opx_moe_route", P(h), P(w), T, H, E, k, P(logits), P(idx), P(wts), S())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"router+topk T={T} H={H} E={E}: {ms:.3f} ms  {2 * T * H * E / ms / 1e9:.1f} TFLOP/s fp32")
