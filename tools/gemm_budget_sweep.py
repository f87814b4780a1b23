"""Debug: the C1 gate|up GEMM (T tokens) under several L2-budget settings of
the band raster (OPX_GEMM_BUDGET_MB), 3 launches each, for ncu DRAM-byte
comparison; prints CUDA-event times."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02317_b200 import check, lib  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H, F = 3584, 18944
A = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
B = torch.randn(2 * F, H, device="cuda", dtype=torch.bfloat16)
D = torch.empty(T, 2 * F, device="cuda", dtype=torch.bfloat16)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
for mb in ("10", "20", "40", "80"):
    os.environ["OPX_GEMM_BUDGET_MB"] = mb
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        check(lib().opx_gemm(T, 2 * F, H, P(A), H, 0, P(B), H, 0, 0, P(D), 2 * F, None, 0, None, 0, 1.0, st))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"budget {mb} MB: {ms:.3f} ms  {2 * T * 2 * F * H / ms / 1e9:.0f} TF/s", flush=True)
