import ctypes, math, sys
import torch
sys.path.insert(0, ".")
from paper_2508_02317_b200 import check, lib
from tests.test_kernels_gpu import _attn_ref, _varlen
def P(t): return ctypes.c_void_p(t.data_ptr())
for (N, lens, hq, hk) in [(128, [128], 1, 1), (256, [256], 1, 1), (256, [256], 2, 1)]:
    torch.manual_seed(0)
    q = torch.randn(N, hq, 128, device="cuda").bfloat16()
    k = torch.randn(N, hk, 128, device="cuda").bfloat16()
    v = torch.randn(N, hk, 128, device="cuda").bfloat16()
    st, en = _varlen(N, lens)
    qr, kr, vr = (t.float().clone().requires_grad_(True) for t in (q, k, v))
    o_ref, lse_ref = _attn_ref(qr, kr, vr, st, hq, hk)
    o = o_ref.detach().bfloat16(); lse = lse_ref.detach().contiguous()
    do = torch.randn(N, hq, 128, device="cuda").bfloat16()
    o_ref.backward(do.float())
    for name in ("opx_attn_bwd_tc",):
        dq = torch.empty(N, hq, 128, device="cuda"); dk = torch.empty(N, hk, 128, device="cuda").bfloat16(); dv = torch.empty_like(dk)
        delta = torch.empty(hq, N, device="cuda")
        check(getattr(lib(), name)(P(q), P(k), P(v), P(o), P(lse), P(do), P(dq), P(dk), P(dv), P(delta), hq*128, hk*128, P(st), P(en), N, hq, hk, 1/math.sqrt(128), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        for tn, got, ref in (("dq", dq, qr.grad), ("dk", dk, kr.grad), ("dv", dv, vr.grad)):
            err = (got.float() - ref).abs()
            m = err.max().item() / ref.abs().max().item()
            idx = (err == err.max()).nonzero()[0].tolist()
            rowerr = err.amax(dim=(1, 2))
            bad = (rowerr > 0.05 * ref.abs().max()).nonzero().flatten().tolist()
            print(f"N={N} hq={hq} {name:16s} {tn}: rel {m:.3e} at {idx}; bad rows {bad[:8]}..{len(bad)} ratio {(got.float()/ref.clamp_min(1e-6)).flatten()[:4].tolist() if tn=='dv' else ''}")
