"""Attention backward precision at the C1 head configuration (28 q / 4 kv
heads of 128, one packed row [763, 90, 171] like the width-parity test):
the tcgen05 kernels against an fp64 reference, next to a torch emulation of
the same bf16 rounding points (P and dS rounded to bf16 before their MMAs,
O and dO bf16) -- separates the kernel's own error from the error any bf16
flash-attention backward has on these inputs."""
import math
import sys

import torch

sys.path.insert(0, ".")
from tests.gpu_util import P, S, call  # noqa: E402

dev = "cuda"


def ref64(q, k, v, do, st, hq, hk, scale, emulate=False):
    N = q.shape[0]
    G = hq // hk
    idx = torch.arange(N, device=dev)
    mask = (idx[None, :] <= idx[:, None]) & (idx[None, :] >= st.long()[:, None])
    dt = torch.float32 if emulate else torch.float64
    qf = q.to(dt).permute(1, 0, 2)
    kf = k.to(dt).repeat_interleave(G, 1).permute(1, 0, 2)
    vf = v.to(dt).repeat_interleave(G, 1).permute(1, 0, 2)
    dof = do.to(dt).permute(1, 0, 2)
    s = (qf @ kf.transpose(1, 2)) * scale
    s = s.masked_fill(~mask[None], float("-inf"))
    lse = torch.logsumexp(s, -1, keepdim=True)
    p = torch.exp(s - lse)
    o = p @ vf
    if emulate:
        o = o.bfloat16().to(dt)
        pb = p.bfloat16().to(dt)
    else:
        pb = p
    dv = pb.transpose(1, 2) @ dof
    dp = dof @ vf.transpose(1, 2)
    delta = (dof * o).sum(-1, keepdim=True)
    ds = p * (dp - delta)
    if emulate:
        ds = ds.bfloat16().to(dt)
    dq = ds @ kf * scale
    dk = ds.transpose(1, 2) @ qf * scale
    dk = dk.view(hk, G, N, 128).sum(1)
    dv = dv.view(hk, G, N, 128).sum(1)
    return (o.permute(1, 0, 2), lse[..., 0], dq.permute(1, 0, 2), dk.permute(1, 0, 2), dv.permute(1, 0, 2))


def err(x, r):
    x, r = x.double().flatten(), r.double().flatten()
    return ((x - r).abs().max() / r.abs().max()).item(), (torch.dot(x, r) / (x.norm() * r.norm())).item()


def main():
    hq, hk = 28, 4
    lens = [763, 90, 171]
    N = sum(lens)
    st = torch.empty(N, dtype=torch.int32)
    en = torch.empty(N, dtype=torch.int32)
    a = 0
    for l in lens:
        st[a:a + l] = a
        en[a:a + l] = a + l
        a += l
    st, en = st.to(dev), en.to(dev)
    scale = 1 / math.sqrt(128)
    for std in (1.0, 1.2, 2.0):
        torch.manual_seed(0)
        q = (torch.randn(N, hq, 128, device=dev) * std).bfloat16()
        k = (torch.randn(N, hk, 128, device=dev) * std).bfloat16()
        v = torch.randn(N, hk, 128, device=dev).bfloat16()
        do = (torch.randn(N, hq, 128, device=dev) * 1e-3).bfloat16()
        o = torch.empty(N, hq, 128, device=dev, dtype=torch.bfloat16)
        lse = torch.empty(hq, N, device=dev)
        call("opx_attn_fwd_tc", P(q), P(k), P(v), P(o), P(lse), hq * 128, hk * 128, hk * 128, hq * 128,
             P(st), P(en), N, hq, hk, scale, S())
        dq = torch.zeros(N, hq, 128, device=dev)
        dk = torch.zeros(N, hk, 128, device=dev)
        dv = torch.zeros(N, hk, 128, device=dev)
        delta = torch.empty(hq, N, device=dev)
        call("opx_attn_bwd_tc_f32kv", P(q), P(k), P(v), P(o), P(lse), P(do), P(dq), P(dk), P(dv),
             P(delta), hq * 128, hk * 128, P(st), P(en), N, hq, hk, scale, 0, S())
        torch.cuda.synchronize()
        R = ref64(q, k, v, do, st, hq, hk, scale)
        E = ref64(q, k, v, do, st, hq, hk, scale, emulate=True)
        print(f"std {std}: o kernel {err(o, R[0])} emul {err(E[0], R[0])}")
        for name, i, g in (("dq", 2, dq), ("dk", 3, dk), ("dv", 4, dv)):
            print(f"   {name}: kernel {err(g, R[i])}  bf16-emulation {err(E[i], R[i])}")
        # the step's consumer rounds dq to bf16 before the wgrad GEMM
        print(f"   dq->bf16: kernel {err(dq.bfloat16(), R[2])}")


if __name__ == "__main__":
    main()
