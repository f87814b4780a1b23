"""Ulysses exchange kernels on two GPUs of one process (no peer barrier, so
safe under ncu kernel replay): rank 0 of an SP2 group sends its C1-shaped
q/k/v rows (seq->head, with RoPE) and the attention output (head->seq) to
itself and to GPU 1 through peer access.  Prints GB/s of the bytes that
leave the GPU ((sp-1)/sp of the payload, comm.cpp:48-60).  Under
ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum the
NVLink counters of the same launches give the link-level rate."""
import ctypes
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02317_b200 import check, lib  # noqa: E402


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def ptrs(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def main():
    from cuda.bindings import runtime as rt

    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    for a, b in ((0, 1), (1, 0)):
        rt.cudaSetDevice(a)
        rt.cudaDeviceEnablePeerAccess(b, 0)
    torch.cuda.set_device(0)
    sp, rank, S, hq, hk, hd = 2, 0, 32768, 28, 4, 128
    T = S // sp
    W = (hq + 2 * hk) * hd
    qkv = torch.randn(T, W, device="cuda:0", dtype=torch.bfloat16)
    pos = torch.arange(S, device="cuda:0", dtype=torch.int32)
    inv = (1.0 / (1e6 ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))).float().to("cuda:0")
    dst = {}
    for g, h in (("q", hq), ("k", hk), ("v", hk)):
        dst[g] = [torch.zeros(S, h // sp, 128, device=f"cuda:{j}", dtype=torch.bfloat16) for j in range(sp)]
    o_heads = torch.randn(S, hq // sp, 128, device="cuda:0", dtype=torch.bfloat16)
    o_dst = [torch.zeros(T, hq * hd, device=f"cuda:{j}", dtype=torch.bfloat16) for j in range(sp)]
    st = torch.cuda.current_stream(0).cuda_stream
    L = lib()

    def s2h():
        check(L.opx_ulysses_seq2head(P(qkv), W, ptrs(dst["q"]), ptrs(dst["k"]), ptrs(dst["v"]), sp, rank, 1, S,
                                     hq, hk, hd, P(pos), P(inv), ctypes.c_void_p(st)))

    def h2s():
        check(L.opx_ulysses_head2seq(P(o_heads), ptrs(o_dst), hq * hd, sp, rank, 1, S, hq, hd,
                                     ctypes.c_void_p(st)))

    frac = (sp - 1) / sp
    for name, fn, payload in (("seq2head q/k/v", s2h, T * W * 2), ("head2seq out", h2s, T * hq * hd * 2)):
        fn()
        torch.cuda.synchronize(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize(0)
        ms = e0.elapsed_time(e1) / n
        print(f"{name:16s} {ms * 1e3:8.1f} us  {payload * frac / ms / 1e6:7.1f} GB/s leaving the GPU "
              f"({payload / 1e6:.1f} MB payload)")
    # correctness spot check: rank 1's q heads of token t (positions 0..T-1 are this rank's)
    t = 5
    x = qkv[t, (hq // sp) * hd:(hq // sp + 1) * hd].float()
    ang = pos[t].float() * inv
    c, s = ang.cos(), ang.sin()
    x1, x2 = x[:hd // 2], x[hd // 2:]
    ref = torch.cat([x1 * c - x2 * s, x2 * c + x1 * s])
    got = dst["q"][1][t, 0].float().to("cuda:0")
    assert (got - ref).abs().max() < 0.05 * ref.abs().max(), "seq2head mismatch"


if __name__ == "__main__":
    main()
