"""Microbenchmark: attention fwd/bwd TFLOP/s on the C1 (Qwen2-7B 32K) shapes."""
import ctypes
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02317_b200 import check, lib  # noqa: E402
from paper_2508_02317_b200.runtime import synthetic_batch  # noqa: E402


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def main():
    S = torch.cuda.current_stream().cuda_stream
    shapes = [(32768, 7, 1, False), (32768, 28, 4, False), (32768, 28, 4, True)]
    if os.environ.get("BENCH_ATTN_SHAPES"):  # e.g. "1,2": a subset of the shapes
        shapes = [shapes[int(i)] for i in os.environ["BENCH_ATTN_SHAPES"].split(",")]
    for (N, hq, hk, single) in shapes:
        b = synthetic_batch(1000, N, 1, seed=2508)
        cu = [0, N] if single else b["cu_rows"][0]
        st = torch.empty(N, dtype=torch.int32)
        en = torch.empty(N, dtype=torch.int32)
        sq = 0
        for a, c in zip(cu[:-1], cu[1:]):
            st[a:c] = a
            en[a:c] = c
            sq += (c - a) ** 2
        st, en = st.cuda(), en.cuda()
        q = torch.randn(N, hq, 128, device="cuda", dtype=torch.bfloat16)
        k = torch.randn(N, hk, 128, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(N, hk, 128, device="cuda", dtype=torch.bfloat16)
        o = torch.empty_like(q)
        lse = torch.empty(hq, N, device="cuda")
        do = torch.randn_like(q)
        dq = torch.empty(N, hq, 128, device="cuda")
        dk = torch.empty_like(k)
        dv = torch.empty_like(v)
        delta = torch.empty(hq, N, device="cuda")
        dk32 = torch.empty(N, hk, 128, device="cuda")
        dv32 = torch.empty_like(dk32)
        flops = 4 * 128 * hq * sq / 2  # causal fwd
        sc = 1 / math.sqrt(128)
        names = ["opx_attn_fwd_tc", "split0"]  # split0: the step's path (fp32 dK/dV, one q head per CTA)
        for name in names:
            def run():
                if name.startswith("split"):
                    check(lib().opx_attn_bwd_tc_f32kv(P(q), P(k), P(v), P(o), P(lse), P(do), P(dq), P(dk32),
                                                      P(dv32), P(delta), hq * 128, hk * 128, P(st), P(en), N,
                                                      hq, hk, ctypes.c_float(sc), int(name[5:]),
                                                      ctypes.c_void_p(S)))
                elif name.startswith("opx_attn_bwd"):
                    check(getattr(lib(), name)(P(q), P(k), P(v), P(o), P(lse), P(do), P(dq), P(dk), P(dv),
                                             P(delta), hq * 128, hk * 128, P(st), P(en), N, hq, hk, sc,
                                             ctypes.c_void_p(S)))
                else:
                    check(getattr(lib(), name)(P(q), P(k), P(v), P(o), P(lse), hq * 128, hk * 128,
                                               hk * 128, hq * 128, P(st), P(en), N, hq, hk, sc,
                                               ctypes.c_void_p(S)))
            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            f = flops * (2.5 if ("bwd" in name or "split" in name) else 1.0)
            tag = " single" if single else ""
            print(f"{name:18s} N={N} hq={hq} hk={hk}{tag}: {ms:8.3f} ms  {f / ms / 1e9:8.1f} TFLOP/s")


if __name__ == "__main__":
    main()
