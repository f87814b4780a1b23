"""Microbenchmark: opx tcgen05 GEMM vs cuBLAS (torch.matmul, comparator only)
on the Qwen2-7B layer shapes (fwd, dgrad, wgrad) at T local tokens."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02317_b200 import check, lib  # noqa: E402


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    H, F, Q = 3584, 18944, 4608
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    # (name, M, N, K, A mn-major, B mn-major, epilogue as used by the step: 0 bf16, 1 fp32)
    shapes = [("qkv fwd", T, Q, H, 0, 0, 0), ("o fwd", T, H, H, 0, 0, 1), ("o fwd+resid", T, H, H, 0, 0, 2),
              ("qkv dgrad", T, H, Q, 0, 1, 1), ("o fwd bf16", T, H, H, 0, 0, 0),
              ("gate|up fwd", T, 2 * F, H, 0, 0, 0),
              ("down fwd", T, H, F, 0, 0, 1), ("down dgrad", T, F, H, 0, 1, 0), ("gu dgrad", T, H, 2 * F, 0, 1, 1),
              ("down wgrad", H, F, T, 1, 1, 1), ("gu wgrad", 2 * F, H, T, 1, 1, 1),
              ("lm_head fwd", 8192, 152064, H, 0, 0, 0)]
    for name, M, N, K, amn, bmn, epi in shapes:
        A = torch.randn(K, M, device="cuda", dtype=torch.bfloat16) if amn else torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(K, N, device="cuda", dtype=torch.bfloat16) if bmn else torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        D = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi else torch.bfloat16)
        R = torch.randn(M, N, device="cuda", dtype=torch.float32) if epi == 2 else None
        ms = timeit(lambda: check(lib().opx_gemm(M, N, K, P(A), A.shape[1], amn, P(B), B.shape[1], bmn, epi, P(D), N,
                                                 P(R) if R is not None else None, N if R is not None else 0,
                                                 None, 0, 1.0, st)))
        At = A.t() if amn else A
        Bt = B if bmn else B.t()
        ms_cub = timeit(lambda: torch.matmul(At, Bt))
        f = 2.0 * M * N * K
        print(f"{name:12s} epi={epi} M={M:6d} N={N:6d} K={K:6d}  opx {ms:7.3f} ms {f / ms / 1e9:7.1f} TF/s | "
              f"cuBLAS {ms_cub:7.3f} ms {f / ms_cub / 1e9:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
