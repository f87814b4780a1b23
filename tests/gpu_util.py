"""Helpers for GPU tests: torch tensors are device-memory plumbing only; every
compute call goes through libopx's C ABI."""
import ctypes

import torch

from paper_2508_02317_b200 import check, lib


def P(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def S():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def rel_err(x, ref):
    x = x.float()
    ref = ref.float()
    return ((x - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


def cosine(x, ref):
    x = x.float().flatten()
    ref = ref.float().flatten()
    return (torch.dot(x, ref) / (x.norm() * ref.norm()).clamp_min(1e-30)).item()
