"""Debug: per-iteration phase durations of one attention-backward CTA
(OPX_ATTN_PROF=<cta> makes k_attn_bwd_tc print clock64 phase averages)."""
import ctypes
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02317_b200 import check, lib  # noqa: E402
from paper_2508_02317_b200.runtime import synthetic_batch  # noqa: E402


def P(t):
    return ctypes.c_void_p(t.data_ptr())


N, hq, hk = 32768, int(sys.argv[1]) if len(sys.argv) > 1 else 7, 1
b = synthetic_batch(1000, N, 1, seed=2508)
cu = b["cu_rows"][0]
st = torch.empty(N, dtype=torch.int32)
en = torch.empty(N, dtype=torch.int32)
for a, c in zip(cu[:-1], cu[1:]):
    st[a:c] = a
    en[a:c] = c
st, en = st.cuda(), en.cuda()
q = torch.randn(N, hq, 128, device="cuda", dtype=torch.bfloat16)
k = torch.randn(N, hk, 128, device="cuda", dtype=torch.bfloat16)
v = torch.randn_like(k)
o = torch.randn_like(q)
lse = torch.randn(hq, N, device="cuda")
do = torch.randn_like(q)
dq = torch.empty(N, hq, 128, device="cuda")
dk = torch.empty(N, hk, 128, device="cuda")
dv = torch.empty_like(dk)
delta = torch.empty(hq, N, device="cuda")
S = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    check(lib().opx_attn_bwd_tc_f32kv(P(q), P(k), P(v), P(o), P(lse), P(do), P(dq), P(dk), P(dv), P(delta),
                                      hq * 128, hk * 128, P(st), P(en), N, hq, hk, ctypes.c_float(1 / math.sqrt(128)),
                                      0, S))
torch.cuda.synchronize()
