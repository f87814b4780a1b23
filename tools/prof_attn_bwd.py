import ctypes, math, sys
import torch
sys.path.insert(0, ".")
from paper_2508_02317_b200 import check, lib
from paper_2508_02317_b200.runtime import synthetic_batch
def P(t): return ctypes.c_void_p(t.data_ptr())
N, hq, hk = int(sys.argv[1]), 7, 1
single = len(sys.argv) > 2
b = synthetic_batch(1000, N, 1, seed=2508, single_sample=single)
cu = b["cu_rows"][0]
st = torch.empty(N, dtype=torch.int32); en = torch.empty(N, dtype=torch.int32)
for a, c in zip(cu[:-1], cu[1:]): st[a:c] = a; en[a:c] = c
st, en = st.cuda(), en.cuda()
q = torch.randn(N, hq, 128, device="cuda", dtype=torch.bfloat16); k = torch.randn(N, hk, 128, device="cuda", dtype=torch.bfloat16); v = torch.randn_like(k)
o = torch.randn_like(q); lse = torch.randn(hq, N, device="cuda"); do = torch.randn_like(q)
dq = torch.empty(N, hq, 128, device="cuda"); dk = torch.empty_like(k); dv = torch.empty_like(k); delta = torch.empty(hq, N, device="cuda")
S = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def run(): check(lib().opx_attn_bwd_tc(P(q), P(k), P(v), P(o), P(lse), P(do), P(dq), P(dk), P(dv), P(delta), hq*128, hk*128, P(st), P(en), N, hq, hk, 1/math.sqrt(128), S))
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [run() for _ in range(3)]; e1.record(); torch.cuda.synchronize()
sq = sum((c-a)**2 for a, c in zip(cu[:-1], cu[1:]))
ms = e0.elapsed_time(e1)/3
print(f"N={N} single={single} bwd_tc {ms:.3f} ms  {2.5*2*128*hq*sq/ms/1e9:.1f} TF/s", flush=True)
