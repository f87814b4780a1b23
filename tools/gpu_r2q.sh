set -x
python -m pytest tests/test_kernels_gpu.py tests/test_moe_gpu.py tests/test_step_gpu.py tests/test_encoder_gpu.py tests/test_widths_gpu.py -q -x -k "not dist and not sp" > gpurun_out/r2_q_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2_q_pytest.log
for st in 0 1 0 1; do CUDA_VISIBLE_DEVICES=0 OPX_GEMM_EPI_STAGED=$st python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('c1 staged=$st', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['node_ms']['fwd.mlp'], d['node_ms']['bwd.recompute'])
" >> gpurun_out/r2_q_bench.log; done
for st in 0 1; do OPX_GEMM_EPI_STAGED=$st python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2965$st bench.py --gpus 4 --steps 5 --warmup 3 --config c2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('c2 staged=$st', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['node_ms'].get('fwd.experts'), d['node_ms'].get('bwd.experts'))
" >> gpurun_out/r2_q_bench.log; done
tail -n 2 gpurun_out/r2_q_pytest.log; cat gpurun_out/r2_q_bench.log
