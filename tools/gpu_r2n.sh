set -x
python -m pytest tests/test_step_gpu.py tests/test_kernels_gpu.py -q -x -k "zero_layer or ulysses or adamw or extreme or rejects or async" > gpurun_out/r2_n_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2_n_pytest.log
for b in 0 2 1 4 0 2; do CUDA_VISIBLE_DEVICES=0 OPX_ADAMW_OVERLAP_BLOCKS=$b python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('c1 bps=$b', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['node_ms'].get('optimizer'))
" >> gpurun_out/r2_n_bench.log; done
for b in 0 2 1; do OPX_ADAMW_OVERLAP_BLOCKS=$b python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2962$b bench.py --gpus 4 --steps 5 --warmup 3 --config c2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('c2 bps=$b', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['node_ms'].get('bwd.combine_bwd'), d['node_ms'].get('optimizer'))
" >> gpurun_out/r2_n_bench.log; done
tail -n 2 gpurun_out/r2_n_pytest.log; cat gpurun_out/r2_n_bench.log
