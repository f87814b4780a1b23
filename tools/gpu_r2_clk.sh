CUDA_VISIBLE_DEVICES=0 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/r2_clk_c2.json
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/r2_clk_c1n2.err | grep '^{' > gpurun_out/r2_clk_c1n2.json
python -c "
import json
for f in ['c2','c1n2']:
    d=json.load(open('gpurun_out/r2_clk_%s.json'%f)); print(f, round(d['value']), d['mfu_exact'], d['clocks'])"
