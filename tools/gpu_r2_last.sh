# last sanity of the committed build on one GPU: smoke, the MoE step parity, C1 + C2 bench lines
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_last_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/r2_last_smoke.log
timeout 600 python -m pytest tests/test_moe_gpu.py -q -x > gpurun_out/r2_last_moe.log 2>&1; echo moe rc=$?; tail -1 gpurun_out/r2_last_moe.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/r2_last_c1.json
python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/r2_last_c2.json
python -c "
import json
for f in ['c1','c2']:
    d=json.load(open('gpurun_out/r2_last_%s.json'%f)); print(f, round(d['value']), d['mfu_exact'], d['clocks']['sm_mhz'], d['gpu_launches'])"
