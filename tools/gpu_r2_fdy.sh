# MoE: dY dispatch fused into the combine backward -- parity (1 and 2 GPUs) and the C2 1-GPU A/B
timeout 1200 python -m pytest tests/test_moe_gpu.py tests/test_step_dist_gpu.py tests/test_report_gpu.py tests/test_widths_gpu.py \
  -q -x -k "moe or c2 or C2" > gpurun_out/r2_z_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2_z_pytest.log
for f in 1 0 1 0; do
  OPX_MOE_FUSED_DY=$f python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/r2_z_c2_$f.json
  python -c "
import json,sys
d=json.load(open('gpurun_out/r2_z_c2_$f.json')); n=d['node_ms']
print('fdy=$f', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], n.get('bwd.combine_bwd'), n.get('bwd.a2a_combine_grad'))"
done
