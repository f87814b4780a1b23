# C2 slice on 4 GPUs: per-half fused dY dispatch (default) vs separate dispatch, then the 2-GPU dy-mode parity test
for f in 1 0; do
  OPX_MOE_FUSED_DY=$f timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2963$f \
    bench.py --gpus 4 --steps 5 --warmup 3 --config c2 --no-cpu-baseline 2>gpurun_out/r2_zb4_$f.err | grep '^{' > gpurun_out/r2_zb4_c2_$f.json
  python -c "
import json
d=json.load(open('gpurun_out/r2_zb4_c2_$f.json')); n=d['node_ms']
print('fdy=$f', round(d['value']), d['mfu_exact'], d['ms_per_step'], d['clocks']['sm_mhz'], n.get('bwd.combine_bwd'), n.get('bwd.a2a_combine_grad'), n.get('bwd.experts'), n.get('bwd.experts_b'), n.get('bwd.a2a_wait'))"
done
timeout 400 python -m pytest tests/test_step_dist_gpu.py -q -x -k "dy_dispatch_modes or ep2_moe_routing" > gpurun_out/r2_zb_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/r2_zb_pytest.log
