# C2 slice on 4 GPUs (EP4): dY dispatch fused into the combine backward (default) vs separate
for f in 1 0; do
  OPX_MOE_FUSED_DY=$f timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2962$f \
    bench.py --gpus 4 --steps 5 --warmup 3 --config c2 --no-cpu-baseline 2>gpurun_out/r2_z4_$f.err | grep '^{' > gpurun_out/r2_z4_c2_$f.json
  python -c "
import json
d=json.load(open('gpurun_out/r2_z4_c2_$f.json')); n=d['node_ms']
print('fdy=$f', round(d['value']), d['mfu_exact'], d['ms_per_step'], d['clocks']['sm_mhz'], n.get('bwd.combine_bwd'), n.get('bwd.a2a_combine_grad'), n.get('bwd.experts'), n.get('bwd.experts_b'), n.get('bwd.a2a_wait'))"
done
