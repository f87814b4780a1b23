# Round-end validation on a fresh box: pass the GPU count as $1 (2 or 4).
#   2: the whole GPU suite (2-GPU plans included), smoke, C1 at 1/2 GPUs with the
#      CPU baseline, the reference arm, the ncu launch list of the 1-GPU bench
#   4: the 4-GPU-only tests and the 4-GPU bench lines (C1, C2 slice, C3, C4 slice)
set -x
N=${1:-2}
O=gpurun_out/final_n$N
mkdir -p $O
if [ "$N" = 2 ]; then
  timeout -s KILL 2400 python -m pytest tests -q -m gpu -rs --durations=20 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$? >> $O/pytest_gpu.log
  timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
  CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > $O/bench_c1_n1.json 2> $O/bench_c1_n1.err
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 10 --warmup 3 > $O/bench_c1_n2.json 2> $O/bench_c1_n2.err
  CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err
  CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_bench.log 2>&1
else
  if [ -z "$SKIP_TESTS" ]; then
    timeout -s KILL 2400 python -m pytest tests/test_step_dist_gpu.py tests/test_encoder_gpu.py -q -rs -k "4-" > $O/pytest_gpu_4.log 2>&1; echo pytest_rc=$? >> $O/pytest_gpu_4.log
  fi
  for cfg in c1 c2 c3 c4; do
    timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2961${cfg:1:1} bench.py --gpus 4 --steps 5 --warmup 3 --config $cfg > $O/bench_${cfg}_n4.json 2> $O/bench_${cfg}_n4.err
  done
fi
tail -n 3 $O/*.log
