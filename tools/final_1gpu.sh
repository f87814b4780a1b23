# Round-end check on one GPU, the way the driver runs it: the GPU suite, smoke,
# the default bench line (+ CPU baseline) and the ncu launch list of one step.
set -x
O=gpurun_out/final_n1
mkdir -p $O
timeout -s KILL 2400 python -m pytest tests -q -m gpu -rs --durations=15 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$? >> $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > $O/bench_c1_n1.json 2> $O/bench_c1_n1.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_bench.log 2>&1
tail -n 3 $O/pytest_gpu.log $O/smoke.log
