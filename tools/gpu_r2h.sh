set -x
python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/r2_h_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2_h_pytest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_h_bench_n1.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2_h_bench_n2.log 2>&1
OPX_BENCH_ASYNC=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2_h_bench_n2_async.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc2 --launch-skip 6 --launch-count 2 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2_h_ncu_mlp.csv 2> gpurun_out/r2_h_ncu_mlp.err
SAN_TIMEOUT=600 ./tools/sanitize.sh > gpurun_out/r2_h_sanitize.txt 2>&1
tail -3 gpurun_out/r2_h_pytest.log; cat gpurun_out/r2_h_sanitize.txt
