set -x
python -m pytest tests/test_encoder_gpu.py tests/test_moe_gpu.py tests/test_step_dist_gpu.py tests/test_widths_gpu.py tests/test_report_gpu.py -q -rs --durations=10 > gpurun_out/r2_i_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2_i_pytest.log
python tools/bench_ulysses.py > gpurun_out/r2_i_ulysses.log 2>&1
ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum --clock-control none -k regex:"seq2head|head2seq" -c 4 --csv python tools/bench_ulysses.py > gpurun_out/r2_i_ulysses_ncu.csv 2> gpurun_out/r2_i_ulysses_ncu.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 5 --warmup 3 --config c2 > gpurun_out/r2_i_bench_c2_n4.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 --steps 3 --warmup 3 --config c3 > gpurun_out/r2_i_bench_c3_n4.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2_i_bench_c1_n4.log 2>&1
tail -3 gpurun_out/r2_i_pytest.log; cat gpurun_out/r2_i_ulysses.log
