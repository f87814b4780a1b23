set -x
python -m pytest tests/test_kernels_gpu.py tests/test_step_gpu.py tests/test_widths_gpu.py -q -rs -x -k "not c2_width and not c4_width" > gpurun_out/r2_k_pytest1.log 2>&1; echo rc=$? >> gpurun_out/r2_k_pytest1.log
OPX_GEMM_LOG=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2_k_gemmlog.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_k_bench_n1.log 2>&1
python bench.py --config c2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_k_bench_c2_n1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"combine|unpermute|dispatch|router" -c 60 --csv python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2_k_c2_moe_kernels.csv 2>/dev/null
python -m pytest tests/test_encoder_gpu.py tests/test_step_dist_gpu.py -q -rs -k "encoder or c0 or structure or plan6 or plan7" > gpurun_out/r2_k_pytest2.log 2>&1; echo rc=$? >> gpurun_out/r2_k_pytest2.log
for f in gpurun_out/r2_k_pytest1.log gpurun_out/r2_k_pytest2.log; do tail -n 3 $f; done
