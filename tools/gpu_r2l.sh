set -x
for st in 0 1; do echo "staged=$st" >> gpurun_out/r2_l_gemm.log; OPX_GEMM_EPI_STAGED=$st python tools/bench_gemm.py 32768 >> gpurun_out/r2_l_gemm.log 2>&1; done
for st in 0 1; do OPX_GEMM_EPI_STAGED=$st OPX_GEMM_LOG=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2_l_gemmlog_$st.log 2>&1; done
python -m pytest tests/test_kernels_gpu.py -q -x -k gemm > gpurun_out/r2_l_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2_l_pytest.log
cat gpurun_out/r2_l_gemm.log; tail -n 2 gpurun_out/r2_l_pytest.log
