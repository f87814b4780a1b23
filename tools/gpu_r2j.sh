set -x
python -m pytest tests/test_step_gpu.py tests/test_moe_gpu.py tests/test_report_gpu.py tests/test_integration_cpp.py -q -rs -x > gpurun_out/r2_j_pytest1.log 2>&1; echo rc=$? >> gpurun_out/r2_j_pytest1.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_j_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2_j_smoke.log
for mode in default serial fused; do
  case $mode in serial) export OPX_MOE_SERIAL_HALVES=1;; fused) unset OPX_MOE_SERIAL_HALVES; export OPX_MOE_FUSED_COMBINE=1;; esac
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$RANDOM_PORT$((${#mode})) bench.py --gpus 4 --steps 5 --warmup 3 --config c2 > gpurun_out/r2_j_bench_c2_$mode.log 2>&1
done
unset OPX_MOE_SERIAL_HALVES OPX_MOE_FUSED_COMBINE
python -m pytest tests/test_step_dist_gpu.py -q -rs -k "moe" > gpurun_out/r2_j_pytest2.log 2>&1; echo rc=$? >> gpurun_out/r2_j_pytest2.log
OPX_GEMM_LOG=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2_j_gemmlog.log 2>&1
tail -3 gpurun_out/r2_j_pytest1.log gpurun_out/r2_j_pytest2.log gpurun_out/r2_j_smoke.log
