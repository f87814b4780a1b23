set -x
for pw in 1 0; do echo "pow2=$pw" >> gpurun_out/r2_m_gemm.log; OPX_GEMM_BAND_POW2=$pw python tools/bench_gemm.py 32768 2>&1 | grep -E "gate|down|lm_head|qkv fwd" >> gpurun_out/r2_m_gemm.log; done
for pw in 1 0 1 0; do OPX_GEMM_BAND_POW2=$pw python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('pow2=$pw', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['node_ms']['fwd.mlp'], d['node_ms']['bwd.mlp.wgrad_gu'])
" >> gpurun_out/r2_m_bench.log; done
for pw in 1 0; do OPX_GEMM_BAND_POW2=$pw ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc2 --launch-skip 6 --launch-count 2 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2_m_ncu_$pw.csv 2>/dev/null; done
cat gpurun_out/r2_m_gemm.log gpurun_out/r2_m_bench.log
