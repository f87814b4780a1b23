python bench.py --steps 5 --warmup 3 --no-cpu-baseline --single-sample > gpurun_out/r2_y_single.json 2>gpurun_out/r2_y_single.err
python -c "
import json
for l in open('gpurun_out/r2_y_single.json'):
    if l.startswith('{'): d=json.loads(l); print(round(d['value']), d['mfu_exact'], d['mfu_ref'], d['clocks']['sm_mhz'], d['roofline_attention'])
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'router|combine|dispatch|unpermute' -c 60 --csv --log-file gpurun_out/r2_y_moe.csv python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2_y_moe.log 2>&1
echo ncu rc=$?
