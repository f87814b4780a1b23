# attention CTA order: plain x-fastest (band 1) vs GQA-group bands walked tile-major (band 0 = g)
for b in 1 0 1 0; do
  echo "band=$b"; OPX_ATTN_FWD_BAND=$b OPX_ATTN_BAND=$b python tools/bench_attn.py 2>&1 | grep TFLOP
done
OPX_ATTN_FWD_BAND=0 OPX_ATTN_BAND=0 timeout 200 python -m pytest tests/test_kernels_gpu.py -q -k "attention" 2>&1 | tail -1
