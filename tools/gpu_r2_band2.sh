# attention CTA order on the 28q/4kv shapes: band 1 / 7 (GQA group) / 28 (all heads tile-major)
for b in 1 28 7 1 28 7; do
  echo "band=$b"; BENCH_ATTN_SHAPES=1,2 OPX_ATTN_FWD_BAND=$b OPX_ATTN_BAND=$b python tools/bench_attn.py 2>&1 | grep TFLOP
done
