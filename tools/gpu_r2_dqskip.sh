# attention bwd: what the dQ drain costs (OPX_DEBUG_SKIP_DQ=1: no TMA reduce, =2: no staging either)
for m in "" 1 2 ""; do
  echo "skip=$m"; env ${m:+OPX_DEBUG_SKIP_DQ=$m} python tools/bench_attn.py 2>&1 | grep -E "bwd_tc |split1 "
done
