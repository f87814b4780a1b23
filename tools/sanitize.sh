#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over the kernel parity
# tests at their small shapes, checking only opx kernels (torch's are
# excluded by the name filter).  Logs -> gpurun_out/sanitize_<tool>.log.
cd "$(dirname "$0")/.."
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
SEL="attention or gemm_bf16 or swiglu or rmsnorm or adamw or embedding or cross_entropy or rope or grouped"
for tool in memcheck racecheck synccheck; do
  timeout ${SAN_TIMEOUT:-900} /usr/local/cuda/bin/compute-sanitizer --tool $tool \
    --kernel-name regex:'(gemm|attn|rmsnorm|adamw|embed|ce_kernel|swiglu|seq2head|head2seq|moe|delta|cast|colsum|init|sum_kernel|grad_accum)' \
    --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_kernels_gpu.py tests/test_moe_gpu.py -q -x -k "$SEL" -p no:cacheprovider \
    > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" | tee -a "$OUT/sanitize_$tool.log"
  tail -4 "$OUT/sanitize_$tool.log"
done
