#!/bin/bash
# Same-box A/B of environment settings: bash scripts/ab_env.sh <out> "<ENV=..>" "<ENV=..>" ...
out=gpurun_out/${1:-abenv}; shift; mkdir -p $out
for rep in 1 2; do
  for v in "$@"; do
    echo "== $v rep $rep" >> $out/ab.log
    env $v timeout 300 python scripts/trace_step.py ${CFG:-gemma2-2b} 2>/dev/null | grep -E "span|lse_kernel|de_kernel|dc_kernel|label_shat" | head -6 >> $out/ab.log
  done
done
cat $out/ab.log
