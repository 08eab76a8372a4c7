#!/bin/bash
# A/B of library variants on one box: bash scripts/ab.sh <out> <variant-file>... (default lib = "base")
out=gpurun_out/${1:-ab}; shift; mkdir -p $out
for rep in 1 2; do
  for v in base "$@"; do
    lib=""; [ "$v" != base ] && lib="$v"
    echo "== $v rep $rep" >> $out/ab.log
    CCE_LIB=$lib timeout 300 python scripts/trace_step.py ${CFG:-gemma2-2b} 2>/dev/null | grep -E "span|lse_kernel|de_kernel|dc_kernel" | head -5 >> $out/ab.log
  done
done
cat $out/ab.log
