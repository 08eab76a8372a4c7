#!/bin/bash
# dE-pass variants (CCE_DE="<chunks>,<order>,<dynamic>"): per-kernel device times from the trace.
out=gpurun_out/${1:-de_var}; mkdir -p $out
for v in 1,0,0 1,1,0 1,0,1 1,1,1 2,0,0 2,1,0 2,0,1 2,1,1; do
  echo "== CCE_DE=$v" >> $out/de_variants.log
  CCE_DE=$v timeout 300 python scripts/trace_step.py 2>/dev/null | grep -E "de_kernel|dc_kernel|span" | head -3 >> $out/de_variants.log
done
cat $out/de_variants.log
