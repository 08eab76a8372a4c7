#!/bin/bash
# dE-pass variants (CCE_DE="<chunks>,<order>,<dynamic>,<prefetch>"): per-kernel device times from the trace.
out=gpurun_out/${1:-de_var}; shift; mkdir -p $out
for v in "$@"; do
  echo "== CCE_DE=$v" >> $out/de_variants.log
  CCE_DE=$v timeout 300 python scripts/trace_step.py ${CFG:-gemma2-2b} 2>/dev/null | grep -E "de_kernel|span" | head -2 >> $out/de_variants.log
done
cat $out/de_variants.log
