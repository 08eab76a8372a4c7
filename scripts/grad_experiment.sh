#!/bin/bash
# B2/B3 load diagnostics: time the gradient kernels with S-hat / operand loads disabled (results invalid)
out=gpurun_out/$1; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1
for dbg in 0 1 2 3; do
  CCE_DEBUG_GRAD=$dbg timeout 300 python scripts/trace_step.py > $out/trace_dbg$dbg.log 2>&1
  echo "== dbg $dbg" >> $out/summary.txt; grep -E "cce_d[ec]_kernel|span" $out/trace_dbg$dbg.log | head -3 >> $out/summary.txt
done
cat $out/summary.txt
