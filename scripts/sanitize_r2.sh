#!/bin/bash
# compute-sanitizer on the streamed path (round-2 build): memcheck + synccheck + racecheck
out=gpurun_out/sanitize_r2; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
sel="not 256000 and not beyond and not changing"
for tool in memcheck synccheck racecheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_stream_gpu.py -q -m gpu -k "$sel" -p no:cacheprovider > $out/sanitize_$tool.log 2>&1
  echo "$tool exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $out/sanitize_$tool.log | tail -2
done
grep -h "Race reported" $out/sanitize_racecheck.log | grep -v tmem_alloc_pair | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head
