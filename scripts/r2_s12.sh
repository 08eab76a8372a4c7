#!/bin/bash
out=gpurun_out/r2s12; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
for seq in "both:0,both:0" "de:0,de:0,de:0" "de:0,dc:0,de:0"; do
  echo "== $seq"
  CCE_STREAM_RING=4096 REPS=1 timeout 60 python scripts/stream_pass_probe.py small $seq 2>&1 | grep "small\|timed" | head -8
done
