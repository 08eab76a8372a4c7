#!/bin/bash
out=gpurun_out/r2s8; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
for cfg in small gemma2-2b; do
  timeout 120 python scripts/stream_pass_probe.py $cfg > $out/probe_$cfg.log 2>&1; echo "exit $?" >> $out/probe_$cfg.log
  cat $out/probe_$cfg.log | grep -v "^ *File\|^frame\|^  " | tail -12
done
