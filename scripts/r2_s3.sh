#!/bin/bash
out=gpurun_out/r2s3; mkdir -p $out
for v in libcce_b200_glag4.so libcce_b200_glag5.so; do
  echo "== $v" >> $out/probe.log
  CCE_LIB=$v timeout 300 python scripts/fwd_gather_probe.py gpt2 gemma2-2b >> $out/probe.log 2>&1
done
cat $out/probe.log
