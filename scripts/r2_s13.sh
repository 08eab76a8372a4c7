#!/bin/bash
for env in "CCE_PDL=0" "CCE_STREAM_ZERO_WS=1" "CUDA_MODULE_LOADING=EAGER"; do
  echo "== $env"
  env $env CCE_STREAM_RING=4096 REPS=1 timeout 60 python scripts/stream_pass_probe.py small de:0,de:0,de:0 2>&1 | grep "small\|timed" | head -8
done
