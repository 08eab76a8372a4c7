#!/bin/bash
out=gpurun_out/r2s10; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 300 python scripts/stream_lists_check.py 2048 512 40000 2>&1 | tail -12
