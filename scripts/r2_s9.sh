#!/bin/bash
out=gpurun_out/r2s9; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
CCE_STREAM_DEBUG=1 timeout 120 python scripts/stream_pass_probe.py small > $out/probe_small.log 2>&1; echo "exit $?" >> $out/probe_small.log
grep -v "^ *File\|^frame\|^  \|^Search\|^CUDA\|^For\|^Compile" $out/probe_small.log | head -40
