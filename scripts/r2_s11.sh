#!/bin/bash
out=gpurun_out/r2s11; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
CCE_STREAM_RING=4096 timeout 120 python scripts/stream_pass_probe.py small > $out/bigring.log 2>&1
grep -v "^ *File\|^frame\|^  \|^Search\|^CUDA\|^For\|^Compile" $out/bigring.log | head -12
CCE_LIB=libcce_b200_trace.so REPS=1 timeout 60 python scripts/stream_pass_probe.py small > $out/trace.log 2>&1
grep "^de cta" $out/trace.log | sort | uniq | head -60
grep -c "^de cta" $out/trace.log
