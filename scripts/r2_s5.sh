#!/bin/bash
out=gpurun_out/r2s5; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 300 python scripts/stream_probe.py gemma2-2b gpt2 > $out/probe.log 2>&1; echo "exit $?" >> $out/probe.log
timeout 600 python -m pytest tests/test_stream_gpu.py -m gpu -v -p no:cacheprovider > $out/stream.log 2>&1; echo "exit $?" >> $out/stream.log
cat $out/probe.log; grep -E "PASS|FAIL|passed|failed|exit" $out/stream.log | tail -20
