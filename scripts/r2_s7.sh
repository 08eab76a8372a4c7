#!/bin/bash
out=gpurun_out/r2s7; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_stream_gpu.py -m gpu -x -v -p no:cacheprovider -k "stream_backward" > $out/stream.log 2>&1; echo "exit $?" >> $out/stream.log
grep -E "PASS|FAIL|Error|error|passed|failed|exit" $out/stream.log | tail -30
timeout 300 python scripts/stream_probe.py gemma2-2b gpt2 > $out/probe.log 2>&1; echo "exit $?" >> $out/probe.log
cat $out/probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k stream > $out/parity.log 2>&1; echo "exit $?" >> $out/parity.log
tail -n 5 $out/parity.log
