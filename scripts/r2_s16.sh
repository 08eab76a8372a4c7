#!/bin/bash
out=gpurun_out/r2s16; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
REPS=3 timeout 120 python scripts/stream_pass_probe.py small > $out/probe_small.log 2>&1
REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b > $out/probe_gemma.log 2>&1
grep "small\|timed" $out/probe_small.log | head; grep "gemma\|timed" $out/probe_gemma.log | head
timeout 600 python -m pytest tests/test_stream_gpu.py -m gpu -q -p no:cacheprovider -k "stream_backward" > $out/stream.log 2>&1; echo "exit $?" >> $out/stream.log
tail -n 3 $out/stream.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k stream > $out/parity.log 2>&1; echo "exit $?" >> $out/parity.log
tail -n 3 $out/parity.log
