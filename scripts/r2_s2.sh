#!/bin/bash
out=gpurun_out/r2s2; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1
timeout 600 python -m pytest tests/test_stream_gpu.py -m gpu -x -v -p no:cacheprovider > $out/stream.log 2>&1; echo "exit $?" >> $out/stream.log
timeout 900 python scripts/fwd_gather_probe.py gpt2 gemma2-2b llama3-8b > $out/probe.log 2>&1; echo "exit $?" >> $out/probe.log
timeout 1500 python -m pytest tests -m gpu -v -p no:cacheprovider --deselect tests/test_baseline_parity_gpu.py --deselect tests/test_stream_gpu.py > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
tail -n 3 $out/*.log
