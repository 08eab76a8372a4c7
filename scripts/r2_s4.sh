#!/bin/bash
out=gpurun_out/r2s4; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_stream_gpu.py -m gpu -x -v -p no:cacheprovider > $out/stream.log 2>&1; echo "exit $?" >> $out/stream.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -v -p no:cacheprovider -k stream > $out/parity.log 2>&1; echo "exit $?" >> $out/parity.log
tail -n 30 $out/stream.log; tail -n 40 $out/parity.log
