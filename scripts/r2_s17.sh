#!/bin/bash
out=gpurun_out/r2s17; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
REPS=5 timeout 200 python scripts/stream_pass_probe.py gemma2-2b > $out/probe_gemma.log 2>&1
grep "gemma\|timed" $out/probe_gemma.log | head
timeout 600 python -m pytest tests/test_stream_gpu.py -m gpu -q -p no:cacheprovider -k "stream_backward" > $out/stream.log 2>&1; echo "exit $?" >> $out/stream.log
tail -n 3 $out/stream.log
REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"stream3|unpermute|gather_rows|window" --csv --log-file $out/ncu.csv python scripts/stream_pass_probe.py gemma2-2b both:1 > /dev/null 2>&1
python3 - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/r2s17/ncu.csv")))
h=None
for r in rows:
    if r and r[0]=="ID": h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d["ID"], d["Kernel Name"][:34], d["Metric Name"], d["Metric Value"])
PY
