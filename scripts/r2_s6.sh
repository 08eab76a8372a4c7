#!/bin/bash
out=gpurun_out/r2s6; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 300 python scripts/stream_pass_probe.py > $out/probe.log 2>&1
REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"stream|gather_rows|unpermute" --csv --log-file $out/ncu.csv python scripts/stream_pass_probe.py > $out/ncu_run.log 2>&1
cat $out/probe.log
python3 - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/r2s6/ncu.csv")))
h=None
for r in rows:
    if r and r[0]=="ID": h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r))
        print(d["ID"], d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"])
PY
