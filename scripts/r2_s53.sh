#!/bin/bash
out=gpurun_out/r2s53; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
   python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $out/launches.log 2>&1
python scripts/launch_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1; head -30 $out/launches_summary.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench.log 2>&1; tail -c 1500 $out/bench.log
for a in "--config gpt2" "--config gpt2 --memory fast" "--memory fast" "--low-memory" "--sigma 2" "--dist zipf" "--dist zipf --memory fast" "--paper-order" "--no-sort" "--config llama3-8b" "--config llama3-8b --memory fast" "--config gemma2-9b" "--config gemma2-9b --memory fast" "--config nemo-12b" "--config nemo-12b --low-memory"; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $a > $out/tmp.log 2>&1
  python3 -c "
import json,sys
for l in open('$out/tmp.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']
        print('$a'.ljust(32), f\"{d['ms_per_step']:8.2f} ms fwd {k['fwd']:7.2f} bwd {k['bwd']:7.2f} skip {d['skip']['skip_rate']:.3f} peak {m['step_peak_transient_bytes']/2**20:7.0f} MiB fwdpk {m['fwd_peak_transient_bytes']/2**20:6.0f} clk {d['clocks']['sm_mhz']}\")
        open('$out/configs.jsonl','a').write(l)
"
done
