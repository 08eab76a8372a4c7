#!/bin/bash
out=gpurun_out/r2s41; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
grep -E "^FAILED|passed|failed|exit" $out/pytest_gpu.log | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench.log 2>&1; echo "exit $?" >> $out/bench.log
tail -c 3000 $out/bench.log
for cfg in gpt2 llama3-8b gemma2-9b nemo-12b; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> $out/configs.log 2>&1; echo "exit $cfg $?" >> $out/configs.log
done
python3 - <<'PY'
import json
for l in open("gpurun_out/r2s41/configs.log"):
    if l.startswith("{"):
        d = json.loads(l); k = d["kernel_ms"]
        print(d["config"]["workload"], f"{d['ms_per_step']:.2f} ms fwd {k['fwd']:.2f} bwd {k['bwd']:.2f} frac {d['roofline']['frac']:.3f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB skip {d['skip']['skip_rate']:.3f}")
    elif l.startswith("exit"): print(l.strip())
PY
