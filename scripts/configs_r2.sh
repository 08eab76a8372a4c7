#!/bin/bash
# every BASELINE head and variant on the final build (profiles/r2/configs_final.jsonl)
out=gpurun_out/configs_r2; mkdir -p $out; rm -f $out/configs.jsonl
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for a in "--config gpt2" "--config gpt2 --memory fast" "" "--memory fast" "--low-memory" "--sigma 2" "--dist zipf" "--paper-order" "--no-sort" \
         "--config llama3-8b" "--config llama3-8b --memory fast" "--config gemma2-9b" "--config gemma2-9b --memory fast" "--config nemo-12b"; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $a > $out/tmp.log 2>&1
  python3 -c "
import json
for l in open('$out/tmp.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']
        d['args'] = '$a'
        print('$a'.ljust(32), f\"{d['ms_per_step']:8.2f} ms fwd {k['fwd']:7.2f} bwd {k['bwd']:7.2f} skip {d['skip']['skip_rate']:.3f} frac {d['roofline']['frac']:.3f} peak {m['step_peak_transient_bytes']/2**20:7.0f} MiB fwdpk {m['fwd_peak_transient_bytes']/2**20:6.0f} clk {d['clocks']['sm_mhz']}\")
        open('$out/configs.jsonl','a').write(json.dumps(d) + '\n')
"
done
