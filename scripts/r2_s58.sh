#!/bin/bash
out=gpurun_out/r2s58; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_memory_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for a in "--config gpt2" "--config llama3-8b" "--config gemma2-9b" "--config nemo-12b" "--config gemma2-9b --memory fast" "--config llama3-8b --memory fast"; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $a > $out/tmp.log 2>&1
  python3 -c "
import json
for l in open('$out/tmp.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']
        print('$a'.ljust(32), f\"{d['ms_per_step']:8.2f} ms fwd {k['fwd']:7.2f} bwd {k['bwd']:7.2f} frac {d['roofline']['frac']:.3f} peak {m['step_peak_transient_bytes']/2**20:7.0f} MiB fwdpk {m['fwd_peak_transient_bytes']/2**20:6.0f} clk {d['clocks']['sm_mhz']}\")
        open('$out/configs.jsonl','a').write(l)
"
done
