#!/bin/bash
out=gpurun_out/r2s56; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_abi_c_gpu.py tests/test_memory_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for a in "--pad 0" "--pad 0.25" "--pad 0.5" "--pad 0 --memory fast" "--pad 0.25 --memory fast"; do
  timeout 900 python bench.py --config llama3-8b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $a > $out/tmp.log 2>&1
  python3 -c "
import json
for l in open('$out/tmp.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']
        print('$a'.ljust(26), f\"{d['ms_per_step']:8.2f} ms fwd {k['fwd']:7.2f} bwd {k['bwd']:7.2f} kept {d['skip']['kept_tiles']} peak {m['step_peak_transient_bytes']/2**20:6.0f} MiB clk {d['clocks']['sm_mhz']}\")
        open('$out/table_a1.jsonl','a').write(l)
"
done
