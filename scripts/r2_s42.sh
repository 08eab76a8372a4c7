#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
run() { env "${@:2}" timeout 600 python bench.py --config $1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.2f} bwd {k['bwd']:.2f} peak {d['memory']['step_peak_transient_bytes']/2**20:.0f} MiB\")
"; }
echo "llama fast: $(run llama3-8b CCE_MEMORY=fast)"
echo "llama ring1024: $(run llama3-8b CCE_STREAM_RING=1024)"
echo "llama ring2048: $(run llama3-8b CCE_STREAM_RING=2048)"
echo "gemma9b fast: $(run gemma2-9b CCE_MEMORY=fast)"
echo "gemma9b ring1024: $(run gemma2-9b CCE_STREAM_RING=1024)"
echo "gpt2 fast: $(run gpt2 CCE_MEMORY=fast)"
echo "gpt2 grouped: $(run gpt2 CCE_MEMORY=grouped)"
echo "nemo fast: $(run nemo-12b CCE_MEMORY=fast)"
echo "nemo grouped: $(run nemo-12b CCE_MEMORY=grouped)"
