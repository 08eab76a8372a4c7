#!/bin/bash
# unpermutation anchor density: 1/64 (default) vs 1/32 vs 1/16
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
python -m paper_2411_09009_b200._build --variant k32 CCE_PERM_K_LOG2=5 > /dev/null 2>&1 || exit 1
python -m paper_2411_09009_b200._build --variant k16 CCE_PERM_K_LOG2=4 > /dev/null 2>&1 || exit 1
for lib in k32 k16; do CCE_LIB=libcce_b200_$lib.so timeout 600 python -m pytest tests/test_stream_gpu.py -k unpermute -q -p no:cacheprovider 2>&1 | tail -1; done
for i in 1 2; do for lib in "" libcce_b200_k32.so libcce_b200_k16.so; do CCE_LIB=$lib timeout 120 python scripts/unpermute_probe.py; done; done
for i in 1 2; do for lib in "" libcce_b200_k32.so libcce_b200_k16.so; do echo "bench $lib: $(CCE_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; m=d['memory']; print(f\"{d['ms_per_step']:.2f} ms  fwd {k['fwd']:.3f} bwd {k['bwd']:.3f} clk {d['clocks']['sm_mhz']} step {m['step_peak_transient_bytes']>>20} MiB\")
")"; done; done
