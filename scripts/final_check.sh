#!/bin/bash
# round-end check: GPU suite, smoke, default bench, reference arm, 2-rank functional bench (gloo, one GPU)
out=gpurun_out/final; mkdir -p $out
python -m paper_2411_09009_b200._build > $out/build.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
grep -E "^FAILED|passed|failed|exit" $out/pytest_gpu.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > $out/bench.log 2>&1; echo "bench exit $?"; grep '^{' $out/bench.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['memory']['step_peak_transient_bytes']/2**20, d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/ref.log 2>&1; echo "ref exit $?"; tail -c 400 $out/ref.log
CCE_BENCH_BACKEND=gloo CCE_BENCH_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $out/multirank.log 2>&1; echo "multirank exit $?"; grep '^{' $out/multirank.log | cut -c1-300
