#!/bin/bash
# ncu --set full of one forward vocabulary-group launch and the stream kernel (Gemma-2-2B default)
out=gpurun_out/ncu_r2; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_lse_kernel" -s 30 -c 1 -o $out/fwd_g2b \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_fwd.log 2>&1; echo "fwd exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_stream3_kernel" -s 1 -c 1 -o $out/stream3 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_stream.log 2>&1; echo "stream exit $?"
for f in fwd_g2b stream3; do python scripts/ncu_summary.py $out/$f.ncu-rep $out/$f.json 2>&1 | tail -1; done
