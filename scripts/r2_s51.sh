#!/bin/bash
out=gpurun_out/r2s51; mkdir -p $out
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_stream3_kernel" -s 1 -c 1 -o $out/stream3 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_stream.log 2>&1; echo "stream exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_lse_kernel" -s 60 -c 1 -o $out/fwd_g2b \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_fwd.log 2>&1; echo "fwd exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_lse_kernel" -s 60 -c 1 -o $out/fwd_g9b \
  python bench.py --config gemma2-9b --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_fwd9.log 2>&1; echo "fwd9 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cce_lse_kernel" -s 60 -c 1 -o $out/fwd_nemo \
  python bench.py --config nemo-12b --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_fwdnemo.log 2>&1; echo "fwdnemo exit $?"
for f in stream3 fwd_g2b fwd_g9b fwd_nemo; do python scripts/ncu_summary.py $out/$f.ncu-rep $out/$f.json 2>&1 | tail -2; done
ls -la $out
