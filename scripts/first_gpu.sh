#!/bin/bash
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
for w in fwd nosort; do
  timeout 120 python scripts/gpu_check.py $w > gpurun_out/chk_$w.log 2>&1; echo "exit $w $?" >> gpurun_out/chk_$w.log
done
for b in 1 4; do
  CCE_GATHER4_BOX_ROWS=$b timeout 120 python scripts/gpu_check.py sort > gpurun_out/chk_sort_b$b.log 2>&1; echo "exit $?" >> gpurun_out/chk_sort_b$b.log
  CCE_GATHER4_BOX_ROWS=$b timeout 120 python scripts/gpu_check.py ignore > gpurun_out/chk_ign_b$b.log 2>&1; echo "exit $?" >> gpurun_out/chk_ign_b$b.log
done
timeout 120 python scripts/gpu_check.py cap > gpurun_out/chk_cap.log 2>&1; echo "exit $?" >> gpurun_out/chk_cap.log
tail -n 5 gpurun_out/chk_*.log
