#!/bin/bash
# where the streamed backward's DRAM traffic comes from: ncu dram bytes of cce_stream3_kernel with
# the dE role's operand loads / epilogue skipped (CCE_STREAM_DEBUG_DE, timing-only builds)
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for dbg in 0 1 2 3 12; do
  CCE_STREAM_DEBUG_DE=$dbg timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"cce_stream3_kernel" -s 1 -c 1 \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "dram__bytes|gpu__time|lts__" | awk -v d=$dbg '{print "dbg " d ": " $1, $(NF-1), $NF}'
done
