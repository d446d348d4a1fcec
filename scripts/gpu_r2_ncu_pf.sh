#!/bin/bash
# DRAM bytes and duration of one-wave (1024x8192) and many-wave (8192^2) gemv launches with the
# L2 prefetch forced off / on (LIFT_VAR_PREFETCH 1 / 2): does the prefetch duplicate DRAM reads?
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for shape in "1024 8192" "8192 8192"; do for pf in 1 2; do
  LIFT_PF=$pf timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum \
    --clock-control none -k regex:gemv -s 2 -c 1 --csv python scripts/ncu_gemv.py $shape 2>/dev/null | grep -E "gpu__time|dram__bytes|lts__" | sed "s|^|$shape pf=$pf |" | cut -c1-220
done; done
