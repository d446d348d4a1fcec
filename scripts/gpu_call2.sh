#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python scripts/ab.py build/liblift_f64.so build/liblift_f32.so build/liblift_g4u2.so build/liblift_g1u8.so > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_probe.csv python scripts/ncu_probe.py 3 > gpurun_out/ncu_probe.log 2>&1
echo "ncu probe rc=$?"; tail -3 gpurun_out/ncu_probe.log; wc -l gpurun_out/launches_probe.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reduce_kernel|gemv_kernel|scal_kernel" -s 4 -c 4 -o gpurun_out/prof_r1 python scripts/ncu_probe.py 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
