#!/bin/bash
# Final round-2 evidence in one gpurun call (after `python scripts/tune.py build` here):
# variant bits + NEXT-4 search, GPU tests, bench (N=1, N=2 gloo, reference arm), ncu launch list
# + --set full captures, sanitizers, size sweep, back-to-back per-op times, gemv stall top.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python scripts/variant_bits.py build/tune/default.so build/tune/tree_smem_tree.so build/tune/load_tma_bulk.so > gpurun_out/variant_bits.txt 2>&1
timeout 2400 python scripts/tune.py measure gpurun_out/tuning.json > gpurun_out/tune.log 2>&1; echo "tune rc=$?"
bash scripts/gpu_r2_final.sh
timeout 600 python scripts/sweep.py > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"
python scripts/ab.py paper_1502_02389_b200/liblift.so > gpurun_out/ab_final.txt 2>&1
bash scripts/gpu_r2_gemvlibs.sh >> gpurun_out/ab_final.txt 2>&1
bash scripts/gpu_r2_midab.sh >> gpurun_out/ab_final.txt 2>&1
echo "ab rc=$?"
