cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python scripts/variant_bits.py build/tune/default.so build/tune/tree_smem_tree.so build/tune/load_tma_bulk.so > gpurun_out/variant_bits.txt 2>&1
timeout 2400 python scripts/tune.py measure gpurun_out/tuning.json > gpurun_out/tune.log 2>&1; echo "tune rc=$?"
bash scripts/gpu_r2_final.sh
