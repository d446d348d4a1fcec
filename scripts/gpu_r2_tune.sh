cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python scripts/variant_bits.py build/tune/default.so build/tune/tree_smem_tree.so build/tune/load_tma_bulk.so build/tune/asum_acc_asum_f64.so build/tune/dot_acc_dot_f32.so build/tune/pdl_pdl_off.so > gpurun_out/variant_bits.txt 2>&1
cat gpurun_out/variant_bits.txt
timeout 2400 python scripts/tune.py measure gpurun_out/tuning.json > gpurun_out/tune.log 2>&1
echo "tune rc=$?"; tail -3 gpurun_out/tune.log
