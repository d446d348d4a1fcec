cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/pt_var.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_var.log
export AB_SHAPES=${AB_SHAPES:-8192x8192,4096x4096,8192x16384,1024x8192,2048x8192,16384x4096,8192x2048}
for l in ${LIBS:-paper_1502_02389_b200/liblift.so build/var_*.so}; do
LIFT_LIB=$PWD/$l timeout 300 python scripts/gemv_xs_ab.py --child 2>&1 >/dev/null | sed "s|^|$(basename $l) |" | cut -c1-260
done
