cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AB_SHAPES=8192x8192,4096x4096,8192x16384
for l in ${LIBS:-paper_1502_02389_b200/liblift.so build/var_*.so}; do
LIFT_LIB=$PWD/$l timeout 300 python scripts/gemv_xs_ab.py --child 2>&1 >/dev/null | sed "s|^|$(basename $l) |" | cut -c1-200
done
