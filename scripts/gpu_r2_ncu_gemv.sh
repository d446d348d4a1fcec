cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in ${VARS:-3}; do
GEMV_X=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -s 2 -c 1 \
  -o gpurun_out/gemv_v$v -f python scripts/ncu_gemv.py ${SHAPE:-8192 8192} > gpurun_out/ncu_gemv_v$v.log 2>&1
echo "ncu v$v rc=$?"
done
