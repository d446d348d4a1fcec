cd "${GRAFT_REPO_ROOT:-/root/repo}"
# the bench step under several builds, interleaved by process (3 rounds)
for r in 1 2 3; do for l in ${LIBS:-paper_1502_02389_b200/liblift.so build/var_*.so}; do
  echo "$(basename $l) $(LIFT_LIB=$PWD/$l python scripts/step_knob_ab.py ${KNOB:-order} ${VALS:-0} 20)"
done; done
