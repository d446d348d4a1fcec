cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=r2 bash scripts/profile_round.sh
bash scripts/gpu_sanitize.sh
