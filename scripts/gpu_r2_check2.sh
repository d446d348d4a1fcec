#!/bin/bash
# Final check of HEAD: GPU tests, smoke(), the default bench line, BlackScholes max error.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
python - <<'PY'
import numpy as np, torch, lift_inputs as gen, oracle, paper_1502_02389_b200 as lift
s = gen.host(4 << 20, 0, gen.TID_X, lo=10.0, hi=200.0)
c, p = lift.blackscholes(torch.from_numpy(s).to("cuda:0"), 100.0, 0.05, 0.2, 1.0)
oc, op = oracle.blackscholes(s, 100.0, 0.05, 0.2, 1.0)
sc = s.astype(np.float64) + 100.0
print("blackscholes max |err|/(s+K): call %.3g put %.3g" % ((np.abs(c.cpu().numpy() - oc) / sc).max(), (np.abs(p.cpu().numpy() - op) / sc).max()))
PY
