#!/bin/bash
# HISTORICAL: A/B of the split-row softmax experiment (TR_ATTN_SPLIT), which
# exists only in commit 44ba687 (check it out to rerun); the result is in
# profiles/r01/split_softmax_ab.log and DESIGN.md section 5.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TR_ATTN_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_execute.py -x -q > gpurun_out/split_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/split_parity.log
tail -3 gpurun_out/split_parity.log
for v in 0 1 0 1; do
  echo "== TR_ATTN_SPLIT=$v"
  TR_ATTN_SPLIT=$v timeout 300 python scripts/probe_attn.py --case 0 1
  TR_ATTN_SPLIT=$v timeout 120 python scripts/power_probe.py attn-full 8
  TR_ATTN_SPLIT=$v timeout 120 python scripts/power_probe.py attn-causal 8
done
